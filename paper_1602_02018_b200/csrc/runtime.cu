// Library-level plumbing behind the C ABI: last-error string, launch counter,
// tuning options, profile counters, device properties, pointer classification.
#include <mutex>
#include <unordered_map>

#include "internal.cuh"

namespace csc {

std::atomic<int64_t> g_launches{0};
Options g_opt;

static thread_local std::string t_last_error;
void set_error(const std::string& msg) { t_last_error = msg; }

static std::mutex g_prof_mu;
static Profile g_prof;
struct PendingLaunch {
  cudaEvent_t e0, e1;
  double bytes;
  int64_t launches;
};
static std::vector<PendingLaunch> g_pending;
static std::vector<cudaEvent_t> g_event_pool;

static cudaEvent_t take_event() {
  // caller holds g_prof_mu
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CSC_CUDA(cudaEventCreate(&e));
  return e;
}

void profile_begin(cudaStream_t s, cudaEvent_t* e0) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  *e0 = take_event();
  CSC_CUDA(cudaEventRecord(*e0, s));
}

void profile_end(cudaStream_t s, cudaEvent_t e0, double bytes, int64_t launches) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t e1 = take_event();
  CSC_CUDA(cudaEventRecord(e1, s));
  g_pending.push_back({e0, e1, bytes, launches});
}

static void resolve_pending() {
  // caller holds g_prof_mu
  for (auto& p : g_pending) {
    CSC_CUDA(cudaEventSynchronize(p.e1));
    float ms = 0.f;
    CSC_CUDA(cudaEventElapsedTime(&ms, p.e0, p.e1));
    g_prof.ms += ms;
    g_prof.launches += p.launches;
    g_prof.bytes += p.bytes;
    g_event_pool.push_back(p.e0);
    g_event_pool.push_back(p.e1);
  }
  g_pending.clear();
}

static std::mutex g_dev_mu;
static std::unordered_map<int, DeviceProps> g_props;
static std::unordered_map<int, bool> g_pool_done;

const DeviceProps& device_props(int dev) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_props.find(dev);
  if (it != g_props.end()) return it->second;
  DeviceProps p;
  CSC_CUDA(cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, dev));
  CSC_CUDA(cudaDeviceGetAttribute(&p.l2_bytes, cudaDevAttrL2CacheSize, dev));
  if (cudaDeviceGetAttribute(&p.max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess) p.max_persist = 0;
  if (cudaDeviceGetAttribute(&p.max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev) != cudaSuccess) p.max_window = 0;
  cudaGetLastError();
  return g_props.emplace(dev, p).first->second;
}

static std::unordered_map<int, int64_t> g_persist_pct;
static std::unordered_map<int, size_t> g_persist_bytes;

size_t persist_bytes(int dev) {
  const int64_t pct = g_opt.l2_persist_pct.load();
  const DeviceProps& p = device_props(dev);
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_persist_pct.find(dev);
  if (it != g_persist_pct.end() && it->second == pct) return g_persist_bytes[dev];
  size_t want = pct > 0 ? (size_t)((double)p.l2_bytes * (double)pct / 100.0) : 0;
  if (want > (size_t)p.max_persist) want = (size_t)p.max_persist;
  if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
    cudaGetLastError();
    want = 0;
  }
  g_persist_pct[dev] = pct;
  g_persist_bytes[dev] = want;
  return want;
}

void ensure_pool(int dev) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (g_pool_done[dev]) return;
  cudaMemPool_t pool;
  CSC_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t threshold = UINT64_MAX;  // keep freed blocks cached across calls
  CSC_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
  g_pool_done[dev] = true;
}

cudaMemPool_t side_pool(int dev) {
  static cudaMemPool_t pools[64] = {};
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (dev < 0 || dev >= 64) fail(CSC_ERR_INVALID, "device index out of range");
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    CSC_CUDA(cudaMemPoolCreate(&pools[dev], &props));
    uint64_t threshold = UINT64_MAX;
    CSC_CUDA(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &threshold));
  }
  return pools[dev];
}

void trim_pools() {
  int dev = 0;
  CSC_CUDA(cudaGetDevice(&dev));
  CSC_CUDA(cudaDeviceSynchronize());
  cudaMemPool_t pool;
  CSC_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  CSC_CUDA(cudaMemPoolTrimTo(pool, 0));
  CSC_CUDA(cudaMemPoolTrimTo(side_pool(dev), 0));
}

bool is_device_ptr(const void* p, int device) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    if (a.type == cudaMemoryTypeDevice && a.device != device)
      fail(CSC_ERR_INVALID, "device pointer belongs to device " + std::to_string(a.device) +
                                ", graph lives on device " + std::to_string(device));
    return true;
  }
  return false;
}

}  // namespace csc

using namespace csc;

extern "C" {

int csc_abi_version(void) { return CSC_ABI_VERSION; }

const char* csc_last_error(void) { return t_last_error.c_str(); }

int csc_launch_count(int64_t* out) {
  return guard([&] {
    if (!out) fail(CSC_ERR_INVALID, "out is NULL");
    *out = g_launches.load();
  });
}

static std::atomic<int64_t>* option_slot(const char* key) {
  if (!key) return nullptr;
  std::string k(key);
  if (k == "panel_width") return &g_opt.panel_width;
  if (k == "recurrence") return &g_opt.recurrence;
  if (k == "cache_hints") return &g_opt.cache_hints;
  if (k == "cg_overlap") return &g_opt.cg_overlap;
  if (k == "lean_mid") return &g_opt.lean_mid;
  if (k == "fast_normalize") return &g_opt.fast_normalize;
  if (k == "l2_policy") return &g_opt.l2_policy;
  if (k == "pdl") return &g_opt.pdl;
  if (k == "h2d_overlap") return &g_opt.h2d_overlap;
  if (k == "block_threads") return &g_opt.block_threads;
  if (k == "profile") return &g_opt.profile;
  if (k == "l2_budget_pct") return &g_opt.l2_budget_pct;
  if (k == "unroll") return &g_opt.unroll;
  if (k == "l2_persist_pct") return &g_opt.l2_persist_pct;
  if (k == "persistent") return &g_opt.persistent;
  if (k == "cg_compact") return &g_opt.cg_compact;
  if (k == "row_order") return &g_opt.row_order;
  return nullptr;
}

int csc_set_option(const char* key, int64_t value) {
  return guard([&] {
    auto* slot = option_slot(key);
    if (!slot) fail(CSC_ERR_INVALID, std::string("unknown option ") + (key ? key : "(null)"));
    std::string k(key);
    if (k == "recurrence" && (value < 0 || value > 1)) fail(CSC_ERR_INVALID, "recurrence must be 0 or 1");
    if (k == "block_threads" && (value < 64 || value > 256 || value % 32))
      fail(CSC_ERR_INVALID, "block_threads must be a multiple of 32 in [64, 256]");
    if (k == "panel_width" && value < 0) fail(CSC_ERR_INVALID, "panel_width must be >= 0");
    if (k == "unroll" && value != 2 && value != 4 && value != 8) fail(CSC_ERR_INVALID, "unroll must be 2, 4 or 8");
    if (k == "l2_persist_pct" && (value < 0 || value > 100)) fail(CSC_ERR_INVALID, "l2_persist_pct in [0, 100]");
    if (k == "persistent" && value != 0 && value != 1) fail(CSC_ERR_INVALID, "persistent must be 0 or 1");
    if (k == "profile" && (value < 0 || value > 2)) fail(CSC_ERR_INVALID, "profile must be 0, 1 or 2");
    if (k == "lean_mid" && value != 0 && value != 1) fail(CSC_ERR_INVALID, "lean_mid must be 0 or 1");
    if (k == "l2_budget_pct" && (value < 1 || value > 100)) fail(CSC_ERR_INVALID, "l2_budget_pct in [1, 100]");
    slot->store(value);
  });
}

int csc_get_option(const char* key, int64_t* value) {
  return guard([&] {
    auto* slot = option_slot(key);
    if (!slot) fail(CSC_ERR_INVALID, std::string("unknown option ") + (key ? key : "(null)"));
    if (!value) fail(CSC_ERR_INVALID, "value is NULL");
    *value = slot->load();
  });
}

int csc_profile_read(double* step_ms, int64_t* step_launches, double* step_bytes) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    resolve_pending();
    if (step_ms) *step_ms = g_prof.ms;
    if (step_launches) *step_launches = g_prof.launches;
    if (step_bytes) *step_bytes = g_prof.bytes;
  });
}

int csc_profile_reset(void) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    resolve_pending();
    g_prof = Profile{};
  });
}

}  // extern "C"
