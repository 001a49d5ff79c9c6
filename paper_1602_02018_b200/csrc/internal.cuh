// Shared internals of libcsc_b200.so: error plumbing at the C-ABI boundary,
// launch accounting, stream-ordered scratch memory, host/device pointer
// classification, and the device graph handle.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/csc_b200.h"

namespace csc {

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error{code, msg}; }

#define CSC_CUDA(call)                                                                         \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) {                                                                   \
      cudaGetLastError();                                                                      \
      ::csc::fail(e_ == cudaErrorMemoryAllocation ? CSC_ERR_NOMEM : CSC_ERR_CUDA,              \
                  std::string(#call) + " failed: " + cudaGetErrorString(e_));                  \
    }                                                                                          \
  } while (0)

void set_error(const std::string& msg);

// Every C-ABI entry point runs its body through guard(): internal failures are
// exceptions, the boundary sees a status code plus csc_last_error().
template <class F>
int guard(F&& f) {
  try {
    f();
    return CSC_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return CSC_ERR_NOMEM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return CSC_ERR_CUDA;
  }
}

// ---- launch accounting / options ------------------------------------------
extern std::atomic<int64_t> g_launches;

#define CSC_LAUNCHED()                   \
  do {                                   \
    ::csc::g_launches.fetch_add(1);      \
    CSC_CUDA(cudaGetLastError());        \
  } while (0)

struct Options {
  std::atomic<int64_t> panel_width{0};    // 0 = auto (L2-sized panels)
  std::atomic<int64_t> recurrence{0};     // 0 Clenshaw (4 streams/step), 1 forward (5 streams/step)
  std::atomic<int64_t> cache_hints{1};    // streaming loads evict-first
  std::atomic<int64_t> block_threads{256};
  std::atomic<int64_t> profile{0};         // 1: events per step launch, 2: per filter span
  std::atomic<int64_t> l2_budget_pct{50}; // auto panel width: panel gather buffer <= pct% of L2
  std::atomic<int64_t> unroll{4};         // neighbour gathers in flight per lane (4 or 8)
  std::atomic<int64_t> row_order{0};      // 0 interleaved row groups, 1 contiguous ranges per warp
  std::atomic<int64_t> l2_persist_pct{0}; // >0: keep the gathered panel in a persisting L2 window
  std::atomic<int64_t> persistent{1};     // 1: step grid = resident CTAs (grid-stride); 0: one CTA per row block
  std::atomic<int64_t> cg_compact{1};     // block CG: move still-active columns into narrower panels
  std::atomic<int64_t> cg_overlap{1};     // block CG: two panels at a time (0 off, 1 auto, 2 no width token)
  std::atomic<int64_t> lean_mid{1};       // K2: lean mid-step kernel (k_cheb_mid) where it applies
  std::atomic<int64_t> fast_normalize{1}; // K3: vectorised single-panel row normalisation
  std::atomic<int64_t> h2d_overlap{1};    // filters of multi-panel pinned host blocks: per-panel uploads overlap
  std::atomic<int64_t> pdl{1};            // step kernels launched with programmatic stream serialization (their CSR prologue overlaps the previous step's drain)
  std::atomic<int64_t> l2_policy{1};      // step kernels: output panel stored evict-first (1) or write-back (0)
};
extern Options g_opt;

struct Profile {
  double ms = 0.0;
  int64_t launches = 0;
  double bytes = 0.0;
};
// Non-blocking kernel profiling: a launch is bracketed by two pooled events
// and its algorithmic bytes are recorded; csc_profile_read resolves them.
void profile_begin(cudaStream_t s, cudaEvent_t* e0);
void profile_end(cudaStream_t s, cudaEvent_t e0, double bytes, int64_t launches = 1);

// ---- device context -------------------------------------------------------
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    CSC_CUDA(cudaGetDevice(&prev));
    if (prev != dev) CSC_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

struct DeviceProps {
  int sms = 0;
  int l2_bytes = 0;
  int max_persist = 0;  // cudaDevAttrMaxPersistingL2CacheSize
  int max_window = 0;   // cudaDevAttrMaxAccessPolicyWindowSize
};
// Persisting-L2 set-aside (bytes) configured on `dev` for the current option; 0 if off/unsupported.
size_t persist_bytes(int dev);
const DeviceProps& device_props(int dev);
void ensure_pool(int dev);  // keep freed stream-ordered memory cached

// Stream-ordered scratch allocation, freed on the same stream at scope exit.
// Synchronise the current device and release the memory its stream-ordered pools cache
// (the default pool and the side pool) back to the driver.  Used when an allocation fails.
void trim_pools();

class Scratch {
 public:
  Scratch() = default;
  Scratch(size_t bytes, cudaStream_t s) { alloc(bytes, s); }
  // from a specific memory pool (e.g. side_pool: work on a side stream that must not
  // share freed blocks -- and thereby stream dependencies -- with the filter's scratch)
  Scratch(size_t bytes, cudaStream_t s, cudaMemPool_t pool) { alloc(bytes, s, pool); }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch() { release(); }
  void alloc(size_t bytes, cudaStream_t s, cudaMemPool_t pool = nullptr) {
    release();
    s_ = s;
    if (bytes == 0) bytes = 16;
    cudaError_t e = pool ? cudaMallocFromPoolAsync(&p_, bytes, pool, s) : cudaMallocAsync(&p_, bytes, s);
    if (e == cudaErrorMemoryAllocation) {  // hand the pools' cached free blocks back, retry once
      cudaGetLastError();
      trim_pools();
      e = pool ? cudaMallocFromPoolAsync(&p_, bytes, pool, s) : cudaMallocAsync(&p_, bytes, s);
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      p_ = nullptr;
      fail(e == cudaErrorMemoryAllocation ? CSC_ERR_NOMEM : CSC_ERR_CUDA,
           std::string("cudaMallocAsync(&p_, bytes, s) failed: ") + cudaGetErrorString(e));
    }
    bytes_ = bytes;
  }
  void release() {
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p_);
  }
  void* get() const { return p_; }
  size_t bytes() const { return bytes_; }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
  cudaStream_t s_ = nullptr;
};

// numpy Generator(PCG64).standard_exponential draws (bit-exact; npzig.cu) into
// device memory; returns the raw uint64 consumed.
int64_t numpy_exponentials(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t count,
                           double* out, cudaStream_t s);

// A second stream-ordered pool per device (never trimmed) for work that runs on a
// side stream concurrently with filters (the parity RNG's scratch).
cudaMemPool_t side_pool(int dev);

// Host or device?  Device pointers must belong to `device`.
bool is_device_ptr(const void* p, int device);

inline size_t dtype_size(int dt) {
  if (dt == CSC_F64) return 8;
  if (dt == CSC_F32) return 4;
  fail(CSC_ERR_INVALID, "unknown dtype " + std::to_string(dt));
}

// Copy n rows of `cols` elements between row-major buffers with leading dims
// dld/sld.  Dense blocks go as one flat copy (a 2D copy with 10^6 short rows
// runs far below link speed).
inline void copy_rows(void* dst, int64_t dld, const void* src, int64_t sld, int64_t n, int64_t cols, size_t es,
                      cudaMemcpyKind kind, cudaStream_t s) {
  if (n <= 0 || cols <= 0) return;
  if (dld == cols && sld == cols) {
    CSC_CUDA(cudaMemcpyAsync(dst, src, es * n * cols, kind, s));
  } else {
    CSC_CUDA(cudaMemcpy2DAsync(dst, es * dld, src, es * sld, es * cols, n, kind, s));
  }
}

// A device copy of a (possibly host) input buffer; passes device pointers through.
class DeviceView {
 public:
  DeviceView(const void* p, size_t bytes, int device, cudaStream_t s) {
    if (p == nullptr) return;
    if (is_device_ptr(p, device)) {
      ptr_ = p;
    } else {
      buf_.alloc(bytes, s);
      CSC_CUDA(cudaMemcpyAsync(buf_.get(), p, bytes, cudaMemcpyHostToDevice, s));
      ptr_ = buf_.get();
    }
  }
  template <class T>
  const T* as() const {
    return static_cast<const T*>(ptr_);
  }

 private:
  const void* ptr_ = nullptr;
  Scratch buf_;
};

// Output that may live on the host: kernels write to `dev()`, finish() copies back.
class DeviceOut {
 public:
  DeviceOut(void* p, size_t bytes, int device, cudaStream_t s) : host_(p), bytes_(bytes), s_(s) {
    if (p == nullptr) return;
    if (is_device_ptr(p, device)) {
      dev_ = p;
      host_ = nullptr;
    } else {
      buf_.alloc(bytes, s);
      dev_ = buf_.get();
    }
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(dev_);
  }
  bool on_host() const { return host_ != nullptr; }
  void finish() {
    if (host_) CSC_CUDA(cudaMemcpyAsync(host_, dev_, bytes_, cudaMemcpyDeviceToHost, s_));
  }

 private:
  void* host_ = nullptr;
  void* dev_ = nullptr;
  size_t bytes_ = 0;
  cudaStream_t s_ = nullptr;
  Scratch buf_;
};

}  // namespace csc

// The opaque handle of the header (global namespace, declared in csc_b200.h).
struct csc_graph {
  int64_t n = 0;
  int64_t nnz = 0;
  int dtype = CSC_F64;  // compute dtype of the normalized operator
  int device = 0;
  int32_t* indptr = nullptr;   // [n+1]
  int32_t* indices = nullptr;  // [nnz], strictly increasing per row
  double* weights = nullptr;   // [nnz] original W (fp64), for export
  void* wv = nullptr;          // [nnz] W in the compute dtype; NULL when every weight is 1 (unit graph)
  void* rs = nullptr;          // [2n] per-row (d^-1/2, d^1/2) in the compute dtype (0, 0 where d == 0)
  double* degrees = nullptr;   // [n] row sums
  double* dis = nullptr;       // [n] d^-1/2 (0 where d == 0)
  bool unit = false;
  int64_t n_global = 0;   // columns / global nodes (== n unless row-sharded)
  int64_t row_begin = 0;  // first global row held (row-sharded operators)
  // row shards (rows.cu): the gather panel holds shard_ranks slots of shard_R rows (rank q's
  // rows at q * shard_R), and `indices` are panel rows, not node ids.  Replicated: 0 / 0.
  int shard_ranks = 0;
  int shard_rank = 0;
  int64_t shard_R = 0;
  int64_t gather_rows = 0;  // rows of the panel a step gathers from (n, or shard_ranks * shard_R)
};

namespace csc {
// graph.cu: allocate + normalize from device-resident canonical CSR arrays
// (takes ownership of indptr/indices/weights).
csc_graph* graph_from_device_csr(int64_t n, int64_t nnz, int32_t* indptr, int32_t* indices, double* weights,
                                 int dtype, int device, cudaStream_t s);
void graph_free(csc_graph* g);
}  // namespace csc
