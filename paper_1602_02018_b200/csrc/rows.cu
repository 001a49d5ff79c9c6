// Row-sharded operator (BASELINE config 5): each rank owns a
// contiguous range of R = ceil(N / ranks) rows of the CSR (global column
// indices); every Chebyshev step reads neighbour rows from the full block, so
// the step's local output is all-gathered over NCCL (NVLink/NVSwitch) into a
// full N x pw gather panel before the next step.  Row norms and row-local
// epilogues need no extra exchange (a rank holds all columns of its rows); the
// eigencount partial is summed by the caller.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2, whichever copy the process
// already has, e.g. torch's), so the library itself has no link-time NCCL
// dependency and loads on machines without it.
//
// Peer transport (csc_peers, csc_cheb_filter_rows_peers): the same recurrence with
// the all-gather fused into the step kernel.  Every rank holds two full gather
// panels (ping-pong) and a flag array in one CUDA-IPC-exported allocation that all
// ranks map; step s gathers from panel s % 2 and its epilogue stores each finished
// row, besides the local copy, into panel (s + 1) % 2 of every rank over NVLink, so
// the exchange overlaps the SpMM row by row.  A one-block barrier kernel (system-
// scope release/acquire flags, monotonically increasing epoch) separates steps:
// after it every rank's rows of step s have landed everywhere (the gather source of
// step s + 1) and every rank has finished reading panel s % 2 (overwritten by step
// s + 1), so one barrier per step suffices.  With one rank it degenerates to the
// replicated path, which is how it is tested on a single GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "filter.cuh"

namespace csc {
csc_graph* graph_create_impl(int64_t num_nodes, int64_t ncols, int64_t nnz, const int32_t* indptr,
                             const int32_t* indices, const double* weights, int dtype, int device, cudaStream_t s);
namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load NCCL: ") + dlerror();
      return;
    }
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.allGather) fail(CSC_ERR_CUDA, err.empty() ? "NCCL symbols missing" : err);
  return api;
}

#define CSC_NCCL(call)                                                                         \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      ::csc::fail(CSC_ERR_CUDA, std::string(#call) + " failed: " + nccl().errorString(r_));    \
  } while (0)

}  // namespace
}  // namespace csc

struct csc_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1;
  int rank = 0;
  int device = 0;
};

// Layout of each rank's allocation: [panel 0 | panel 1 | flags (nranks x uint64)].
struct csc_peers {
  static constexpr int kMax = 32;
  int nranks = 1;
  int rank = 0;
  int device = 0;
  size_t panel_bytes = 0;      // one gather panel (R * nranks rows of the widest panel)
  size_t stride = 0;           // panel_bytes rounded up to 4 KB
  void* base = nullptr;        // own allocation
  void* peer[kMax] = {};       // every rank's allocation in this address space (own included)
  bool opened[kMax] = {};      // IPC-opened (to close on destroy)
  void** dptrs = nullptr;      // device: [2][nranks] panel pointers + [nranks] flag pointers
  uint64_t epoch = 0;
  bool ready = false;
  // optional host-side barrier (csc_peers_set_host_barrier): the step boundary becomes
  // stream synchronise + callback instead of the flag kernel, so no kernel waits on another
  // rank's kernel (ranks of different processes time-sliced on one GPU)
  csc_host_barrier_fn host_barrier = nullptr;
  void* host_barrier_ctx = nullptr;
};

namespace csc {
namespace rows_impl {

// One Clenshaw filter (the recurrence of filter_panel, filters.py:140-155) as a list of
// steps over named per-rank buffers, shared by the three exchanges below: every step but the
// last is followed by an all-gather of its output rows into the next gather panel, and the
// scaled input Xs is all-gathered before the first step (when p >= 1).
enum Buf : int { B_NONE = 0, B_X, B_XS, B_Y, B_0, B_1 };

struct PlanStep {
  double ka = 0.0, ks = 0.0, kx = 0.0;
  Buf S = B_NONE, X = B_NONE, O = B_NONE;
  bool gather = false;  // G = the current gather panel
  bool last = false;
};

std::vector<PlanStep> clenshaw_plan(const double* c, int nc) {
  const int p = nc - 1;
  std::vector<PlanStep> v;
  auto step = [&](bool G, double ka, Buf S, double ks, Buf X, double kx, Buf O, bool last) {
    PlanStep t;
    t.gather = G;
    t.ka = ka;
    t.S = S;
    t.ks = ks;
    t.X = X;
    t.kx = kx;
    t.O = O;
    t.last = last;
    v.push_back(t);
  };
  if (p == 0) {
    step(false, 0.0, B_NONE, 0.0, B_X, c[0], B_Y, true);
    return v;
  }
  if (p == 1) {
    step(true, -c[1], B_NONE, 0.0, B_X, c[0], B_Y, true);
    return v;
  }
  step(true, -2.0 * c[p], B_NONE, 0.0, B_XS, c[p - 1], B_0, false);
  if (p == 2) {
    step(true, -1.0, B_NONE, 0.0, B_X, c[0] - c[2], B_Y, true);
    return v;
  }
  step(true, -2.0, B_NONE, 0.0, B_XS, c[p - 2] - c[p], B_1, false);
  Buf prv = B_0, cur = B_1;
  for (int l = p - 3; l >= 1; --l) {  // in place: b_l overwrites b_{l+2}
    step(true, -2.0, prv, -1.0, B_XS, c[l], prv, false);
    std::swap(cur, prv);
  }
  step(true, -1.0, prv, -1.0, B_X, c[0], B_Y, true);
  return v;
}

double filter_hz(const double* c, int nc) {  // h(1): the filter on isolated nodes
  double hz = 0.0;
  for (int l = 0; l < nc; l += 2) hz += ((l / 2) % 2 ? -c[l] : c[l]);
  return hz;
}

// one rank's R x pw panels of one column panel
struct RankPanels {
  const csc_graph* g = nullptr;
  void* buf[6] = {};  // indexed by Buf
  double* part = nullptr;
  template <typename T>
  T* at(Buf b) const { return static_cast<T*>(buf[b]); }
};

template <typename T>
StepArgs plan_args(const RankPanels& rp, const PlanStep& st, const void* G, int wc, double hz, int epi) {
  StepArgs a{};
  const csc_graph* g = rp.g;
  a.indptr = g->indptr;
  a.indices = g->indices;
  a.wv = g->wv;
  a.rs = g->rs;
  a.n = g->n;  // local rows
  a.wc = wc;
  a.hz = hz;
  a.G = st.gather ? G : nullptr;
  a.ka = st.ka;
  a.S = st.S ? rp.at<T>(st.S) : nullptr;
  a.ks = st.ks;
  a.X = rp.at<T>(st.X);
  a.kx = st.kx;
  a.O = rp.at<T>(st.O);
  a.last = st.last ? 1 : 0;
  if (st.last && epi != EPI_NONE) a.part = rp.part;
  return a;
}

// NCCL: every rank runs the plan on its own stream; ncclAllGather after each step.
template <typename T>
void filter_panel_nccl(csc_comm* cm, const RankPanels& rp, const double* c, int nc, T* F, int64_t R, int pw, int wc,
                       int epi, cudaStream_t s) {
  const ncclDataType_t dt = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
  auto gather = [&](Buf b) {  // local R x pw rows -> full (nranks R) x pw panel
    CSC_NCCL(nccl().allGather(rp.at<T>(b), F, (size_t)R * pw, dt, cm->comm, s));
  };
  const double hz = filter_hz(c, nc);
  if (nc > 1) gather(B_XS);
  for (const PlanStep& st : clenshaw_plan(c, nc)) {
    launch_step<T>(rp.g, plan_args<T>(rp, st, F, wc, hz, epi), pw, st.last ? epi : EPI_NONE, s);
    if (!st.last) gather(st.O);
  }
}

// Emulated ranks (one process, one device): the shards step in lockstep on one stream and the
// all-gather is a device copy of each shard's R rows into its slot of the shared panel -- the
// multi-rank exchange without ranks that wait on one another (B200_PROFILING.md).  Same kernels,
// same per-rank arguments, same panel layout as the NCCL path.
template <typename T>
void filter_panel_group(const std::vector<RankPanels>& ranks, const double* c, int nc, T* F, int64_t R, int pw,
                        int wc, int epi, cudaStream_t s) {
  auto gather = [&](Buf b) {
    for (size_t q = 0; q < ranks.size(); ++q)
      CSC_CUDA(cudaMemcpyAsync(F + (size_t)q * R * pw, ranks[q].at<T>(b), sizeof(T) * (size_t)R * pw,
                               cudaMemcpyDeviceToDevice, s));
  };
  const double hz = filter_hz(c, nc);
  if (nc > 1) gather(B_XS);
  for (const PlanStep& st : clenshaw_plan(c, nc)) {
    for (const RankPanels& rp : ranks)
      launch_step<T>(rp.g, plan_args<T>(rp, st, F, wc, hz, epi), pw, st.last ? epi : EPI_NONE, s);
    if (!st.last) gather(st.O);
  }
}

// every rank publishes `epoch` in its slot of every rank's flag array, then waits
// until all ranks have published it in its own array (system-scope release/acquire;
// the fence orders this rank's earlier peer stores -- the preceding kernel on the
// stream -- before the release)
__global__ void k_peer_barrier(void* const* flag_ptrs, int nranks, int rank, uint64_t epoch) {
  const int q = threadIdx.x;
  if (q >= nranks) return;
  __threadfence_system();
  uint64_t* slot = static_cast<uint64_t*>(flag_ptrs[q]) + rank;
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot), "l"(epoch) : "memory");
  const uint64_t* mine = static_cast<const uint64_t*>(flag_ptrs[rank]) + q;
  uint64_t v = 0;
  const long long t0 = clock64();
  do {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
    // a peer that never arrives (died, or called with a different block) would hang the
    // GPU: after ~1 minute of cycles fail the launch instead
    if (v < epoch && clock64() - t0 > 120000000000ll) __trap();
  } while (v < epoch);
}

void peer_barrier(csc_peers* pe, cudaStream_t s) {
  ++pe->epoch;
  if (pe->host_barrier) {
    CSC_CUDA(cudaStreamSynchronize(s));  // this rank's peer stores have landed
    if (pe->host_barrier(pe->host_barrier_ctx) != 0) fail(CSC_ERR_INVALID, "host barrier callback failed");
    return;
  }
  k_peer_barrier<<<1, 32, 0, s>>>(pe->dptrs + 2 * pe->nranks, pe->nranks, pe->rank, pe->epoch);
  CSC_LAUNCHED();
}

// this rank's R x pw rows -> rows [rank R, rank R + R) of panel `which` on every rank
template <typename T>
void peer_put(csc_peers* pe, int which, const T* local, int64_t R, int pw, cudaStream_t s) {
  const size_t bytes = sizeof(T) * (size_t)R * pw;
  const size_t off = (size_t)which * pe->stride + sizeof(T) * (size_t)pe->rank * R * pw;
  for (int q = 0; q < pe->nranks; ++q)
    CSC_CUDA(cudaMemcpyAsync(static_cast<char*>(pe->peer[q]) + off, local, bytes, cudaMemcpyDeviceToDevice, s));
}

// Peer transport: the all-gather fused into each non-last step (its epilogue stores the
// step's rows into every rank's other panel), a flag barrier after it.
template <typename T>
void filter_panel_peers(csc_peers* pe, const RankPanels& rp, const double* c, int nc, int64_t R, int pw, int wc,
                        int epi, cudaStream_t s) {
  const double hz = filter_hz(c, nc);
  auto panel = [&](int which) {
    return static_cast<T*>(static_cast<void*>(static_cast<char*>(pe->base) + (size_t)which * pe->stride));
  };
  int cur_panel = 0;  // gather source of the next step
  if (nc > 1) {
    peer_barrier(pe, s);  // every rank is done with the previous call's panels
    peer_put<T>(pe, 0, rp.at<T>(B_XS), R, pw, s);
    peer_barrier(pe, s);
  }
  for (const PlanStep& st : clenshaw_plan(c, nc)) {
    StepArgs a = plan_args<T>(rp, st, panel(cur_panel), wc, hz, epi);
    if (st.last) {
      launch_step<T>(rp.g, a, pw, epi, s);
      continue;
    }
    a.peers = pe->dptrs + (size_t)(1 - cur_panel) * pe->nranks;
    a.npeers = pe->nranks;
    a.peer_row0 = (int64_t)pe->rank * R;
    launch_step<T>(rp.g, a, pw, EPI_NONE, s);
    peer_barrier(pe, s);
    cur_panel = 1 - cur_panel;
  }
}

template <typename Ti, typename To>
__global__ void k_pack_rows(const Ti* __restrict__ src, int64_t ld, int c0, int wc, int pw, int64_t n,
                            const double* __restrict__ dis, To* __restrict__ dst, To* __restrict__ scaled) {
  const int64_t total = n * pw;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / pw;
    const int c = (int)(t - row * pw);
    const double v = c < wc ? (double)src[row * ld + c0 + c] : 0.0;
    dst[t] = static_cast<To>(v);
    scaled[t] = static_cast<To>(v * dis[row]);
  }
}

template <typename Ti, typename To>
__global__ void k_unpack_rows(const Ti* __restrict__ src, int c0, int wc, int pw, int64_t n, To* __restrict__ dst,
                              int64_t ld, const double* __restrict__ rowsq_part, double* __restrict__ rowsq) {
  const int64_t total = n * wc;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / wc;
    const int c = (int)(t - row * wc);
    dst[row * ld + c0 + c] = static_cast<To>(src[row * pw + c]);
    if (rowsq && c == 0) rowsq[row] += rowsq_part[row];
  }
}

// Per-rank scratch of one filter call: packed input (symmetric and scaled), output and the
// two recurrence panels, R x max_pw each, zeroed so the pad rows a rank sends are zeros.
struct RankScratch {
  Scratch x, xs, y, b0, b1, part;
  RankScratch(size_t panel_bytes, size_t part_bytes, cudaStream_t s)
      : x(panel_bytes, s), xs(panel_bytes, s), y(panel_bytes, s), b0(panel_bytes, s), b1(panel_bytes, s),
        part(part_bytes, s) {
    for (Scratch* b : {&x, &xs, &y, &b0, &b1}) CSC_CUDA(cudaMemsetAsync(b->get(), 0, b->bytes(), s));
  }
};

// One rank's call (NCCL or peers) or all emulated ranks' calls (group): pack, run every column
// panel's plan, unpack; mode 0 Y = h(L) X, 1 sum of squares per rank, 2 Y + row sums of squares.
template <typename T, typename Tio>
void run_rows(const std::vector<const csc_graph*>& gs, csc_comm* cm, csc_peers* pe, const double* coeffs, int nc,
              const std::vector<const Tio*>& X, const std::vector<int64_t>& ldx, const std::vector<Tio*>& Y,
              const std::vector<int64_t>& ldy, int ncols, int mode, const std::vector<double*>& outs,
              cudaStream_t s) {
  const csc_graph* g0 = gs[0];
  const int nranks = g0->shard_ranks;
  const int64_t R = g0->shard_R;
  int64_t nnz_all = 0;
  for (const csc_graph* g : gs) nnz_all += g->nnz;
  if (gs.size() == 1) nnz_all = g0->nnz * nranks;  // one rank of many: estimate
  const PanelPlan pp = plan_panels(g0->gather_rows, ncols, g0->dtype, g0->device, nnz_all);
  if (pe && sizeof(T) * (size_t)R * nranks * pp.max_pw > pe->panel_bytes)
    fail(CSC_ERR_INVALID, "peer panels too small for this block (see csc_panel_row_bytes)");
  const int cap = step_grid_cap(g0->device);
  const size_t pbytes = sizeof(T) * (size_t)R * pp.max_pw;
  std::vector<std::unique_ptr<RankScratch>> sc;
  for (const csc_graph* g : gs)
    sc.emplace_back(new RankScratch(pbytes, sizeof(double) * std::max<int64_t>((int64_t)cap * pp.np, g->n), s));
  Scratch full(pe ? 16 : sizeof(T) * (size_t)R * nranks * pp.max_pw, s);
  for (size_t q = 0; q < gs.size(); ++q) {
    if (mode == 1) CSC_CUDA(cudaMemsetAsync(sc[q]->part.get(), 0, sc[q]->part.bytes(), s));
    if (mode == 2) CSC_CUDA(cudaMemsetAsync(outs[q], 0, sizeof(double) * gs[q]->n, s));
  }
  const int epi = mode == 1 ? EPI_SUMSQ : (mode == 2 ? EPI_ROWSQ : EPI_NONE);
  for (int j = 0; j < pp.np; ++j) {
    const int pw = pp.pw[j], wc = pp.wc[j];
    std::vector<RankPanels> rps(gs.size());
    for (size_t q = 0; q < gs.size(); ++q) {
      const csc_graph* g = gs[q];
      const int64_t n = g->n;
      RankScratch& r = *sc[q];
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n * pw + 255) / 256, 148 * 64));
      k_pack_rows<Tio, T><<<grid, 256, 0, s>>>(X[q], ldx[q], pp.c0[j], wc, pw, n, g->dis, r.x.as<T>(), r.xs.as<T>());
      CSC_LAUNCHED();
      RankPanels& rp = rps[q];
      rp.g = g;
      rp.buf[B_X] = r.x.get();
      rp.buf[B_XS] = r.xs.get();
      rp.buf[B_Y] = mode == 1 ? nullptr : r.y.get();  // SUMSQ: the partials only
      rp.buf[B_0] = r.b0.get();
      rp.buf[B_1] = r.b1.get();
      rp.part = mode == 1 ? r.part.as<double>() + (size_t)cap * j : (mode == 2 ? r.part.as<double>() : nullptr);
    }
    if (pe)
      filter_panel_peers<T>(pe, rps[0], coeffs, nc, R, pw, wc, epi, s);
    else if (cm)
      filter_panel_nccl<T>(cm, rps[0], coeffs, nc, full.as<T>(), R, pw, wc, epi, s);
    else
      filter_panel_group<T>(rps, coeffs, nc, full.as<T>(), R, pw, wc, epi, s);
    if (mode == 0 || mode == 2) {
      for (size_t q = 0; q < gs.size(); ++q) {
        const int64_t n = gs[q]->n;
        k_unpack_rows<T, Tio><<<(int)std::max<int64_t>(1, std::min<int64_t>((n * wc + 255) / 256, 148 * 64)), 256,
                                0, s>>>(sc[q]->y.as<T>(), pp.c0[j], wc, pw, n, Y[q], ldy[q], sc[q]->part.as<double>(),
                                        mode == 2 ? outs[q] : nullptr);
        CSC_LAUNCHED();
      }
    }
  }
  if (mode == 1)
    for (size_t q = 0; q < gs.size(); ++q)
      reduce_sum(sc[q]->part.as<double>(), (int64_t)cap * pp.np, outs[q], s);
}

}  // namespace rows_impl
}  // namespace csc

using namespace csc;
using namespace csc::rows_impl;

extern "C" {

int csc_comm_unique_id(uint8_t* out) {
  return guard([&] {
    if (!out) fail(CSC_ERR_INVALID, "out is NULL");
    ncclUniqueId id;
    CSC_NCCL(nccl().getUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  });
}

int csc_comm_create(const uint8_t* unique_id, int nranks, int rank, int device, csc_comm** out) {
  return guard([&] {
    if (!unique_id || !out) fail(CSC_ERR_INVALID, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(CSC_ERR_INVALID, "bad rank / nranks");
    DeviceGuard dg(device);
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    csc_comm* c = new csc_comm();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclResult_t r = nccl().commInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      delete c;
      fail(CSC_ERR_CUDA, std::string("ncclCommInitRank failed: ") + nccl().errorString(r));
    }
    *out = c;
  });
}

int csc_comm_destroy(csc_comm* c) {
  return guard([&] {
    if (!c) return;
    if (c->comm) nccl().commDestroy(c->comm);
    delete c;
  });
}

int csc_graph_create_row_shard(int64_t num_nodes, int nranks, int rank, const int64_t* row_starts, int64_t nnz,
                               const int32_t* indptr, const int32_t* indices, const double* weights, int dtype,
                               int device, void* stream, csc_graph** out) {
  return guard([&] {
    if (!out || !indptr || !row_starts) fail(CSC_ERR_INVALID, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(CSC_ERR_INVALID, "bad rank / nranks");
    if (dtype != CSC_F64 && dtype != CSC_F32) fail(CSC_ERR_INVALID, "dtype must be CSC_F64 or CSC_F32");
    if (row_starts[0] != 0 || row_starts[nranks] != num_nodes) fail(CSC_ERR_INVALID, "row_starts must span [0, N]");
    int64_t R = 0;
    for (int q = 0; q < nranks; ++q) {
      if (row_starts[q + 1] < row_starts[q]) fail(CSC_ERR_INVALID, "row_starts must be non-decreasing");
      R = std::max<int64_t>(R, row_starts[q + 1] - row_starts[q]);
    }
    if (nnz > 0 && !indices) fail(CSC_ERR_INVALID, "indices is NULL");
    const int64_t n = row_starts[rank + 1] - row_starts[rank];
    // node id -> gather-panel row: rank q's rows occupy slots [q R, q R + rows_q) (monotone, so
    // every row's columns stay sorted)
    std::vector<int32_t> panel_idx((size_t)std::max<int64_t>(nnz, 1));
    if ((int64_t)nranks * R >= (int64_t(1) << 31)) fail(CSC_ERR_INVALID, "gather panel rows exceed int32");
    for (int64_t e = 0; e < nnz; ++e) {
      const int64_t j = indices[e];
      if (j < 0 || j >= num_nodes) fail(CSC_ERR_GRAPH, "column index out of range");
      const int64_t q = std::upper_bound(row_starts, row_starts + nranks + 1, j) - row_starts - 1;
      panel_idx[e] = (int32_t)(q * R + (j - row_starts[q]));
    }
    csc_graph* g = graph_create_impl(n, (int64_t)nranks * R, nnz, indptr, panel_idx.data(), weights, dtype, device,
                                     static_cast<cudaStream_t>(stream));
    g->n_global = num_nodes;
    g->row_begin = row_starts[rank];
    g->shard_ranks = nranks;
    g->shard_rank = rank;
    g->shard_R = R;
    g->gather_rows = (int64_t)nranks * R;
    *out = g;
  });
}

}  // extern "C"

namespace {
// shards: one (NCCL / peers: this rank's) or all (group emulation) row shards of one graph
void filter_rows_entry(const std::vector<const csc_graph*>& gs, csc_comm* comm, csc_peers* pe, const double* coeffs,
                       int ncoeffs, const void* const* X, const int64_t* ldx, void* const* Y, const int64_t* ldy,
                       int ncols, int io_dtype, int mode, double* const* out, void* stream) {
  if (gs.empty() || !gs[0]) fail(CSC_ERR_INVALID, "graph is NULL");
  if (ncoeffs < 1 || !coeffs) fail(CSC_ERR_INVALID, "need coefficients");
  if (mode < 0 || mode > 2) fail(CSC_ERR_INVALID, "mode must be 0 (filter), 1 (sum of squares), 2 (row sums)");
  if (io_dtype != CSC_F64 && io_dtype != CSC_F32) fail(CSC_ERR_INVALID, "io_dtype must be CSC_F64 or CSC_F32");
  const csc_graph* g0 = gs[0];
  if (g0->shard_ranks < 1) fail(CSC_ERR_INVALID, "not a row shard (csc_graph_create_row_shard)");
  const int nranks = pe ? pe->nranks : (comm ? comm->nranks : (int)gs.size());
  if (g0->shard_ranks != nranks) fail(CSC_ERR_INVALID, "shard count and transport rank count differ");
  if (!pe && !comm && (int)gs.size() != nranks) fail(CSC_ERR_INVALID, "group needs every shard");
  const int my_rank = pe ? pe->rank : (comm ? comm->rank : -1);
  for (size_t q = 0; q < gs.size(); ++q) {
    const csc_graph* g = gs[q];
    if (!g) fail(CSC_ERR_INVALID, "graph is NULL");
    if (g->device != g0->device || g->dtype != g0->dtype || g->shard_ranks != nranks || g->shard_R != g0->shard_R ||
        g->n_global != g0->n_global)
      fail(CSC_ERR_INVALID, "shards of different graphs / devices / dtypes");
    if (g->shard_rank != (my_rank >= 0 ? my_rank : (int)q)) fail(CSC_ERR_INVALID, "shard / rank mismatch");
    // (a shard without rows may pass NULL blocks)
    if (ncols < 1 || ldx[q] < ncols || (mode != 1 && (ldy[q] < ncols || (!Y[q] && g->n > 0))))
      fail(CSC_ERR_INVALID, "bad block");
    if (mode != 0 && !out[q]) fail(CSC_ERR_INVALID, "out is NULL");
    if ((g->n > 0 && !is_device_ptr(X[q], g->device)) || (mode != 1 && g->n > 0 && !is_device_ptr(Y[q], g->device)))
      fail(CSC_ERR_INVALID, "row-sharded blocks must be device buffers");
  }
  const int dev = g0->device;
  if ((pe && pe->device != dev) || (comm && comm->device != dev))
    fail(CSC_ERR_INVALID, "transport and graph on different devices");
  if (pe && !pe->ready) fail(CSC_ERR_INVALID, "peer transport not attached to every rank (csc_peers_attach)");
  DeviceGuard dg(dev);
  ensure_pool(dev);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<std::unique_ptr<DeviceOut>> os;
  std::vector<double*> douts(gs.size(), nullptr);
  for (size_t q = 0; q < gs.size(); ++q)
    if (mode != 0) {
      os.emplace_back(new DeviceOut(out[q], sizeof(double) * (mode == 2 ? std::max<int64_t>(gs[q]->n, 1) : 1), dev, s));
      douts[q] = os.back()->as<double>();
    }
  std::vector<int64_t> lx(ldx, ldx + gs.size()), ly(gs.size(), 0);
  for (size_t q = 0; q < gs.size(); ++q) ly[q] = mode == 1 ? 0 : ldy[q];
  auto go = [&](auto tag_t, auto tag_io) {
    using T = decltype(tag_t);
    using Tio = decltype(tag_io);
    std::vector<const Tio*> xs(gs.size());
    std::vector<Tio*> ys(gs.size(), nullptr);
    for (size_t q = 0; q < gs.size(); ++q) {
      xs[q] = static_cast<const Tio*>(X[q]);
      if (mode != 1) ys[q] = static_cast<Tio*>(Y[q]);
    }
    run_rows<T, Tio>(gs, comm, pe, coeffs, ncoeffs, xs, lx, ys, ly, ncols, mode, douts, s);
  };
  if (g0->dtype == CSC_F64 && io_dtype == CSC_F64) go(double(), double());
  else if (g0->dtype == CSC_F32 && io_dtype == CSC_F32) go(float(), float());
  else if (g0->dtype == CSC_F32) go(float(), double());
  else go(double(), float());
  for (auto& o : os) o->finish();
  CSC_CUDA(cudaStreamSynchronize(s));
}
}  // namespace

extern "C" {

int csc_cheb_filter_rows(const csc_graph* g, csc_comm* comm, const double* coeffs, int ncoeffs, const void* X,
                         int64_t ldx, void* Y, int64_t ldy, int ncols, int io_dtype, int mode, double* out,
                         void* stream) {
  return guard([&] {
    if (!comm) fail(CSC_ERR_INVALID, "comm is NULL");
    filter_rows_entry({g}, comm, nullptr, coeffs, ncoeffs, &X, &ldx, &Y, &ldy, ncols, io_dtype, mode, &out, stream);
  });
}

int csc_cheb_filter_rows_peers(const csc_graph* g, csc_peers* peers, const double* coeffs, int ncoeffs,
                               const void* X, int64_t ldx, void* Y, int64_t ldy, int ncols, int io_dtype, int mode,
                               double* out, void* stream) {
  return guard([&] {
    if (!peers) fail(CSC_ERR_INVALID, "peers is NULL");
    filter_rows_entry({g}, nullptr, peers, coeffs, ncoeffs, &X, &ldx, &Y, &ldy, ncols, io_dtype, mode, &out, stream);
  });
}

int csc_cheb_filter_rows_group(const csc_graph* const* shards, int nshards, const double* coeffs, int ncoeffs,
                               const void* const* X, const int64_t* ldx, void* const* Y, const int64_t* ldy, int ncols,
                               int io_dtype, int mode, double* const* out, void* stream) {
  return guard([&] {
    if (!shards || nshards < 1 || !X || !ldx || (mode != 1 && (!Y || !ldy)) || (mode != 0 && !out))
      fail(CSC_ERR_INVALID, "NULL argument");
    std::vector<const csc_graph*> gs(shards, shards + nshards);
    std::vector<void*> ys(nshards, nullptr);
    std::vector<int64_t> lys(nshards, 0);
    std::vector<double*> outs(nshards, nullptr);
    for (int q = 0; q < nshards; ++q) {
      if (mode != 1) {
        ys[q] = Y[q];
        lys[q] = ldy[q];
      }
      if (mode != 0) outs[q] = out[q];
    }
    filter_rows_entry(gs, nullptr, nullptr, coeffs, ncoeffs, X, ldx, ys.data(), lys.data(), ncols, io_dtype, mode,
                      outs.data(), stream);
  });
}

int csc_panel_row_bytes(int64_t num_nodes, int ncols, int dtype, int device, int64_t nnz, int64_t* out) {
  return guard([&] {
    if (!out || num_nodes < 1 || ncols < 1) fail(CSC_ERR_INVALID, "bad arguments");
    const PanelPlan pp = plan_panels(num_nodes, ncols, dtype, device, nnz);
    *out = (int64_t)pp.max_pw * (int64_t)dtype_size(dtype);
  });
}

int csc_peers_create(int nranks, int rank, int device, size_t panel_bytes, csc_peers** out) {
  return guard([&] {
    if (!out) fail(CSC_ERR_INVALID, "out is NULL");
    if (nranks < 1 || nranks > csc_peers::kMax || rank < 0 || rank >= nranks)
      fail(CSC_ERR_INVALID, "bad rank / nranks (at most 32 ranks)");
    if (panel_bytes == 0) fail(CSC_ERR_INVALID, "panel_bytes must be > 0");
    DeviceGuard dg(device);
    auto* pe = new csc_peers();
    pe->nranks = nranks;
    pe->rank = rank;
    pe->device = device;
    pe->panel_bytes = panel_bytes;
    pe->stride = (panel_bytes + 4095) / 4096 * 4096;
    const size_t total = 2 * pe->stride + 4096;
    cudaError_t e = cudaMalloc(&pe->base, total);  // plain cudaMalloc: IPC-exportable
    if (e != cudaSuccess) {
      delete pe;
      CSC_CUDA(e);
    }
    CSC_CUDA(cudaMemset(pe->base, 0, total));  // flags start at epoch 0
    CSC_CUDA(cudaMalloc(reinterpret_cast<void**>(&pe->dptrs), sizeof(void*) * 3 * nranks));
    pe->peer[rank] = pe->base;
    CSC_CUDA(cudaDeviceSynchronize());
    if (nranks == 1) {
      void* h[3] = {pe->base, static_cast<char*>(pe->base) + pe->stride, static_cast<char*>(pe->base) + 2 * pe->stride};
      CSC_CUDA(cudaMemcpy(pe->dptrs, h, sizeof(h), cudaMemcpyHostToDevice));
      pe->ready = true;
    }
    *out = pe;
  });
}

int csc_peers_handle(const csc_peers* pe, uint8_t* out) {
  return guard([&] {
    if (!pe || !out) fail(CSC_ERR_INVALID, "NULL argument");
    DeviceGuard dg(pe->device);
    cudaIpcMemHandle_t h;
    CSC_CUDA(cudaIpcGetMemHandle(&h, pe->base));
    std::memcpy(out, &h, sizeof(h));
  });
}

int csc_peers_attach(csc_peers* pe, int peer_rank, const uint8_t* handle) {
  return guard([&] {
    if (!pe || !handle) fail(CSC_ERR_INVALID, "NULL argument");
    if (peer_rank < 0 || peer_rank >= pe->nranks) fail(CSC_ERR_INVALID, "peer rank out of range");
    DeviceGuard dg(pe->device);
    if (peer_rank != pe->rank && !pe->peer[peer_rank]) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handle, sizeof(h));
      CSC_CUDA(cudaIpcOpenMemHandle(&pe->peer[peer_rank], h, cudaIpcMemLazyEnablePeerAccess));
      pe->opened[peer_rank] = true;
    }
    bool all = true;
    for (int q = 0; q < pe->nranks; ++q) all = all && pe->peer[q] != nullptr;
    if (all) {  // device pointer table: panel 0 of every rank, panel 1 of every rank, flags of every rank
      std::vector<void*> h(3 * (size_t)pe->nranks);
      for (int q = 0; q < pe->nranks; ++q) {
        h[q] = pe->peer[q];
        h[pe->nranks + q] = static_cast<char*>(pe->peer[q]) + pe->stride;
        h[2 * pe->nranks + q] = static_cast<char*>(pe->peer[q]) + 2 * pe->stride;
      }
      CSC_CUDA(cudaMemcpy(pe->dptrs, h.data(), sizeof(void*) * h.size(), cudaMemcpyHostToDevice));
      pe->ready = true;
    }
  });
}

int csc_peers_set_host_barrier(csc_peers* pe, csc_host_barrier_fn fn, void* ctx) {
  return guard([&] {
    if (!pe) fail(CSC_ERR_INVALID, "NULL argument");
    pe->host_barrier = fn;
    pe->host_barrier_ctx = ctx;
  });
}

int csc_peers_destroy(csc_peers* pe) {
  return guard([&] {
    if (!pe) return;
    DeviceGuard dg(pe->device);
    cudaDeviceSynchronize();
    for (int q = 0; q < pe->nranks; ++q)
      if (pe->opened[q]) cudaIpcCloseMemHandle(pe->peer[q]);
    if (pe->dptrs) cudaFree(pe->dptrs);
    if (pe->base) cudaFree(pe->base);
    delete pe;
  });
}

}  // extern "C"
