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
};

namespace csc {
namespace rows_impl {

// per-rank row range of an N-row block over `nranks` (equal counts; the last rank may be short)
int64_t rows_per_rank(int64_t n, int nranks) { return (n + nranks - 1) / nranks; }

template <typename T>
void filter_panel_rows(const csc_graph* g, csc_comm* cm, const double* c, int nc, const T* X, const T* Xs, T* Y,
                       T* B0, T* B1, T* F, int64_t R, int pw, int wc, int epi, double* part, cudaStream_t s) {
  const int p = nc - 1;
  double hz = 0.0;
  for (int l = 0; l < nc; l += 2) hz += ((l / 2) % 2 ? -c[l] : c[l]);
  const ncclDataType_t dt = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
  auto gather = [&](const T* local) {  // local R x pw rows -> full (nranks R) x pw panel
    CSC_NCCL(nccl().allGather(local, F, (size_t)R * pw, dt, cm->comm, s));
  };
  auto base = [&]() {
    StepArgs a{};
    a.indptr = g->indptr;
    a.indices = g->indices;
    a.wv = g->wv;
    a.rs = g->rs;
    a.n = g->n;  // local rows
    a.wc = wc;
    a.hz = hz;
    return a;
  };
  auto run = [&](StepArgs a, int e) {
    if (e != EPI_NONE) {
      a.part = part;
      a.last = 1;
    }
    launch_step<T>(g, a, pw, e, s);
  };
  if (p == 0) {
    StepArgs a = base();
    a.X = X;
    a.kx = c[0];
    a.O = Y;
    a.last = 1;
    run(a, epi);
    return;
  }
  gather(Xs);
  if (p == 1) {
    StepArgs a = base();
    a.G = F;
    a.ka = -c[1];
    a.X = X;
    a.kx = c[0];
    a.O = Y;
    a.last = 1;
    run(a, epi);
    return;
  }
  StepArgs a = base();
  a.G = F;
  a.ka = -2.0 * c[p];
  a.X = Xs;
  a.kx = c[p - 1];
  a.O = B0;
  run(a, EPI_NONE);
  gather(B0);
  if (p == 2) {
    StepArgs f = base();
    f.G = F;
    f.ka = -1.0;
    f.X = X;
    f.kx = c[0] - c[2];
    f.O = Y;
    f.last = 1;
    run(f, epi);
    return;
  }
  StepArgs b = base();
  b.G = F;
  b.ka = -2.0;
  b.X = Xs;
  b.kx = c[p - 2] - c[p];
  b.O = B1;
  run(b, EPI_NONE);
  gather(B1);
  T* cur = B1;
  T* prv = B0;
  for (int l = p - 3; l >= 1; --l) {
    StepArgs m = base();
    m.G = F;
    m.ka = -2.0;
    m.S = prv;
    m.ks = -1.0;
    m.X = Xs;
    m.kx = c[l];
    m.O = prv;
    run(m, EPI_NONE);
    gather(prv);
    std::swap(cur, prv);
  }
  StepArgs f = base();
  f.G = F;
  f.ka = -1.0;
  f.S = prv;
  f.ks = -1.0;
  f.X = X;
  f.kx = c[0];
  f.O = Y;
  f.last = 1;
  run(f, epi);
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

template <typename T>
void filter_panel_peers(const csc_graph* g, csc_peers* pe, const double* c, int nc, const T* X, const T* Xs, T* Y,
                        T* B0, T* B1, int64_t R, int pw, int wc, int epi, double* part, cudaStream_t s) {
  const int p = nc - 1;
  double hz = 0.0;
  for (int l = 0; l < nc; l += 2) hz += ((l / 2) % 2 ? -c[l] : c[l]);
  int cur_panel = 0;  // gather source of the next step
  auto panel = [&](int which) { return static_cast<T*>(static_cast<void*>(static_cast<char*>(pe->base) +
                                                                          (size_t)which * pe->stride)); };
  auto base = [&]() {
    StepArgs a{};
    a.indptr = g->indptr;
    a.indices = g->indices;
    a.wv = g->wv;
    a.rs = g->rs;
    a.n = g->n;  // local rows
    a.wc = wc;
    a.hz = hz;
    return a;
  };
  // a mid step: gather panel cur, O = local rows, fused stores into every rank's other panel
  auto mid = [&](StepArgs a) {
    a.G = panel(cur_panel);
    a.peers = pe->dptrs + (size_t)(1 - cur_panel) * pe->nranks;
    a.npeers = pe->nranks;
    a.peer_row0 = (int64_t)pe->rank * R;
    launch_step<T>(g, a, pw, EPI_NONE, s);
    peer_barrier(pe, s);
    cur_panel = 1 - cur_panel;
  };
  auto last = [&](StepArgs a) {
    a.G = a.G ? panel(cur_panel) : nullptr;
    a.last = 1;
    if (epi != EPI_NONE) a.part = part;
    launch_step<T>(g, a, pw, epi, s);
  };
  if (p == 0) {
    StepArgs a = base();
    a.X = X;
    a.kx = c[0];
    a.O = Y;
    last(a);
    return;
  }
  peer_barrier(pe, s);  // every rank is done with the previous call's panels
  peer_put<T>(pe, 0, Xs, R, pw, s);
  peer_barrier(pe, s);
  cur_panel = 0;
  if (p == 1) {
    StepArgs a = base();
    a.G = Xs;  // placeholder: replaced by the gather panel
    a.ka = -c[1];
    a.X = X;
    a.kx = c[0];
    a.O = Y;
    last(a);
    return;
  }
  StepArgs a = base();
  a.ka = -2.0 * c[p];
  a.X = Xs;
  a.kx = c[p - 1];
  a.O = B0;
  mid(a);
  if (p == 2) {
    StepArgs f = base();
    f.G = Xs;
    f.ka = -1.0;
    f.X = X;
    f.kx = c[0] - c[2];
    f.O = Y;
    last(f);
    return;
  }
  StepArgs b = base();
  b.ka = -2.0;
  b.X = Xs;
  b.kx = c[p - 2] - c[p];
  b.O = B1;
  mid(b);
  T* prv = B0;
  T* cur = B1;
  for (int l = p - 3; l >= 1; --l) {
    StepArgs m = base();
    m.ka = -2.0;
    m.S = prv;
    m.ks = -1.0;
    m.X = Xs;
    m.kx = c[l];
    m.O = prv;
    mid(m);
    std::swap(cur, prv);
  }
  StepArgs f = base();
  f.G = Xs;
  f.ka = -1.0;
  f.S = prv;
  f.ks = -1.0;
  f.X = X;
  f.kx = c[0];
  f.O = Y;
  last(f);
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

// one of cm (NCCL all-gather after each step) / pe (peer stores fused into the step)
template <typename T, typename Tio>
void run_rows(const csc_graph* g, csc_comm* cm, csc_peers* pe, const double* coeffs, int nc, const Tio* X,
              int64_t ldx, Tio* Y, int64_t ldy, int ncols, int mode, double* count_or_rowsq, cudaStream_t s) {
  const int64_t n = g->n;
  const int nranks = pe ? pe->nranks : cm->nranks;
  const int64_t R = rows_per_rank(g->n_global, nranks);
  const PanelPlan pp = plan_panels(g->n_global, ncols, g->dtype, g->device, g->nnz * nranks);
  if (pe && sizeof(T) * (size_t)R * nranks * pp.max_pw > pe->panel_bytes)
    fail(CSC_ERR_INVALID, "peer panels too small for this block (see csc_panel_row_bytes)");
  const int cap = step_grid_cap(g->device);
  Scratch x(sizeof(T) * R * pp.max_pw, s), xs(sizeof(T) * R * pp.max_pw, s), y(sizeof(T) * R * pp.max_pw, s),
      b0(sizeof(T) * R * pp.max_pw, s), b1(sizeof(T) * R * pp.max_pw, s),
      full(pe ? 16 : sizeof(T) * (size_t)R * nranks * pp.max_pw, s);
  Scratch part(sizeof(double) * std::max<int64_t>((int64_t)cap * pp.np, n), s);
  CSC_CUDA(cudaMemsetAsync(x.get(), 0, x.bytes(), s));
  CSC_CUDA(cudaMemsetAsync(xs.get(), 0, xs.bytes(), s));
  CSC_CUDA(cudaMemsetAsync(b0.get(), 0, b0.bytes(), s));
  CSC_CUDA(cudaMemsetAsync(b1.get(), 0, b1.bytes(), s));
  if (mode == 1) CSC_CUDA(cudaMemsetAsync(part.get(), 0, part.bytes(), s));
  if (mode == 2) CSC_CUDA(cudaMemsetAsync(count_or_rowsq, 0, sizeof(double) * n, s));
  for (int j = 0; j < pp.np; ++j) {
    const int pw = pp.pw[j], wc = pp.wc[j];
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n * pw + 255) / 256, 148 * 64));
    k_pack_rows<Tio, T><<<grid, 256, 0, s>>>(X, ldx, pp.c0[j], wc, pw, n, g->dis, x.as<T>(), xs.as<T>());
    CSC_LAUNCHED();
    const int epi = mode == 1 ? EPI_SUMSQ : (mode == 2 ? EPI_ROWSQ : EPI_NONE);
    double* pj = mode == 1 ? part.as<double>() + (size_t)cap * j : part.as<double>();
    if (pe)
      filter_panel_peers<T>(g, pe, coeffs, nc, x.as<T>(), xs.as<T>(), mode == 1 ? nullptr : y.as<T>(), b0.as<T>(),
                            b1.as<T>(), R, pw, wc, epi, pj, s);
    else
      filter_panel_rows<T>(g, cm, coeffs, nc, x.as<T>(), xs.as<T>(), mode == 1 ? nullptr : y.as<T>(), b0.as<T>(),
                           b1.as<T>(), full.as<T>(), R, pw, wc, epi, pj, s);
    if (mode != 1) {
      k_unpack_rows<T, Tio><<<(int)std::max<int64_t>(1, std::min<int64_t>((n * wc + 255) / 256, 148 * 64)), 256, 0,
                              s>>>(y.as<T>(), pp.c0[j], wc, pw, n, Y, ldy, part.as<double>(),
                                   mode == 2 ? count_or_rowsq : nullptr);
      CSC_LAUNCHED();
    }
  }
  if (mode == 1) reduce_sum(part.as<double>(), (int64_t)cap * pp.np, count_or_rowsq, s);
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

int csc_graph_create_rows(int64_t num_nodes, int64_t row_begin, int64_t num_rows, int64_t nnz, const int32_t* indptr,
                          const int32_t* indices, const double* weights, int dtype, int device, void* stream,
                          csc_graph** out) {
  return guard([&] {
    if (!out || !indptr) fail(CSC_ERR_INVALID, "NULL argument");
    if (row_begin < 0 || num_rows < 0 || row_begin + num_rows > num_nodes) fail(CSC_ERR_INVALID, "bad row range");
    if (dtype != CSC_F64 && dtype != CSC_F32) fail(CSC_ERR_INVALID, "dtype must be CSC_F64 or CSC_F32");
    // the local CSR is an ordinary num_rows x num_nodes CSR with global column indices
    csc_graph* g = graph_create_impl(num_rows, num_nodes, nnz, indptr, indices, weights, dtype, device,
                                     static_cast<cudaStream_t>(stream));
    g->n_global = num_nodes;
    g->row_begin = row_begin;
    *out = g;
  });
}

}  // extern "C"

namespace {
void filter_rows_entry(const csc_graph* g, csc_comm* comm, csc_peers* pe, const double* coeffs, int ncoeffs,
                       const void* X, int64_t ldx, void* Y, int64_t ldy, int ncols, int io_dtype, int mode, double* out,
                       void* stream) {
  if (!g) fail(CSC_ERR_INVALID, "graph is NULL");
  if (ncoeffs < 1 || !coeffs) fail(CSC_ERR_INVALID, "need coefficients");
  if (mode < 0 || mode > 2) fail(CSC_ERR_INVALID, "mode must be 0 (filter), 1 (sum of squares), 2 (row sums)");
  if (ncols < 1 || ldx < ncols || (mode != 1 && (ldy < ncols || !Y))) fail(CSC_ERR_INVALID, "bad block");
  if (mode != 0 && !out) fail(CSC_ERR_INVALID, "out is NULL");
  const int dev = pe ? pe->device : comm->device;
  if (dev != g->device) fail(CSC_ERR_INVALID, "transport and graph on different devices");
  if (pe && !pe->ready) fail(CSC_ERR_INVALID, "peer transport not attached to every rank (csc_peers_attach)");
  if (!is_device_ptr(X, g->device) || (mode != 1 && !is_device_ptr(Y, g->device)))
    fail(CSC_ERR_INVALID, "row-sharded blocks must be device buffers");
  DeviceGuard dg(g->device);
  ensure_pool(g->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DeviceOut o(out, sizeof(double) * (mode == 2 ? g->n : 1), g->device, s);
  double* dout = mode == 0 ? nullptr : o.as<double>();
  if (g->dtype == CSC_F64 && io_dtype == CSC_F64)
    run_rows<double, double>(g, comm, pe, coeffs, ncoeffs, (const double*)X, ldx, (double*)Y, ldy, ncols, mode, dout,
                             s);
  else if (g->dtype == CSC_F32 && io_dtype == CSC_F32)
    run_rows<float, float>(g, comm, pe, coeffs, ncoeffs, (const float*)X, ldx, (float*)Y, ldy, ncols, mode, dout, s);
  else if (g->dtype == CSC_F32 && io_dtype == CSC_F64)
    run_rows<float, double>(g, comm, pe, coeffs, ncoeffs, (const double*)X, ldx, (double*)Y, ldy, ncols, mode, dout,
                            s);
  else
    run_rows<double, float>(g, comm, pe, coeffs, ncoeffs, (const float*)X, ldx, (float*)Y, ldy, ncols, mode, dout, s);
  if (mode != 0) o.finish();
  CSC_CUDA(cudaStreamSynchronize(s));
}
}  // namespace

extern "C" {

int csc_cheb_filter_rows(const csc_graph* g, csc_comm* comm, const double* coeffs, int ncoeffs, const void* X,
                         int64_t ldx, void* Y, int64_t ldy, int ncols, int io_dtype, int mode, double* out,
                         void* stream) {
  return guard([&] {
    if (!comm) fail(CSC_ERR_INVALID, "comm is NULL");
    filter_rows_entry(g, comm, nullptr, coeffs, ncoeffs, X, ldx, Y, ldy, ncols, io_dtype, mode, out, stream);
  });
}

int csc_cheb_filter_rows_peers(const csc_graph* g, csc_peers* peers, const double* coeffs, int ncoeffs,
                               const void* X, int64_t ldx, void* Y, int64_t ldy, int ncols, int io_dtype, int mode,
                               double* out, void* stream) {
  return guard([&] {
    if (!peers) fail(CSC_ERR_INVALID, "peers is NULL");
    filter_rows_entry(g, nullptr, peers, coeffs, ncoeffs, X, ldx, Y, ldy, ncols, io_dtype, mode, out, stream);
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
