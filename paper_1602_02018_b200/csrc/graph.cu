// K1: graph ingestion and symmetric normalization on the device.
//
//   csc_graph_build_coo : edge triples -> canonical CSR   (reference graph.py:73-125)
//   csc_graph_create    : canonical CSR -> operator        (reference graph.py:58-70, 164-169)
//
// Canonicalization is sort + segmented reduce, the data-parallel form of
// scipy's coo->csr + sum_duplicates + maximum(A, A^T) + eliminate_zeros:
//   1. key = src * N + dst, radix-sort (stable) and sum runs of equal keys
//      (per-direction duplicates are summed, graph.py:122-123);
//   2. emit every entry twice, as (i,j) and (j,i), sort again and take the max
//      of each run (W = max(A, A^T), graph.py:124; absent entries are 0 and all
//      weights are >= 0, so max over the present ones is the same);
//   3. drop explicit zeros (graph.py:62), split keys into row/column.
// Degrees are fp64 row sums in the summation order scipy's CSR row sum uses
// (np.add.reduceat, graph.py:63), so they are bit-identical.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "internal.cuh"

namespace csc {
namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t work, int threads = kThreads) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > (1 << 30)) g = 1 << 30;
  return static_cast<int>(g);
}

// numpy's pairwise summation (the add-reduce inner loop): sequential below 8
// terms, 8 interleaved accumulators up to 128, halving recursion above.
__device__ double np_pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

// degrees and d^-1/2 (graph.py:63, 168).  scipy's CSR row sum is
// np.add.reduceat(data, indptr), i.e. a[0] + pairwise(a[1:]) per row; the same
// order here makes the degrees bit-identical for arbitrary weights.
__global__ void k_degrees(const int32_t* __restrict__ indptr, const double* __restrict__ w, int64_t n,
                          double* __restrict__ deg, double* __restrict__ dis) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = indptr[i], e = indptr[i + 1];
    const double s = e > b ? w[b] + np_pairwise_sum(w + b + 1, e - b - 1) : 0.0;
    deg[i] = s;
    dis[i] = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
  }
}

// Per-row scales of the scaled-basis recurrence (filter.cuh): (d^-1/2, d^1/2).
template <typename T>
__global__ void k_row_scales(const double* __restrict__ deg, const double* __restrict__ dis, int64_t n,
                             T* __restrict__ rs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    rs[2 * i] = static_cast<T>(dis[i]);
    rs[2 * i + 1] = static_cast<T>(deg[i] > 0.0 ? sqrt(deg[i]) : 0.0);
  }
}

template <typename T>
__global__ void k_cast_weights(const double* __restrict__ w, int64_t nnz, T* __restrict__ out, int* __restrict__ nonunit) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    out[e] = static_cast<T>(w[e]);
    if (w[e] != 1.0) atomicOr(nonunit, 1);
  }
}

// CSR sanity for user-supplied arrays: flags[0] bad indptr, flags[1] bad index.
__global__ void k_check_csr(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t n,
                            int64_t ncols, int64_t nnz, int* flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = indptr[i], e = indptr[i + 1];
    if (b < 0 || e < b || e > nnz) {
      atomicOr(&flags[0], 1);
      continue;
    }
    for (int32_t k = b; k < e; ++k) {
      const int32_t j = indices[k];
      if (j < 0 || j >= ncols) atomicOr(&flags[1], 1);
    }
  }
}

// First offending edge per category: 0 negative weight, 1 negative index,
// 2 index >= N, 3 self loop (checked in the reference's order, graph.py:104-118).
__global__ void k_check_edges(const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                              const double* __restrict__ w, int64_t m, int64_t n, unsigned long long* first) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = src[e], b = dst[e];
    if (w && w[e] < 0.0) atomicMin(&first[0], (unsigned long long)e);
    if (a < 0 || b < 0) atomicMin(&first[1], (unsigned long long)e);
    if (a >= n || b >= n) atomicMin(&first[2], (unsigned long long)e);
    if (a == b) atomicMin(&first[3], (unsigned long long)e);
  }
}

__global__ void k_make_keys(const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                            const double* __restrict__ w, int64_t m, uint64_t n, int drop_loops,
                            uint64_t* __restrict__ keys, double* __restrict__ vals) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = (uint64_t)src[e], b = (uint64_t)dst[e];
    const bool loop = a == b;
    // dropped self loops become weight-0 entries on (a, a); they vanish at the
    // zero-elimination step and never meet a real entry (no loops survive).
    keys[e] = a * n + b;
    vals[e] = (loop && drop_loops) ? 0.0 : (w ? w[e] : 1.0);
  }
}

__global__ void k_mirror(const uint64_t* __restrict__ keys, const double* __restrict__ vals, int64_t m,
                         uint64_t n, uint64_t* __restrict__ keys2, double* __restrict__ vals2) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[e];
    const uint64_t r = k / n, c = k % n;
    keys2[e] = k;
    vals2[e] = vals[e];
    keys2[m + e] = c * n + r;
    vals2[m + e] = vals[e];
  }
}

struct NonZero {
  const double* v;
  __device__ bool operator()(const int64_t& i) const { return v[i] != 0.0; }
};

__global__ void k_split_keys(const uint64_t* __restrict__ keys, const double* __restrict__ vals,
                             const int64_t* __restrict__ sel, int64_t nnz, uint64_t n,
                             int32_t* __restrict__ rows, int32_t* __restrict__ cols, double* __restrict__ w) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = sel[e];
    const uint64_t k = keys[s];
    rows[e] = (int32_t)(k / n);
    cols[e] = (int32_t)(k % n);
    w[e] = vals[s];
  }
}

// indptr[i] = first entry with row >= i (rows sorted ascending).
__global__ void k_indptr(const int32_t* __restrict__ rows, int64_t nnz, int64_t n, int32_t* __restrict__ indptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (rows[mid] < i)
        lo = mid + 1;
      else
        hi = mid;
    }
    indptr[i] = (int32_t)lo;
  }
}

struct MaxOp {
  __device__ double operator()(const double& a, const double& b) const { return a < b ? b : a; }
};

int key_bits(uint64_t n) {
  const unsigned __int128 top = (unsigned __int128)n * n;
  int bits = 1;
  while (bits < 64 && ((unsigned __int128)1 << bits) < top) ++bits;
  return bits;
}

}  // namespace

csc_graph* graph_from_device_csr(int64_t n, int64_t nnz, int32_t* indptr, int32_t* indices, double* weights,
                                 int dtype, int device, cudaStream_t s) {
  csc_graph* g = new csc_graph();
  g->n = n;
  g->nnz = nnz;
  g->dtype = dtype;
  g->device = device;
  g->indptr = indptr;
  g->indices = indices;
  g->weights = weights;
  g->n_global = n;
  g->gather_rows = n;
  try {
    const size_t es = dtype_size(dtype);
    CSC_CUDA(cudaMalloc(&g->degrees, sizeof(double) * (n > 0 ? n : 1)));
    CSC_CUDA(cudaMalloc(&g->dis, sizeof(double) * (n > 0 ? n : 1)));
    CSC_CUDA(cudaMalloc(&g->rs, 2 * es * (n > 0 ? n : 1)));
    if (n > 0) {
      k_degrees<<<grid_for(n), kThreads, 0, s>>>(indptr, weights, n, g->degrees, g->dis);
      CSC_LAUNCHED();
      if (dtype == CSC_F64)
        k_row_scales<double><<<grid_for(n), kThreads, 0, s>>>(g->degrees, g->dis, n, static_cast<double*>(g->rs));
      else
        k_row_scales<float><<<grid_for(n), kThreads, 0, s>>>(g->degrees, g->dis, n, static_cast<float*>(g->rs));
      CSC_LAUNCHED();
    }
    // weights in the compute dtype, dropped entirely for unit-weight graphs
    g->unit = true;
    if (nnz > 0) {
      void* wv = nullptr;
      CSC_CUDA(cudaMalloc(&wv, es * nnz));
      int* flag = nullptr;
      CSC_CUDA(cudaMalloc(&flag, sizeof(int)));
      CSC_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
      if (dtype == CSC_F64)
        k_cast_weights<double><<<grid_for(nnz), kThreads, 0, s>>>(weights, nnz, static_cast<double*>(wv), flag);
      else
        k_cast_weights<float><<<grid_for(nnz), kThreads, 0, s>>>(weights, nnz, static_cast<float*>(wv), flag);
      CSC_LAUNCHED();
      int nonunit = 0;
      CSC_CUDA(cudaMemcpyAsync(&nonunit, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
      CSC_CUDA(cudaStreamSynchronize(s));
      cudaFree(flag);
      if (nonunit) {
        g->wv = wv;
        g->unit = false;
      } else {
        cudaFree(wv);
      }
    }
    CSC_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    graph_free(g);
    throw;
  }
  return g;
}

void graph_free(csc_graph* g) {
  if (!g) return;
  DeviceGuard dg(g->device);
  cudaFree(g->indptr);
  cudaFree(g->indices);
  cudaFree(g->weights);
  cudaFree(g->wv);
  cudaFree(g->rs);
  cudaFree(g->degrees);
  cudaFree(g->dis);
  delete g;
}

}  // namespace csc

using namespace csc;

static void check_common(int64_t num_nodes, int dtype, int device, csc_graph** out) {
  if (!out) fail(CSC_ERR_INVALID, "out is NULL");
  if (num_nodes < 0) fail(CSC_ERR_INVALID, "num_nodes must be >= 0");
  if (num_nodes >= (int64_t(1) << 31) - 1) fail(CSC_ERR_INVALID, "num_nodes must fit int32 CSR indices");
  if (dtype != CSC_F64 && dtype != CSC_F32) fail(CSC_ERR_INVALID, "dtype must be CSC_F64 or CSC_F32");
  int ndev = 0;
  CSC_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) fail(CSC_ERR_INVALID, "device " + std::to_string(device) + " not present");
}

namespace csc {
// canonical CSR with num_nodes rows and column indices < ncols -> device operator
csc_graph* graph_create_impl(int64_t num_nodes, int64_t ncols, int64_t nnz, const int32_t* indptr,
                             const int32_t* indices, const double* weights, int dtype, int device, cudaStream_t s);
}  // namespace csc

extern "C" {

int csc_graph_create(int64_t num_nodes, int64_t nnz, const int32_t* indptr, const int32_t* indices,
                     const double* weights, int dtype, int device, void* stream, csc_graph** out) {
  return guard([&] {
    check_common(num_nodes, dtype, device, out);
    *out = graph_create_impl(num_nodes, num_nodes, nnz, indptr, indices, weights, dtype, device,
                             static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"

csc_graph* csc::graph_create_impl(int64_t num_nodes, int64_t ncols, int64_t nnz, const int32_t* indptr,
                                  const int32_t* indices, const double* weights, int dtype, int device,
                                  cudaStream_t s) {
  csc_graph* result = nullptr;
  {
    if (nnz < 0 || nnz >= (int64_t(1) << 31)) fail(CSC_ERR_INVALID, "nnz out of int32 range");
    if (!indptr || (nnz > 0 && (!indices || !weights))) fail(CSC_ERR_INVALID, "CSR array is NULL");
    DeviceGuard dg(device);
    ensure_pool(device);
    int32_t *d_ptr = nullptr, *d_idx = nullptr;
    double* d_w = nullptr;
    try {
      CSC_CUDA(cudaMalloc(&d_ptr, sizeof(int32_t) * (num_nodes + 1)));
      CSC_CUDA(cudaMalloc(&d_idx, sizeof(int32_t) * (nnz > 0 ? nnz : 1)));
      CSC_CUDA(cudaMalloc(&d_w, sizeof(double) * (nnz > 0 ? nnz : 1)));
      CSC_CUDA(cudaMemcpyAsync(d_ptr, indptr, sizeof(int32_t) * (num_nodes + 1), cudaMemcpyDefault, s));
      if (nnz > 0) {
        CSC_CUDA(cudaMemcpyAsync(d_idx, indices, sizeof(int32_t) * nnz, cudaMemcpyDefault, s));
        CSC_CUDA(cudaMemcpyAsync(d_w, weights, sizeof(double) * nnz, cudaMemcpyDefault, s));
      }
      int32_t ends[2];
      CSC_CUDA(cudaMemcpyAsync(&ends[0], d_ptr, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      CSC_CUDA(cudaMemcpyAsync(&ends[1], d_ptr + num_nodes, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      Scratch flags(2 * sizeof(int), s);
      CSC_CUDA(cudaMemsetAsync(flags.get(), 0, 2 * sizeof(int), s));
      if (num_nodes > 0) {
        k_check_csr<<<grid_for(num_nodes), kThreads, 0, s>>>(d_ptr, d_idx, num_nodes, ncols, nnz, flags.as<int>());
        CSC_LAUNCHED();
      }
      int hflags[2];
      CSC_CUDA(cudaMemcpyAsync(hflags, flags.get(), sizeof(hflags), cudaMemcpyDeviceToHost, s));
      CSC_CUDA(cudaStreamSynchronize(s));
      if (ends[0] != 0 || ends[1] != nnz) fail(CSC_ERR_GRAPH, "indptr must start at 0 and end at nnz");
      if (hflags[0]) fail(CSC_ERR_GRAPH, "indptr is not non-decreasing");
      if (hflags[1]) fail(CSC_ERR_GRAPH, "column index out of range");
      result = graph_from_device_csr(num_nodes, nnz, d_ptr, d_idx, d_w, dtype, device, s);
      d_ptr = nullptr;
      d_idx = nullptr;
      d_w = nullptr;
    } catch (...) {
      cudaFree(d_ptr);
      cudaFree(d_idx);
      cudaFree(d_w);
      throw;
    }
  }
  return result;
}

extern "C" {

int csc_graph_build_coo(int64_t num_nodes, int64_t num_edges, const int64_t* src, const int64_t* dst,
                        const double* weights, int self_loops, int dtype, int device, void* stream,
                        csc_graph** out) {
  return guard([&] {
    check_common(num_nodes, dtype, device, out);
    if (num_edges < 0) fail(CSC_ERR_INVALID, "num_edges must be >= 0");
    if (num_edges > 0 && (!src || !dst)) fail(CSC_ERR_INVALID, "edge arrays are NULL");
    if (self_loops != CSC_SELF_LOOPS_ERROR && self_loops != CSC_SELF_LOOPS_DROP)
      fail(CSC_ERR_INVALID, "self_loops must be 'error' or 'drop'");
    if (2 * num_edges >= (int64_t(1) << 31)) fail(CSC_ERR_INVALID, "too many edges for int32 CSR");
    DeviceGuard dg(device);
    ensure_pool(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t m = num_edges;
    const uint64_t n = (uint64_t)num_nodes;

    int32_t *d_ptr = nullptr, *d_idx = nullptr;
    double* d_w = nullptr;
    int64_t nnz = 0;
    try {
      CSC_CUDA(cudaMalloc(&d_ptr, sizeof(int32_t) * (num_nodes + 1)));
      if (m == 0) {
        CSC_CUDA(cudaMemsetAsync(d_ptr, 0, sizeof(int32_t) * (num_nodes + 1), s));
        CSC_CUDA(cudaMalloc(&d_idx, sizeof(int32_t)));
        CSC_CUDA(cudaMalloc(&d_w, sizeof(double)));
      } else {
        DeviceView vs(src, sizeof(int64_t) * m, device, s);
        DeviceView vd(dst, sizeof(int64_t) * m, device, s);
        DeviceView vw(weights, sizeof(double) * m, device, s);

        // validation (first offending edge per category)
        Scratch first(4 * sizeof(unsigned long long), s);
        CSC_CUDA(cudaMemsetAsync(first.get(), 0xff, 4 * sizeof(unsigned long long), s));
        k_check_edges<<<grid_for(m), kThreads, 0, s>>>(vs.as<int64_t>(), vd.as<int64_t>(), vw.as<double>(), m,
                                                       num_nodes, first.as<unsigned long long>());
        CSC_LAUNCHED();
        unsigned long long hf[4];
        CSC_CUDA(cudaMemcpyAsync(hf, first.get(), sizeof(hf), cudaMemcpyDeviceToHost, s));
        CSC_CUDA(cudaStreamSynchronize(s));
        auto edge_str = [&](unsigned long long e) {
          int64_t a, b;
          CSC_CUDA(cudaMemcpyAsync(&a, vs.as<int64_t>() + e, sizeof(a), cudaMemcpyDeviceToHost, s));
          CSC_CUDA(cudaMemcpyAsync(&b, vd.as<int64_t>() + e, sizeof(b), cudaMemcpyDeviceToHost, s));
          CSC_CUDA(cudaStreamSynchronize(s));
          return std::make_pair(a, b);
        };
        if (hf[0] != ~0ull) {
          double wv;
          CSC_CUDA(cudaMemcpyAsync(&wv, vw.as<double>() + hf[0], sizeof(wv), cudaMemcpyDeviceToHost, s));
          CSC_CUDA(cudaStreamSynchronize(s));
          auto ab = edge_str(hf[0]);
          fail(CSC_ERR_GRAPH, "negative weight " + std::to_string(wv) + " on edge (" + std::to_string(ab.first) +
                                  ", " + std::to_string(ab.second) + ")");
        }
        if (hf[1] != ~0ull) fail(CSC_ERR_GRAPH, "negative node index");
        if (hf[2] != ~0ull) fail(CSC_ERR_GRAPH, "node index out of range for num_nodes=" + std::to_string(num_nodes));
        if (hf[3] != ~0ull && self_loops == CSC_SELF_LOOPS_ERROR)
          fail(CSC_ERR_GRAPH, "self-loop on node " + std::to_string(edge_str(hf[3]).first));

        const int bits = key_bits(n > 1 ? n : 2);
        // 1. sort by (src, dst) and sum per-direction duplicates
        Scratch k0(sizeof(uint64_t) * m, s), v0(sizeof(double) * m, s);
        Scratch k1(sizeof(uint64_t) * m, s), v1(sizeof(double) * m, s);
        k_make_keys<<<grid_for(m), kThreads, 0, s>>>(vs.as<int64_t>(), vd.as<int64_t>(), vw.as<double>(), m, n,
                                                     self_loops == CSC_SELF_LOOPS_DROP, k0.as<uint64_t>(),
                                                     v0.as<double>());
        CSC_LAUNCHED();
        size_t tmp_sort = 0, tmp_red = 0, tmp_sel = 0;
        CSC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, k0.as<uint64_t>(), k1.as<uint64_t>(),
                                                 v0.as<double>(), v1.as<double>(), (int64_t)2 * m, 0, bits, s));
        CSC_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, tmp_red, k1.as<uint64_t>(), k0.as<uint64_t>(),
                                                v1.as<double>(), v0.as<double>(), (int64_t*)nullptr,
                                                cub::Sum(), (int64_t)2 * m, s));
        Scratch tmp(std::max(tmp_sort, tmp_red), s);
        size_t tb = tmp.bytes();
        CSC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, k0.as<uint64_t>(), k1.as<uint64_t>(),
                                                 v0.as<double>(), v1.as<double>(), m, 0, bits, s));
        CSC_LAUNCHED();
        Scratch cnt(sizeof(int64_t), s);
        tb = tmp.bytes();
        CSC_CUDA(cub::DeviceReduce::ReduceByKey(tmp.get(), tb, k1.as<uint64_t>(), k0.as<uint64_t>(),
                                                v1.as<double>(), v0.as<double>(), cnt.as<int64_t>(), cub::Sum(),
                                                m, s));
        CSC_LAUNCHED();
        int64_t m1 = 0;
        CSC_CUDA(cudaMemcpyAsync(&m1, cnt.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CSC_CUDA(cudaStreamSynchronize(s));

        // 2. W = max(A, A^T): mirror, sort, max per run
        Scratch k2(sizeof(uint64_t) * 2 * m1, s), v2(sizeof(double) * 2 * m1, s);
        Scratch k3(sizeof(uint64_t) * 2 * m1, s), v3(sizeof(double) * 2 * m1, s);
        k_mirror<<<grid_for(m1), kThreads, 0, s>>>(k0.as<uint64_t>(), v0.as<double>(), m1, n, k2.as<uint64_t>(),
                                                   v2.as<double>());
        CSC_LAUNCHED();
        tb = tmp.bytes();
        CSC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, k2.as<uint64_t>(), k3.as<uint64_t>(),
                                                 v2.as<double>(), v3.as<double>(), 2 * m1, 0, bits, s));
        CSC_LAUNCHED();
        tb = tmp.bytes();
        CSC_CUDA(cub::DeviceReduce::ReduceByKey(tmp.get(), tb, k3.as<uint64_t>(), k2.as<uint64_t>(),
                                                v3.as<double>(), v2.as<double>(), cnt.as<int64_t>(), MaxOp(),
                                                2 * m1, s));
        CSC_LAUNCHED();
        int64_t m2 = 0;
        CSC_CUDA(cudaMemcpyAsync(&m2, cnt.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CSC_CUDA(cudaStreamSynchronize(s));

        // 3. eliminate zeros, split keys
        Scratch sel(sizeof(int64_t) * (m2 > 0 ? m2 : 1), s);
        thrust::counting_iterator<int64_t> it(0);
        NonZero nz{v2.as<double>()};
        CSC_CUDA(cub::DeviceSelect::If(nullptr, tmp_sel, it, sel.as<int64_t>(), cnt.as<int64_t>(), m2, nz, s));
        Scratch tmp2(tmp_sel, s);
        CSC_CUDA(cub::DeviceSelect::If(tmp2.get(), tmp_sel, it, sel.as<int64_t>(), cnt.as<int64_t>(), m2, nz, s));
        CSC_LAUNCHED();
        CSC_CUDA(cudaMemcpyAsync(&nnz, cnt.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CSC_CUDA(cudaStreamSynchronize(s));

        Scratch rows(sizeof(int32_t) * (nnz > 0 ? nnz : 1), s);
        CSC_CUDA(cudaMalloc(&d_idx, sizeof(int32_t) * (nnz > 0 ? nnz : 1)));
        CSC_CUDA(cudaMalloc(&d_w, sizeof(double) * (nnz > 0 ? nnz : 1)));
        if (nnz > 0) {
          k_split_keys<<<grid_for(nnz), kThreads, 0, s>>>(k2.as<uint64_t>(), v2.as<double>(), sel.as<int64_t>(),
                                                          nnz, n, rows.as<int32_t>(), d_idx, d_w);
          CSC_LAUNCHED();
        }
        k_indptr<<<grid_for(num_nodes + 1), kThreads, 0, s>>>(rows.as<int32_t>(), nnz, num_nodes, d_ptr);
        CSC_LAUNCHED();
        CSC_CUDA(cudaStreamSynchronize(s));
      }
      csc_graph* g = graph_from_device_csr(num_nodes, nnz, d_ptr, d_idx, d_w, dtype, device, s);
      d_ptr = nullptr;
      d_idx = nullptr;
      d_w = nullptr;
      *out = g;
    } catch (...) {
      cudaFree(d_ptr);
      cudaFree(d_idx);
      cudaFree(d_w);
      throw;
    }
  });
}

int csc_graph_destroy(csc_graph* g) {
  return guard([&] { graph_free(g); });
}

int csc_graph_info(const csc_graph* g, int64_t* num_nodes, int64_t* nnz, int* dtype, int* device) {
  return guard([&] {
    if (!g) fail(CSC_ERR_INVALID, "graph is NULL");
    if (num_nodes) *num_nodes = g->n;
    if (nnz) *nnz = g->nnz;
    if (dtype) *dtype = g->dtype;
    if (device) *device = g->device;
  });
}

int csc_graph_export(const csc_graph* g, int32_t* indptr, int32_t* indices, double* weights, double* degrees,
                     double* d_inv_sqrt, void* stream) {
  return guard([&] {
    if (!g) fail(CSC_ERR_INVALID, "graph is NULL");
    DeviceGuard dg(g->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (indptr)
      CSC_CUDA(cudaMemcpyAsync(indptr, g->indptr, sizeof(int32_t) * (g->n + 1), cudaMemcpyDefault, s));
    if (indices && g->nnz)
      CSC_CUDA(cudaMemcpyAsync(indices, g->indices, sizeof(int32_t) * g->nnz, cudaMemcpyDefault, s));
    if (weights && g->nnz)
      CSC_CUDA(cudaMemcpyAsync(weights, g->weights, sizeof(double) * g->nnz, cudaMemcpyDefault, s));
    if (degrees && g->n) CSC_CUDA(cudaMemcpyAsync(degrees, g->degrees, sizeof(double) * g->n, cudaMemcpyDefault, s));
    if (d_inv_sqrt && g->n) CSC_CUDA(cudaMemcpyAsync(d_inv_sqrt, g->dis, sizeof(double) * g->n, cudaMemcpyDefault, s));
    CSC_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
