// K7: Lloyd iterations of the reduced k-means on the device (reference kmeans.py:64-93).
//
// One call runs one replicate from given initial centroids (the k-means++ seeding
// stays on the host, where it must consume numpy's generator exactly like the
// reference, kmeans.py:46-61).  Per iteration:
//   k_sqnorm     |c_j|^2 in numpy's pairwise-summation order
//   k_assign     D_ij = max(|p_i|^2 + |c_j|^2 - 2 p_i.c_j, 0) (kmeans.py:39-43); labels =
//                first argmin; point_d2; one warp per point
//   k_inertia    sum of point_d2 in numpy's pairwise order (kmeans.py:76)
//   k_update     centroid_j = mean of its points, summed in point order (kmeans.py:80-82)
//   repair       empty clusters take the farthest point, successively (kmeans.py:84-88)
// The convergence test (kmeans.py:89-92) runs on the host on the returned inertia.
#include <cmath>
#include <vector>

#include "internal.cuh"

namespace csc {
namespace {

// numpy's add-reduce order over a contiguous run (see graph.cu)
__device__ double pairwise(const double* a, int64_t n, int64_t stride) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i * stride];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j * stride];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[(i + j) * stride];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i * stride];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise(a, n2, stride) + pairwise(a + n2 * stride, n - n2, stride);
}

// |row|^2 with the squares summed in numpy's order: (x*x).sum(axis=1) squares
// first, then a pairwise reduction of the squared row
__device__ double sq_row(const double* x, int d) {
  double buf[8];
  // reproduce pairwise() on the squared values without materialising them
  if (d < 8) {
    double r = 0.0;
    for (int i = 0; i < d; ++i) r += x[i] * x[i];
    return r;
  }
  if (d <= 128) {
    for (int j = 0; j < 8; ++j) buf[j] = x[j] * x[j];
    int i = 8;
    for (; i < d - (d % 8); i += 8)
      for (int j = 0; j < 8; ++j) buf[j] += x[i + j] * x[i + j];
    double res = ((buf[0] + buf[1]) + (buf[2] + buf[3])) + ((buf[4] + buf[5]) + (buf[6] + buf[7]));
    for (; i < d; ++i) res += x[i] * x[i];
    return res;
  }
  int n2 = d / 2;
  n2 -= n2 % 8;
  return sq_row(x, n2) + sq_row(x + n2, d - n2);
}

__global__ void k_sqnorm(const double* __restrict__ X, int rows, int d, double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x)
    out[i] = sq_row(X + (int64_t)i * d, d);
}

// one warp per point: distances to all centroids, first argmin
__global__ void k_assign(const double* __restrict__ P, const double* __restrict__ pp, const double* __restrict__ C,
                         const double* __restrict__ cc, int n, int k, int d, int64_t* __restrict__ labels,
                         double* __restrict__ pd2) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < n; i += nw) {
    const double* p = P + (int64_t)i * d;
    double best = INFINITY;
    int bj = 0;
    for (int j0 = 0; j0 < k; j0 += 32) {
      const int j = j0 + lane;
      double dist = INFINITY;
      if (j < k) {
        const double* c = C + (int64_t)j * d;
        double dot = 0.0;
        for (int t = 0; t < d; ++t) dot = fma(p[t], c[t], dot);
        dist = fmax(pp[i] + cc[j] - 2.0 * dot, 0.0);
      }
      // warp argmin with first-index ties
      double v = dist;
      int vj = j < k ? j : INT_MAX;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oj = __shfl_xor_sync(0xffffffffu, vj, o);
        if (ov < v || (ov == v && oj < vj)) {
          v = ov;
          vj = oj;
        }
      }
      if (v < best) {  // strictly smaller: earlier chunks keep ties
        best = v;
        bj = vj;
      }
    }
    if (lane == 0) {
      labels[i] = bj;
      pd2[i] = best;
    }
  }
}

__global__ void k_inertia(const double* __restrict__ pd2, int n, double* __restrict__ out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = pairwise(pd2, n, 1);
}

// centroid_j[t] = sum over points with label j (in point order) / count_j; counts out
__global__ void k_update(const double* __restrict__ P, const int64_t* __restrict__ labels, int n, int k, int d,
                         double* __restrict__ C, int* __restrict__ counts) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < (int64_t)k * d;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(u / d), t = (int)(u % d);
    double s = 0.0;
    int cnt = 0;
    for (int i = 0; i < n; ++i)
      if (labels[i] == j) {
        s += P[(int64_t)i * d + t];
        ++cnt;
      }
    if (cnt > 0) C[u] = s / cnt;
    if (t == 0) counts[j] = cnt;
  }
}

// empty clusters: successively take the farthest point (first max), zero its distance
__global__ void k_repair(const double* __restrict__ P, int n, int k, int d, const int* __restrict__ counts,
                         double* __restrict__ pd2, double* __restrict__ C, int* __restrict__ repaired) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int rep = 0;
  for (int j = 0; j < k; ++j) {
    if (counts[j] > 0) continue;
    int far = 0;
    for (int i = 1; i < n; ++i)
      if (pd2[i] > pd2[far]) far = i;
    for (int t = 0; t < d; ++t) C[(int64_t)j * d + t] = P[(int64_t)far * d + t];
    pd2[far] = 0.0;
    rep = 1;
  }
  *repaired = rep;
}

}  // namespace
}  // namespace csc

using namespace csc;

extern "C" int csc_kmeans_lloyd(const double* points, int64_t n, int d, const double* init, int k, int64_t max_iters,
                                double tol, int64_t* labels_out, double* centroids_out, double* inertia_out,
                                int64_t* iters_out, int device, void* stream) {
  return guard([&] {
    if (n < 1 || d < 1 || k < 1) fail(CSC_ERR_INVALID, "kmeans: n, d and k must be >= 1");
    if (n < k) fail(CSC_ERR_INVALID, "need at least k points");
    if (!points || !init || !labels_out) fail(CSC_ERR_INVALID, "NULL buffer");
    if (max_iters < 0) fail(CSC_ERR_INVALID, "max_iters must be >= 0");
    DeviceGuard dg(device);
    ensure_pool(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DeviceView dP(points, sizeof(double) * n * d, device, s);
    DeviceView dC0(init, sizeof(double) * k * d, device, s);
    Scratch C(sizeof(double) * k * d, s), pp(sizeof(double) * n, s), cc(sizeof(double) * k, s),
        pd2(sizeof(double) * n, s), inert(sizeof(double), s), counts(sizeof(int) * k, s), rep(sizeof(int), s);
    DeviceOut lab(labels_out, sizeof(int64_t) * n, device, s);
    CSC_CUDA(cudaMemcpyAsync(C.get(), dC0.as<double>(), sizeof(double) * k * d, cudaMemcpyDeviceToDevice, s));
    CSC_CUDA(cudaMemsetAsync(lab.as<int64_t>(), 0, sizeof(int64_t) * n, s));
    const int ng = (int)std::min<int64_t>((n + 255) / 256, 1024);
    k_sqnorm<<<ng, 256, 0, s>>>(dP.as<double>(), (int)n, d, pp.as<double>());
    CSC_LAUNCHED();
    const double tiny = 2.2250738585072014e-308;
    double inertia = INFINITY;
    int64_t iters = 0;
    for (int64_t it = 0; it < max_iters; ++it) {
      k_sqnorm<<<(k + 255) / 256, 256, 0, s>>>(C.as<double>(), k, d, cc.as<double>());
      CSC_LAUNCHED();
      k_assign<<<(int)std::min<int64_t>((n + 7) / 8, 2048), 256, 0, s>>>(dP.as<double>(), pp.as<double>(),
                                                                          C.as<double>(), cc.as<double>(), (int)n, k,
                                                                          d, lab.as<int64_t>(), pd2.as<double>());
      CSC_LAUNCHED();
      k_inertia<<<1, 32, 0, s>>>(pd2.as<double>(), (int)n, inert.as<double>());
      CSC_LAUNCHED();
      k_update<<<(int)std::min<int64_t>(((int64_t)k * d + 255) / 256, 4096), 256, 0, s>>>(
          dP.as<double>(), lab.as<int64_t>(), (int)n, k, d, C.as<double>(), counts.as<int>());
      CSC_LAUNCHED();
      k_repair<<<1, 1, 0, s>>>(dP.as<double>(), (int)n, k, d, counts.as<int>(), pd2.as<double>(), C.as<double>(),
                               rep.as<int>());
      CSC_LAUNCHED();
      double h_inert = 0.0;
      int h_rep = 0;
      CSC_CUDA(cudaMemcpyAsync(&h_inert, inert.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
      CSC_CUDA(cudaMemcpyAsync(&h_rep, rep.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
      CSC_CUDA(cudaStreamSynchronize(s));
      iters = it + 1;
      const bool settled = inertia - h_inert <= tol * std::max(h_inert, tiny);
      inertia = h_inert;
      if (!h_rep && settled) break;
    }
    lab.finish();
    if (centroids_out)
      CSC_CUDA(cudaMemcpyAsync(centroids_out, C.get(), sizeof(double) * k * d, cudaMemcpyDefault, s));
    CSC_CUDA(cudaStreamSynchronize(s));
    if (inertia_out) *inertia_out = inertia;
    if (iters_out) *iters_out = iters;
  });
}
