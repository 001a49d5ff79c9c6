// K7: the reduced k-means on the device (reference kmeans.py).
//
// One CTA per replicate runs the whole replicate without returning to the host:
//   seeding   k-means++ D^2 sampling with numpy's arithmetic (kmeans.py:46-61):
//             d2 = ((P - c)**2).sum(axis=1) and d2.sum() in numpy's pairwise order,
//             rng.choice(q, p=d2/total) == searchsorted(cumsum(p)/cumsum(p)[-1],
//             random(), 'right') with random() drawn from the replicate's PCG64
//             state (the first centroid, rng.integers(q), is drawn on the host);
//   Lloyd     (kmeans.py:64-93) per iteration: |c_j|^2; D_ij = max(|p_i|^2 + |c_j|^2
//             - 2 p_i.c_j, 0) (kmeans.py:39-43), first argmin; inertia = pairwise sum;
//             centroid_j = mean of its points summed in point order; empty clusters
//             take the farthest point, successively; relative-inertia stop.
// Replicates run concurrently on separate SMs; the host picks the lowest inertia
// (first minimum, kmeans.py:121-123).  A replicate whose D^2 total is not positive
// (the reference's rng.integers fallback, kmeans.py:57-58) is flagged for the host.
#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.cuh"
#include "pcg64.cuh"

namespace csc {
namespace {

// numpy's pairwise add-reduce of v(off .. off+n-1) (numpy pairwise_sum; see graph.cu).
// Products are rounded before the adds (__dmul_rn / __dadd_rn: no FMA contraction).
template <class F>
__device__ double pw_leaf(const F& v, int64_t off, int64_t n) {  // n <= 128
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, v(off + i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = v(off + j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v(off + i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, v(off + i));
  return res;
}

// The recursion sum(a, n2) + sum(a + n2, n - n2), n2 = n/2 rounded down to a multiple
// of 8, walked iteratively (device recursion would need a dynamic stack).
template <class F>
__device__ double pw_sum(const F& v, int64_t off, int64_t n) {
  if (n <= 128) return pw_leaf(v, off, n);
  int64_t fo[32], fn[32];
  double left[32];
  int st[32];
  int sp = 0;
  fo[0] = off;
  fn[0] = n;
  st[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    int64_t n2 = fn[sp] / 2;
    n2 -= n2 % 8;
    if (st[sp] == 0) {  // left half
      st[sp] = 1;
      if (n2 > 128) {
        ++sp;
        fo[sp] = fo[sp - 1];
        fn[sp] = n2;
        st[sp] = 0;
        continue;
      }
      ret = pw_leaf(v, fo[sp], n2);
    }
    if (st[sp] == 1) {  // ret = left sum; right half
      left[sp] = ret;
      st[sp] = 2;
      if (fn[sp] - n2 > 128) {
        ++sp;
        fo[sp] = fo[sp - 1] + n2;
        fn[sp] = fn[sp - 1] - n2;
        st[sp] = 0;
        continue;
      }
      ret = pw_leaf(v, fo[sp] + n2, fn[sp] - n2);
    }
    ret = __dadd_rn(left[sp], ret);  // ret = right sum
    --sp;
  }
  return ret;
}

// numpy's pairwise sum over n elements evaluated by a whole CTA: the leaves of the
// recursion (blocks of <= 128 elements, each summed with pw_leaf's 8 accumulators) are
// independent, so threads sum them in parallel; one thread then combines the leaf sums in
// the recursion's order (a postfix program built once per kernel).  Bit-identical to pw_sum.
constexpr int kMaxLeaves = 512;
struct PwPlan {
  int nleaf, nprog;  // nleaf < 0: too many leaves, use pw_sum
  int off[kMaxLeaves];
  int len[kMaxLeaves];
  short prog[2 * kMaxLeaves];  // >= 0: push leaf sum, -1: add the top two
};

__device__ void pw_plan_build(PwPlan& pl, int64_t n) {  // one thread
  pl.nleaf = pl.nprog = 0;
  if (n <= 128) {
    pl.off[0] = 0;
    pl.len[0] = (int)n;
    pl.prog[0] = 0;
    pl.nleaf = pl.nprog = 1;
    return;
  }
  int64_t so[48], sn[48];
  int ss[48];
  int sp = 0;
  so[0] = 0;
  sn[0] = n;
  ss[0] = 0;
  while (sp >= 0) {
    int64_t n2 = sn[sp] / 2;
    n2 -= n2 % 8;
    if (ss[sp] == 0 || ss[sp] == 1) {  // 0: left half, 1: right half
      const int64_t o = ss[sp] == 0 ? so[sp] : so[sp] + n2;
      const int64_t m = ss[sp] == 0 ? n2 : sn[sp] - n2;
      ++ss[sp];
      if (m > 128) {
        ++sp;
        so[sp] = o;
        sn[sp] = m;
        ss[sp] = 0;
        continue;
      }
      if (pl.nleaf >= kMaxLeaves) {
        pl.nleaf = -1;
        return;
      }
      pl.off[pl.nleaf] = (int)o;
      pl.len[pl.nleaf] = (int)m;
      pl.prog[pl.nprog++] = (short)pl.nleaf++;
      continue;
    }
    pl.prog[pl.nprog++] = -1;  // both halves done: left + right
    --sp;
  }
}

// Called by every thread of the CTA; returns the sum to all of them.
template <class F>
__device__ double pw_sum_block(const F& v, int64_t n, const PwPlan& pl, double* leafval) {
  __shared__ double s_res;
  if (pl.nleaf < 0) {
    if (threadIdx.x == 0) s_res = pw_sum(v, 0, n);
    __syncthreads();
    const double r = s_res;
    __syncthreads();
    return r;
  }
  for (int l = threadIdx.x; l < pl.nleaf; l += blockDim.x) leafval[l] = pw_leaf(v, pl.off[l], pl.len[l]);
  __syncthreads();
  if (threadIdx.x == 0) {
    double st[64];
    int sp = 0;
    for (int t = 0; t < pl.nprog; ++t) {
      const int op = pl.prog[t];
      if (op >= 0) {
        st[sp++] = leafval[op];
      } else {
        const double b = st[--sp];
        st[sp - 1] = __dadd_rn(st[sp - 1], b);
      }
    }
    s_res = st[0];
  }
  __syncthreads();
  const double r = s_res;
  __syncthreads();  // s_res / leafval reused by the next call
  return r;
}

// (x * x).sum() of one row
__device__ double sq_row(const double* x, int d) {
  return pw_sum([x](int64_t t) { return __dmul_rn(x[t], x[t]); }, 0, d);
}

// the same on column j of a transposed (d x k) centroid block
__device__ double sq_col(const double* C, int64_t k, int j, int d) {
  return pw_sum([C, k, j](int64_t t) {
    const double x = C[t * k + j];
    return __dmul_rn(x, x);
  }, 0, d);
}

__device__ double sqdiff_col(const double* a, const double* C, int64_t k, int j, int d) {
  return pw_sum([a, C, k, j](int64_t t) {
    const double u = __dsub_rn(a[t], C[t * k + j]);
    return __dmul_rn(u, u);
  }, 0, d);
}

// sqdiff_col evaluated by the 8 lanes of an octet (8 <= d <= 128, pw_leaf's case): lane o
// keeps pw_leaf's accumulator r[o] (its coordinates o, o + 8, ... in order), the tree
// ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)) is built with xor shuffles (a + b == b + a
// exactly), and the d % 8 tail is added in order -- bit-identical to sqdiff_col, with the
// point's row read coalesced.  Every lane of the octet returns the sum.
__device__ double sqdiff_col_oct(const double* a, const double* C, int64_t k, int j, int d, int o) {
  const int n8 = d - d % 8;
  auto v = [a, C, k, j](int t) {
    const double u = __dsub_rn(a[t], C[(int64_t)t * k + j]);
    return __dmul_rn(u, u);
  };
  double r = v(o);
  for (int i = 8; i < n8; i += 8) r = __dadd_rn(r, v(i + o));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
  for (int i = n8; i < d; ++i) r = __dadd_rn(r, v(i));
  return r;
}

// seeding's D^2 update near[i] (= or min=) ||p_i - c_j||^2 over all points (whole CTA)
__device__ void d2_update(const double* __restrict__ P, int64_t n, int d, const double* C, int64_t k, int j,
                          double* near, bool first) {
  const int tid = threadIdx.x;
  if (d >= 8 && d <= 128) {  // four points per warp, one octet each
    const int lane = tid & 31, oct = lane >> 3, o = lane & 7;
    const int64_t per = (int64_t)(blockDim.x >> 5) * 4;
    for (int64_t base = (int64_t)(tid >> 5) * 4; base < n; base += per) {
      const int64_t i = base + oct;
      const double v = sqdiff_col_oct(P + (i < n ? i : n - 1) * d, C, k, j, d, o);
      if (o == 0 && i < n) near[i] = first ? v : fmin(near[i], v);
    }
  } else {
    for (int64_t i = tid; i < n; i += blockDim.x) {
      const double v = sqdiff_col(P + i * d, C, k, j, d);
      near[i] = first ? v : fmin(near[i], v);
    }
  }
}

__global__ void k_sqnorm(const double* __restrict__ X, int64_t rows, int d, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sq_row(X + i * d, d);
}

constexpr int kThreads = 1024;
constexpr int kQP = 4;  // points per warp in the Lloyd assignment

// Byte offsets of the per-replicate arrays in dynamic shared memory (-1: global slice).
// The seeding walks near/cdf sequentially in one thread and Lloyd scans lab per
// cluster, so those go to shared memory first, then the centroids.
struct SmemPlan {
  int64_t near = -1, cdf = -1, lab = -1, C = -1;
  size_t bytes = 0;
};

struct RepScratch {
  double* C;      // k x d centroids (global slice, used when they do not fit in shared memory)
  double* near;   // n: D^2 of the seeding / point_d2 of Lloyd
  double* cdf;    // n
  int* lab;       // n
  int* members;   // n: point indices grouped by cluster, point order within a cluster
};

__global__ void __launch_bounds__(kThreads) k_kmeans_rep(
    const double* __restrict__ P, const double* __restrict__ pp, int64_t n, int d, int k, const int64_t* first,
    const uint64_t* pcg, const double* init, int64_t max_iters, double tol, double* Cg, double* near_g, double* cdf_g,
    int* lab_g, int* mem_g, SmemPlan sp, int64_t* labels_out, double* centroids_out, double* inertia_out,
    int64_t* iters_out, int* status_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int r = blockIdx.x, tid = threadIdx.x;
  double* cc = reinterpret_cast<double*>(smem_raw);  // k
  int* counts = reinterpret_cast<int*>(cc + k);      // k
  int* offs = counts + k;                            // k
  // per-warp copy of the point being assigned (read once per point, not once per centroid chunk)
  double* pbuf = reinterpret_cast<double*>(smem_raw + (((size_t)k * 16 + 15) / 16) * 16);
  // centroids stored transposed (d x k): conflict-free shared-memory reads in the assignment
  double* C = sp.C >= 0 ? reinterpret_cast<double*>(smem_raw + sp.C) : Cg + (int64_t)r * k * d;
  double* near = sp.near >= 0 ? reinterpret_cast<double*>(smem_raw + sp.near) : near_g + (int64_t)r * n;
  double* cdf = sp.cdf >= 0 ? reinterpret_cast<double*>(smem_raw + sp.cdf) : cdf_g + (int64_t)r * n;
  int* lab = sp.lab >= 0 ? reinterpret_cast<int*>(smem_raw + sp.lab) : lab_g + (int64_t)r * n;
  int* members = mem_g + (int64_t)r * n;
  __shared__ int64_t s_pick;
  __shared__ double s_inertia;
  __shared__ int s_rep;
  __shared__ PwPlan s_plan;  // numpy's pairwise-sum tree over n points
  __shared__ double s_leaf[kMaxLeaves];
  int status = 0;
  if (tid == 0) pw_plan_build(s_plan, n);
  __syncthreads();

  if (first) {
    // ---- k-means++ seeding (kmeans.py:52-61)
    u128 st = 0, inc = 0;
    if (tid == 0) {
      st = make128(pcg[4 * r], pcg[4 * r + 1]);
      inc = make128(pcg[4 * r + 2], pcg[4 * r + 3]);
    }
    const double* p0 = P + first[r] * d;
    for (int t = tid; t < d; t += kThreads) C[(int64_t)t * k] = p0[t];
    __syncthreads();
    d2_update(P, n, d, C, k, 0, near, true);
    __syncthreads();
    for (int j = 1; j < k; ++j) {
      const double total_all = pw_sum_block([near](int64_t i) { return near[i]; }, n, s_plan, s_leaf);
      if (tid == 0) {
        const double total = total_all;
        s_pick = (total > 0.0 && total < INFINITY) ? 0 : -1;
        s_inertia = total;
      }
      __syncthreads();
      if (s_pick < 0) {
        status = 1;
        break;
      }
      const double total = s_inertia;
      for (int64_t i = tid; i < n; i += kThreads) cdf[i] = __ddiv_rn(near[i], total);  // p = d2 / total
      __syncthreads();
      if (tid == 0) {
        double acc = 0.0;  // cdf = p.cumsum() (sequential; loads batched ahead of the adds)
        int64_t i = 0;
        for (; i + 8 <= n; i += 8) {
          double v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = cdf[i + j];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            acc = __dadd_rn(acc, v[j]);
            cdf[i + j] = acc;
          }
        }
        for (; i < n; ++i) {
          acc = __dadd_rn(acc, cdf[i]);
          cdf[i] = acc;
        }
        const double u = pcg_next_double(st, inc);
        // searchsorted(cdf / cdf[-1], u, side='right'): first i with cdf[i]/last > u
        int64_t lo = 0, hi = n;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (__ddiv_rn(cdf[mid], acc) <= u) lo = mid + 1;
          else hi = mid;
        }
        s_pick = lo;
      }
      __syncthreads();
      const double* pj = P + s_pick * d;
      for (int t = tid; t < d; t += kThreads) C[(int64_t)t * k + j] = pj[t];
      __syncthreads();
      d2_update(P, n, d, C, k, j, near, false);
      __syncthreads();
    }
  } else {
    const double* ci = init + (int64_t)r * k * d;
    for (int64_t u = tid; u < (int64_t)k * d; u += kThreads) C[(u % d) * k + u / d] = ci[u];
    __syncthreads();
  }

  double inertia = INFINITY;
  int64_t iters = 0;
  if (status == 0) {
    for (int64_t i = tid; i < n; i += kThreads) lab[i] = 0;
    const double tiny = 2.2250738585072014e-308;
    const int lane = tid & 31, warp = tid >> 5;
    for (int64_t it = 0; it < max_iters; ++it) {
      for (int j = tid; j < k; j += kThreads) {
        cc[j] = sq_col(C, k, j, d);
        counts[j] = 0;
      }
      __syncthreads();
      // assignment: four points per warp (kQP), lanes over centroids, first argmin.  Each
      // (point, centroid) distance is the same sequential fma chain over the coordinates as
      // one point per warp; a centroid coordinate loaded once serves the four points, and the
      // points sit coordinate-major in pbuf ([t][q]: two 16-B broadcast loads per t).
      double* p4 = pbuf + (size_t)warp * kQP * d;
      for (int64_t i0 = (int64_t)warp * kQP; i0 < n; i0 += (int64_t)(kThreads / 32) * kQP) {
        for (int u = lane; u < kQP * d; u += 32) {  // the four rows are contiguous in P
          const int q = u / d, t = u - q * d;
          p4[t * kQP + q] = i0 + q < n ? P[i0 * d + u] : 0.0;
        }
        __syncwarp();
        double best[kQP], ppi[kQP];
        int bj[kQP];
#pragma unroll
        for (int q = 0; q < kQP; ++q) {
          best[q] = INFINITY;
          bj[q] = 0;
          ppi[q] = i0 + q < n ? pp[i0 + q] : 0.0;
        }
        for (int j0 = 0; j0 < k; j0 += 32) {
          const int j = j0 + lane;
          double dot[kQP];
#pragma unroll
          for (int q = 0; q < kQP; ++q) dot[q] = 0.0;
          if (j < k) {  // C is d x k: the warp's 32 centroids are contiguous per coordinate
            for (int t = 0; t < d; ++t) {
              const double c = C[(int64_t)t * k + j];
              const double2 pa = *reinterpret_cast<const double2*>(p4 + t * kQP);
              const double2 pb = *reinterpret_cast<const double2*>(p4 + t * kQP + 2);
              dot[0] = fma(pa.x, c, dot[0]);
              dot[1] = fma(pa.y, c, dot[1]);
              dot[2] = fma(pb.x, c, dot[2]);
              dot[3] = fma(pb.y, c, dot[3]);
            }
          }
#pragma unroll
          for (int q = 0; q < kQP; ++q) {
            double v = j < k ? fmax(__dsub_rn(__dadd_rn(ppi[q], cc[j]), 2.0 * dot[q]), 0.0) : INFINITY;
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
            if (v < best[q]) {  // strictly smaller: earlier chunks keep ties
              best[q] = v;
              bj[q] = vj;
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kQP; ++q)
          if (lane == q && i0 + q < n) {
            lab[i0 + q] = bj[q];
            near[i0 + q] = best[q];
            atomicAdd(&counts[bj[q]], 1);
          }
        __syncwarp();  // p4 is overwritten by the next points
      }
      __syncthreads();
      const double inert_all = pw_sum_block([near](int64_t i) { return near[i]; }, n, s_plan, s_leaf);
      if (tid == 0) {
        s_inertia = inert_all;
        int acc = 0;
        for (int j = 0; j < k; ++j) {
          offs[j] = acc;
          acc += counts[j];
        }
      }
      __syncthreads();
      // members of each cluster in point order
      for (int j = tid; j < k; j += kThreads) {
        int pos = offs[j];
        if (counts[j] > 0)
          for (int64_t i = 0; i < n; ++i)
            if (lab[i] == j) members[pos++] = (int)i;
      }
      __syncthreads();
      // centroid_j = points[labels == j].mean(axis=0): sum in point order, then / count
      for (int64_t u = tid; u < (int64_t)k * d; u += kThreads) {
        const int t = (int)(u / k), j = (int)(u % k);
        const int cnt = counts[j];
        if (cnt > 0) {
          const int* mj = members + offs[j];
          double s = 0.0;
          for (int m = 0; m < cnt; ++m) s = __dadd_rn(s, P[(int64_t)mj[m] * d + t]);
          C[(int64_t)t * k + j] = __ddiv_rn(s, (double)cnt);
        }
      }
      __syncthreads();
      if (tid == 0) {
        int rep = 0;
        for (int j = 0; j < k; ++j) {
          if (counts[j] > 0) continue;
          int64_t far = 0;  // first argmax of point_d2
          for (int64_t i = 1; i < n; ++i)
            if (near[i] > near[far]) far = i;
          for (int t = 0; t < d; ++t) C[(int64_t)t * k + j] = P[far * d + t];
          near[far] = 0.0;
          rep = 1;
        }
        s_rep = rep;
      }
      __syncthreads();
      const double ni = s_inertia;
      iters = it + 1;
      const bool settled = inertia - ni <= tol * fmax(ni, tiny);
      inertia = ni;
      if (!s_rep && settled) break;
      __syncthreads();  // s_inertia / s_rep reused next iteration
    }
  }
  for (int64_t i = tid; i < n; i += kThreads) labels_out[(int64_t)r * n + i] = status == 0 ? lab[i] : 0;
  if (centroids_out)
    for (int64_t u = tid; u < (int64_t)k * d; u += kThreads)
      centroids_out[(int64_t)r * k * d + u] = C[(u % d) * k + u / d];
  if (tid == 0) {
    inertia_out[r] = inertia;
    iters_out[r] = iters;
    status_out[r] = status;
  }
}

void run_replicates(const double* points, int64_t n, int d, int k, int reps, const int64_t* first,
                    const uint64_t* pcg, const double* init, int64_t max_iters, double tol, int64_t* labels_out,
                    double* centroids_out, double* inertia_out, int64_t* iters_out, int32_t* status_out, int device,
                    void* stream) {
  if (n < 1 || d < 1 || k < 1 || reps < 1) fail(CSC_ERR_INVALID, "kmeans: n, d, k and replicates must be >= 1");
  if (n < k) fail(CSC_ERR_INVALID, "need at least k points");
  if (n > INT32_MAX) fail(CSC_ERR_INVALID, "kmeans: too many points");
  if (!points || !labels_out || !inertia_out || !iters_out) fail(CSC_ERR_INVALID, "NULL buffer");
  if (!first && !init) fail(CSC_ERR_INVALID, "kmeans: need either seeding states or initial centroids");
  if (first && !pcg) fail(CSC_ERR_INVALID, "kmeans: seeding needs the PCG64 states");
  if (max_iters < 0) fail(CSC_ERR_INVALID, "max_iters must be >= 0");
  DeviceGuard dg(device);
  ensure_pool(device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (first)
    for (int r = 0; r < reps; ++r)
      if (first[r] < 0 || first[r] >= n) fail(CSC_ERR_INVALID, "kmeans: first centroid index out of range");
  DeviceView dP(points, sizeof(double) * n * d, device, s);
  DeviceView dFirst(first, first ? sizeof(int64_t) * reps : 0, device, s);
  DeviceView dPcg(pcg, first ? sizeof(uint64_t) * 4 * reps : 0, device, s);
  DeviceView dInit(first ? nullptr : init, first ? 0 : sizeof(double) * reps * k * d, device, s);
  const size_t c_bytes = sizeof(double) * k * d;
  // dynamic shared memory: the opt-in per-block maximum less the kernel's static arrays
  cudaFuncAttributes fa;
  CSC_CUDA(cudaFuncGetAttributes(&fa, k_kmeans_rep));
  int optin = 0;
  CSC_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  const size_t limit = (size_t)std::max<int64_t>(0, (int64_t)optin - (int64_t)fa.sharedSizeBytes - 1024);
  SmemPlan sp;
  sp.bytes = (((size_t)k * 16 + 15) / 16) * 16 + sizeof(double) * (kThreads / 32) * kQP * d;  // cc, counts, offs, points
  if (sp.bytes > limit) fail(CSC_ERR_INVALID, "kmeans: k or d too large for the device kernel");
  auto place = [&](int64_t& off, size_t bytes) {
    bytes = (bytes + 15) / 16 * 16;
    if (sp.bytes + bytes <= limit) {
      off = (int64_t)sp.bytes;
      sp.bytes += bytes;
    }
  };
  place(sp.near, sizeof(double) * n);
  place(sp.cdf, sizeof(double) * n);
  place(sp.lab, sizeof(int) * n);
  place(sp.C, c_bytes);
  const bool c_smem = sp.C >= 0;
  const size_t smem = sp.bytes;
  Scratch pp(sizeof(double) * n, s), Cg(c_smem ? 16 : c_bytes * reps, s), near(sizeof(double) * n * reps, s),
      cdf(sizeof(double) * n * reps, s), lab(sizeof(int) * n * reps, s), mem(sizeof(int) * n * reps, s),
      inert(sizeof(double) * reps, s), its(sizeof(int64_t) * reps, s), st(sizeof(int) * reps, s);
  DeviceOut dLab(labels_out, sizeof(int64_t) * n * reps, device, s);
  DeviceOut dCen(centroids_out, centroids_out ? c_bytes * reps : 0, device, s);
  k_sqnorm<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, s>>>(dP.as<double>(), n, d, pp.as<double>());
  CSC_LAUNCHED();
  CSC_CUDA(cudaFuncSetAttribute(k_kmeans_rep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_kmeans_rep<<<reps, kThreads, smem, s>>>(
      dP.as<double>(), pp.as<double>(), n, d, k, first ? dFirst.as<int64_t>() : nullptr,
      first ? dPcg.as<uint64_t>() : nullptr, first ? nullptr : dInit.as<double>(), max_iters, tol, Cg.as<double>(),
      near.as<double>(), cdf.as<double>(), lab.as<int>(), mem.as<int>(), sp, dLab.as<int64_t>(),
      centroids_out ? dCen.as<double>() : nullptr, inert.as<double>(), its.as<int64_t>(), st.as<int>());
  CSC_LAUNCHED();
  dLab.finish();
  if (centroids_out) dCen.finish();
  CSC_CUDA(cudaMemcpyAsync(inertia_out, inert.get(), sizeof(double) * reps, cudaMemcpyDefault, s));
  CSC_CUDA(cudaMemcpyAsync(iters_out, its.get(), sizeof(int64_t) * reps, cudaMemcpyDefault, s));
  std::vector<int32_t> hst(reps);
  CSC_CUDA(cudaMemcpyAsync(hst.data(), st.get(), sizeof(int) * reps, cudaMemcpyDeviceToHost, s));
  CSC_CUDA(cudaStreamSynchronize(s));
  if (status_out) std::copy(hst.begin(), hst.end(), status_out);
}

}  // namespace
}  // namespace csc

using namespace csc;

extern "C" int csc_kmeans_lloyd(const double* points, int64_t n, int d, const double* init, int k, int64_t max_iters,
                                double tol, int64_t* labels_out, double* centroids_out, double* inertia_out,
                                int64_t* iters_out, int device, void* stream) {
  return guard([&] {
    if (!init) fail(CSC_ERR_INVALID, "NULL buffer");
    double inertia = 0.0;
    int64_t iters = 0;
    run_replicates(points, n, d, k, 1, nullptr, nullptr, init, max_iters, tol, labels_out, centroids_out, &inertia,
                   &iters, nullptr, device, stream);
    if (inertia_out) *inertia_out = inertia;
    if (iters_out) *iters_out = iters;
  });
}

extern "C" int csc_kmeans_replicates(const double* points, int64_t n, int d, int k, int replicates,
                                     const int64_t* first_index, const uint64_t* pcg_states, const double* init,
                                     int64_t max_iters, double tol, int64_t* labels_out, double* centroids_out,
                                     double* inertia_out, int64_t* iters_out, int32_t* status_out, int device,
                                     void* stream) {
  return guard([&] {
    run_replicates(points, n, d, k, replicates, first_index, pcg_states, init, max_iters, tol, labels_out,
                   centroids_out, inertia_out, iters_out, status_out, device, stream);
  });
}
