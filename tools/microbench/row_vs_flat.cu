// Row-structured vs edge-balanced ("merge") gathers on the real graph, 128-B fp32 rows.
// One Chebyshev-step-shaped pass per launch: every row's neighbour rows summed and the row
// sum stored (evict-first), no S/X streams.  Three schedules, 8 CTAs x 256 threads per SM:
//   flat   edges in CSR order, 4 per warp slot, U slots in flight (no row structure, no store)
//   rows   k_cheb_mid's schedule: 4 rows per warp (8 lanes per row), the warp loops to its
//          longest row in chunks of 8 slots (indices loaded cooperatively, shuffled)
//   merge  4 rows per warp, but the warp's contiguous edge span is split into 4 equal
//          contiguous quarters, one per 8-lane group; a group's running sum is flushed to
//          shared memory when its quarter crosses a row boundary, and row k's owner group adds
//          the partials of the groups that touched row k (in group order) before the store
//
//   row_vs_flat <indptr.bin> <indices.bin> [repeats]     (tools/dump_csr.py writes the files)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o row_vs_flat row_vs_flat.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                          \
  do {                                                                 \
    cudaError_t e = (x);                                               \
    if (e != cudaSuccess) {                                            \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                   \
      exit(1);                                                         \
    }                                                                  \
  } while (0)

constexpr unsigned FULL = 0xffffffffu;

template <int U>
__global__ void __launch_bounds__(256, 8) k_flat(const float4* __restrict__ G, const int* __restrict__ idx, long nnz,
                                                 float* __restrict__ sink) {
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long e0 = warp * 4 * U; e0 < nnz; e0 += nw * 4 * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long e = e0 + u * 4 + grp;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < nnz) v[u] = __ldg(G + (size_t)__ldg(idx + e) * 8 + sub);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc.x += v[u].x;
      acc.y += v[u].y;
      acc.z += v[u].z;
      acc.w += v[u].w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[0] = acc.x;
}

// k_cheb_mid's row schedule (LPR 8, CH 8, one index per lane per chunk, next chunk's indices
// loaded before this chunk's gathers)
__global__ void __launch_bounds__(256, 8) k_rows(const float4* __restrict__ G, const int* __restrict__ indptr,
                                                 const int* __restrict__ idx, int n, float4* __restrict__ O) {
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  const int ngroups = (n + 3) / 4;
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  for (int gi = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); gi < ngroups; gi += nwarps) {
    const int row = gi * 4 + grp;
    int nbeg = 0, nend = 0;
    if (row < n) {
      nbeg = __ldg(indptr + row);
      nend = __ldg(indptr + row + 1);
    }
    const int cnt = nend - nbeg;
    const int maxcnt = __reduce_max_sync(FULL, cnt);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int jj = sub < cnt ? __ldcs(idx + nbeg + sub) : -1;
    for (int base = 0; base < maxcnt; base += 8) {
      const int e = base + 8 + sub;
      const int jn = (base + 8 < maxcnt && e < cnt) ? __ldcs(idx + nbeg + e) : -1;
      float4 gv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = __shfl_sync(FULL, jj, k, 8);
        gv[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j >= 0) gv[k] = __ldg(G + (uint32_t)j * 8u + sub);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        acc.x += gv[k].x;
        acc.y += gv[k].y;
        acc.z += gv[k].z;
        acc.w += gv[k].w;
      }
      jj = jn;
    }
    if (row < n) __stcs(O + (uint32_t)row * 8u + sub, acc);
  }
}

// k_rows without the store (the row sums only kept alive)
__global__ void __launch_bounds__(256, 8) k_rows_nostore(const float4* __restrict__ G, const int* __restrict__ indptr,
                                                         const int* __restrict__ idx, int n, float* __restrict__ sink) {
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  const int ngroups = (n + 3) / 4;
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  float4 tot = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int gi = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); gi < ngroups; gi += nwarps) {
    const int row = gi * 4 + grp;
    int nbeg = 0, nend = 0;
    if (row < n) {
      nbeg = __ldg(indptr + row);
      nend = __ldg(indptr + row + 1);
    }
    const int cnt = nend - nbeg;
    const int maxcnt = __reduce_max_sync(FULL, cnt);
    int jj = sub < cnt ? __ldcs(idx + nbeg + sub) : -1;
    for (int base = 0; base < maxcnt; base += 8) {
      const int e = base + 8 + sub;
      const int jn = (base + 8 < maxcnt && e < cnt) ? __ldcs(idx + nbeg + e) : -1;
      float4 gv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = __shfl_sync(FULL, jj, k, 8);
        gv[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j >= 0) gv[k] = __ldg(G + (uint32_t)j * 8u + sub);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        tot.x += gv[k].x;
        tot.y += gv[k].y;
        tot.z += gv[k].z;
        tot.w += gv[k].w;
      }
      jj = jn;
    }
  }
  if (tot.x + tot.y + tot.z + tot.w == 12345.f) sink[0] = tot.x;
}

// two consecutive rows per 8-lane group, streamed back to back (8 rows per warp)
__global__ void __launch_bounds__(256, 8) k_rows2(const float4* __restrict__ G, const int* __restrict__ indptr,
                                                  const int* __restrict__ idx, int n, float4* __restrict__ O) {
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  const int ngroups = (n + 7) / 8;
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  for (int gi = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); gi < ngroups; gi += nwarps) {
    const int ra = gi * 8 + 2 * grp;
    const int sa = __ldg(indptr + min(ra, n)), m = __ldg(indptr + min(ra + 1, n)), s1 = __ldg(indptr + min(ra + 2, n));
    const int cnt = s1 - sa;
    const int maxcnt = __reduce_max_sync(FULL, cnt);
    float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
    int jj = sub < cnt ? __ldcs(idx + sa + sub) : -1;
    for (int base = 0; base < maxcnt; base += 8) {
      const int e = base + 8 + sub;
      const int jn = (base + 8 < maxcnt && e < cnt) ? __ldcs(idx + sa + e) : -1;
      float4 gv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = __shfl_sync(FULL, jj, k, 8);
        gv[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j >= 0) gv[k] = __ldg(G + (uint32_t)j * 8u + sub);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (sa + base + k < m) {
          a0.x += gv[k].x;
          a0.y += gv[k].y;
          a0.z += gv[k].z;
          a0.w += gv[k].w;
        } else {
          a1.x += gv[k].x;
          a1.y += gv[k].y;
          a1.z += gv[k].z;
          a1.w += gv[k].w;
        }
      }
      jj = jn;
    }
    if (ra < n) __stcs(O + (uint32_t)ra * 8u + sub, a0);
    if (ra + 1 < n) __stcs(O + (uint32_t)(ra + 1) * 8u + sub, a1);
  }
}

// k_rows with a choice of output store: 0 st.global.cs (evict-first, as K2), 1 st.global (write-back),
// 2 st.global into a 1 MB window (stays in L2: the store's issue cost without DRAM write-back),
// 3 per-warp TMA bulk store of the warp's 4 rows (512 contiguous bytes) staged in shared memory
template <int MODE>
__global__ void __launch_bounds__(256, 8) k_rows_st(const float4* __restrict__ G, const int* __restrict__ indptr,
                                                    const int* __restrict__ idx, int n, float4* __restrict__ O) {
  __shared__ __align__(128) float4 stage[8][2][32];  // [warp][buffer][lane]: 4 rows x 128 B
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3, wib = threadIdx.x >> 5;
  const int ngroups = (n + 3) / 4;
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  int it = 0;
  for (int gi = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); gi < ngroups; gi += nwarps, ++it) {
    const int row = gi * 4 + grp;
    int nbeg = 0, nend = 0;
    if (row < n) {
      nbeg = __ldg(indptr + row);
      nend = __ldg(indptr + row + 1);
    }
    const int cnt = nend - nbeg;
    const int maxcnt = __reduce_max_sync(FULL, cnt);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int jj = sub < cnt ? __ldcs(idx + nbeg + sub) : -1;
    for (int base = 0; base < maxcnt; base += 8) {
      const int e = base + 8 + sub;
      const int jn = (base + 8 < maxcnt && e < cnt) ? __ldcs(idx + nbeg + e) : -1;
      float4 gv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = __shfl_sync(FULL, jj, k, 8);
        gv[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j >= 0) gv[k] = __ldg(G + (uint32_t)j * 8u + sub);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        acc.x += gv[k].x;
        acc.y += gv[k].y;
        acc.z += gv[k].z;
        acc.w += gv[k].w;
      }
      jj = jn;
    }
    if constexpr (MODE == 0) {
      if (row < n) __stcs(O + (uint32_t)row * 8u + sub, acc);
    } else if constexpr (MODE == 1) {
      if (row < n) O[(uint32_t)row * 8u + sub] = acc;
    } else if constexpr (MODE == 2) {
      if (row < n) O[((uint32_t)row & 8191u) * 8u + sub] = acc;
    } else {
      const int b = it & 1;
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // buffer b free again
      __syncwarp();
      stage[wib][b][lane] = acc;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0 && gi * 4 + 4 <= n) {
        const uint32_t src = (uint32_t)__cvta_generic_to_shared(&stage[wib][b][0]);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(O + (size_t)gi * 32), "r"(src)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
  }
  if constexpr (MODE == 3) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// edge-balanced: the warp's 4 rows' contiguous edge span in 4 equal quarters
__global__ void __launch_bounds__(256, 8) k_merge(const float4* __restrict__ G, const int* __restrict__ indptr,
                                                  const int* __restrict__ idx, int n, float4* __restrict__ O) {
  __shared__ float4 part[8][4][4][8];  // [warp][group][row][lane]
  __shared__ int sb[8][8];             // [warp][k] = indptr[r0 + k], k = 0..4
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3, wib = threadIdx.x >> 5;
  const int ngroups = (n + 3) / 4;
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  for (int gi = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); gi < ngroups; gi += nwarps) {
    const int r0 = gi * 4;
    __syncwarp();
    if (lane < 5) sb[wib][lane] = __ldg(indptr + min(r0 + lane, n));
    __syncwarp();
    const int b0 = sb[wib][0], T = sb[wib][4] - b0;
    const int s0 = b0 + (T * grp) / 4, s1 = b0 + (T * (grp + 1)) / 4;  // this group's quarter
    const int len = s1 - s0;
    const int maxlen = __reduce_max_sync(FULL, len);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int cur = 0;  // row of the quarter's next edge, and that row's end
    while (cur < 3 && s0 >= sb[wib][cur + 1]) ++cur;
    int nextb = sb[wib][cur + 1];
    int jj = sub < len ? __ldcs(idx + s0 + sub) : -1;
    for (int base = 0; base < maxlen; base += 8) {
      const int e = base + 8 + sub;
      const int jn = (base + 8 < maxlen && e < len) ? __ldcs(idx + s0 + e) : -1;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float4 gv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int j = __shfl_sync(FULL, jj, 4 * h + k, 8);
          gv[k] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (j >= 0) gv[k] = __ldg(G + (uint32_t)j * 8u + sub);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int ee = s0 + base + 4 * h + k;
          if (ee < s1) {
            if (ee >= nextb) {
              part[wib][grp][cur][sub] = acc;
              acc = make_float4(0.f, 0.f, 0.f, 0.f);
              do {
                ++cur;
                nextb = sb[wib][cur + 1];
              } while (ee >= nextb);
            }
            acc.x += gv[k].x;
            acc.y += gv[k].y;
            acc.z += gv[k].z;
            acc.w += gv[k].w;
          }
        }
      }
      jj = jn;
    }
    if (len > 0) part[wib][grp][cur][sub] = acc;
    __syncwarp();
    // row grp: edges [bk, bk1), touched by the quarters that overlap it
    const int bk = sb[wib][grp], bk1 = sb[wib][grp + 1];
    const int row = r0 + grp;
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    if (bk1 > bk) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int q0 = b0 + (T * q) / 4, q1 = b0 + (T * (q + 1)) / 4;
        if (q0 < bk1 && q1 > bk && q1 > q0) {
          const float4 p = part[wib][q][grp][sub];
          sum.x += p.x;
          sum.y += p.y;
          sum.z += p.z;
          sum.w += p.w;
        }
      }
    }
    if (row < n) __stcs(O + (uint32_t)row * 8u + sub, sum);
  }
}

static std::vector<int> load(const char* path) {
  FILE* f = fopen(path, "rb");
  if (!f) {
    printf("cannot open %s\n", path);
    exit(1);
  }
  fseek(f, 0, SEEK_END);
  long bytes = ftell(f);
  fseek(f, 0, SEEK_SET);
  std::vector<int> v(bytes / 4);
  if (fread(v.data(), 4, v.size(), f) != v.size()) exit(1);
  fclose(f);
  return v;
}

template <typename F>
static double timeit(F launch, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  launch();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) launch();
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  CK(cudaGetLastError());
  return 1e3 * ms / reps;
}

int main(int argc, char** argv) {
  if (argc < 3) {
    printf("usage: %s indptr.bin indices.bin [repeats]\n", argv[0]);
    return 1;
  }
  std::vector<int> ip = load(argv[1]), ix = load(argv[2]);
  const int reps = argc > 3 ? atoi(argv[3]) : 20;
  const int n = (int)ip.size() - 1;
  const long nnz = (long)ix.size();
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  printf("N=%d nnz=%ld (mean degree %.2f), %d SMs, 128-B rows\n", n, nnz, (double)nnz / n, sms);
  float4 *G, *O1, *O2;
  float* sink;
  int *dip, *dix;
  const size_t panel = (size_t)n * 8 * sizeof(float4);
  CK(cudaMalloc(&G, panel));
  CK(cudaMalloc(&O1, panel));
  CK(cudaMalloc(&O2, panel));
  {
    std::vector<float> h((size_t)n * 32);
    uint32_t x = 12345u;
    for (auto& v : h) {
      x = x * 1664525u + 1013904223u;
      v = (float)(x >> 8) * (1.0f / 16777216.0f) - 0.5f;
    }
    CK(cudaMemcpy(G, h.data(), panel, cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&sink, 64));
  CK(cudaMalloc(&dip, sizeof(int) * (n + 1)));
  CK(cudaMalloc(&dix, sizeof(int) * nnz));
  CK(cudaMemcpy(dip, ip.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dix, ix.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice));
  const int grid = sms * 8;
  for (int round = 0; round < 2; ++round) {
    printf("flat  U=4  %8.1f us\n", timeit([&] { k_flat<4><<<grid, 256>>>(G, dix, nnz, sink); }, reps));
    printf("rows       %8.1f us\n", timeit([&] { k_rows<<<grid, 256>>>(G, dip, dix, n, O1); }, reps));
    printf("merge      %8.1f us\n", timeit([&] { k_merge<<<grid, 256>>>(G, dip, dix, n, O2); }, reps));
    printf("rows nostr %8.1f us\n", timeit([&] { k_rows_nostore<<<grid, 256>>>(G, dip, dix, n, sink); }, reps));
    printf("rows2      %8.1f us\n", timeit([&] { k_rows2<<<grid, 256>>>(G, dip, dix, n, O1); }, reps));
    printf("rows st.cs %8.1f us\n", timeit([&] { k_rows_st<0><<<grid, 256>>>(G, dip, dix, n, O1); }, reps));
    printf("rows st.wb %8.1f us\n", timeit([&] { k_rows_st<1><<<grid, 256>>>(G, dip, dix, n, O1); }, reps));
    printf("rows st1MB %8.1f us\n", timeit([&] { k_rows_st<2><<<grid, 256>>>(G, dip, dix, n, O1); }, reps));
    printf("rows tma   %8.1f us\n", timeit([&] { k_rows_st<3><<<grid, 256>>>(G, dip, dix, n, O2); }, reps));
  }
  k_rows<<<grid, 256>>>(G, dip, dix, n, O1);  // O1 = rows, O2 = TMA-stored rows
  CK(cudaDeviceSynchronize());
  // the two schedules sum the same rows (different association): compare
  std::vector<float> a((size_t)n * 32), b((size_t)n * 32);
  CK(cudaMemcpy(a.data(), O1, panel, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b.data(), O2, panel, cudaMemcpyDeviceToHost));
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (double)(a[i] - b[i]) * (a[i] - b[i]);
    den += (double)a[i] * a[i];
  }
  printf("tma-stored vs rows: relative difference %.3e\n", std::sqrt(num / (den > 0 ? den : 1.0)));
  return 0;
}
