// Speed of light of K2's gathers on the real graph: read every CSR entry's neighbour row
// (the `valid` leading floats of a `stride`-float panel row) in CSR order, exactly the
// gather stream of one Chebyshev step, with nothing else (no S/X/O streams, no epilogue).
//
//   csr_gather_sol <indptr.bin> <indices.bin> [repeats]
//
// indptr/indices: raw int32 files (tools/dump_csr.py writes them for a BASELINE config).
// Each configuration: LPR lanes (16 B each) per edge, 32/LPR edges per warp, U edges in
// flight per lane group, B CTAs of 256 threads per SM (grid-stride).  Prints the time per
// pass, row gathers/s and gathered bytes/s (valid bytes).  Also times a sequential copy of
// the panel (HBM reference) for the same bytes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o csr_gather_sol csr_gather_sol.cu
#include <cuda_runtime.h>

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

template <int LPR, int U>
__global__ void __launch_bounds__(256) k_gather(const float* __restrict__ G, int stride, int valid,
                                                const int* __restrict__ idx, long nnz, float* __restrict__ sink) {
  constexpr int EPW = 32 / LPR;  // edges per warp per slot
  const int lane = threadIdx.x & 31, sub = lane % LPR, grp = lane / LPR;
  const bool on = grp < EPW && sub * 4 < valid;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long e0 = warp * EPW * U; e0 < nnz; e0 += nw * EPW * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long e = e0 + u * EPW + grp;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (on && e < nnz) v[u] = __ldg(reinterpret_cast<const float4*>(G + (size_t)__ldg(idx + e) * stride) + sub);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc.x += v[u].x;
      acc.y += v[u].y;
      acc.z += v[u].z;
      acc.w += v[u].w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[0] = acc.x;  // keep the loads alive
}

// 32-byte lanes: ld.global.nc.v8.f32 (LDG.E.ENL2.256), LPR lanes of 32 B per row
template <int LPR, int U>
__global__ void __launch_bounds__(256) k_gather8(const float* __restrict__ G, int stride, int valid,
                                                 const int* __restrict__ idx, long nnz, float* __restrict__ sink) {
  constexpr int EPW = 32 / LPR;
  const int lane = threadIdx.x & 31, sub = lane % LPR, grp = lane / LPR;
  const bool on = grp < EPW && sub * 8 < valid;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (long e0 = warp * EPW * U; e0 < nnz; e0 += nw * EPW * U) {
    float v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long e = e0 + u * EPW + grp;
#pragma unroll
      for (int c = 0; c < 8; ++c) v[u][c] = 0.f;
      if (on && e < nnz) {
        const float* p = G + (size_t)__ldg(idx + e) * stride + sub * 8;
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3]), "=f"(v[u][4]), "=f"(v[u][5]),
                       "=f"(v[u][6]), "=f"(v[u][7])
                     : "l"(p));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] += v[u][c];
  }
  float t = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) t += acc[c];
  if (t == 12345.f) sink[0] = t;
}

template <int LPR, int U>
static void run8(const float* G, int stride, int valid, const int* idx, long nnz, long n, float* sink, int blocks_per_sm,
                 int sms, int reps, const char* tag) {
  const int grid = sms * blocks_per_sm;
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gather8<LPR, U>, 256, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_gather8<LPR, U><<<grid, 256>>>(G, stride, valid, idx, nnz, sink);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) k_gather8<LPR, U><<<grid, 256>>>(G, stride, valid, idx, nnz, sink);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double us = 1e3 * ms / reps;
  printf("%-8s v8 (32-B lanes) stride %3d valid %3d  LPR %2d U %d  %d CTAs/SM (resident %d)  %8.1f us/pass  %6.2f G rows/s\n",
         tag, stride, valid, LPR, U, blocks_per_sm, occ, us, nnz / us / 1e3);
  CK(cudaEventDestroy(e0));
  CK(cudaEventDestroy(e1));
}

// cp.async ring: per warp D batches of B slots (slot = 32 lanes x 16 B = EPW edges' row slices).
// Gathers land in shared memory, so the in-flight depth is not bounded by registers; the
// neighbour indices of a batch are loaded one iteration before its copies are issued.
template <int LPR, int D>
__global__ void __launch_bounds__(256) k_gather_cpa(const float* __restrict__ G, int stride, int valid,
                                                    const int* __restrict__ idx, long nnz, float* __restrict__ sink) {
  constexpr int EPW = 32 / LPR, B = 4;
  extern __shared__ float4 ring[];  // [warps][D][B][32]
  const int lane = threadIdx.x & 31, sub = lane % LPR, grp = lane / LPR, wib = threadIdx.x >> 5;
  const bool on = grp < EPW && sub * 4 < valid;
  float4* my = ring + (size_t)wib * D * B * 32;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  // batch t of this warp covers edges ((warp + t * nw) * B + b) * EPW + grp, b < B
  auto edge = [&](long t, int b) { return ((warp + t * nw) * B + b) * EPW + grp; };
  int nxt[B];
  auto load_idx = [&](long t) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const long e = edge(t, b);
      nxt[b] = (on && e < nnz) ? __ldg(idx + e) : -1;
    }
  };
  auto issue = [&](int slot) {
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (nxt[b] >= 0) {
        const float4* src = reinterpret_cast<const float4*>(G + (size_t)nxt[b] * stride) + sub;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(my + (slot * B + b) * 32 + lane)),
                     "l"(src)
                     : "memory");
      }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const long nb = (nnz / (EPW * B) + nw) / nw + 1;
  for (int t = 0; t < D - 1; ++t) {
    load_idx(t);
    issue(t);
  }
  load_idx(D - 1);
  for (long t = 0; t < nb; ++t) {
    issue((int)((t + D - 1) % D));
    load_idx(t + D);
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const long e = edge(t, b);
      if (on && e < nnz) {
        const float4 v = my[((t % D) * B + b) * 32 + lane];
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[0] = acc.x;
}

template <int LPR, int D>
static void run_cpa(const float* G, int stride, int valid, const int* idx, long nnz, long n, float* sink,
                    int blocks_per_sm, int sms, int reps, const char* tag) {
  const int grid = sms * blocks_per_sm;
  const size_t smem = (size_t)8 * D * 4 * 32 * 16;
  CK(cudaFuncSetAttribute(k_gather_cpa<LPR, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gather_cpa<LPR, D>, 256, smem));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_gather_cpa<LPR, D><<<grid, 256, smem>>>(G, stride, valid, idx, nnz, sink);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) k_gather_cpa<LPR, D><<<grid, 256, smem>>>(G, stride, valid, idx, nnz, sink);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double us = 1e3 * ms / reps;
  const int vb = ((valid + 3) / 4) * 16;
  printf("%-8s cp.async ring D=%2d  stride %3d valid %3d  LPR %2d  %d CTAs/SM (resident %d, %zu KB smem/CTA)  %8.1f us/pass  "
         "%6.2f G rows/s  %6.2f TB/s valid\n",
         tag, D, stride, valid, LPR, blocks_per_sm, occ, smem / 1024, us, nnz / us / 1e3, nnz * (double)vb / us / 1e6);
  CK(cudaEventDestroy(e0));
  CK(cudaEventDestroy(e1));
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
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

template <int LPR, int U>
static void run(const float* G, int stride, int valid, const int* idx, long nnz, long n, float* sink, int blocks_per_sm,
                int sms, int reps, const char* tag) {
  const int grid = sms * blocks_per_sm;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gather<LPR, U>, 256, 0));
  if (occ < blocks_per_sm) printf("  (only %d CTAs/SM resident)\n", occ);
  k_gather<LPR, U><<<grid, 256>>>(G, stride, valid, idx, nnz, sink);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) k_gather<LPR, U><<<grid, 256>>>(G, stride, valid, idx, nnz, sink);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double us = 1e3 * ms / reps;
  const int vb = ((valid + 3) / 4) * 16;
  printf("%-8s stride %3d floats valid %3d  LPR %2d U %d  %2d CTAs/SM  %8.1f us/pass  %6.2f G rows/s  %6.2f TB/s valid  "
         "(panel %.0f MB)\n",
         tag, stride, valid, LPR, U, blocks_per_sm, us, nnz / us / 1e3, nnz * (double)vb / us / 1e6,
         n * (double)stride * 4 / 1e6);
  CK(cudaEventDestroy(e0));
  CK(cudaEventDestroy(e1));
}

int main(int argc, char** argv) {
  if (argc < 3) {
    printf("usage: %s indptr.bin indices.bin [repeats]\n", argv[0]);
    return 1;
  }
  std::vector<int> ip = load(argv[1]), ix = load(argv[2]);
  const int reps = argc > 3 ? atoi(argv[3]) : 10;
  const long n = (long)ip.size() - 1, nnz = (long)ix.size();
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  printf("N=%ld nnz=%ld (mean degree %.2f), %d SMs\n", n, nnz, (double)nnz / n, sms);
  float *G, *sink, *B;
  int* idx;
  const size_t panel = (size_t)n * 128 * sizeof(float);
  CK(cudaMalloc(&G, panel));
  CK(cudaMalloc(&B, panel));
  {
    std::vector<float> h((size_t)n * 128);
    uint32_t x = 12345u;
    for (auto& v : h) {
      x = x * 1664525u + 1013904223u;
      v = (float)(x >> 8) * (1.0f / 16777216.0f) - 0.5f;
    }
    CK(cudaMemcpy(G, h.data(), panel, cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&sink, 64));
  CK(cudaMalloc(&idx, sizeof(int) * nnz));
  CK(cudaMemcpy(idx, ix.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice));

  // sequential HBM reference: copy of the N x 64 fp32 panel
  {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const long n4 = n * 64 / 4;
    k_copy<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(G), reinterpret_cast<float4*>(B), n4);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r)
      k_copy<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(G), reinterpret_cast<float4*>(B), n4);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("copy     N x 64 fp32 panel: %.1f us, %.2f TB/s (read + write)\n", 1e3 * ms / reps,
           2.0 * n4 * 16 / (1e-3 * ms / reps) / 1e12);
  }
  const bool quick = getenv("SOL_QUICK") != nullptr;
  if (getenv("SOL_SPLIT")) {
    // source-split passes: the edges into each of P source ranges, in CSR order, one pass per
    // range (a range's gather rows can stay in L2 while its pass runs)
    for (int P : {1, 2, 3, 4}) {
      std::vector<std::vector<int>> parts(P);
      for (long e = 0; e < nnz; ++e) parts[(long)ix[e] * P / n].push_back(ix[e]);
      double tot = 0.0;
      for (int q = 0; q < P; ++q) {
        int* d = nullptr;
        CK(cudaMalloc(&d, sizeof(int) * parts[q].size()));
        CK(cudaMemcpy(d, parts[q].data(), sizeof(int) * parts[q].size(), cudaMemcpyHostToDevice));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        k_gather<16, 4><<<sms * 6, 256>>>(G, 64, 56, d, (long)parts[q].size(), sink);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int r = 0; r < reps; ++r) k_gather<16, 4><<<sms * 6, 256>>>(G, 64, 56, d, (long)parts[q].size(), sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        tot += 1e3 * ms / reps;
        CK(cudaFree(d));
      }
      printf("split P=%d: d=56 (64-float stride) gathers in %d source ranges of %.0f MB: %.1f us total\n", P, P,
             n * 256.0 / P / 1e6, tot);
    }
    return 0;
  }
  run<16, 4>(G, 64, 56, idx, nnz, n, sink, 6, sms, reps, "d=56");
  run<16, 4>(G, 64, 56, idx, nnz, n, sink, 8, sms, reps, "d=56");
  run<16, 6>(G, 64, 56, idx, nnz, n, sink, 6, sms, reps, "d=56");
  run_cpa<16, 2>(G, 64, 56, idx, nnz, n, sink, 6, sms, reps, "d=56");
  run_cpa<16, 2>(G, 64, 56, idx, nnz, n, sink, 4, sms, reps, "d=56");
  run_cpa<16, 3>(G, 64, 56, idx, nnz, n, sink, 4, sms, reps, "d=56");
  run_cpa<16, 4>(G, 64, 56, idx, nnz, n, sink, 3, sms, reps, "d=56");
  run_cpa<16, 6>(G, 64, 56, idx, nnz, n, sink, 2, sms, reps, "d=56");
  run_cpa<8, 2>(G, 32, 28, idx, nnz, n, sink, 6, sms, reps, "d=28");
  run_cpa<8, 3>(G, 32, 28, idx, nnz, n, sink, 4, sms, reps, "d=28");
  run8<8, 1>(G, 64, 56, idx, nnz, n, sink, 6, sms, reps, "d=56");
  run8<8, 2>(G, 64, 56, idx, nnz, n, sink, 6, sms, reps, "d=56");
  run8<8, 2>(G, 64, 56, idx, nnz, n, sink, 8, sms, reps, "d=56");
  run8<8, 3>(G, 64, 56, idx, nnz, n, sink, 6, sms, reps, "d=56");
  run8<8, 4>(G, 64, 56, idx, nnz, n, sink, 4, sms, reps, "d=56");
  run8<4, 2>(G, 32, 28, idx, nnz, n, sink, 6, sms, reps, "d=28");
  run8<4, 2>(G, 32, 28, idx, nnz, n, sink, 8, sms, reps, "d=28");
  run<8, 4>(G, 32, 28, idx, nnz, n, sink, 6, sms, reps, "d=28");
  if (quick) return 0;
  // K2's layouts: d=56 (one 64-wide panel), d=36 (64-wide), d=28 (32-wide), 16-wide, 128-wide
  for (int bps : {6, 8}) {
    run<16, 4>(G, 64, 56, idx, nnz, n, sink, bps, sms, reps, "d=56");
    run<16, 8>(G, 64, 56, idx, nnz, n, sink, bps, sms, reps, "d=56");
    run<16, 4>(G, 64, 36, idx, nnz, n, sink, bps, sms, reps, "d=36");
    run<16, 4>(G, 64, 64, idx, nnz, n, sink, bps, sms, reps, "d=64");
    run<8, 4>(G, 32, 28, idx, nnz, n, sink, bps, sms, reps, "d=28");
    run<8, 8>(G, 32, 28, idx, nnz, n, sink, bps, sms, reps, "d=28");
    run<4, 4>(G, 16, 16, idx, nnz, n, sink, bps, sms, reps, "d=16");
    run<32, 4>(G, 128, 100, idx, nnz, n, sink, bps, sms, reps, "d=100");
  }
  // compact 56-float stride (no padding): LPR 14 lanes active of 16
  run<16, 4>(G, 56, 56, idx, nnz, n, sink, 6, sms, reps, "d=56c");
  run<16, 8>(G, 56, 56, idx, nnz, n, sink, 8, sms, reps, "d=56c");
  return 0;
}
