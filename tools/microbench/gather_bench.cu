// Gather microbenchmark: random 64-byte row gathers from an L2-sized panel.
//   A: LDG.128 per lane (4 lanes per row), 4 gathers in flight per lane (the K2 scheme)
//   B: TMA tile::gather4 into shared memory, mbarrier completion, 1 issuing lane per row
//   C: cp.async (LDGSTS.128, L2-only) into a per-warp ring of STAGES chunk buffers
//      (8 rows x 4 neighbours x 64 B = 2 KB each): in-flight depth set by shared memory
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int PW = 16;      // floats per row (64 B)
constexpr int DEG = 16;     // neighbours per row

__global__ void k_ldg(const float* __restrict__ G, const int* __restrict__ idx, int n, float* __restrict__ out) {
  const int lane = threadIdx.x & 31, sub = lane & 3, grp = lane >> 2;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long rb = warp * 8; rb < n; rb += nw * 8) {
    const long row = rb + grp;
    float4 acc = make_float4(0, 0, 0, 0);
    if (row < n) {
      for (int e = 0; e < DEG; e += 4) {
        float4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = __ldg(reinterpret_cast<const float4*>(G + (size_t)idx[row * DEG + e + k] * PW) + sub);
#pragma unroll
        for (int k = 0; k < 4; ++k) { acc.x += v[k].x; acc.y += v[k].y; acc.z += v[k].z; acc.w += v[k].w; }
      }
      reinterpret_cast<float4*>(out + row * PW)[sub] = acc;
    }
  }
}

__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* map, int r0, int r1, int r2, int r3, uint32_t mbar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               :: "r"(dst), "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(b), "r"(phase) : "memory");
}

// B: each warp handles 8 rows per batch; batch = 8 rows x 16 nbrs x 64 B = 8 KB smem; STAGES batches in flight.
template <int STAGES>
__global__ void __launch_bounds__(128) k_tma(const __grid_constant__ CUtensorMap map, const int* __restrict__ idx, int n, float* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, sub = lane & 3, grp = lane >> 2;
  unsigned char* wbuf = smem + (size_t)wid * STAGES * 8192;
  __shared__ __align__(8) uint64_t bars[4][STAGES];
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bars[wid][s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const long nbatch = (n + 7) / 8;
  // batches for this warp: b = warp, warp + nw, ...
  auto issue = [&](long b, int s) {
    uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[wid][s]);
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(8192) : "memory");
    __syncwarp();
    // 32 gather4 per batch (8 rows x 4 groups of 4 nbrs): lane l issues one
    const long row = b * 8 + (lane >> 2);
    const int q = lane & 3;
    const int* ip = idx + (row < n ? row : 0) * DEG + q * 4;
    uint32_t dst = (uint32_t)__cvta_generic_to_shared(wbuf + s * 8192 + ((lane >> 2) * DEG + q * 4) * 64);
    gather4(dst, &map, ip[0], ip[1], ip[2], ip[3], bar);
  };
  int s = 0; uint32_t phase[STAGES] = {0};
  long b = warp;
  long bi = warp;
  for (int k = 0; k < STAGES - 1 && bi < nbatch; ++k, bi += nw) issue(bi, k);
  int cs = 0;
  for (; b < nbatch; b += nw) {
    if (bi < nbatch) { issue(bi, (cs + STAGES - 1) % STAGES); }
    bi += nw;
    mbar_wait((uint32_t)__cvta_generic_to_shared(&bars[wid][cs]), phase[cs]);
    phase[cs] ^= 1;
    const float4* rowbuf = reinterpret_cast<const float4*>(wbuf + cs * 8192 + grp * DEG * 64);
    float4 acc = make_float4(0, 0, 0, 0);
#pragma unroll
    for (int e = 0; e < DEG; ++e) { float4 v = rowbuf[e * 4 + sub]; acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
    const long row = b * 8 + grp;
    if (row < n) reinterpret_cast<float4*>(out + row * PW)[sub] = acc;
    __syncwarp();
    cs = (cs + 1) % STAGES;
  }
}

// C: work item = (row batch of 8, chunk of 4 neighbours); items of a warp are pipelined
template <int STAGES>
__global__ void __launch_bounds__(256) k_cpasync(const float* __restrict__ G, const int* __restrict__ idx, int n,
                                                  float* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, sub = lane & 3, grp = lane >> 2;
  unsigned char* ring = smem + (size_t)wid * STAGES * 2048;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  const long nbatch = (n + 7) / 8;
  const long mybatches = warp < nbatch ? (nbatch - warp + nw - 1) / nw : 0;
  const long items = mybatches * (DEG / 4);
  auto issue = [&](long it) {
    if (it < items) {
      const long b = warp + (it / (DEG / 4)) * nw;
      const int e = (int)(it % (DEG / 4));
      const long row = b * 8 + grp;
      const int st = (int)(it % STAGES);
      const uint32_t base = (uint32_t)__cvta_generic_to_shared(ring + st * 2048 + grp * 256 + sub * 16);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = row < n ? idx[row * DEG + e * 4 + k] : 0;
        const float* src = G + (size_t)j * PW + sub * 4;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(base + k * 64), "l"(src) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int k = 0; k < STAGES - 1; ++k) issue(k);
  float4 acc = make_float4(0, 0, 0, 0);
  for (long it = 0; it < items; ++it) {
    issue(it + STAGES - 1);
    asm volatile("cp.async.wait_group %0;" :: "n"(STAGES - 1) : "memory");
    __syncwarp();
    const float4* buf = reinterpret_cast<const float4*>(ring + (it % STAGES) * 2048 + grp * 256);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 v = buf[k * 4 + sub];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if ((it % (DEG / 4)) == DEG / 4 - 1) {
      const long row = (warp + (it / (DEG / 4)) * nw) * 8 + grp;
      if (row < n) reinterpret_cast<float4*>(out + row * PW)[sub] = acc;
      acc = make_float4(0, 0, 0, 0);
    }
    __syncwarp();
  }
}

int main() {
  const int n = 1000000;
  std::vector<int> h(n * (size_t)DEG);
  std::mt19937 rng(1);
  for (auto& v : h) v = rng() % n;
  float *G, *out; int* idx;
  CK(cudaMalloc(&G, sizeof(float) * n * PW)); CK(cudaMalloc(&out, sizeof(float) * n * PW));
  CK(cudaMalloc(&idx, sizeof(int) * h.size()));
  CK(cudaMemcpy(idx, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(G, 0, sizeof(float) * n * PW));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto report = [&](const char* name, float ms) {
    double bytes = (double)n * DEG * 64;
    printf("%-28s %8.1f us  gather %6.2f TB/s\n", name, ms * 1000, bytes / (ms * 1e-3) / 1e12);
  };
  for (int blocks_per_sm : {4, 6, 8}) {
    for (int it = 0; it < 2; ++it) k_ldg<<<sms * blocks_per_sm, 256>>>(G, idx, n, out);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) k_ldg<<<sms * blocks_per_sm, 256>>>(G, idx, n, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    char nm[64]; snprintf(nm, 64, "LDG blocks/SM=%d", blocks_per_sm);
    report(nm, ms / 10);
  }
  CUtensorMap map;
  cuuint64_t dims[2] = {PW, (cuuint64_t)n};
  cuuint64_t strides[1] = {PW * sizeof(float)};
  cuuint32_t box[2] = {PW, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, G, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  // correctness check vs LDG
  std::vector<float> hg((size_t)n * PW);
  for (size_t i = 0; i < hg.size(); ++i) hg[i] = (float)(i % 97) * 0.01f;
  CK(cudaMemcpy(G, hg.data(), sizeof(float) * hg.size(), cudaMemcpyHostToDevice));
  k_ldg<<<sms * 4, 256>>>(G, idx, n, out);
  std::vector<float> ref((size_t)n * PW), got((size_t)n * PW);
  CK(cudaMemcpy(ref.data(), out, sizeof(float) * ref.size(), cudaMemcpyDeviceToHost));
  auto run_tma = [&](auto kern, int stages, int bps, bool timed) {
    size_t smem = (size_t)4 * stages * 8192;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<sms * bps, 128, smem>>>(map, idx, n, out);
    CK(cudaGetLastError());
    if (!timed) return 0.f;
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) kern<<<sms * bps, 128, smem>>>(map, idx, n, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 10;
  };
  CK(cudaMemset(out, 0, sizeof(float) * n * PW));
  run_tma(k_tma<3>, 3, 1, false); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(got.data(), out, sizeof(float) * got.size(), cudaMemcpyDeviceToHost));
  double maxd = 0; for (size_t i = 0; i < got.size(); ++i) maxd = fmax(maxd, fabs(got[i] - ref[i]));
  printf("TMA vs LDG max abs diff %.3g\n", maxd);
  auto run_cp = [&](auto kern, int stages, bool timed) {
    size_t smem = (size_t)8 * stages * 2048;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem));
    kern<<<sms * occ, 256, smem>>>(G, idx, n, out);
    CK(cudaGetLastError());
    if (!timed) return 0.f;
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) kern<<<sms * occ, 256, smem>>>(G, idx, n, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("  (cp.async stages=%d: %d CTAs/SM = %d warps, %zu KB in flight/SM)\n", stages, occ, occ * 8,
           (size_t)occ * smem / 1024);
    return ms / 10;
  };
  CK(cudaMemset(out, 0, sizeof(float) * n * PW));
  run_cp(k_cpasync<3>, 3, false); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(got.data(), out, sizeof(float) * got.size(), cudaMemcpyDeviceToHost));
  maxd = 0; for (size_t i = 0; i < got.size(); ++i) maxd = fmax(maxd, fabs(got[i] - ref[i]));
  printf("cp.async vs LDG max abs diff %.3g\n", maxd);
  report("cp.async stages=2", run_cp(k_cpasync<2>, 2, true));
  report("cp.async stages=3", run_cp(k_cpasync<3>, 3, true));
  report("cp.async stages=4", run_cp(k_cpasync<4>, 4, true));
  report("cp.async stages=6", run_cp(k_cpasync<6>, 6, true));
  report("cp.async stages=8", run_cp(k_cpasync<8>, 8, true));
  report("TMA gather4 stages=2 bps=2", run_tma(k_tma<2>, 2, 2, true));
  report("TMA gather4 stages=3 bps=1", run_tma(k_tma<3>, 3, 1, true));
  report("TMA gather4 stages=3 bps=2", run_tma(k_tma<3>, 3, 2, true));
  report("TMA gather4 stages=4 bps=1", run_tma(k_tma<4>, 4, 1, true));
  report("TMA gather4 stages=6 bps=1", run_tma(k_tma<6>, 6, 1, true));
  return 0;
}
