// Effective L2 capacity for a randomly gathered working set read by every SM.
// Each 8-lane group gathers 128-byte rows at hashed (uniform) indices from a source of S MB;
// no index stream, no stores.  Run under
//   ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none
// to read the DRAM bytes per pass: with G gathers of 128 B over a source of S bytes, a cache that
// holds C bytes of it reads about S + (1 - C/S) * 128 G from DRAM once warm.
//   l2_capacity [gathers_in_millions] [mode: 0 all SMs, 1 smid < half, 2 even smid, 3 smid >= half] [persisting set-aside %]
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_capacity l2_capacity.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                        \
  do {                                                               \
    cudaError_t e = (x);                                             \
    if (e != cudaSuccess) {                                          \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                 \
      exit(1);                                                       \
    }                                                                \
  } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// mode 0: every SM gathers; 1: SMs with %smid < half only; 2: SMs with even %smid only
// (the participating CTAs split the same number of gathers among themselves through a counter)
__device__ unsigned long long g_next;

__global__ void __launch_bounds__(256, 8) k_gather_sel(const float4* __restrict__ G, uint32_t rows, long gathers,
                                                       uint32_t salt, float* __restrict__ sink, int mode, int half) {
  unsigned smid;
  asm("mov.u32 %0, %%smid;" : "=r"(smid));
  if (mode == 1 && (int)smid >= half) return;
  if (mode == 2 && (smid & 1)) return;
  if (mode == 3 && (int)smid < half) return;
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (;;) {
    unsigned long long e0 = 0;
    if (lane == 0) e0 = atomicAdd(&g_next, 256ull);
    e0 = __shfl_sync(0xffffffffu, e0, 0);
    if ((long)e0 >= gathers) break;
#pragma unroll 4
    for (int r = 0; r < 16; ++r) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t e = (uint32_t)(e0 + r * 16 + u * 4 + grp);
        const uint32_t j = (uint32_t)(((uint64_t)mix(e ^ salt) * rows) >> 32);
        v[u] = __ldcg(G + (size_t)j * 8 + sub);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[0] = acc.x;
}

__global__ void __launch_bounds__(256, 8) k_gather(const float4* __restrict__ G, uint32_t rows, long gathers,
                                                   uint32_t salt, float* __restrict__ sink) {
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long e0 = warp * 16; e0 < gathers; e0 += nw * 16) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t e = (uint32_t)(e0 + u * 4 + grp);
      const uint32_t j = (uint32_t)(((uint64_t)mix(e ^ salt) * rows) >> 32);
      v[u] = __ldcg(G + (size_t)j * 8 + sub);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc.x += v[u].x;
      acc.y += v[u].y;
      acc.z += v[u].z;
      acc.w += v[u].w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[0] = acc.x;
}

int main(int argc, char** argv) {
  const long gathers = (argc > 1 ? atol(argv[1]) : 16) * 1000000L;
  const int mode = argc > 2 ? atoi(argv[2]) : 0;  // SM subset (see k_gather_sel)
  // persisting-L2 window over the source: percent of the set-aside maximum to reserve (0 = none)
  const int persist_pct = argc > 3 ? atoi(argv[3]) : 0;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  printf("%s, %d SMs, L2 %.1f MiB; %ld gathers of 128 B per pass; SM subset mode %d\n", prop.name,
         prop.multiProcessorCount, prop.l2CacheSize / 1048576.0, gathers, mode);
  float* sink;
  CK(cudaMalloc(&sink, 4));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  size_t set_aside = 0;
  if (persist_pct > 0) {
    set_aside = (size_t)prop.persistingL2CacheMaxSize * persist_pct / 100;
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, set_aside));
    printf("persisting set-aside %.1f MB (max %.1f MB), max window %.1f MB\n", set_aside / 1e6,
           prop.persistingL2CacheMaxSize / 1e6, prop.accessPolicyMaxWindowSize / 1e6);
  }
  const int sizes_mb[] = {16, 32, 48, 56, 64, 72, 80, 96, 112, 128, 160, 192, 256};
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int mb : sizes_mb) {
    const size_t bytes = (size_t)mb * 1000000;
    const uint32_t rows = (uint32_t)(bytes / 128);
    float4* G;
    CK(cudaMalloc(&G, (size_t)rows * 128));
    CK(cudaMemset(G, 0, (size_t)rows * 128));
    const int grid = prop.multiProcessorCount * 8;
    if (persist_pct > 0) {
      cudaStreamAttrValue av = {};
      av.accessPolicyWindow.base_ptr = G;
      av.accessPolicyWindow.num_bytes = std::min<size_t>((size_t)rows * 128, (size_t)prop.accessPolicyMaxWindowSize);
      av.accessPolicyWindow.hitRatio = std::min(1.0f, (float)((double)set_aside / (double)av.accessPolicyWindow.num_bytes));
      av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
    }
    for (int pass = 0; pass < 3; ++pass) {  // pass 0 warms; passes 1 and 2 use fresh index sequences
      CK(cudaEventRecord(e0, st));
      if (mode == 0) {
        k_gather<<<grid, 256, 0, st>>>(G, rows, gathers, 0x9e3779b9u * (pass + 1), sink);
      } else {
        unsigned long long zero = 0;
        CK(cudaMemcpyToSymbol(g_next, &zero, sizeof(zero)));
        k_gather_sel<<<grid, 256, 0, st>>>(G, rows, gathers, 0x9e3779b9u * (pass + 1), sink, mode, prop.multiProcessorCount / 2);
      }
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (pass) printf("source %4d MB  pass %d  %8.1f us  %6.2f TB/s L2->SM\n", mb, pass, ms * 1e3, gathers * 128.0 / ms / 1e9);
    }
    CK(cudaStreamSynchronize(st));
    if (persist_pct > 0) CK(cudaCtxResetPersistingL2Cache());
    CK(cudaFree(G));
  }
  return 0;
}
