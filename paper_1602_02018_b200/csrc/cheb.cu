// K2 implementation: fused Chebyshev step kernel, panel planning, packing, and
// the filter-level C-ABI entry points (Laplacian apply, filter, eigencount,
// features).  See filter.cuh for the formulation.
#include <atomic>
#include <algorithm>
#include <chrono>
#include <memory>
#include <mutex>

#include "filter.cuh"

namespace csc {

// ---------------------------------------------------------------------------
// vector access helpers (16-byte lanes)
template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  using type = float4;
  static constexpr int n = 4;
  __device__ static void unpack(const float4& v, float (&a)[4]) {
    a[0] = v.x;
    a[1] = v.y;
    a[2] = v.z;
    a[3] = v.w;
  }
  __device__ static float4 make(const float (&a)[4]) { return make_float4(a[0], a[1], a[2], a[3]); }
  __device__ static float4 zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
};
template <>
struct Vec16<double> {
  using type = double2;
  static constexpr int n = 2;
  __device__ static void unpack(const double2& v, double (&a)[2]) {
    a[0] = v.x;
    a[1] = v.y;
  }
  __device__ static double2 make(const double (&a)[2]) { return make_double2(a[0], a[1]); }
  __device__ static double2 zero() { return make_double2(0.0, 0.0); }
};

template <typename V>
__device__ __forceinline__ V ld_stream(bool hint, const V* p) {
  return hint ? __ldcs(p) : *p;  // evict-first: read once per step
}
template <typename V>
__device__ __forceinline__ void st_stream(bool hint, V* p, const V& v) {
  if (hint)
    __stcs(p, v);
  else
    *p = v;
}
template <typename S>
__device__ __forceinline__ S ld_csr(bool hint, const S* p) {
  return hint ? __ldcs(p) : __ldg(p);
}

// ---------------------------------------------------------------------------
// The step kernel.  LPR lanes own one row of a panel (VEC elements each);
// 32/LPR rows per warp; warps stride over row groups.
//
// Memory-level parallelism is the whole game for this kernel (it streams
// ~4 N x pw blocks per step and gathers N x deg rows at random), so a row group
// is processed as:
//   1. its row-local operands (S, X, row scales) are loaded first, so their
//      latency overlaps the neighbour gathers;
//   2. neighbours go in chunks of CH = max(LPR, 4|8) per row: the row's lanes
//      load the chunk's column indices cooperatively (CH/LPR each, coalesced)
//      and broadcast them with shuffles; the next chunk's indices are loaded
//      before this chunk's CH independent 16-byte gathers are issued.  Chunks
//      run to the warp's largest degree, so short rows waste < CH slots;
//   3. the next row group's indptr pair is fetched before the epilogue.
template <int LPR, int CHUNK>
struct Rounds {
  // neighbours per chunk: max(LPR, CHUNK), but 8 for 32-lane rows (a 32-slot chunk runs
  // to the warp's largest degree and is mostly empty slots: C4 k = 250 CG filter -20 %;
  // 8-slot chunks for 16-lane rows measured neutral at degree 16, -3 % at degree 5.5)
  static constexpr int CH = LPR > CHUNK ? (LPR < 32 ? LPR : 8) : CHUNK;
  static constexpr int UC = (CH + LPR - 1) / LPR;  // indices held per lane per chunk
  static constexpr bool PART = CH < LPR;           // only lanes sub < CH hold an index
};

template <typename T>
struct Pair;
template <>
struct Pair<float> {
  using type = float2;
};
template <>
struct Pair<double> {
  using type = double2;
};

// The neighbour-row gather load: L2 only (ld.global.cg).  Gathered rows are not reused within an
// SM (L1 hit rate 3.6 % at C3), so allocating them in L1 only costs L1 fill bandwidth: C3 features
// -0.8 %, 16-B rows -6 %, 32-B rows -3.4 %, k = 100 block -1.8 %, fp64 -1 %, C3 CG -2.5 %, C4/C5
// -0.5 %, C2 (L1 hits on a 12.8 MB panel) +0.7 % (profiles/r02_ab_gather_ld.txt; the
// ld.global.nc.L1::no_allocate / L1::evict_first forms were 15 % slower).
template <typename V>
__device__ __forceinline__ V gather_ld(const V* p) {
#ifdef CSC_GATHER_NC  // A/B builds only: the read-only path, allocating in L1
  return __ldg(p);
#else
  return __ldcg(p);
#endif
}

// Programmatic dependent launch (sm_90+): a step kernel lets its successor in the stream be
// scheduled at once and waits for its predecessor's completion (and memory flush) only
// after its own CSR prologue.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// <<<grid, threads, 0, s>>> with the programmatic-stream-serialization attribute (option pdl)
template <typename K>
static void launch_pdl(K kern, int grid, int threads, cudaStream_t s, const StepArgs& a) {
  if (g_opt.pdl.load() == 0) {
    kern<<<grid, threads, 0, s>>>(a);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CSC_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
}

template <typename T, int LPR, int EPI, int CHUNK, int MINB, bool UNIT>
__global__ void __launch_bounds__(256, MINB) k_cheb_step(const StepArgs a) {
  using VT = Vec16<T>;
  using V = typename VT::type;
  using V2 = typename Pair<T>::type;
  constexpr int VEC = VT::n;
  constexpr int PW = LPR * VEC;
  constexpr int GPW = 32 / LPR;
  constexpr int CH = Rounds<LPR, CHUNK>::CH;
  constexpr int UC = Rounds<LPR, CHUNK>::UC;
  constexpr bool PART = Rounds<LPR, CHUNK>::PART;
  const bool HINTS = a.hints != 0;
  constexpr unsigned FULL = 0xffffffffu;

  const int lane = threadIdx.x & 31;
  const int sub = lane % LPR;
  const int grp = lane / LPR;
  const int gbase = lane & ~(LPR - 1);
  const int col0 = sub * VEC;
  const bool lane_on = col0 < a.wc;
  // 32-bit row / group / vector-offset arithmetic (n * LPR < 2^32 for every supported
  // size): fewer registers in the neighbour loop
  const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  constexpr uint32_t SV = LPR;  // row stride in vectors
  const V* __restrict__ Gv = static_cast<const V*>(a.G) + sub;

  const T* __restrict__ G = static_cast<const T*>(a.G);
  const T* S = static_cast<const T*>(a.S);
  const T* __restrict__ X = static_cast<const T*>(a.X);
  const T* Yin = static_cast<const T*>(a.Yin);
  T* O = static_cast<T*>(a.O);
  T* Y = static_cast<T*>(a.Y);
  const int32_t* __restrict__ indices = a.indices;
  const T* __restrict__ wv = static_cast<const T*>(a.wv);
  const V2* __restrict__ rs = static_cast<const V2*>(a.rs);
  const T ka = static_cast<T>(a.ka), ks = static_cast<T>(a.ks), kx = static_cast<T>(a.kx);
  const T ky0 = static_cast<T>(a.ky0), ky = static_cast<T>(a.ky), hz = static_cast<T>(a.hz);
  const bool last = a.last != 0;
  const bool sym = last && !a.fwd;  // Clenshaw's last step returns to the symmetric basis
  const bool want_x = X != nullptr && (a.kx != 0.0 || EPI == EPI_CGAP || last);

  double ssq = 0.0;
  double cd[VEC];
#pragma unroll
  for (int c = 0; c < VEC; ++c) cd[c] = 0.0;

  // row-group schedule: interleaved (warp w takes groups w, w + nwarps, ...) or
  // contiguous (each warp owns one contiguous run of groups, so an SM works on
  // neighbouring rows and their shared neighbours can hit in L1)
  const int n = (int)a.n;
  const int ngroups = (n + GPW - 1) / GPW;
  int gfirst, gstep, glast;
  if (a.contig) {
    const int per = (ngroups + nwarps - 1) / nwarps;
    gfirst = warp * per;
    glast = min(ngroups, gfirst + per);
    gstep = 1;
  } else {
    gfirst = warp;
    glast = ngroups;
    gstep = nwarps;
  }
  int gi = gfirst;
  int32_t nbeg = 0, nend = 0;  // indptr pair of the next row group (prefetched)
  pdl_trigger();
  if (G != nullptr && gi < glast && gi * GPW + grp < n) {
    nbeg = __ldg(a.indptr + gi * GPW + grp);
    nend = __ldg(a.indptr + gi * GPW + grp + 1);
  }
  pdl_wait();  // earlier kernels' panels are read and written only below
  for (; gi < glast; gi += gstep) {
    const int row = gi * GPW + grp;
    const bool rok = row < n;
    const bool on = rok && lane_on;
    const int cnt = nend - nbeg;
    const uint32_t voff = (uint32_t)row * SV + sub;  // this lane's vector in row-local streams
    const size_t off = (size_t)voff * VEC;

    // 1. row-local operands: loaded after the neighbour loop (latency hidden by
    //    the other resident warps; keeping them live across it costs occupancy)
    T sv[VEC], xv[VEC], yv[VEC];
    V2 sc = {T(0), T(0)};

    // 2. neighbour chunks: CH neighbours per chunk (the row's lanes hold UC
    //    indices each), next chunk's indices loaded before this chunk's gathers
    T acc[VEC];
#pragma unroll
    for (int c = 0; c < VEC; ++c) acc[c] = T(0);
    if (G != nullptr) {
      const int maxcnt = __reduce_max_sync(FULL, cnt);
      const int32_t* ip = indices + nbeg;
      const T* wp = wv + nbeg;
      int32_t jj[UC];
      T ww[UC];
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int e = u * LPR + sub;
        const bool ok = e < cnt && (!PART || sub < CH);
        jj[u] = ok ? ld_csr(HINTS, ip + e) : -1;
        if constexpr (!UNIT) ww[u] = ok ? ld_csr(HINTS, wp + e) : T(0);
      }
      for (int base = 0; base < maxcnt; base += CH) {
        int32_t jn[UC];
        T wn[UC];
        const bool more = base + CH < maxcnt;  // warp-uniform
#pragma unroll
        for (int u = 0; u < UC; ++u) {
          const int e = base + CH + u * LPR + sub;
          const bool ok = more && e < cnt && (!PART || sub < CH);
          jn[u] = ok ? ld_csr(HINTS, ip + e) : -1;
          if constexpr (!UNIT) wn[u] = ok ? ld_csr(HINTS, wp + e) : T(0);
        }
        int32_t jc[CH];
        T wc[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) {  // slot k is entry k / LPR of lane gbase + k % LPR
          // width-LPR shuffles: the source lane k % LPR is relative to this row's lane segment
          jc[k] = LPR == 1 ? jj[k] : __shfl_sync(FULL, jj[k / LPR], k % LPR, LPR);
          wc[k] = T(1);
          if constexpr (!UNIT) wc[k] = LPR == 1 ? ww[k] : __shfl_sync(FULL, ww[k / LPR], k % LPR, LPR);
        }
        V gv[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          gv[k] = VT::zero();
          if (jc[k] >= 0 && lane_on) gv[k] = gather_ld(Gv + (uint32_t)jc[k] * SV);
        }
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          T g[VEC];
          VT::unpack(gv[k], g);
#pragma unroll
          for (int c = 0; c < VEC; ++c) {
            if constexpr (UNIT)
              acc[c] += g[c];
            else
              acc[c] = fma(wc[k], g[c], acc[c]);
          }
        }
#pragma unroll
        for (int u = 0; u < UC; ++u) {
          jj[u] = jn[u];
          if constexpr (!UNIT) ww[u] = wn[u];
        }
      }
    }

    // 3. prefetch the next row group's indptr pair
    {
      const int nrow = (gi + gstep) * GPW + grp;
      if (G != nullptr && gi + gstep < glast && nrow < n) {
        nbeg = __ldg(a.indptr + nrow);
        nend = __ldg(a.indptr + nrow + 1);
      } else {
        nbeg = nend = 0;
      }
    }

    // 4. epilogue
    double rsq = 0.0;
#pragma unroll
    for (int c = 0; c < VEC; ++c) sv[c] = xv[c] = yv[c] = T(0);
    if (on) {
      sc = rs[row];
      if (S != nullptr) VT::unpack(ld_stream(HINTS, reinterpret_cast<const V*>(S + off)), sv);
      if (want_x) VT::unpack(ld_stream(HINTS, reinterpret_cast<const V*>(X + off)), xv);
      if (a.fwd) VT::unpack(ld_stream(HINTS, reinterpret_cast<const V*>(Yin + off)), yv);
    }
    if (on) {
      const T si = sc.x, sdi = sc.y;
      const bool isolated = si == T(0);
      T out[VEC], res[VEC];
      const T kacc = ka * (sym ? si : si * si);
      const T kss = sym ? ks * sdi : ks;
#pragma unroll
      for (int c = 0; c < VEC; ++c) {
        out[c] = kacc * acc[c];
        if (S != nullptr) out[c] = fma(kss, sv[c], out[c]);
        if (want_x) out[c] = fma(kx, xv[c], out[c]);
        res[c] = out[c];
      }
      if (a.fwd) {
#pragma unroll
        for (int c = 0; c < VEC; ++c) res[c] = fma(ky, sdi * out[c], ky0 * yv[c]);
      }
      if (last && isolated) {  // L - I = 0 on an isolated node: Y = h(1) X
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          res[c] = hz * xv[c];
          if (!a.fwd) out[c] = res[c];
        }
      }
      if (a.fwd && Y != nullptr) st_stream(HINTS, reinterpret_cast<V*>(Y + off), VT::make(res));
      if (O != nullptr) {
        // this panel is the next step's gather source; evict-first unless option l2_policy = 0
        // (it would push this step's gather source out of L2; measured in k_cheb_mid)
        st_stream(a.pol != 0, reinterpret_cast<V*>(O + off), VT::make(out));
      }
      if constexpr (EPI == EPI_NONE) {  // (peer stores happen on mid steps only)
      if (a.npeers > 0) {  // fused all-gather: this row into every rank's next gather panel
        const size_t poff = (size_t)(a.peer_row0 + row) * (SV * VEC) + col0;
        for (int q = 0; q < a.npeers; ++q)
          *reinterpret_cast<V*>(static_cast<T*>(a.peers[q]) + poff) = VT::make(out);
      }
      }
      if constexpr (EPI == EPI_SUMSQ || EPI == EPI_ROWSQ) {
#pragma unroll
        for (int c = 0; c < VEC; ++c)
          if (col0 + c < a.wc) rsq += (double)res[c] * (double)res[c];
        if constexpr (EPI == EPI_SUMSQ) ssq += rsq;
      }
      if constexpr (EPI == EPI_CGAP) {
        const T m = a.mask[row] ? T(1) : T(0);
        const double gam = a.gamma, rho = a.ridge;
        T ap[VEC];
#pragma unroll
        for (int c = 0; c < VEC; ++c) {
          // AP = mask*P + gamma*(g(L)P + ridge*P), sampling.py:120-121
          const double reg = (double)res[c] + rho * (double)xv[c];
          ap[c] = static_cast<T>((double)(m * xv[c]) + gam * reg);
          if (col0 + c < a.wc) cd[c] += (double)xv[c] * (double)ap[c];
        }
        st_stream(HINTS, reinterpret_cast<V*>(static_cast<T*>(a.E) + off), VT::make(ap));
      }
    }
    if constexpr (EPI == EPI_ROWSQ) {
#pragma unroll
      for (int o = LPR / 2; o >= 1; o >>= 1) rsq += __shfl_xor_sync(FULL, rsq, o);
      if (sub == 0 && rok) a.part[row] = rsq;
    }
  }

  // block-level epilogue reductions (fixed order -> deterministic)
  if constexpr (EPI == EPI_SUMSQ) {
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ssq += __shfl_xor_sync(FULL, ssq, o);
    if (lane == 0) red[threadIdx.x >> 5] = ssq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      a.part[blockIdx.x] = t;
    }
  }
  if constexpr (EPI == EPI_CGAP) {
    __shared__ double red[8][PW];  // <= 256 threads (launch bounds)
#pragma unroll
    for (int c = 0; c < VEC; ++c) {
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1) cd[c] += __shfl_xor_sync(FULL, cd[c], o);
    }
    if (grp == 0) {
#pragma unroll
      for (int c = 0; c < VEC; ++c) red[threadIdx.x >> 5][col0 + c] = cd[c];
    }
    __syncthreads();
    const int pwr = (int)SV * VEC;  // the partials' row stride is the panel width
    for (int t = threadIdx.x; t < pwr; t += blockDim.x) {
      double sum = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sum += red[w][t];
      a.part[(size_t)blockIdx.x * pwr + t] = sum;
    }
  }
}

// ---------------------------------------------------------------------------
// Lean mid step (the hot case: unit-weight graph, Clenshaw or first steps in the scaled
// basis, no epilogue, no forward accumulator, no peer stores):
//   out~_i = ka d_i^-1 sum_j G~_j + ks S~_i + kx X~_i
// Same schedule and chunking as k_cheb_step, with only the state that case needs, so it
// fits 32 registers and runs 64 warps per SM (8 CTAs of 256 threads); 256-B rows use the
// 40-register / 6-CTA build (five gathers in flight per lane).
// OUT_EF: the output panel (the next step's gather source) is stored evict-first, so it does not
// push this step's gather source out of an L2 it barely fits (option l2_policy)
template <typename T, int LPR, int MINB, bool UNIT, bool OUT_EF = false>
__global__ void __launch_bounds__(256, MINB) k_cheb_mid(const StepArgs a) {
  using VT = Vec16<T>;
  using V = typename VT::type;
  using V2 = typename Pair<T>::type;
  constexpr int VEC = VT::n;
  constexpr int GPW = 32 / LPR;
  constexpr int CH = Rounds<LPR, 4>::CH;
  constexpr int UC = Rounds<LPR, 4>::UC;  // indices held per lane per chunk
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int sub = lane % LPR;
  const int grp = lane / LPR;
  const bool lane_on = sub * VEC < a.wc;
  const int n = (int)a.n;
  const int ngroups = (n + GPW - 1) / GPW;
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  constexpr uint32_t SV = LPR;  // row stride in vectors
  const V* __restrict__ Gv = static_cast<const V*>(a.G) + sub;
  const T ka = static_cast<T>(a.ka), ks = static_cast<T>(a.ks), kx = static_cast<T>(a.kx);
  int gi = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  int32_t nbeg = 0, nend = 0;
  pdl_trigger();
  if (gi < ngroups && gi * GPW + grp < n) {
    nbeg = __ldg(a.indptr + gi * GPW + grp);
    nend = __ldg(a.indptr + gi * GPW + grp + 1);
  }
  // the first chunk's column indices (and weights) of the warp's next row group, loaded one
  // group ahead so a group starts with its gathers instead of an index round trip
  int32_t jf[UC];
  T wf[UC];
  auto first_chunk = [&]() {
#pragma unroll
    for (int u = 0; u < UC; ++u) {  // slot k of a chunk is entry k / LPR of lane k % LPR
      const int e = u * LPR + sub;
      const bool ok = e < nend - nbeg && (UC > 1 || sub < CH);
      jf[u] = ok ? __ldcs(a.indices + nbeg + e) : -1;
      if constexpr (!UNIT) wf[u] = ok ? __ldcs(static_cast<const T*>(a.wv) + nbeg + e) : T(0);
    }
  };
  first_chunk();
  // programmatic dependent launch: everything above reads only the CSR, so it overlaps the
  // previous step's drain; the panels written by earlier kernels are touched after the wait
  // (a no-op for a launch without the attribute)
  pdl_wait();
  for (; gi < ngroups; gi += nwarps) {
    const int row = gi * GPW + grp;
    const int cnt = nend - nbeg;
    T acc[VEC];
#pragma unroll
    for (int c = 0; c < VEC; ++c) acc[c] = T(0);
    {
      const int maxcnt = __reduce_max_sync(FULL, cnt);
      const int32_t* ip = a.indices + nbeg;
      const T* wp = static_cast<const T*>(a.wv) + nbeg;  // edge weights (weighted graphs only)
      int32_t jj[UC];
      T ww[UC];
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        jj[u] = jf[u];
        if constexpr (!UNIT) ww[u] = wf[u];
      }
      for (int base = 0; base < maxcnt; base += CH) {
        int32_t jn[UC];
        T wn[UC];
        const bool more = base + CH < maxcnt;  // warp-uniform
#pragma unroll
        for (int u = 0; u < UC; ++u) {
          const int e = base + CH + u * LPR + sub;
          const bool ok = more && e < cnt && (UC > 1 || sub < CH);
          jn[u] = ok ? __ldcs(ip + e) : -1;
          if constexpr (!UNIT) wn[u] = ok ? __ldcs(wp + e) : T(0);
        }
        V gv[CH];
        T wk[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          const int32_t j = LPR == 1 ? jj[k] : __shfl_sync(FULL, jj[k / LPR], k % LPR, LPR);
          if constexpr (!UNIT) wk[k] = LPR == 1 ? ww[k] : __shfl_sync(FULL, ww[k / LPR], k % LPR, LPR);
          gv[k] = VT::zero();
          if (j >= 0 && lane_on) gv[k] = gather_ld(Gv + (uint32_t)j * SV);
        }
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          T g[VEC];
          VT::unpack(gv[k], g);
#pragma unroll
          for (int c = 0; c < VEC; ++c) {
            if constexpr (UNIT)
              acc[c] += g[c];
            else
              acc[c] = fma(wk[k], g[c], acc[c]);  // as k_cheb_step
          }
        }
#pragma unroll
        for (int u = 0; u < UC; ++u) {
          jj[u] = jn[u];
          if constexpr (!UNIT) ww[u] = wn[u];
        }
      }
    }
    {  // next row group's indptr pair
      const int nrow = (gi + nwarps) * GPW + grp;
      if (gi + nwarps < ngroups && nrow < n) {
        nbeg = __ldg(a.indptr + nrow);
        nend = __ldg(a.indptr + nrow + 1);
      } else {
        nbeg = nend = 0;
      }
    }
    first_chunk();  // (nbeg / nend now belong to the next group)
    if (row < n && lane_on) {
      const uint32_t off = ((uint32_t)row * SV + sub) * VEC;
      const T si = static_cast<const V2*>(a.rs)[row].x;
      const T kacc = ka * (si * si);  // as k_cheb_step (bit-identical results)
      T out[VEC], sv[VEC], xv[VEC];
#pragma unroll
      for (int c = 0; c < VEC; ++c) sv[c] = xv[c] = T(0);
      if (a.S) VT::unpack(__ldcs(reinterpret_cast<const V*>(static_cast<const T*>(a.S) + off)), sv);
      if (a.X && a.kx != 0.0) VT::unpack(__ldcs(reinterpret_cast<const V*>(static_cast<const T*>(a.X) + off)), xv);
#pragma unroll
      for (int c = 0; c < VEC; ++c) out[c] = fma(kx, xv[c], fma(ks, sv[c], kacc * acc[c]));
      V* op = reinterpret_cast<V*>(static_cast<T*>(a.O) + off);
      if constexpr (OUT_EF)
        __stcs(op, VT::make(out));
      else
        *op = VT::make(out);
    }
  }
}

// 6 CTAs/SM at 40 registers (five gathers in flight per lane) vs 8 CTAs at 32 (three): 64-, 256-
// and 512-B rows are faster with 6 (C3 16 columns -4.8 %, C4 k = 250 -8 %), 128-B rows with 8
// (C3 features +1.4 % with 6), 16-B rows keep 8 (profiles/r02_ab_minb.txt)
template <typename T, int LPR, int MINB = (LPR == 8 || LPR == 1 ? 8 : 6)>
static int launch_mid(const StepArgs& a, int device, cudaStream_t s) {
  const bool unit = a.wv == nullptr;
  auto kern = unit ? k_cheb_mid<T, LPR, MINB, true> : k_cheb_mid<T, LPR, MINB, false>;
  if (a.pol) kern = unit ? k_cheb_mid<T, LPR, MINB, true, true> : k_cheb_mid<T, LPR, MINB, false, true>;
  // per (device, unit) occupancy, published atomically: concurrent host threads (the CG
  // overlap worker) either see 0 and compute the same value or read the stored one
  static std::atomic<int> occ_cache[64][2];
  std::atomic<int>& slot = occ_cache[device & 63][unit ? 1 : 0];
  int occ = slot.load(std::memory_order_acquire);
  if (occ == 0) {
    int o = 0;
    CSC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, 256, 0));
    occ = std::max(o, 1);
    slot.store(occ, std::memory_order_release);
  }
  const int64_t rows_per_block = 8 * (32 / LPR);
  const int64_t need = (a.n + rows_per_block - 1) / rows_per_block;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)device_props(device).sms * occ));
  launch_pdl(kern, grid, 256, s, a);
  CSC_LAUNCHED();
  return grid;
}

// ---------------------------------------------------------------------------
// dispatch
template <typename T, int LPR, int EPI, int CHUNK, int MINB, bool UNIT>
static int launch_typed(const StepArgs& a, int threads, int device, cudaStream_t s) {
  auto kern = k_cheb_step<T, LPR, EPI, CHUNK, MINB, UNIT>;
  static std::mutex mu;
  static int occ_cache[64] = {0};  // per device
  int occ;
  {
    std::lock_guard<std::mutex> lk(mu);
    const int slot = (device & 7) * 8 + ((threads / 32 - 1) & 7);
    if (occ_cache[slot] == 0) {
      int o = 0;
      CSC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, 0));
      occ_cache[slot] = std::max(o, 1);
    }
    occ = occ_cache[slot];
  }
  const int64_t rows_per_block = (int64_t)(threads / 32) * (32 / LPR);
  int64_t need = (a.n + rows_per_block - 1) / rows_per_block;
  const int64_t cap = g_opt.persistent.load() ? std::min<int64_t>((int64_t)device_props(device).sms * occ,
                                                                    step_grid_cap(device))
                                              : (int64_t)INT32_MAX;
  const int grid = (int)std::max<int64_t>(1, std::min(need, cap));
  const size_t persist = a.G ? persist_bytes(device) : 0;
  if (persist > 0) {
    // keep the gathered panel in the persisting L2 set-aside; everything else streams
    constexpr int VEC = 16 / sizeof(T);
    const size_t win = std::min<size_t>((size_t)a.n * LPR * VEC * sizeof(T), (size_t)device_props(device).max_window);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(a.G);
    attr[0].val.accessPolicyWindow.num_bytes = win;
    attr[0].val.accessPolicyWindow.hitRatio = std::min(1.0f, (float)((double)persist / (double)win));
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CSC_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  } else {
    launch_pdl(kern, grid, threads, s, a);
  }
  CSC_LAUNCHED();
  return grid;
}

template <typename T, int EPI, int CHUNK, int MINB, bool UNIT>
static int launch_lpr(const StepArgs& a, int lpr, int threads, int device, cudaStream_t s) {
  switch (lpr) {
    case 1: return launch_typed<T, 1, EPI, CHUNK, MINB, UNIT>(a, threads, device, s);
    case 2: return launch_typed<T, 2, EPI, CHUNK, MINB, UNIT>(a, threads, device, s);
    case 4: return launch_typed<T, 4, EPI, CHUNK, MINB, UNIT>(a, threads, device, s);
    case 8: return launch_typed<T, 8, EPI, CHUNK, MINB, UNIT>(a, threads, device, s);
    case 16: return launch_typed<T, 16, EPI, CHUNK, MINB, UNIT>(a, threads, device, s);
    case 32: return launch_typed<T, 32, EPI, CHUNK, MINB, UNIT>(a, threads, device, s);
  }
  fail(CSC_ERR_INVALID, "unsupported panel width");
}

template <typename T, int EPI>
static int launch_epi(const StepArgs& a, int lpr, int threads, int device, cudaStream_t s) {
  // UNIT: unit-weight graph, no per-edge values are read
  // unroll: 8 -> 8 gathers in flight (2 CTAs/SM); 4 -> 4 in flight at 6 CTAs/SM (40 regs);
  // 2 -> 4 in flight at 8 CTAs/SM (32 regs, full occupancy)
  const int64_t mode = g_opt.unroll.load();
  const bool unit = a.wv == nullptr;
  if (mode == 8) {
    if (unit) return launch_lpr<T, EPI, 8, 2, true>(a, lpr, threads, device, s);
    return launch_lpr<T, EPI, 8, 2, false>(a, lpr, threads, device, s);
  }
  if (mode == 2) {
    if (unit) return launch_lpr<T, EPI, 4, 8, true>(a, lpr, threads, device, s);
    return launch_lpr<T, EPI, 4, 8, false>(a, lpr, threads, device, s);
  }

  if (unit) return launch_lpr<T, EPI, 4, 6, true>(a, lpr, threads, device, s);
  return launch_lpr<T, EPI, 4, 6, false>(a, lpr, threads, device, s);
}

int step_grid_cap(int device) {
  // 2048 resident threads per SM at most; block_threads >= 64
  return device_props(device).sms * 32;
}

static double step_bytes(const csc_graph* g, const StepArgs& a, int epi) {
  const double s = (double)dtype_size(g->dtype);
  const double nw = (double)a.n * a.wc * s;
  double b = 0.0;
  if (a.G) {  // CSR (indptr + indices [+ weights]) + per-row scales + one compulsory read of G
    b += 4.0 * (g->n + 1) + (double)g->nnz * (4.0 + (a.wv ? s : 0.0)) + 2.0 * s * a.n + nw;
  }
  if (a.S) b += nw;
  if (a.X && (a.kx != 0.0 || epi == EPI_CGAP)) b += nw;
  if (a.O) b += nw;
  if (a.fwd) b += nw + (a.Y ? nw : 0.0);
  if (epi == EPI_CGAP) b += nw + (double)a.n;  // AP write + mask
  if (epi == EPI_ROWSQ) b += 8.0 * a.n;
  return b;
}

template <typename T>
int launch_step(const csc_graph* g, const StepArgs& a_in, int pw, int epi, cudaStream_t s) {
  StepArgs a = a_in;
  a.hints = g_opt.cache_hints.load() != 0;
  a.contig = g_opt.row_order.load() == 1;
  a.pol = (int)g_opt.l2_policy.load();
  constexpr int VEC = 16 / sizeof(T);
  if (pw < VEC || pw % VEC != 0 || pw > 32 * VEC) fail(CSC_ERR_INVALID, "unsupported panel width");
  a.sv = pw / VEC;
  int lpr = 1;  // lanes per row: the power of two >= the row's vectors
  while (lpr < a.sv) lpr *= 2;
  // rows of the gathered panel: the local rows, or every rank's slots of a row shard
  const int64_t gsrc = std::max<int64_t>(a.n, g->gather_rows);
  if (gsrc > 0 && (uint64_t)gsrc * (uint64_t)lpr >= (1ull << 32))
    fail(CSC_ERR_INVALID, "panel too large for 32-bit vector offsets (rows x lanes >= 2^32)");
  const int threads = (int)g_opt.block_threads.load();
  const bool prof = g_opt.profile.load() == 1 && a.G != nullptr;  // 2: per filter span (filter_panel)
  cudaEvent_t e0 = nullptr;
  if (prof) profile_begin(s, &e0);
  int grid = 0;
  // Lean mid-step kernel (32 registers, 64 warps/SM) for the hot case: 16- to 512-B rows whose
  // gather panel is at most 4x L2 (32-B rows since the final round-2 kernel: C3 8 columns -3.4 %,
  // C4 -25 %, C2 -6 %, fp64 4 columns -8 % at 6 CTAs/SM, profiles/r02_ab_lean_lpr2.txt).
  // A/B on B200 (profiles/r01_panel_sweeps.txt): C3 d=56 -1.7 %, CG k=100 -4.7 %, probe d=28
  // -5.8 %, fp64 d=56 -8.3 %, 16-B rows -4.3 %, 64-B rows -4.6 %, 512-B rows -4.5 % (C4 k=250) to
  // -20 % (C2 fp64); a 2 GB C5 panel (DRAM-bound random gathers) is 3.7 % slower with it and
  // keeps k_cheb_step.
  // Weighted graphs: fp32 -3.5 to -5 %, fp64 +5 % (weights cost the fp64 build its buffers).
  const bool lean = g_opt.lean_mid.load() != 0 && epi == EPI_NONE && (a.wv == nullptr || sizeof(T) == 4) &&
                    !a.fwd && !a.last &&
                    a.npeers == 0 && a.G != nullptr && a.O != nullptr && !a.contig && threads == 256 &&
                    g_opt.unroll.load() == 4 && g_opt.persistent.load() && persist_bytes(g->device) == 0 &&
                    (double)gsrc * a.sv * 16.0 <= 4.0 * (double)device_props(g->device).l2_bytes;
  if (lean) {
    switch (lpr) {
      case 1: grid = launch_mid<T, 1>(a, g->device, s); break;
      case 2: grid = launch_mid<T, 2>(a, g->device, s); break;
      case 4: grid = launch_mid<T, 4>(a, g->device, s); break;
      case 8: grid = launch_mid<T, 8>(a, g->device, s); break;
      case 16: grid = launch_mid<T, 16>(a, g->device, s); break;
      default: grid = launch_mid<T, 32>(a, g->device, s); break;
    }
    if (prof) profile_end(s, e0, step_bytes(g, a, epi));
    return grid;
  }
  switch (epi) {
    case EPI_NONE: grid = launch_epi<T, EPI_NONE>(a, lpr, threads, g->device, s); break;
    case EPI_SUMSQ: grid = launch_epi<T, EPI_SUMSQ>(a, lpr, threads, g->device, s); break;
    case EPI_ROWSQ: grid = launch_epi<T, EPI_ROWSQ>(a, lpr, threads, g->device, s); break;
    case EPI_CGAP: grid = launch_epi<T, EPI_CGAP>(a, lpr, threads, g->device, s); break;
    default: fail(CSC_ERR_INVALID, "bad epilogue");
  }
  if (prof) profile_end(s, e0, step_bytes(g, a, epi));
  return grid;
}

template int launch_step<float>(const csc_graph*, const StepArgs&, int, int, cudaStream_t);
template int launch_step<double>(const csc_graph*, const StepArgs&, int, int, cudaStream_t);

// ---------------------------------------------------------------------------
// filter drivers

// h(1) = sum_l c_l T_l(0), T_l(0) = 1, 0, -1, 0, 1, ...: the filter on an isolated node.
static double value_at_one(const double* c, int nc) {
  double h = 0.0;
  for (int l = 0; l < nc; l += 2) h += ((l / 2) % 2 ? -c[l] : c[l]);
  return h;
}

template <typename T>
int filter_panel(const csc_graph* g, const double* c, int nc, const T* X, const T* Xs, T* Y, T* B0, T* B1, T* Yacc,
                 int pw, int wc, int epi, const EpiExtra& ex, cudaStream_t s) {
  const int p = nc - 1;
  const double hz = value_at_one(c, nc);
  auto base = [&]() {
    StepArgs a{};
    a.indptr = g->indptr;
    a.indices = g->indices;
    a.wv = g->wv;
    a.rs = g->rs;
    a.n = g->n;
    a.wc = wc;
    a.hz = hz;
    return a;
  };
  // profile mode 2: one event pair around the whole filter (the step launches back to back),
  // counted as its SpMM launches -- per-launch events cost ~2 % of a step at C3
  const bool span = g_opt.profile.load() == 2;
  cudaEvent_t span_e0 = nullptr;
  double span_bytes = 0.0;
  int64_t span_launches = 0;
  if (span) profile_begin(s, &span_e0);
  auto run = [&](StepArgs a, int e) {
    if (e != EPI_NONE) {
      a.part = ex.part;
      a.last = 1;
    }
    if (e == EPI_CGAP) {
      a.mask = ex.mask;
      a.gamma = ex.gamma;
      a.ridge = ex.ridge;
      a.E = ex.ap;
    }
    if (span && a.G != nullptr) {
      span_bytes += step_bytes(g, a, e);
      ++span_launches;
    }
    const int grid = launch_step<T>(g, a, pw, e, s);
    if (span && a.last) profile_end(s, span_e0, span_bytes, span_launches);  // the filter's final step
    return grid;
  };

  if (p == 0) {  // order 0: Y = c_0 X (filters.py:147)
    StepArgs a = base();
    a.X = X;
    a.kx = c[0];
    a.O = Y;
    a.last = 1;
    return run(a, epi);
  }
  const bool forward = g_opt.recurrence.load() == 1;
  if (!forward) {
    // Clenshaw: b_l = c_l X + 2A b_{l+1} - b_{l+2}, A = L - I; Y = c_0 X + A b_1 - b_2
    if (p == 1) {
      StepArgs a = base();
      a.G = Xs;
      a.ka = -c[1];
      a.X = X;
      a.kx = c[0];
      a.O = Y;
      a.last = 1;
      return run(a, epi);
    }
    StepArgs a = base();  // b_{p-1} = c_{p-1} X + 2 c_p A X
    a.G = Xs;
    a.ka = -2.0 * c[p];
    a.X = Xs;
    a.kx = c[p - 1];
    a.O = B0;
    run(a, EPI_NONE);
    if (p == 2) {  // Y = c_0 X + A b_1 - b_2 with b_2 = c_2 X
      StepArgs f = base();
      f.G = B0;
      f.ka = -1.0;
      f.X = X;
      f.kx = c[0] - c[2];
      f.O = Y;
      f.last = 1;
      return run(f, epi);
    }
    StepArgs b = base();  // b_{p-2} = c_{p-2} X + 2A b_{p-1} - c_p X
    b.G = B0;
    b.ka = -2.0;
    b.X = Xs;
    b.kx = c[p - 2] - c[p];
    b.O = B1;
    run(b, EPI_NONE);
    T* cur = B1;  // b~_{l+1}
    T* prv = B0;  // b~_{l+2}
    for (int l = p - 3; l >= 1; --l) {
      StepArgs m = base();
      m.G = cur;
      m.ka = -2.0;
      m.S = prv;
      m.ks = -1.0;
      m.X = Xs;
      m.kx = c[l];
      m.O = prv;  // b~_l overwrites b~_{l+2} row by row
      run(m, EPI_NONE);
      std::swap(cur, prv);
    }
    StepArgs f = base();
    f.G = cur;
    f.ka = -1.0;
    f.S = prv;
    f.ks = -1.0;
    f.X = X;
    f.kx = c[0];
    f.O = Y;
    f.last = 1;
    return run(f, epi);
  }

  // forward recurrence (filters.py:148-154), T~ in the scaled basis, Y symmetric
  T* acc = Y ? Y : Yacc;
  if (!acc) fail(CSC_ERR_INVALID, "forward recurrence needs an accumulator panel");
  {
    StepArgs a = base();  // T_1 = (L - I) X;  Y = c_0 X + c_1 T_1
    a.G = Xs;
    a.ka = -1.0;
    a.O = (p == 1) ? nullptr : B0;
    a.fwd = 1;
    a.Yin = X;
    a.ky0 = c[0];
    a.ky = c[1];
    a.Y = (p == 1) ? Y : acc;
    if (p == 1) {
      a.X = X;  // isolated-node fixup / CGAP operand
      a.last = 1;
      return run(a, epi);
    }
    run(a, EPI_NONE);
  }
  const T* t_prev = Xs;  // T~_{l-2}
  T* t_cur = B0;         // T~_{l-1}
  for (int l = 2; l <= p; ++l) {
    const bool last = l == p;
    StepArgs a = base();
    a.G = t_cur;
    a.ka = -2.0;
    a.S = t_prev;
    a.ks = -1.0;
    T* dst = (t_prev == Xs) ? B1 : const_cast<T*>(t_prev);
    a.O = last ? nullptr : dst;
    a.fwd = 1;
    a.Yin = acc;
    a.ky0 = 1.0;
    a.ky = c[l];
    a.Y = last ? Y : acc;
    if (last) {
      a.X = X;
      a.last = 1;
      return run(a, epi);
    }
    run(a, EPI_NONE);
    t_prev = t_cur;
    t_cur = dst;
  }
  return 0;  // unreachable
}

template int filter_panel<float>(const csc_graph*, const double*, int, const float*, const float*, float*, float*,
                                 float*, float*, int, int, int, const EpiExtra&, cudaStream_t);
template int filter_panel<double>(const csc_graph*, const double*, int, const double*, const double*, double*,
                                  double*, double*, double*, int, int, int, const EpiExtra&, cudaStream_t);

// ---------------------------------------------------------------------------
// panels
PanelPlan plan_panels(int64_t n, int w, int dtype, int device, int64_t nnz) {
  const int vec = 16 / (int)dtype_size(dtype);
  const int max_lpr = 32;
  int max_pw = vec * max_lpr;
  const int64_t forced = g_opt.panel_width.load();
  if (forced > 0) {
    int pw = vec;
    while (pw < forced && pw < max_pw) pw *= 2;
    max_pw = pw;
  } else {
    // Gathers cost per L2 request more than per byte (64-B rows run at ~2/3 the speed of
    // 128-B rows per request), and every panel re-reads the CSR, so: panel rows of at
    // least 128 B; wider when the panel still fits the L2 budget (which grows as
    // 16 / mean degree, <= 4x: low-degree graphs re-read gathered rows less often); and
    // the whole block in one panel when its rows are <= 256 B.  Measured on B200 at
    // BASELINE C2-C5, fp32 and fp64 (profiles/r01_panel_sweeps.txt): 10-23 % faster than
    // L2-fit-only panels at C3/C5, equal where the block is L2-resident.
    const double deg = n > 0 ? (double)nnz / (double)n : 16.0;
    const double relax = std::min(4.0, std::max(1.0, 16.0 / std::max(deg, 1.0)));
    const double budget =
        relax * (double)device_props(device).l2_bytes * (double)g_opt.l2_budget_pct.load() / 100.0;
    int pw_l2 = vec;
    while (pw_l2 * 2 <= max_pw && (double)n * (pw_l2 * 2) * dtype_size(dtype) <= budget) pw_l2 *= 2;
    int pw = std::max(pw_l2, 128 / (int)dtype_size(dtype));
    if ((size_t)w * dtype_size(dtype) <= 256) {
      int one = vec;
      while (one < w) one *= 2;
      pw = std::max(pw, one);
      // ... unless that one panel's gather source spills L2 while 128-B-row panels fit it
      // (fp32): C3 d = 56 as 2 x 32 columns, 24.55 -> 23.89 ms per filter, the inter-community
      // gathers then hit L2; fp64 (256-B rows: 44.3 -> 49.4 ms) and L2-resident blocks (C4:
      // 6.04 -> 7.64 ms) keep one panel (profiles/r02_ab_two_panels.txt)
      const double l2 = (double)device_props(device).l2_bytes;
      const int p128 = 128 / (int)dtype_size(dtype);
      // (round-2 final kernels, fp64 too: C3 ds = 28 as 16 + 12 columns 23.7 -> 22.3 ms,
      // gpurun sweep in profiles/r02_plan_sweep_final.txt)
      if (one > p128 && (double)n * one * dtype_size(dtype) > l2 && (double)n * 128.0 <= l2) pw = p128;
      // ... and in the DRAM-random regime (gather source > 4x L2, C5), where a gathered row
      // costs per 128-B line, a block just over 128 B runs as one 128-B-row panel plus a narrow
      // remainder rather than one 256-B-row panel (C5 probe, 34 columns: 496 -> 401 ms per
      // filter, profiles/r02_c5_panels.txt)
      if (dtype == CSC_F32 && one > p128 && (double)n * one * dtype_size(dtype) > 4.0 * l2 &&
          (size_t)(w - p128) * dtype_size(dtype) <= 32)
        pw = p128;
    }
    max_pw = std::min(pw, max_pw);
  }
  PanelPlan pp;
  int c0 = 0;
  int64_t off = 0;
  while (c0 < w) {
    const int rem = w - c0;
    int pw;
    if (rem >= max_pw) {
      pw = max_pw;
    } else {
      pw = vec;
      while (pw < rem) pw *= 2;
    }
    const int wc = std::min(pw, rem);
    pp.pw.push_back(pw);
    pp.wc.push_back(wc);
    pp.c0.push_back(c0);
    pp.off.push_back(off);
    off += (int64_t)n * pw;
    pp.max_pw = std::max(pp.max_pw, pw);
    c0 += wc;
  }
  pp.np = (int)pp.pw.size();
  pp.total = off;
  return pp;
}

// one thread per (row, panel column); `scaled` (optional) gets row i times d_i^-1/2
template <typename Ti, typename To>
__global__ void k_pack(const Ti* __restrict__ src, int64_t ld, int c0, int wc, int pw, int64_t n,
                       const double* __restrict__ dis, To* __restrict__ dst, To* __restrict__ scaled) {
  const int64_t total = n * pw;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / pw;
    const int c = (int)(t - row * pw);
    const double v = c < wc ? (double)src[row * ld + c0 + c] : 0.0;
    dst[t] = static_cast<To>(v);
    if (scaled) scaled[t] = static_cast<To>(v * dis[row]);
  }
}

template <typename Ti, typename To>
__global__ void k_unpack(const Ti* __restrict__ src, int c0, int wc, int pw, int64_t n, To* __restrict__ dst, int64_t ld) {
  const int64_t total = n * wc;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / wc;
    const int c = (int)(t - row * wc);
    dst[row * ld + c0 + c] = static_cast<To>(src[row * pw + c]);
  }
}

static int ew_grid(int64_t work) {
  int64_t g = (work + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 64));
}

template <typename Ti, typename To>
static void pack_typed(const void* src, int64_t ld, void* dst, void* scaled, const csc_graph* g, const PanelPlan& pp,
                       cudaStream_t s) {
  for (int j = 0; j < pp.np; ++j) {
    const int64_t work = g->n * pp.pw[j];
    if (work == 0) continue;
    k_pack<Ti, To><<<ew_grid(work), 256, 0, s>>>(static_cast<const Ti*>(src), ld, pp.c0[j], pp.wc[j], pp.pw[j], g->n,
                                                 g->dis, static_cast<To*>(dst) + pp.off[j],
                                                 scaled ? static_cast<To*>(scaled) + pp.off[j] : nullptr);
    CSC_LAUNCHED();
  }
}

void pack_panels(const void* src, int io_dtype, int64_t ld, void* dst, void* scaled, const csc_graph* g,
                 const PanelPlan& pp, cudaStream_t s) {
  if (io_dtype == CSC_F64 && g->dtype == CSC_F64)
    pack_typed<double, double>(src, ld, dst, scaled, g, pp, s);
  else if (io_dtype == CSC_F64 && g->dtype == CSC_F32)
    pack_typed<double, float>(src, ld, dst, scaled, g, pp, s);
  else if (io_dtype == CSC_F32 && g->dtype == CSC_F64)
    pack_typed<float, double>(src, ld, dst, scaled, g, pp, s);
  else
    pack_typed<float, float>(src, ld, dst, scaled, g, pp, s);
}

void unpack_panels(const void* src, int dtype, const PanelPlan& pp, int64_t n, void* dst, int io_dtype, int64_t ld,
                   cudaStream_t s) {
  for (int j = 0; j < pp.np; ++j) {
    const int64_t work = n * pp.wc[j];
    if (work == 0) continue;
    const int gsz = ew_grid(work);
    if (dtype == CSC_F64 && io_dtype == CSC_F64)
      k_unpack<double, double><<<gsz, 256, 0, s>>>((const double*)src + pp.off[j], pp.c0[j], pp.wc[j], pp.pw[j], n,
                                                   (double*)dst, ld);
    else if (dtype == CSC_F32 && io_dtype == CSC_F64)
      k_unpack<float, double><<<gsz, 256, 0, s>>>((const float*)src + pp.off[j], pp.c0[j], pp.wc[j], pp.pw[j], n,
                                                  (double*)dst, ld);
    else if (dtype == CSC_F64 && io_dtype == CSC_F32)
      k_unpack<double, float><<<gsz, 256, 0, s>>>((const double*)src + pp.off[j], pp.c0[j], pp.wc[j], pp.pw[j], n,
                                                  (float*)dst, ld);
    else
      k_unpack<float, float><<<gsz, 256, 0, s>>>((const float*)src + pp.off[j], pp.c0[j], pp.wc[j], pp.pw[j], n,
                                                 (float*)dst, ld);
    CSC_LAUNCHED();
  }
}

// fixed-order reductions
__global__ void k_reduce_sum(const double* __restrict__ in, int64_t count, double* __restrict__ out) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) acc += in[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o >= 1; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

void reduce_sum(const double* in, int64_t count, double* out, cudaStream_t s) {
  k_reduce_sum<<<1, 256, 0, s>>>(in, count, out);
  CSC_LAUNCHED();
}


// features: sum the panel row norms in panel order, normalise, flag zero rows
template <typename T, typename To>
__global__ void k_normalize_rows(const T* __restrict__ Yp, const double* __restrict__ rowsq, int np,
                                 const int* __restrict__ pw, const int* __restrict__ wc, const int* __restrict__ c0,
                                 const int64_t* __restrict__ off, int64_t n, To* __restrict__ F, int64_t ldf,
                                 uint8_t* __restrict__ zflag, unsigned long long* __restrict__ nzero) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = warp; row < n; row += nw) {
    double t = 0.0;
    for (int j = 0; j < np; ++j) t += rowsq[(int64_t)j * n + row];
    const double nrm = sqrt(t);
    const bool zero = nrm <= 1e-300;  // features.py:23, 81
    for (int j = 0; j < np; ++j) {
      const T* src = Yp + off[j] + row * pw[j];
      for (int c = lane; c < wc[j]; c += 32) {
        const double v = (double)src[c];
        F[row * ldf + c0[j] + c] = zero ? To(0) : static_cast<To>(v / nrm);
      }
    }
    if (lane == 0) {
      if (zflag) zflag[row] = zero ? 1 : 0;
      if (zero) atomicAdd(nzero, 1ull);
    }
  }
}

// Single-panel features (the whole block in one panel, e.g. C3's d = 56 in one 64-wide
// panel): LPR lanes per row move 16-byte vectors, several rows per warp, stores vectorised;
// same arithmetic as k_normalize_rows (fp64 v / ||row||, features.py:84-87).
// Also multi-panel blocks whose panels share one width (C3's d = 56 as 2 x 32 columns): panel
// j's rows follow panel j-1's, its columns start at j * pw, and a row's norm sums the panels'
// partial squares in panel order, as k_normalize_rows does.
template <typename T, typename To, int LPR>
__global__ void __launch_bounds__(256) k_normalize_1p(const T* __restrict__ Yp, int pw, int np, int ncols,
                                                      const double* __restrict__ rowsq,
                                                      int64_t n, To* __restrict__ F, int64_t ldf,
                                                      uint8_t* __restrict__ zflag,
                                                      unsigned long long* __restrict__ nzero) {
  constexpr int VEC = 16 / (int)sizeof(T);
  constexpr int GPW = 32 / LPR;
  const int lane = threadIdx.x & 31, sub = lane % LPR, grp = lane / LPR;
  const int col0 = sub * VEC;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned zeros = 0;
  for (int64_t row = warp * GPW + grp; row - grp < n; row += nw * GPW) {
    if (row < n) {
      double t = rowsq[row];
      for (int j = 1; j < np; ++j) t += rowsq[(int64_t)j * n + row];
      const double nrm = sqrt(t);
      const bool zero = nrm <= 1e-300;  // features.py:23, 81
      for (int j = 0; j < np; ++j) {
      const int wc = min(pw, ncols - j * pw);
      T v[VEC];
      if (col0 < wc) {
        const T* src = Yp + ((int64_t)j * n + row) * pw + col0;
        if constexpr (sizeof(T) == 4) {
          const float4 q = __ldcs(reinterpret_cast<const float4*>(src));
          v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
        } else {
          const double2 q = __ldcs(reinterpret_cast<const double2*>(src));
          v[0] = q.x, v[1] = q.y;
        }
      }
      if (col0 < wc) {
        To o[VEC];
#pragma unroll
        for (int c = 0; c < VEC; ++c) o[c] = zero ? To(0) : static_cast<To>((double)v[c] / nrm);
        To* dst = F + row * ldf + j * pw + col0;
        if (col0 + VEC <= wc) {  // 16-B aligned: ldf * sizeof(To) and col0 * sizeof(To) are multiples of 16
          if constexpr (sizeof(To) == 4 && VEC == 4) {
            __stcs(reinterpret_cast<float4*>(dst), make_float4(o[0], o[1], o[2], o[3]));
          } else if constexpr (sizeof(To) == 8 && VEC == 4) {
            __stcs(reinterpret_cast<double2*>(dst), make_double2(o[0], o[1]));
            __stcs(reinterpret_cast<double2*>(dst) + 1, make_double2(o[2], o[3]));
          } else if constexpr (sizeof(To) == 8 && VEC == 2) {
            __stcs(reinterpret_cast<double2*>(dst), make_double2(o[0], o[1]));
          } else {
#pragma unroll
            for (int c = 0; c < VEC; ++c) dst[c] = o[c];
          }
        } else {
          for (int c = 0; c < wc - col0; ++c) dst[c] = o[c];
        }
      }
      }
      if (sub == 0) {
        if (zflag) zflag[row] = zero ? 1 : 0;
        zeros += zero ? 1u : 0u;
      }
    }
  }
  if (zeros) atomicAdd(nzero, (unsigned long long)zeros);
}

template <typename T, typename To>
static bool launch_normalize_1p(const PanelPlan& pp, const T* Yp, const double* rowsq, int64_t n, To* F, int64_t ldf,
                                uint8_t* zflag, unsigned long long* nzero, int device, cudaStream_t s) {
  constexpr int VEC = 16 / (int)sizeof(T);
  if (((size_t)ldf * sizeof(To)) % 16 != 0 || reinterpret_cast<uintptr_t>(F) % 16 != 0) return false;
  int ncols = 0;
  for (int j = 0; j < pp.np; ++j) {  // equal-width panels, back to back (every panel but the last full)
    if (pp.pw[j] != pp.pw[0] || pp.off[j] != (int64_t)j * n * pp.pw[0] || pp.c0[j] != j * pp.pw[0]) return false;
    if (j + 1 < pp.np && pp.wc[j] != pp.pw[j]) return false;
    ncols += pp.wc[j];
  }
  if ((VEC * sizeof(To)) % 16 != 0 && VEC * sizeof(To) != 8) return false;
  int lpr = 1;
  while (lpr < pp.pw[0] / VEC) lpr *= 2;
  const int64_t rows_per_block = 8 * (32 / lpr);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + rows_per_block - 1) / rows_per_block,
                                                               (int64_t)device_props(device).sms * 8));
  switch (lpr) {
#define CSC_NORM1P(L)                                                                                        \
  case L:                                                                                                    \
    k_normalize_1p<T, To, L><<<grid, 256, 0, s>>>(Yp, pp.pw[0], pp.np, ncols, rowsq, n, F, ldf, zflag, nzero); \
    break;
    CSC_NORM1P(1)
    CSC_NORM1P(2)
    CSC_NORM1P(4)
    CSC_NORM1P(8)
    CSC_NORM1P(16)
    CSC_NORM1P(32)
#undef CSC_NORM1P
    default:
      return false;
  }
  CSC_LAUNCHED();
  return true;
}

__global__ void k_sum_panels(const double* __restrict__ rowsq, int np, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int j = 0; j < np; ++j) t += rowsq[(int64_t)j * n + i];
    out[i] = t;
  }
}

template <typename T>
__global__ void k_normalize_rowmajor(const T* __restrict__ Y, int64_t ldy, int64_t n, int w,
                                     const double* __restrict__ rowsq, T* __restrict__ F, int64_t ldf,
                                     uint8_t* __restrict__ zflag, unsigned long long* __restrict__ nzero) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = warp; row < n; row += nw) {
    const double nrm = sqrt(rowsq[row]);
    const bool zero = nrm <= 1e-300;
    for (int c = lane; c < w; c += 32) {
      const double v = (double)Y[row * ldy + c];
      F[row * ldf + c] = zero ? T(0) : static_cast<T>(v / nrm);
    }
    if (lane == 0) {
      if (zflag) zflag[row] = zero ? 1 : 0;
      if (zero) atomicAdd(nzero, 1ull);
    }
  }
}

}  // namespace csc

using namespace csc;

// ---------------------------------------------------------------------------
// C ABI (filter level)
namespace {

void check_graph(const csc_graph* g) {
  if (!g) fail(CSC_ERR_INVALID, "graph is NULL");
}

void check_block(const csc_graph* g, const void* p, int64_t ld, int ncols, int io, const char* what) {
  if (ncols < 0) fail(CSC_ERR_INVALID, std::string(what) + ": ncols must be >= 0");
  if (io != CSC_F64 && io != CSC_F32) fail(CSC_ERR_INVALID, "io_dtype must be CSC_F64 or CSC_F32");
  if (ld < ncols) fail(CSC_ERR_INVALID, std::string(what) + ": leading dimension smaller than ncols");
  if (p == nullptr && g->n > 0 && ncols > 0) fail(CSC_ERR_INVALID, std::string(what) + " is NULL");
}

void check_coeffs(const double* c, int nc) {
  if (nc < 1) fail(CSC_ERR_INVALID, "need at least one coefficient");
  if (!c) fail(CSC_ERR_INVALID, "coefficients are NULL");
}

// Stage a row-major (n x ncols, ld) input on the device; returns pointer + ld.
struct StagedIn {
  const void* p = nullptr;
  int64_t ld = 0;
  Scratch buf;
};
void stage_in(const void* src, int64_t ld, int64_t n, int ncols, int io, int device, cudaStream_t s, StagedIn& out) {
  const size_t es = dtype_size(io);
  if (is_device_ptr(src, device)) {
    out.p = src;
    out.ld = ld;
    return;
  }
  out.buf.alloc(es * n * ncols, s);
  copy_rows(out.buf.get(), ncols, src, ld, n, ncols, es, cudaMemcpyHostToDevice, s);
  out.p = out.buf.get();
  out.ld = ncols;
}

struct StagedOut {
  void* p = nullptr;  // device target
  int64_t ld = 0;
  void* host = nullptr;
  int64_t host_ld = 0;
  Scratch buf;
};
void stage_out(void* dst, int64_t ld, int64_t n, int ncols, int io, int device, cudaStream_t s, StagedOut& out) {
  const size_t es = dtype_size(io);
  if (is_device_ptr(dst, device)) {
    out.p = dst;
    out.ld = ld;
    return;
  }
  out.buf.alloc(es * n * ncols, s);
  out.p = out.buf.get();
  out.ld = ncols;
  out.host = dst;
  out.host_ld = ld;
}
void finish_out(StagedOut& o, int64_t n, int ncols, int io, cudaStream_t s) {
  if (!o.host) return;
  copy_rows(o.host, o.host_ld, o.p, ncols, n, ncols, dtype_size(io), cudaMemcpyDeviceToHost, s);
}

// Pinned host memory (cudaMemcpy2DAsync from it is asynchronous)?
static bool is_pinned_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// One copy stream per device for overlapped uploads (created once, never destroyed).
static cudaStream_t upload_stream(int device) {
  static std::mutex mu;
  static cudaStream_t st[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (!st[device & 63]) CSC_CUDA(cudaStreamCreateWithFlags(&st[device & 63], cudaStreamNonBlocking));
  return st[device & 63];
}

static void pack_one(const void* src, int io, int64_t ld, int wc, int pw, void* dst, void* scaled, const csc_graph* g,
                     cudaStream_t s) {
  const int64_t work = g->n * pw;
  if (work == 0) return;
#define CSC_PACK1(Ti, To)                                                                                    \
  k_pack<Ti, To><<<ew_grid(work), 256, 0, s>>>(static_cast<const Ti*>(src), ld, 0, wc, pw, g->n, g->dis,   \
                                               static_cast<To*>(dst), static_cast<To*>(scaled))
  if (io == CSC_F64 && g->dtype == CSC_F64)
    CSC_PACK1(double, double);
  else if (io == CSC_F64)
    CSC_PACK1(double, float);
  else if (g->dtype == CSC_F64)
    CSC_PACK1(float, double);
  else
    CSC_PACK1(float, float);
#undef CSC_PACK1
  CSC_LAUNCHED();
}

// A row-major input block packed into symmetric and scaled panels.
//
// Lazy mode (filter entry points that run the panels through run_filter_all): a multi-panel
// block in pinned host memory is uploaded panel by panel -- a 2-D copy of the panel's columns
// (~50 GB/s, as a contiguous copy) on the device's upload stream -- and panel j is packed only
// when its filter starts (ready(j)), so later panels' uploads overlap earlier panels' filters.
// Narrower panels go first (C3 features: 24 columns, 3.9 ms, then 32 columns behind the first
// filter).  Every panel writes its own output / partials, so the order changes no result.
struct PackedInput {
  PanelPlan pp;
  Scratch x, xs;
  std::vector<int> order;  // panel processing order
  PackedInput(const csc_graph* g, const void* src, int64_t ld, int ncols, int io, cudaStream_t s, bool lazy = false)
      : g_(g), io_(io), s_(s) {
    pp = plan_panels(g->n, ncols, g->dtype, g->device, g->nnz);
    const size_t cs = dtype_size(g->dtype);
    for (int j = 0; j < pp.np; ++j) order.push_back(j);
    x.alloc(cs * pp.total, s);
    xs.alloc(cs * pp.total, s);
    if (lazy && pp.np >= 2 && g->n > 0 && g_opt.h2d_overlap.load() != 0 && !is_device_ptr(src, g->device) &&
        is_pinned_host(src)) {
      const size_t es = dtype_size(io);
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return pp.wc[a] < pp.wc[b]; });
      ev_.assign(pp.np, nullptr);
      for (int j = 0; j < pp.np; ++j) stage_.push_back(std::make_unique<Scratch>(es * g->n * pp.wc[j], s));
      cudaStream_t us = upload_stream(g->device);
      cudaEvent_t allocd = nullptr;
      CSC_CUDA(cudaEventCreateWithFlags(&allocd, cudaEventDisableTiming));
      CSC_CUDA(cudaEventRecord(allocd, s));  // the stream-ordered staging allocations
      CSC_CUDA(cudaStreamWaitEvent(us, allocd, 0));
      CSC_CUDA(cudaEventDestroy(allocd));
      for (int j : order) {
        copy_rows(stage_[j]->get(), pp.wc[j], static_cast<const char*>(src) + es * pp.c0[j], ld, g->n, pp.wc[j], es,
                  cudaMemcpyHostToDevice, us);
        CSC_CUDA(cudaEventCreateWithFlags(&ev_[j], cudaEventDisableTiming));
        CSC_CUDA(cudaEventRecord(ev_[j], us));
      }
      return;
    }
    StagedIn in;
    stage_in(src, ld, g->n, ncols, io, g->device, s, in);
    pack_panels(in.p, io, in.ld, x.get(), xs.get(), g, pp, s);
  }
  // before panel j's first step: its upload has landed, pack it
  void ready(int j, cudaStream_t s) const {
    if (ev_.empty()) return;
    CSC_CUDA(cudaStreamWaitEvent(s, ev_[j], 0));
    const size_t cs = dtype_size(g_->dtype);
    pack_one(stage_[j]->get(), io_, pp.wc[j], pp.wc[j], pp.pw[j], static_cast<char*>(x.get()) + cs * pp.off[j],
             static_cast<char*>(xs.get()) + cs * pp.off[j], g_, s);
  }
  ~PackedInput() {  // (an early exit left panels unread: their uploads still precede the frees)
    for (cudaEvent_t e : ev_)
      if (e) {
        cudaStreamWaitEvent(s_, e, 0);
        cudaEventDestroy(e);
      }
  }
  PackedInput(const PackedInput&) = delete;
  PackedInput& operator=(const PackedInput&) = delete;

 private:
  const csc_graph* g_;
  int io_;
  cudaStream_t s_;
  std::vector<std::unique_ptr<Scratch>> stage_;  // per-panel staged columns (lazy mode), freed on s_
  std::vector<cudaEvent_t> ev_;
};

template <typename T>
void run_filter_all(const csc_graph* g, const double* coeffs, int nc, const PackedInput& in, T* Yp, int epi,
                    double* part, int64_t part_stride, cudaStream_t s) {
  const PanelPlan& pp = in.pp;
  Scratch b0(sizeof(T) * g->n * pp.max_pw, s), b1(sizeof(T) * g->n * pp.max_pw, s);
  Scratch yacc;
  if (!Yp && g_opt.recurrence.load() == 1) yacc.alloc(sizeof(T) * g->n * pp.max_pw, s);
  for (int j : in.order) {
    in.ready(j, s);
    EpiExtra ex;
    ex.part = part ? part + part_stride * j : nullptr;
    filter_panel<T>(g, coeffs, nc, in.x.as<T>() + pp.off[j], in.xs.as<T>() + pp.off[j],
                    Yp ? Yp + pp.off[j] : nullptr, b0.as<T>(), b1.as<T>(), yacc.as<T>(), pp.pw[j], pp.wc[j], epi, ex, s);
  }
}

void unpack_out(const csc_graph* g, const PanelPlan& pp, const Scratch& yp, void* Y, int64_t ldy, int ncols, int io,
                cudaStream_t s) {
  StagedOut yo;
  stage_out(Y, ldy, g->n, ncols, io, g->device, s, yo);
  unpack_panels(yp.get(), g->dtype, pp, g->n, yo.p, io, yo.ld, s);
  finish_out(yo, g->n, ncols, io, s);
  if (yo.host) CSC_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

extern "C" {

int csc_laplacian_apply(const csc_graph* g, const void* X, int64_t ldx, void* Y, int64_t ldy, int ncols, int io_dtype,
                        void* stream) {
  return guard([&] {
    check_graph(g);
    check_block(g, X, ldx, ncols, io_dtype, "X");
    check_block(g, Y, ldy, ncols, io_dtype, "Y");
    if (g->n == 0 || ncols == 0) return;
    DeviceGuard dg(g->device);
    ensure_pool(g->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PackedInput in(g, X, ldx, ncols, io_dtype, s);
    const PanelPlan& pp = in.pp;
    Scratch yp(dtype_size(g->dtype) * pp.total, s);
    for (int j = 0; j < pp.np; ++j) {  // L X = X - Wn X  (graph.py:154-155); isolated rows: L x = x
      StepArgs a{};
      a.indptr = g->indptr;
      a.indices = g->indices;
      a.wv = g->wv;
      a.rs = g->rs;
      a.n = g->n;
      a.wc = pp.wc[j];
      a.ka = -1.0;
      a.kx = 1.0;
      a.hz = 1.0;
      a.last = 1;
      if (g->dtype == CSC_F64) {
        a.G = in.xs.as<double>() + pp.off[j];
        a.X = in.x.as<double>() + pp.off[j];
        a.O = yp.as<double>() + pp.off[j];
        launch_step<double>(g, a, pp.pw[j], EPI_NONE, s);
      } else {
        a.G = in.xs.as<float>() + pp.off[j];
        a.X = in.x.as<float>() + pp.off[j];
        a.O = yp.as<float>() + pp.off[j];
        launch_step<float>(g, a, pp.pw[j], EPI_NONE, s);
      }
    }
    unpack_out(g, pp, yp, Y, ldy, ncols, io_dtype, s);
  });
}

int csc_cheb_filter(const csc_graph* g, const double* coeffs, int ncoeffs, const void* X, int64_t ldx, void* Y,
                    int64_t ldy, int ncols, int io_dtype, void* stream) {
  return guard([&] {
    check_graph(g);
    check_coeffs(coeffs, ncoeffs);
    check_block(g, X, ldx, ncols, io_dtype, "X");
    check_block(g, Y, ldy, ncols, io_dtype, "Y");
    if (g->n == 0 || ncols == 0) return;
    DeviceGuard dg(g->device);
    ensure_pool(g->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PackedInput in(g, X, ldx, ncols, io_dtype, s, true);
    Scratch yp(dtype_size(g->dtype) * in.pp.total, s);
    if (g->dtype == CSC_F64)
      run_filter_all<double>(g, coeffs, ncoeffs, in, yp.as<double>(), EPI_NONE, nullptr, 0, s);
    else
      run_filter_all<float>(g, coeffs, ncoeffs, in, yp.as<float>(), EPI_NONE, nullptr, 0, s);
    unpack_out(g, in.pp, yp, Y, ldy, ncols, io_dtype, s);
  });
}

int csc_eigencount(const csc_graph* g, const double* coeffs, int ncoeffs, const void* R, int64_t ldr, int ncols,
                   int io_dtype, double* count, void* stream) {
  return guard([&] {
    check_graph(g);
    check_coeffs(coeffs, ncoeffs);
    check_block(g, R, ldr, ncols, io_dtype, "R");
    if (!count) fail(CSC_ERR_INVALID, "count is NULL");
    DeviceGuard dg(g->device);
    ensure_pool(g->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DeviceOut co(count, sizeof(double), g->device, s);
    if (g->n == 0 || ncols == 0) {
      CSC_CUDA(cudaMemsetAsync(co.as<double>(), 0, sizeof(double), s));
    } else {
      PackedInput in(g, R, ldr, ncols, io_dtype, s, true);
      const int cap = step_grid_cap(g->device);
      Scratch part(sizeof(double) * (size_t)cap * in.pp.np, s);
      CSC_CUDA(cudaMemsetAsync(part.get(), 0, part.bytes(), s));
      if (g->dtype == CSC_F64)
        run_filter_all<double>(g, coeffs, ncoeffs, in, nullptr, EPI_SUMSQ, part.as<double>(), cap, s);
      else
        run_filter_all<float>(g, coeffs, ncoeffs, in, nullptr, EPI_SUMSQ, part.as<double>(), cap, s);
      reduce_sum(part.as<double>(), (int64_t)cap * in.pp.np, co.as<double>(), s);
    }
    co.finish();
    if (co.on_host()) CSC_CUDA(cudaStreamSynchronize(s));
  });
}

int csc_filter_rowsq(const csc_graph* g, const double* coeffs, int ncoeffs, const void* R, int64_t ldr, int ncols,
                     int io_dtype, void* Y, int64_t ldy, double* rowsq, void* stream) {
  return guard([&] {
    check_graph(g);
    check_coeffs(coeffs, ncoeffs);
    check_block(g, R, ldr, ncols, io_dtype, "R");
    check_block(g, Y, ldy, ncols, io_dtype, "Y");
    if (!rowsq && g->n > 0) fail(CSC_ERR_INVALID, "rowsq is NULL");
    DeviceGuard dg(g->device);
    ensure_pool(g->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t n = g->n;
    if (n == 0) return;
    DeviceOut ro(rowsq, sizeof(double) * n, g->device, s);
    if (ncols == 0) {
      CSC_CUDA(cudaMemsetAsync(ro.as<double>(), 0, sizeof(double) * n, s));
    } else {
      PackedInput in(g, R, ldr, ncols, io_dtype, s, true);
      Scratch yp(dtype_size(g->dtype) * in.pp.total, s), part(sizeof(double) * n * in.pp.np, s);
      if (g->dtype == CSC_F64)
        run_filter_all<double>(g, coeffs, ncoeffs, in, yp.as<double>(), EPI_ROWSQ, part.as<double>(), n, s);
      else
        run_filter_all<float>(g, coeffs, ncoeffs, in, yp.as<float>(), EPI_ROWSQ, part.as<double>(), n, s);
      k_sum_panels<<<ew_grid(n), 256, 0, s>>>(part.as<double>(), in.pp.np, n, ro.as<double>());
      CSC_LAUNCHED();
      unpack_out(g, in.pp, yp, Y, ldy, ncols, io_dtype, s);
    }
    ro.finish();
    CSC_CUDA(cudaStreamSynchronize(s));
  });
}

int csc_normalize_rows(const void* Y, int64_t ldy, int64_t num_rows, int ncols, int io_dtype, const double* rowsq,
                       void* F, int64_t ldf, uint8_t* zero_flags, int64_t* num_zero, int device, void* stream) {
  return guard([&] {
    if (num_rows < 0 || ncols < 0 || ldy < ncols || ldf < ncols) fail(CSC_ERR_INVALID, "bad block shape");
    dtype_size(io_dtype);
    if (num_rows == 0) {
      if (num_zero) *num_zero = 0;
      return;
    }
    if (!Y || !F || !rowsq) fail(CSC_ERR_INVALID, "NULL buffer");
    DeviceGuard dg(device);
    ensure_pool(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    StagedIn yin;
    stage_in(Y, ldy, num_rows, ncols, io_dtype, device, s, yin);
    DeviceView rq(rowsq, sizeof(double) * num_rows, device, s);
    StagedOut fo;
    stage_out(F, ldf, num_rows, ncols, io_dtype, device, s, fo);
    DeviceOut zo(zero_flags, (size_t)num_rows, device, s);
    Scratch nz(sizeof(unsigned long long), s);
    CSC_CUDA(cudaMemsetAsync(nz.get(), 0, sizeof(unsigned long long), s));
    const int grid = (int)std::min<int64_t>((num_rows + 7) / 8, (int64_t)device_props(device).sms * 16);
    if (io_dtype == CSC_F64)
      k_normalize_rowmajor<double><<<grid, 256, 0, s>>>((const double*)yin.p, yin.ld, num_rows, ncols,
                                                        rq.as<double>(), (double*)fo.p, fo.ld, zo.as<uint8_t>(),
                                                        nz.as<unsigned long long>());
    else
      k_normalize_rowmajor<float><<<grid, 256, 0, s>>>((const float*)yin.p, yin.ld, num_rows, ncols,
                                                       rq.as<double>(), (float*)fo.p, fo.ld, zo.as<uint8_t>(),
                                                       nz.as<unsigned long long>());
    CSC_LAUNCHED();
    finish_out(fo, num_rows, ncols, io_dtype, s);
    zo.finish();
    unsigned long long hz = 0;
    CSC_CUDA(cudaMemcpyAsync(&hz, nz.get(), sizeof(hz), cudaMemcpyDeviceToHost, s));
    CSC_CUDA(cudaStreamSynchronize(s));
    if (num_zero) *num_zero = (int64_t)hz;
  });
}

int csc_system_apply(const csc_graph* g, const double* hp_coeffs, int ncoeffs, double gamma, double ridge,
                     const uint8_t* mask, const void* X, int64_t ldx, void* AP, int64_t ldap, int ncols, int io_dtype,
                     void* stream) {
  return guard([&] {
    check_graph(g);
    check_coeffs(hp_coeffs, ncoeffs);
    check_block(g, X, ldx, ncols, io_dtype, "X");
    check_block(g, AP, ldap, ncols, io_dtype, "AP");
    if (g->n == 0 || ncols == 0) return;
    if (!mask) fail(CSC_ERR_INVALID, "mask is NULL");
    DeviceGuard dg(g->device);
    ensure_pool(g->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PackedInput in(g, X, ldx, ncols, io_dtype, s);
    const PanelPlan& pp = in.pp;
    const size_t cs = dtype_size(g->dtype);
    DeviceView dm(mask, (size_t)g->n, g->device, s);
    Scratch ap(cs * pp.total, s);
    const int cap = step_grid_cap(g->device);
    Scratch part(sizeof(double) * (size_t)cap * pp.max_pw, s);
    Scratch b0(cs * g->n * pp.max_pw, s), b1(cs * g->n * pp.max_pw, s), yacc;
    if (g_opt.recurrence.load() == 1) yacc.alloc(cs * g->n * pp.max_pw, s);
    for (int j = 0; j < pp.np; ++j) {
      EpiExtra ex;
      ex.part = part.as<double>();
      ex.mask = dm.as<uint8_t>();
      ex.gamma = gamma;
      ex.ridge = ridge;
      if (g->dtype == CSC_F64) {
        ex.ap = ap.as<double>() + pp.off[j];
        filter_panel<double>(g, hp_coeffs, ncoeffs, in.x.as<double>() + pp.off[j], in.xs.as<double>() + pp.off[j],
                             nullptr, b0.as<double>(), b1.as<double>(), yacc.as<double>(), pp.pw[j], pp.wc[j],
                             EPI_CGAP, ex, s);
      } else {
        ex.ap = ap.as<float>() + pp.off[j];
        filter_panel<float>(g, hp_coeffs, ncoeffs, in.x.as<float>() + pp.off[j], in.xs.as<float>() + pp.off[j],
                            nullptr, b0.as<float>(), b1.as<float>(), yacc.as<float>(), pp.pw[j], pp.wc[j], EPI_CGAP,
                            ex, s);
      }
    }
    unpack_out(g, pp, ap, AP, ldap, ncols, io_dtype, s);
    CSC_CUDA(cudaStreamSynchronize(s));
  });
}

int csc_build_features(const csc_graph* g, const double* coeffs, int ncoeffs, const void* R, int64_t ldr, int ncols,
                       int io_dtype, void* F, int64_t ldf, uint8_t* zero_flags, int64_t* num_zero, void* stream) {
  return guard([&] {
    check_graph(g);
    check_coeffs(coeffs, ncoeffs);
    check_block(g, R, ldr, ncols, io_dtype, "R");
    check_block(g, F, ldf, ncols, io_dtype, "F");
    DeviceGuard dg(g->device);
    ensure_pool(g->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (g->n == 0 || ncols == 0) {
      if (num_zero) *num_zero = 0;
      return;
    }
    const int64_t n = g->n;
    PackedInput in(g, R, ldr, ncols, io_dtype, s, true);
    const PanelPlan& pp = in.pp;
    Scratch yp(dtype_size(g->dtype) * pp.total, s), rowsq(sizeof(double) * n * pp.np, s);
    if (g->dtype == CSC_F64)
      run_filter_all<double>(g, coeffs, ncoeffs, in, yp.as<double>(), EPI_ROWSQ, rowsq.as<double>(), n, s);
    else
      run_filter_all<float>(g, coeffs, ncoeffs, in, yp.as<float>(), EPI_ROWSQ, rowsq.as<double>(), n, s);
    StagedOut fo;
    stage_out(F, ldf, n, ncols, io_dtype, g->device, s, fo);
    DeviceOut zo(zero_flags, (size_t)n, g->device, s);
    Scratch nz(sizeof(unsigned long long), s);
    CSC_CUDA(cudaMemsetAsync(nz.get(), 0, sizeof(unsigned long long), s));
    const int grid = (int)std::min<int64_t>((n + 7) / 8, (int64_t)device_props(g->device).sms * 16);
    bool done = false;
    if (g_opt.fast_normalize.load()) {
      if (g->dtype == CSC_F64 && io_dtype == CSC_F64)
        done = launch_normalize_1p<double, double>(pp, yp.as<double>(), rowsq.as<double>(), n, (double*)fo.p, fo.ld,
                                                   zo.as<uint8_t>(), nz.as<unsigned long long>(), g->device, s);
      else if (g->dtype == CSC_F32 && io_dtype == CSC_F64)
        done = launch_normalize_1p<float, double>(pp, yp.as<float>(), rowsq.as<double>(), n, (double*)fo.p, fo.ld,
                                                  zo.as<uint8_t>(), nz.as<unsigned long long>(), g->device, s);
      else if (g->dtype == CSC_F64 && io_dtype == CSC_F32)
        done = launch_normalize_1p<double, float>(pp, yp.as<double>(), rowsq.as<double>(), n, (float*)fo.p, fo.ld,
                                                  zo.as<uint8_t>(), nz.as<unsigned long long>(), g->device, s);
      else
        done = launch_normalize_1p<float, float>(pp, yp.as<float>(), rowsq.as<double>(), n, (float*)fo.p, fo.ld,
                                                 zo.as<uint8_t>(), nz.as<unsigned long long>(), g->device, s);
    }
    // panel tables for the general normaliser (pageable copies: only when it runs)
    Scratch dmeta, doff;
    const int *pw = nullptr, *wc = nullptr, *c0 = nullptr;
    if (!done) {
      std::vector<int> meta(3 * pp.np);
      for (int j = 0; j < pp.np; ++j) {
        meta[j] = pp.pw[j];
        meta[pp.np + j] = pp.wc[j];
        meta[2 * pp.np + j] = pp.c0[j];
      }
      dmeta.alloc(sizeof(int) * meta.size(), s);
      doff.alloc(sizeof(int64_t) * pp.np, s);
      CSC_CUDA(cudaMemcpyAsync(dmeta.get(), meta.data(), sizeof(int) * meta.size(), cudaMemcpyHostToDevice, s));
      CSC_CUDA(cudaMemcpyAsync(doff.get(), pp.off.data(), sizeof(int64_t) * pp.np, cudaMemcpyHostToDevice, s));
      pw = dmeta.as<int>();
      wc = pw + pp.np;
      c0 = pw + 2 * pp.np;
    }
    if (done) {
    } else if (g->dtype == CSC_F64 && io_dtype == CSC_F64)
      k_normalize_rows<double, double><<<grid, 256, 0, s>>>(yp.as<double>(), rowsq.as<double>(), pp.np, pw, wc, c0,
                                                            doff.as<int64_t>(), n, (double*)fo.p, fo.ld,
                                                            zo.as<uint8_t>(), nz.as<unsigned long long>());
    else if (g->dtype == CSC_F32 && io_dtype == CSC_F64)
      k_normalize_rows<float, double><<<grid, 256, 0, s>>>(yp.as<float>(), rowsq.as<double>(), pp.np, pw, wc, c0,
                                                           doff.as<int64_t>(), n, (double*)fo.p, fo.ld,
                                                           zo.as<uint8_t>(), nz.as<unsigned long long>());
    else if (g->dtype == CSC_F64 && io_dtype == CSC_F32)
      k_normalize_rows<double, float><<<grid, 256, 0, s>>>(yp.as<double>(), rowsq.as<double>(), pp.np, pw, wc, c0,
                                                           doff.as<int64_t>(), n, (float*)fo.p, fo.ld,
                                                           zo.as<uint8_t>(), nz.as<unsigned long long>());
    else
      k_normalize_rows<float, float><<<grid, 256, 0, s>>>(yp.as<float>(), rowsq.as<double>(), pp.np, pw, wc, c0,
                                                          doff.as<int64_t>(), n, (float*)fo.p, fo.ld,
                                                          zo.as<uint8_t>(), nz.as<unsigned long long>());
    if (!done) CSC_LAUNCHED();
    finish_out(fo, n, ncols, io_dtype, s);
    zo.finish();
    // num_zero NULL with device outputs: no host readback, the call stays asynchronous
    if (num_zero || fo.host || zo.on_host()) {
      unsigned long long hz = 0;
      CSC_CUDA(cudaMemcpyAsync(&hz, nz.get(), sizeof(hz), cudaMemcpyDeviceToHost, s));
      CSC_CUDA(cudaStreamSynchronize(s));
      if (num_zero) *num_zero = (int64_t)hz;
    }
  });
}

}  // extern "C"
