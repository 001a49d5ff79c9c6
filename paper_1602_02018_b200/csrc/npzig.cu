// Parity RNG on the device: numpy's Generator(PCG64).standard_normal, bit-exact.
//
// The reference draws its probe and feature signals from seeded numpy streams
// (spectrum.py:84, features.py:63); on the host that is ~90 M normals/s, the
// dominant cost of run_csc at N = 1e6.  The stream is reproduced here:
//   1. device: PCG64 raw outputs u_i (128-bit LCG jump-ahead per thread chunk,
//      XSL-RR output); a raw is "special" if, as the start of a draw, it fails
//      the ziggurat's fast test (rabs >= ki[layer]) -- ~1 % of positions;
//   2. device: every special is evaluated as if it started a draw (wedge tests
//      with numpy's operation order; CUDA's exp decides only comparisons that
//      clear an 8-ulp margin); draws reaching a tail (their value needs libm's
//      log1p) or a closer call are evaluated on the host with the C library's
//      exp / log1p -- the functions numpy's own C code calls -- in one round trip;
//   3. device: which specials start a draw (a prefix max of the positions their
//      slow paths reach; short sequential walks inside clusters), positions
//      consumed inside slow paths are masked, a scan numbers the starts, fast
//      draws are +-rabs * wi[layer], and every value is divided by `divisor`.
// The caller advances its numpy generator by the returned raw count, so later
// host draws continue the same stream.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "internal.cuh"
#include "pcg64.cuh"

namespace csc {
namespace {

constexpr double kZigR = 3.6541528853610087963519472518;
constexpr double kZigInvR = 0.27366123732975827203338247596;
constexpr double kZigExpR = 7.69711747013104972;  // tail start of the 256-layer exponential ziggurat

// which numpy distribution a stream of draws follows
enum class Dist { Normal, Exponential };

__constant__ uint64_t c_ki[256];  // normal:      ki / wi
__constant__ double c_wi[256];
__constant__ uint64_t c_ke[256];  // exponential: ke / we
__constant__ double c_we[256];
__constant__ double c_fi[256];    // wedge tables (slow paths on the device)
__constant__ double c_fe[256];

struct Tables {
  uint64_t k[256];
  double w[256];
  double f[256];
  bool set = false;
};
Tables g_tab, g_exp;
std::mutex g_tab_mu;

// the fast-path test of numpy's random_standard_normal / random_standard_exponential
template <Dist D>
__device__ inline bool is_special(uint64_t u) {
  if (D == Dist::Normal) {
    const uint64_t rabs = ((u >> 8) >> 1) & 0x000fffffffffffffull;
    return rabs >= c_ki[u & 0xff];
  } else {
    return (u >> 11) >= c_ke[(u >> 3) & 0xff];
  }
}

template <Dist D>
__device__ inline double fast_value(uint64_t u) {
  if (D == Dist::Normal) {
    const uint64_t r = u >> 8;
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    const double v = (double)rabs * c_wi[u & 0xff];
    return (r & 1) ? -v : v;
  } else {
    return (double)(u >> 11) * c_we[(u >> 3) & 0xff];
  }
}


template <Dist D>
__global__ void k_pcg_raw(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, int64_t m,
                          uint64_t* __restrict__ raw, uint8_t* __restrict__ special) {
  // Thread t of T produces raws t, t + T, t + 2T, ...: consecutive threads write consecutive
  // positions (coalesced stores).  Raw p is the output of the state after p + 1 LCG steps;
  // moving T positions ahead is the affine map st -> A st + C of T steps.
  const u128 inc = make128(i_hi, i_lo);
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  if (t >= m) return;
  u128 A = 1, C = 0, cur_mult = pcg_mult(), cur_plus = inc;
  for (uint64_t delta = (uint64_t)T; delta; delta >>= 1) {
    if (delta & 1) {
      A *= cur_mult;
      C = C * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
  }
  u128 st = pcg_advance(make128(s_hi, s_lo), inc, (uint64_t)t + 1);
  for (int64_t i = t; i < m; i += T) {
    const uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st;  // numpy's XSL-RR output of st
    const uint64_t x = hi ^ lo;
    const unsigned r = (unsigned)(hi >> 58);
    const uint64_t u = (x >> r) | (x << ((64u - r) & 63u));
    raw[i] = u;
    special[i] = is_special<D>(u) ? 1 : 0;
    st = A * st + C;
  }
}

__global__ void k_gather_near(const uint64_t* __restrict__ raw, const int64_t* __restrict__ pos, int64_t nspec,
                              int64_t m, int near, uint64_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nspec * near; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = t / near;
    const int64_t p = pos[q] + (t - q * near);
    out[t] = raw[p < m ? p : m - 1];
  }
}

__global__ void k_init_starts(int64_t m, uint32_t* __restrict__ is_start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    is_start[i] = 1;
}

template <Dist D>
__global__ void k_emit(const uint64_t* __restrict__ raw, const uint8_t* __restrict__ special,
                       const uint32_t* __restrict__ is_start, const uint32_t* __restrict__ index, int64_t m,
                       int64_t count, const int64_t* __restrict__ sp_pos, const double* __restrict__ sp_val,
                       int64_t nsp, double divisor, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    if (!is_start[i]) continue;
    const int64_t j = index[i];
    if (j >= count) continue;
    double v;
    if (special[i]) {
      int64_t lo = 0, hi = nsp;  // sp_pos sorted
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (sp_pos[mid] < i)
          lo = mid + 1;
        else
          hi = mid;
      }
      v = sp_val[lo];
    } else {
      v = fast_value<D>(raw[i]);
    }
    out[j] = v / divisor;
  }
}

// Host evaluation of one draw starting at raw position `pos` (the slow path of
// numpy's random_standard_normal); `raw` holds the device-generated stream,
// positions beyond it are produced by jump-ahead.  Returns the value and sets
// the number of raws consumed.
struct HostStream {
  const uint64_t* near;  // raws pos .. pos + nnear - 1
  int64_t nnear;
  int64_t pos;
  u128 s0, inc;
  int64_t k = 0;
  uint64_t next() {
    const int64_t i = k++;
    if (i < nnear) return near[i];
    u128 st = pcg_advance(s0, inc, (uint64_t)(pos + i));
    return pcg_next(st, inc);
  }
  double next_double() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
};

// numpy's random_standard_normal, whole draw (fast and slow paths)
double slow_normal(HostStream& hs, const Tables& t) {
  for (;;) {
    uint64_t r = hs.next();
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * t.w[idx];
    if (sign) x = -x;
    if (rabs < t.k[idx]) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = -kZigInvR * std::log1p(-hs.next_double());
        const double yy = -std::log1p(-hs.next_double());
        if (yy + yy > xx * xx) return ((rabs >> 8) & 1) ? -(kZigR + xx) : kZigR + xx;
      }
    } else {
      if ((t.f[idx - 1] - t.f[idx]) * hs.next_double() + t.f[idx] < std::exp(-0.5 * x * x)) return x;
    }
  }
}

// numpy's random_standard_exponential (standard_exponential_unlikely retries the whole draw)
double slow_exponential(HostStream& hs, const Tables& t) {
  for (;;) {
    uint64_t ri = hs.next() >> 3;
    const int idx = (int)(ri & 0xff);
    ri >>= 8;
    const double x = (double)ri * t.w[idx];
    if (ri < t.k[idx]) return x;
    if (idx == 0) return kZigExpR - std::log1p(-hs.next_double());
    if ((t.f[idx - 1] - t.f[idx]) * hs.next_double() + t.f[idx] < std::exp(-x)) return x;
  }
}

template <Dist D>
double slow_draw(HostStream& hs, const Tables& t) {
  return D == Dist::Normal ? slow_normal(hs, t) : slow_exponential(hs, t);
}

// grow-only pinned host staging, one per thread
template <typename T>
T* pinned_buffer(size_t count, int slot) {
  static thread_local void* buf[4] = {nullptr, nullptr, nullptr, nullptr};
  static thread_local size_t cap[4] = {0, 0, 0, 0};
  const size_t bytes = sizeof(T) * std::max<size_t>(count, 1);
  if (cap[slot] < bytes) {
    if (buf[slot]) cudaFreeHost(buf[slot]);
    buf[slot] = nullptr;
    CSC_CUDA(cudaMallocHost(&buf[slot], bytes + bytes / 4));
    cap[slot] = bytes + bytes / 4;
  }
  return static_cast<T*>(buf[slot]);
}

// raw output at stream position i (from the generated buffer, else by jump-ahead)
__device__ inline uint64_t raw_at(const uint64_t* __restrict__ raw, int64_t m, int64_t i, u128 s0, u128 inc) {
  if (i < m) return raw[i];
  u128 st = pcg_advance(s0, inc, (uint64_t)i);
  return pcg_next(st, inc);
}

__device__ inline double raw_double(uint64_t u) { return (double)(u >> 11) * (1.0 / 9007199254740992.0); }

// The wedge test compares against libm's exp in the reference; CUDA's exp is within
// 1 ulp and glibc's within ~0.5 ulp of the true value, so a comparison that clears
// 8 ulp is decided identically.  Closer calls go to the host.
__device__ inline bool too_close(double lhs, double rhs) {
  return fabs(lhs - rhs) <= 8.0 * 2.220446049250313e-16 * fabs(rhs);
}

// Every special position evaluated as if it started a draw (numpy's slow paths, same
// operation order as the C code: no FMA contraction): value and raws consumed; draws
// that reach a tail (libm log1p) or a too-close wedge test are flagged for the host.
template <Dist D>
__global__ void k_slow_eval(const uint64_t* __restrict__ raw, int64_t m, const int64_t* __restrict__ pos,
                            int64_t nspec, uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo,
                            double* __restrict__ val, int32_t* __restrict__ cons, uint8_t* __restrict__ flag) {
  const u128 s0 = make128(s_hi, s_lo), inc = make128(i_hi, i_lo);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nspec; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pos[q];
    int k = 0;
    bool host = true;
    double v = 0.0;
    for (int tries = 0; tries < 32; ++tries) {
      const uint64_t u = raw_at(raw, m, p + k, s0, inc);
      ++k;
      double x, lhs, rhs;
      if (D == Dist::Normal) {
        const int idx = (int)(u & 0xff);
        const uint64_t r = u >> 8;
        const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
        x = (double)rabs * c_wi[idx];
        if (r & 1) x = -x;
        if (rabs < c_ki[idx]) { v = x; host = false; break; }
        if (idx == 0) break;  // tail: libm log1p decides value and consumption
        const double uu = raw_double(raw_at(raw, m, p + k, s0, inc));
        ++k;
        lhs = __dadd_rn(__dmul_rn(__dsub_rn(c_fi[idx - 1], c_fi[idx]), uu), c_fi[idx]);
        rhs = exp(__dmul_rn(__dmul_rn(-0.5, x), x));
      } else {
        uint64_t ri = u >> 3;
        const int idx = (int)(ri & 0xff);
        ri >>= 8;
        x = (double)ri * c_we[idx];
        if (ri < c_ke[idx]) { v = x; host = false; break; }
        if (idx == 0) break;  // tail: ziggurat_exp_r - log1p(-u)
        const double uu = raw_double(raw_at(raw, m, p + k, s0, inc));
        ++k;
        lhs = __dadd_rn(__dmul_rn(__dsub_rn(c_fe[idx - 1], c_fe[idx]), uu), c_fe[idx]);
        rhs = exp(-x);
      }
      if (too_close(lhs, rhs)) break;
      if (lhs < rhs) { v = x; host = false; break; }
      // rejected: numpy retries the whole draw from the next raw
    }
    val[q] = v;
    cons[q] = k;
    flag[q] = host ? 1 : 0;
  }
}

__global__ void k_flag_pos(const int64_t* __restrict__ pos, const int64_t* __restrict__ fidx,
                           const int64_t* __restrict__ nfl_p, int64_t* __restrict__ fpos) {
  const int64_t nfl = *nfl_p;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nfl; t += (int64_t)gridDim.x * blockDim.x)
    fpos[t] = pos[fidx[t]];
}

__global__ void k_scatter_host(const int64_t* __restrict__ fidx, int64_t nfl, const double* __restrict__ hv,
                               const int32_t* __restrict__ hc, double* __restrict__ val, int32_t* __restrict__ cons) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nfl; t += (int64_t)gridDim.x * blockDim.x) {
    val[fidx[t]] = hv[t];
    cons[fidx[t]] = hc[t];
  }
}

__global__ void k_reach(const int64_t* __restrict__ pos, const int32_t* __restrict__ cons, int64_t nspec,
                        int64_t* __restrict__ reach) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nspec; q += (int64_t)gridDim.x * blockDim.x)
    reach[q] = pos[q] + cons[q];
}

// Which specials start a draw: a special that no earlier special's slow path reaches
// (prefix max of reach <= its position) heads a cluster and starts a draw; inside a
// cluster the starts follow sequentially (clusters are a few specials long).
__global__ void k_resolve(const int64_t* __restrict__ pos, const int32_t* __restrict__ cons,
                          const int64_t* __restrict__ pmax, int64_t nspec, uint8_t* __restrict__ start) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nspec; q += (int64_t)gridDim.x * blockDim.x) {
    if (pmax[q] > pos[q]) continue;  // not a cluster head
    start[q] = 1;
    int64_t next_free = pos[q] + cons[q];
    for (int64_t r = q + 1; r < nspec && pmax[r] > pos[r]; ++r) {
      if (pos[r] >= next_free) {
        start[r] = 1;
        next_free = pos[r] + cons[r];
      } else {
        start[r] = 0;
      }
    }
  }
}

// positions consumed inside a starting special's slow path are not draw starts;
// covered specials are not starts either
__global__ void k_mark_consumed(const int64_t* __restrict__ pos, const int32_t* __restrict__ cons,
                                const uint8_t* __restrict__ start, int64_t nspec, int64_t m,
                                uint32_t* __restrict__ is_start) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nspec; q += (int64_t)gridDim.x * blockDim.x) {
    if (!start[q]) {
      is_start[pos[q]] = 0;
      continue;
    }
    for (int j = 1; j < cons[q]; ++j)
      if (pos[q] + j < m) is_start[pos[q] + j] = 0;
  }
}

// the count-th draw: its position and the raws it consumed
__global__ void k_find_end(const uint32_t* __restrict__ is_start, const uint32_t* __restrict__ index, int64_t m,
                           int64_t count, const uint8_t* __restrict__ special, const int64_t* __restrict__ pos,
                           const int32_t* __restrict__ cons, int64_t nspec, int64_t* __restrict__ end) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    if (!is_start[i] || (int64_t)index[i] != count - 1) continue;
    int64_t c = 1;
    if (special[i]) {
      int64_t lo = 0, hi = nspec;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (pos[mid] < i) lo = mid + 1;
        else hi = mid;
      }
      c = cons[lo];
    }
    end[0] = i;
    end[1] = c;
  }
}

inline int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 65535)); }

// The first `count` draws of numpy's Generator(PCG64) stream of distribution D
// from state (s0, inc), divided by `divisor`, into device memory; returns the
// number of raw uint64 the draws consumed.  Everything runs on the device except
// the few slow paths k_slow_eval flags (one host round trip).
template <Dist D>
int64_t numpy_draws(const Tables& t, u128 s0, u128 inc, int64_t count, double divisor, double* out, cudaStream_t s) {
  const uint64_t inc_hi = (uint64_t)(inc >> 64), inc_lo = (uint64_t)inc;
  const uint64_t s_hi = (uint64_t)(s0 >> 64), s_lo = (uint64_t)s0;
  int dev = 0;
  CSC_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t mp = side_pool(dev);
  if (D == Dist::Normal) {
    CSC_CUDA(cudaMemcpyToSymbolAsync(c_ki, t.k, sizeof(t.k), 0, cudaMemcpyHostToDevice, s));
    CSC_CUDA(cudaMemcpyToSymbolAsync(c_wi, t.w, sizeof(t.w), 0, cudaMemcpyHostToDevice, s));
    CSC_CUDA(cudaMemcpyToSymbolAsync(c_fi, t.f, sizeof(t.f), 0, cudaMemcpyHostToDevice, s));
  } else {
    CSC_CUDA(cudaMemcpyToSymbolAsync(c_ke, t.k, sizeof(t.k), 0, cudaMemcpyHostToDevice, s));
    CSC_CUDA(cudaMemcpyToSymbolAsync(c_we, t.w, sizeof(t.w), 0, cudaMemcpyHostToDevice, s));
    CSC_CUDA(cudaMemcpyToSymbolAsync(c_fe, t.f, sizeof(t.f), 0, cudaMemcpyHostToDevice, s));
  }
  const bool timing = std::getenv("CSC_RNG_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  auto t_start = now();
  int64_t m = count + count / 16 + 4096;  // ~2 % of raws are consumed inside slow paths
  for (int attempt = 0; attempt < 4; ++attempt, m = m * 2) {
    // 1. raws + special flags; compact the special positions (stable)
    Scratch raw(sizeof(uint64_t) * m, s, mp), special(m, s, mp);
    int dev_now = 0;
    CSC_CUDA(cudaGetDevice(&dev_now));
    const int64_t pblocks = std::min<int64_t>((m + 255) / 256, (int64_t)device_props(dev_now).sms * 8);
    k_pcg_raw<D><<<(int)std::max<int64_t>(pblocks, 1), 256, 0, s>>>(
        s_hi, s_lo, inc_hi, inc_lo, m, raw.as<uint64_t>(), special.as<uint8_t>());
    CSC_LAUNCHED();
    Scratch pos(sizeof(int64_t) * m, s, mp), nsel(2 * sizeof(int64_t), s, mp);
    thrust::counting_iterator<int64_t> it(0);
    {
      size_t tb = 0;
      CSC_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, special.as<uint8_t>(), pos.as<int64_t>(),
                                          nsel.as<int64_t>(), m, s));
      Scratch tmp(tb, s, mp);
      CSC_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, it, special.as<uint8_t>(), pos.as<int64_t>(),
                                          nsel.as<int64_t>(), m, s));
      CSC_LAUNCHED();
    }
    int64_t nspec = 0;
    CSC_CUDA(cudaMemcpyAsync(&nspec, nsel.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CSC_CUDA(cudaStreamSynchronize(s));
    // 2. slow paths on the device
    const int64_t ns1 = std::max<int64_t>(nspec, 1);
    Scratch val(sizeof(double) * ns1, s, mp), cons(sizeof(int32_t) * ns1, s, mp), flag(ns1, s, mp),
        fidx(sizeof(int64_t) * ns1, s, mp);
    int64_t nfl = 0;
    if (nspec > 0) {
      k_slow_eval<D><<<grid_of(nspec), 256, 0, s>>>(raw.as<uint64_t>(), m, pos.as<int64_t>(), nspec, s_hi, s_lo,
                                                    inc_hi, inc_lo, val.as<double>(), cons.as<int32_t>(),
                                                    flag.as<uint8_t>());
      CSC_LAUNCHED();
      size_t tb = 0;
      CSC_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, flag.as<uint8_t>(), fidx.as<int64_t>(),
                                          nsel.as<int64_t>() + 1, nspec, s));
      Scratch tmp(tb, s, mp);
      CSC_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, it, flag.as<uint8_t>(), fidx.as<int64_t>(),
                                          nsel.as<int64_t>() + 1, nspec, s));
      CSC_LAUNCHED();
      CSC_CUDA(cudaMemcpyAsync(&nfl, nsel.as<int64_t>() + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      CSC_CUDA(cudaStreamSynchronize(s));
    }
    {
      auto t_gen = now();
      // 3. flagged slow paths on the host (libm), results scattered back
      if (nfl > 0) {
        constexpr int kNear = 8;
        Scratch fpos(sizeof(int64_t) * nfl, s, mp), gath(sizeof(uint64_t) * nfl * kNear, s, mp);
        k_flag_pos<<<grid_of(nfl), 256, 0, s>>>(pos.as<int64_t>(), fidx.as<int64_t>(), nsel.as<int64_t>() + 1,
                                                fpos.as<int64_t>());
        CSC_LAUNCHED();
        k_gather_near<<<grid_of(nfl * kNear), 256, 0, s>>>(raw.as<uint64_t>(), fpos.as<int64_t>(), nfl, m, kNear,
                                                          gath.as<uint64_t>());
        CSC_LAUNCHED();
        int64_t* hpos = pinned_buffer<int64_t>(nfl, 0);
        uint64_t* hraw = pinned_buffer<uint64_t>((size_t)nfl * kNear, 1);
        double* hv = pinned_buffer<double>(nfl, 2);
        int32_t* hc = pinned_buffer<int32_t>(nfl, 3);
        CSC_CUDA(cudaMemcpyAsync(hpos, fpos.get(), sizeof(int64_t) * nfl, cudaMemcpyDeviceToHost, s));
        CSC_CUDA(cudaMemcpyAsync(hraw, gath.get(), sizeof(uint64_t) * nfl * kNear, cudaMemcpyDeviceToHost, s));
        CSC_CUDA(cudaStreamSynchronize(s));
        for (int64_t q = 0; q < nfl; ++q) {
          HostStream hs{hraw + q * kNear, std::min<int64_t>(kNear, m - hpos[q]), hpos[q], s0, inc};
          hv[q] = slow_draw<D>(hs, t);
          hc[q] = (int32_t)hs.k;
        }
        Scratch dv(sizeof(double) * nfl, s, mp), dc(sizeof(int32_t) * nfl, s, mp);
        CSC_CUDA(cudaMemcpyAsync(dv.get(), hv, sizeof(double) * nfl, cudaMemcpyHostToDevice, s));
        CSC_CUDA(cudaMemcpyAsync(dc.get(), hc, sizeof(int32_t) * nfl, cudaMemcpyHostToDevice, s));
        k_scatter_host<<<grid_of(nfl), 256, 0, s>>>(fidx.as<int64_t>(), nfl, dv.as<double>(), dc.as<int32_t>(),
                                                   val.as<double>(), cons.as<int32_t>());
        CSC_LAUNCHED();
        CSC_CUDA(cudaStreamSynchronize(s));  // pinned staging is reused by the next call
      }
      auto t_eval = now();
      // 4. which specials start a draw; mask consumed positions; number the starts
      Scratch reach(sizeof(int64_t) * std::max<int64_t>(nspec, 1), s, mp),
          pmax(sizeof(int64_t) * std::max<int64_t>(nspec, 1), s, mp), start(std::max<int64_t>(nspec, 1), s, mp);
      Scratch is_start(sizeof(uint32_t) * m, s, mp), index(sizeof(uint32_t) * m, s, mp), end(2 * sizeof(int64_t), s, mp);
      k_init_starts<<<grid_of(m), 256, 0, s>>>(m, is_start.as<uint32_t>());
      CSC_LAUNCHED();
      if (nspec > 0) {
        k_reach<<<grid_of(nspec), 256, 0, s>>>(pos.as<int64_t>(), cons.as<int32_t>(), nspec, reach.as<int64_t>());
        CSC_LAUNCHED();
        size_t tb2 = 0;
        CSC_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, tb2, reach.as<int64_t>(), pmax.as<int64_t>(), cub::Max(),
                                                (int64_t)-1, nspec, s));
        Scratch tmp2(tb2, s, mp);
        CSC_CUDA(cub::DeviceScan::ExclusiveScan(tmp2.get(), tb2, reach.as<int64_t>(), pmax.as<int64_t>(), cub::Max(),
                                                (int64_t)-1, nspec, s));
        CSC_LAUNCHED();
        k_resolve<<<grid_of(nspec), 256, 0, s>>>(pos.as<int64_t>(), cons.as<int32_t>(), pmax.as<int64_t>(), nspec,
                                                start.as<uint8_t>());
        CSC_LAUNCHED();
        k_mark_consumed<<<grid_of(nspec), 256, 0, s>>>(pos.as<int64_t>(), cons.as<int32_t>(), start.as<uint8_t>(),
                                                      nspec, m, is_start.as<uint32_t>());
        CSC_LAUNCHED();
      }
      size_t tb3 = 0;
      CSC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb3, is_start.as<uint32_t>(), index.as<uint32_t>(), m, s));
      Scratch tmp3(tb3, s, mp);
      CSC_CUDA(cub::DeviceScan::ExclusiveSum(tmp3.get(), tb3, is_start.as<uint32_t>(), index.as<uint32_t>(), m, s));
      CSC_LAUNCHED();
      CSC_CUDA(cudaMemsetAsync(end.get(), 0xff, 2 * sizeof(int64_t), s));
      k_find_end<<<grid_of(m), 256, 0, s>>>(is_start.as<uint32_t>(), index.as<uint32_t>(), m, count,
                                            special.as<uint8_t>(), pos.as<int64_t>(), cons.as<int32_t>(), nspec,
                                            end.as<int64_t>());
      CSC_LAUNCHED();
      // 5. emit (the values of special starts come from val)
      k_emit<D><<<grid_of(m), 256, 0, s>>>(raw.as<uint64_t>(), special.as<uint8_t>(), is_start.as<uint32_t>(),
                                           index.as<uint32_t>(), m, count, pos.as<int64_t>(), val.as<double>(), nspec,
                                           divisor, out);
      CSC_LAUNCHED();
      int64_t hend[2] = {-1, -1};
      CSC_CUDA(cudaMemcpyAsync(hend, end.get(), sizeof(hend), cudaMemcpyDeviceToHost, s));
      CSC_CUDA(cudaStreamSynchronize(s));
      if (timing)
        std::fprintf(stderr, "parity RNG (%s): n=%lld specials=%lld host=%lld gen %.2f eval %.2f emit %.2f ms\n",
                     D == Dist::Normal ? "normal" : "exponential", (long long)count, (long long)nspec,
                     (long long)nfl, ms(t_start, t_gen), ms(t_gen, t_eval), ms(t_eval, now()));
      if (hend[0] < 0) continue;  // fewer than `count` starts in the generated raws: retry with more
      return hend[0] + hend[1];
    }
  }
  fail(CSC_ERR_CUDA, "parity RNG: raw margin exhausted");
}

Tables tables_of(const Tables& g, const char* what) {
  std::lock_guard<std::mutex> lk(g_tab_mu);
  if (!g.set) fail(CSC_ERR_INVALID, std::string(what) + " tables not set");
  return g;
}

}  // namespace

int64_t numpy_exponentials(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t count,
                           double* out, cudaStream_t s) {
  if (count <= 0) return 0;
  const Tables t = tables_of(g_exp, "exponential ziggurat");
  return numpy_draws<Dist::Exponential>(t, make128(state_hi, state_lo), make128(inc_hi, inc_lo), count, 1.0, out, s);
}

}  // namespace csc

using namespace csc;

extern "C" {

int csc_set_normal_tables(const uint64_t* ki, const double* wi, const double* fi) {
  return guard([&] {
    if (!ki || !wi || !fi) fail(CSC_ERR_INVALID, "NULL table");
    std::lock_guard<std::mutex> lk(g_tab_mu);
    std::memcpy(g_tab.k, ki, sizeof(g_tab.k));
    std::memcpy(g_tab.w, wi, sizeof(g_tab.w));
    std::memcpy(g_tab.f, fi, sizeof(g_tab.f));
    g_tab.set = true;
  });
}

int csc_set_exponential_tables(const uint64_t* ke, const double* we, const double* fe) {
  return guard([&] {
    if (!ke || !we || !fe) fail(CSC_ERR_INVALID, "NULL table");
    std::lock_guard<std::mutex> lk(g_tab_mu);
    std::memcpy(g_exp.k, ke, sizeof(g_exp.k));
    std::memcpy(g_exp.w, we, sizeof(g_exp.w));
    std::memcpy(g_exp.f, fe, sizeof(g_exp.f));
    g_exp.set = true;
  });
}

int csc_numpy_normals(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t count,
                      double divisor, double* out, int64_t* raw_consumed, int device, void* stream) {
  return guard([&] {
    if (count < 0) fail(CSC_ERR_INVALID, "count must be >= 0");
    if (!out && count > 0) fail(CSC_ERR_INVALID, "out is NULL");
    if (!raw_consumed) fail(CSC_ERR_INVALID, "raw_consumed is NULL");
    const Tables t = tables_of(g_tab, "normal ziggurat (csc_set_normal_tables)");
    if (count == 0) {
      *raw_consumed = 0;
      return;
    }
    DeviceGuard dg(device);
    ensure_pool(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DeviceOut dout(out, sizeof(double) * count, device, s);
    *raw_consumed = numpy_draws<Dist::Normal>(t, make128(state_hi, state_lo), make128(inc_hi, inc_lo), count, divisor,
                                              dout.as<double>(), s);
    dout.finish();
    CSC_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
