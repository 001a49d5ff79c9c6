// Parity RNG on the device: numpy's Generator(PCG64).standard_normal, bit-exact.
//
// The reference draws its probe and feature signals from seeded numpy streams
// (spectrum.py:84, features.py:63); on the host that is ~90 M normals/s, the
// dominant cost of run_csc at N = 1e6.  The stream is reproduced here:
//   1. device: PCG64 raw outputs u_i (128-bit LCG jump-ahead per thread chunk,
//      XSL-RR output); a raw is "special" if, as the start of a draw, it fails
//      the ziggurat's fast test (rabs >= ki[layer]) -- ~1 % of positions;
//   2. host: a sequential walk over the special positions decides which are
//      draw starts and evaluates their wedge / tail paths with the C library's
//      exp / log1p (the functions numpy's own C code calls), recording each
//      start's value and how many raws it consumed;
//   3. device: positions consumed inside slow paths are masked, a scan numbers
//      the remaining starts, fast draws are +-rabs * wi[layer], and every value
//      is divided by `divisor` into the output.
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
#include <thread>
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

constexpr int kChunk = 64;  // raws per thread

template <Dist D>
__global__ void k_pcg_raw(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, int64_t m,
                          uint64_t* __restrict__ raw, uint8_t* __restrict__ special) {
  const u128 inc = make128(i_hi, i_lo);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c * kChunk < m; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = c * kChunk;
    u128 st = pcg_advance(make128(s_hi, s_lo), inc, (uint64_t)i0);
    const int64_t i1 = min(m, i0 + kChunk);
    for (int64_t i = i0; i < i1; ++i) {
      const uint64_t u = pcg_next(st, inc);
      raw[i] = u;
      special[i] = is_special<D>(u) ? 1 : 0;
    }
  }
}

// positions consumed inside slow paths are not draw starts
__global__ void k_mark_skips(const int64_t* __restrict__ skip_begin, const int32_t* __restrict__ skip_len, int64_t nskip,
                             int64_t m, uint32_t* __restrict__ is_start) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nskip; t += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < skip_len[t]; ++k) {
      const int64_t p = skip_begin[t] + k;
      if (p < m) is_start[p] = 0;
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

// The first `count` draws of numpy's Generator(PCG64) stream of distribution D
// from state (s0, inc), divided by `divisor`, into device memory; returns the
// number of raw uint64 the draws consumed.
template <Dist D>
int64_t numpy_draws(const Tables& t, u128 s0, u128 inc, int64_t count, double divisor, double* out, cudaStream_t s) {
  const uint64_t inc_hi = (uint64_t)(inc >> 64), inc_lo = (uint64_t)inc;
  int dev = 0;
  CSC_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t mp = side_pool(dev);
  if (D == Dist::Normal) {
    CSC_CUDA(cudaMemcpyToSymbolAsync(c_ki, t.k, sizeof(t.k), 0, cudaMemcpyHostToDevice, s));
    CSC_CUDA(cudaMemcpyToSymbolAsync(c_wi, t.w, sizeof(t.w), 0, cudaMemcpyHostToDevice, s));
  } else {
    CSC_CUDA(cudaMemcpyToSymbolAsync(c_ke, t.k, sizeof(t.k), 0, cudaMemcpyHostToDevice, s));
    CSC_CUDA(cudaMemcpyToSymbolAsync(c_we, t.w, sizeof(t.w), 0, cudaMemcpyHostToDevice, s));
  }
    const bool timing = std::getenv("CSC_RNG_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    auto t_start = now();
    int64_t m = count + count / 16 + 4096;  // ~2.2 % of raws are consumed inside slow paths
    for (int attempt = 0; attempt < 4; ++attempt, m = m * 2) {
      Scratch raw(sizeof(uint64_t) * m, s, mp), special(m, s, mp);
      const int64_t chunks = (m + kChunk - 1) / kChunk;
      k_pcg_raw<D><<<(int)std::min<int64_t>((chunks + 255) / 256, 65535), 256, 0, s>>>(
          (uint64_t)(s0 >> 64), (uint64_t)s0, inc_hi, inc_lo, m, raw.as<uint64_t>(), special.as<uint8_t>());
      CSC_LAUNCHED();
      // compact the special positions (stable)
      Scratch pos(sizeof(int64_t) * m, s, mp), nsel(sizeof(int64_t), s, mp);
      size_t tb = 0;
      thrust::counting_iterator<int64_t> it(0);
      CSC_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, special.as<uint8_t>(), pos.as<int64_t>(),
                                          nsel.as<int64_t>(), m, s));
      Scratch tmp(tb, s, mp);
      CSC_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, it, special.as<uint8_t>(), pos.as<int64_t>(),
                                          nsel.as<int64_t>(), m, s));
      CSC_LAUNCHED();
      int64_t nspec = 0;
      CSC_CUDA(cudaMemcpyAsync(&nspec, nsel.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      CSC_CUDA(cudaStreamSynchronize(s));
      auto t_gen = now();
      int64_t* hpos = pinned_buffer<int64_t>(nspec, 0);
      if (nspec) CSC_CUDA(cudaMemcpyAsync(hpos, pos.get(), sizeof(int64_t) * nspec, cudaMemcpyDeviceToHost, s));
      // raws following each special position (slow paths read a few more)
      constexpr int kNear = 8;
      uint64_t* hraw = pinned_buffer<uint64_t>((size_t)nspec * kNear, 1);
      Scratch gath(sizeof(uint64_t) * std::max<int64_t>(nspec * kNear, 1), s, mp);
      if (nspec) {
        k_gather_near<<<(int)std::min<int64_t>((nspec * kNear + 255) / 256, 65535), 256, 0, s>>>(
            raw.as<uint64_t>(), pos.as<int64_t>(), nspec, m, kNear, gath.as<uint64_t>());
        CSC_LAUNCHED();
        CSC_CUDA(cudaMemcpyAsync(hraw, gath.get(), sizeof(uint64_t) * nspec * kNear, cudaMemcpyDeviceToHost, s));
      }
      CSC_CUDA(cudaStreamSynchronize(s));
      auto t_d2h = now();
      // every special evaluated as if it started a draw (its value and consumption
      // depend only on its own raws): in parallel host threads with the C library's
      // exp / log1p, then a sequential pass keeps the real starts
      std::vector<double> val(nspec);
      std::vector<int32_t> cons_all(nspec);
      {
        const int nth = (int)std::max<int64_t>(1, std::min<int64_t>(16, nspec / 8192));
        std::vector<std::thread> pool;
        auto work = [&](int th) {
          for (int64_t q = th; q < nspec; q += nth) {
            HostStream hs{hraw + q * kNear, std::min<int64_t>(kNear, m - hpos[q]), hpos[q], s0, inc};
            val[q] = slow_draw<D>(hs, t);
            cons_all[q] = (int32_t)hs.k;
          }
        };
        for (int th = 1; th < nth; ++th) pool.emplace_back(work, th);
        work(0);
        for (auto& th : pool) th.join();
      }
      std::vector<int64_t> sp_pos, skip_begin;
      std::vector<double> sp_val;
      std::vector<int32_t> skip_len;
      int64_t next_free = 0, skipped = 0;
      for (int64_t q = 0; q < nspec; ++q) {
        const int64_t p = hpos[q];
        if (p < next_free) continue;      // consumed by an earlier slow path
        if (p - skipped >= count) break;  // draws before p already complete the request
        sp_pos.push_back(p);
        sp_val.push_back(val[q]);
        if (cons_all[q] > 1) {
          skip_begin.push_back(p + 1);
          skip_len.push_back(cons_all[q] - 1);
          skipped += cons_all[q] - 1;
        }
        next_free = p + cons_all[q];
      }
      auto t_walk = now();
      // position of the count-th draw start
      // starts are all positions not inside a skip run; the j-th start (0-based) is at
      // j + (skipped raws before it).  Walk the skip runs to locate start `count - 1`.
      int64_t before = 0;  // skipped raws before the current position
      int64_t end_pos = -1;
      {
        int64_t target = count - 1;  // draw index
        size_t r = 0;
        int64_t cur = 0;  // candidate position = target + before
        for (;;) {
          cur = target + before;
          if (r < skip_begin.size() && skip_begin[r] <= cur) {
            before += skip_len[r];
            ++r;
            continue;
          }
          break;
        }
        end_pos = cur;
      }
      if (end_pos >= m) continue;  // not enough raws generated: retry with more
      // consumption of the last draw
      int64_t cons = 1;
      auto itp = std::lower_bound(sp_pos.begin(), sp_pos.end(), end_pos);
      if (itp != sp_pos.end() && *itp == end_pos) {
        // its consumption is recorded in the skip run that follows it (if any)
        auto itb = std::lower_bound(skip_begin.begin(), skip_begin.end(), end_pos + 1);
        if (itb != skip_begin.end() && *itb == end_pos + 1) cons = 1 + skip_len[itb - skip_begin.begin()];
      }
      // device: mask skipped positions, number the starts, emit
      Scratch is_start(sizeof(uint32_t) * m, s, mp), index(sizeof(uint32_t) * m, s, mp);
      k_init_starts<<<(int)std::min<int64_t>((m + 255) / 256, 65535), 256, 0, s>>>(m, is_start.as<uint32_t>());
      CSC_LAUNCHED();
      const int64_t nskip = (int64_t)skip_begin.size();
      Scratch dsb(sizeof(int64_t) * std::max<int64_t>(nskip, 1), s, mp), dsl(sizeof(int32_t) * std::max<int64_t>(nskip, 1), s, mp);
      if (nskip) {
        CSC_CUDA(cudaMemcpyAsync(dsb.get(), skip_begin.data(), sizeof(int64_t) * nskip, cudaMemcpyHostToDevice, s));
        CSC_CUDA(cudaMemcpyAsync(dsl.get(), skip_len.data(), sizeof(int32_t) * nskip, cudaMemcpyHostToDevice, s));
        k_mark_skips<<<(int)std::min<int64_t>((nskip + 255) / 256, 65535), 256, 0, s>>>(
            dsb.as<int64_t>(), dsl.as<int32_t>(), nskip, m, is_start.as<uint32_t>());
        CSC_LAUNCHED();
      }
      size_t tb2 = 0;
      CSC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, is_start.as<uint32_t>(), index.as<uint32_t>(), m, s));
      Scratch tmp2(tb2, s, mp);
      CSC_CUDA(cub::DeviceScan::ExclusiveSum(tmp2.get(), tb2, is_start.as<uint32_t>(), index.as<uint32_t>(), m, s));
      CSC_LAUNCHED();
      const int64_t nsp = (int64_t)sp_pos.size();
      Scratch dsp(sizeof(int64_t) * std::max<int64_t>(nsp, 1), s, mp), dsv(sizeof(double) * std::max<int64_t>(nsp, 1), s, mp);
      if (nsp) {
        CSC_CUDA(cudaMemcpyAsync(dsp.get(), sp_pos.data(), sizeof(int64_t) * nsp, cudaMemcpyHostToDevice, s));
        CSC_CUDA(cudaMemcpyAsync(dsv.get(), sp_val.data(), sizeof(double) * nsp, cudaMemcpyHostToDevice, s));
      }
      k_emit<D><<<(int)std::min<int64_t>((m + 255) / 256, 65535), 256, 0, s>>>(
          raw.as<uint64_t>(), special.as<uint8_t>(), is_start.as<uint32_t>(), index.as<uint32_t>(), m, count,
          dsp.as<int64_t>(), dsv.as<double>(), nsp, divisor, out);
      CSC_LAUNCHED();
      CSC_CUDA(cudaStreamSynchronize(s));
      if (timing)
        std::fprintf(stderr, "parity RNG (%s): n=%lld specials=%lld gen %.2f d2h %.2f walk %.2f emit %.2f ms\n",
                     D == Dist::Normal ? "normal" : "exponential", (long long)count, (long long)nspec, ms(t_start, t_gen), ms(t_gen, t_d2h), ms(t_d2h, t_walk),
                     ms(t_walk, now()));
      return end_pos + cons;
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
