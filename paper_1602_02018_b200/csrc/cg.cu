// K5: blocked conjugate gradient for the interpolation step (reference
// interpolate_all, sampling.py:124-180).
//
// The reference runs per-column CG with shared filtering passes: each column
// has its own alpha/beta, converged columns are frozen (alpha = beta = 0, so X
// and R never change again).  Columns never interact, so the device runs the
// iteration panel by panel: each panel's loop stops when its own columns have
// converged (or at max_iters).  Per-column arithmetic, iteration counts and the
// frozen-column semantics are unchanged; a panel whose columns are all done
// stops costing filter passes (the reference keeps filtering them).
//
// Per iteration and panel: one high-pass filter whose last step fuses
// AP = mask*P + gamma*(g(L)P + ridge*P) and the per-column P.AP partials
// (EPI_CGAP), then alpha (fixed-order reduce), X/R update with ||R||^2
// partials, beta + freeze bookkeeping, and P = R + beta P.
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <functional>
#include <future>
#include <memory>
#include <thread>
#include <vector>

#include "filter.cuh"

namespace csc {
namespace {

constexpr double kTiny = 2.2250738585072014e-308;  // np.finfo(np.float64).tiny, sampling.py:154

int colred_grid(int device) { return device_props(device).sms * 8; }

// thread -> (row slot, column) mapping shared by the column-reduction kernels:
// column c = tid % pw, row slot = tid / pw; 256 / pw rows per block pass.
template <typename T>
__global__ void k_colsumsq(const T* __restrict__ A, int64_t n, int pw, int wc, double* __restrict__ part) {
  __shared__ double red[256];
  const int c = threadIdx.x % pw;
  const int rs = threadIdx.x / pw;
  const int rpb = blockDim.x / pw;
  double s = 0.0;
  if (c < wc && rs < rpb)
    for (int64_t r = (int64_t)blockIdx.x * rpb + rs; r < n; r += (int64_t)gridDim.x * rpb) {
      const double v = (double)A[r * pw + c];
      s += v * v;
    }
  red[threadIdx.x] = s;
  __syncthreads();
  if ((int)threadIdx.x < pw) {
    double t = 0.0;
    for (int k = 0; k < rpb; ++k) t += red[k * pw + threadIdx.x];
    part[(size_t)blockIdx.x * pw + threadIdx.x] = t;
  }
}

// X += alpha P; R -= alpha AP; partial ||R||^2  (sampling.py:161-163)
template <typename T>
__global__ void k_cg_update(T* __restrict__ X, T* __restrict__ R, const T* __restrict__ P, const T* __restrict__ AP,
                            const double* __restrict__ alpha, int64_t n, int pw, int wc, double* __restrict__ part) {
  __shared__ double red[256];
  const int c = threadIdx.x % pw;
  const int rs = threadIdx.x / pw;
  const int rpb = blockDim.x / pw;
  double s = 0.0;
  if (c < wc && rs < rpb) {
    const double a = alpha[c];
    for (int64_t r = (int64_t)blockIdx.x * rpb + rs; r < n; r += (int64_t)gridDim.x * rpb) {
      const size_t o = (size_t)r * pw + c;
      const double p = (double)P[o], ap = (double)AP[o];
      const T x = static_cast<T>((double)X[o] + a * p);
      const T rr = static_cast<T>((double)R[o] - a * ap);
      X[o] = x;
      R[o] = rr;
      s += (double)rr * (double)rr;
    }
  }
  red[threadIdx.x] = s;
  __syncthreads();
  if ((int)threadIdx.x < pw) {
    double t = 0.0;
    for (int k = 0; k < rpb; ++k) t += red[k * pw + threadIdx.x];
    part[(size_t)blockIdx.x * pw + threadIdx.x] = t;
  }
}

// P = R + beta P  (sampling.py:164), also written in the filter's scaled basis
// Ps = D^-1/2 P.  beta == NULL: P = R (initial direction, sampling.py:149).
template <typename T>
__global__ void k_cg_direction(T* __restrict__ P, T* __restrict__ Ps, const T* __restrict__ R,
                               const double* __restrict__ beta, const double* __restrict__ dis, int64_t n, int pw,
                               int wc) {
  const int64_t total = n * pw;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / pw;
    const int c = (int)(t - row * pw);
    if (c >= wc) continue;
    const T p = beta ? static_cast<T>((double)R[t] + beta[c] * (double)P[t]) : R[t];
    P[t] = p;
    Ps[t] = static_cast<T>((double)p * dis[row]);
  }
}

struct ColState {
  double* rs;      // current ||R||^2
  double* t2;      // (tol ||B||)^2
  double* alpha;
  double* beta;
  int64_t* conv_at;
  uint8_t* active;
  int* nactive;    // device counter
};

// Fixed-order sum over the per-block partials of column c (one CTA per column):
// thread t adds blocks t, t + 256, ... sequentially, then a fixed tree.
__device__ double column_total(const double* __restrict__ part, int64_t nblocks, int pw, int c) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t b = threadIdx.x; b < nblocks; b += blockDim.x) s += part[b * pw + c];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o >= 1; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  return red[0];
}

// rs = ||B||^2, target^2, initial active set (sampling.py:150-153); grid = wc CTAs
__global__ void k_cg_init(const double* __restrict__ part, int64_t nblocks, int pw, int wc, double tol, ColState st) {
  const int c = blockIdx.x;
  const double s = column_total(part, nblocks, pw, c);
  if (threadIdx.x != 0) return;
  st.rs[c] = s;
  const double t = tol * sqrt(s);
  st.t2[c] = t * t;
  st.conv_at[c] = 0;
  const bool act = s > st.t2[c];
  st.active[c] = act ? 1 : 0;
  if (act) atomicAdd(st.nactive, 1);
}

// alpha = rs / (P.AP) on active columns with |denom| > tiny (sampling.py:159-160);
// also clears the active counter that k_cg_beta refills
__global__ void k_cg_alpha(const double* __restrict__ part, int64_t nblocks, int pw, int wc, ColState st) {
  const int c = blockIdx.x;
  const double d = column_total(part, nblocks, pw, c);
  if (threadIdx.x != 0) return;
  if (c == 0) *st.nactive = 0;
  const bool ok = st.active[c] && fabs(d) > kTiny;
  st.alpha[c] = ok ? st.rs[c] / d : 0.0;
}

// beta, rs update, freeze newly converged columns (sampling.py:164-170)
__global__ void k_cg_beta(const double* __restrict__ part, int64_t nblocks, int pw, int wc, int64_t iter, ColState st) {
  const int c = blockIdx.x;
  const double rsn = column_total(part, nblocks, pw, c);
  if (threadIdx.x != 0) return;
  const bool act = st.active[c] != 0;
  st.beta[c] = act ? rsn / fmax(st.rs[c], kTiny) : 0.0;
  st.rs[c] = rsn;
  const bool done = act && rsn <= st.t2[c];
  if (done) st.conv_at[c] = iter;
  const bool still = act && !done;
  st.active[c] = still ? 1 : 0;
  if (still) atomicAdd(st.nactive, 1);
}

// residuals, converged flags, iterations of unconverged columns (sampling.py:172-175)
__global__ void k_cg_finish(ColState st, int wc, int64_t iters, double* __restrict__ resid, uint8_t* __restrict__ conv,
                            int64_t* __restrict__ its) {
  const int c = threadIdx.x;
  if (c >= wc) return;
  const double r = sqrt(st.rs[c]);
  resid[c] = r;
  conv[c] = r <= sqrt(st.t2[c]) + kTiny ? 1 : 0;
  its[c] = st.active[c] ? iters : st.conv_at[c];
}

// residuals / flags / iterations of the current columns, written at their panel columns cmap[c]
__global__ void k_cg_finish_map(ColState st, int wc, int64_t iters, const int* __restrict__ cmap,
                                double* __restrict__ resid, uint8_t* __restrict__ conv, int64_t* __restrict__ its) {
  const int c = threadIdx.x;
  if (c >= wc) return;
  const int o = cmap[c];
  const double r = sqrt(st.rs[c]);
  resid[o] = r;
  conv[o] = r <= sqrt(st.t2[c]) + kTiny ? 1 : 0;
  its[o] = st.active[c] ? iters : st.conv_at[c];
}

// per-column state of the kept columns: dst[j] = src[map[j]]
__global__ void k_gather_state(ColState src, ColState dst, const int* __restrict__ map, int wc) {
  const int j = threadIdx.x;
  if (j >= wc) return;
  const int c = map[j];
  dst.rs[j] = src.rs[c];
  dst.t2[j] = src.t2[c];
  dst.alpha[j] = src.alpha[c];
  dst.beta[j] = src.beta[c];
  dst.conv_at[j] = src.conv_at[c];
  dst.active[j] = src.active[c];
}

template <typename T>
__global__ void k_scatter_rhs(const double* __restrict__ reduced, int k, const int64_t* __restrict__ idx, int64_t n,
                              int c0, int wc, int pw, T* __restrict__ B) {
  const int64_t total = n * wc;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / wc;
    const int c = (int)(t - i * wc);
    B[(size_t)idx[i] * pw + c] = static_cast<T>(reduced[i * k + c0 + c]);
  }
}

__global__ void k_mask(const int64_t* __restrict__ idx, int64_t n, int64_t N, uint8_t* __restrict__ mask,
                       int* __restrict__ bad) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx[t];
    if (i < 0 || i >= N) {
      atomicOr(bad, 1);
      continue;
    }
    const unsigned int word = atomicOr(reinterpret_cast<unsigned int*>(mask + (i & ~3ll)), 1u << (8 * (i & 3)));
    if (word & (1u << (8 * (i & 3)))) atomicOr(bad, 2);
  }
}

// --- column compaction: once at most half of a panel's columns are still active, they
// move into a panel half as wide (or narrower), so later filter passes stop paying for
// frozen columns.  Per-column arithmetic is unchanged.

// dst[:, j] = src[:, map[j]] for j < wc (zero padding up to pw_dst)
template <typename T>
__global__ void k_gather_cols(const T* __restrict__ src, int pw_src, T* __restrict__ dst, int pw_dst,
                              const int* __restrict__ map, int wc, int64_t n) {
  const int64_t total = n * pw_dst;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / pw_dst;
    const int j = (int)(t - r * pw_dst);
    dst[t] = j < wc ? src[r * pw_src + map[j]] : T(0);
  }
}

// dst[:, map[j]] = src[:, j] for j < wc
template <typename T>
__global__ void k_scatter_cols(const T* __restrict__ src, int pw_src, T* __restrict__ dst, int pw_dst,
                               const int* __restrict__ map, int wc, int64_t n) {
  const int64_t total = n * wc;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / wc;
    const int j = (int)(t - r * wc);
    dst[r * pw_dst + map[j]] = src[r * pw_src + j];
  }
}

// per-column state carved out of one allocation of `w` columns
ColState carve_state(Scratch& mem, int w, cudaStream_t s) {
  const size_t head = ((sizeof(double) * 4 * w + sizeof(int64_t) * w + w + 15) / 16) * 16;
  mem.alloc(head + 16, s);
  ColState st;
  st.rs = mem.as<double>();
  st.t2 = st.rs + w;
  st.alpha = st.t2 + w;
  st.beta = st.alpha + w;
  st.conv_at = reinterpret_cast<int64_t*>(st.beta + w);
  st.active = reinterpret_cast<uint8_t*>(st.conv_at + w);
  st.nactive = reinterpret_cast<int*>(mem.as<char>() + head);
  return st;
}

template <typename T>
void cg_panel(const csc_graph* g, const double* hp, int nc, double gamma, double ridge, const uint8_t* mask,
              const int64_t* idx, int64_t n, const double* reduced, int k, double tol, int64_t max_iters, int c0,
              int pw, int wc, T* Xp, double* resid, uint8_t* conv, int64_t* its, int64_t* iters_run, cudaStream_t s,
              const std::function<void()>* on_narrow = nullptr) {
  const int64_t N = g->n;
  const size_t pb = sizeof(T) * (size_t)N * pw;
  Scratch R(pb, s), P(pb, s), Ps(pb, s), AP(pb, s), B0(pb, s), B1(pb, s), Yacc;
  if (g_opt.recurrence.load() == 1) Yacc.alloc(pb, s);
  const int cg = colred_grid(g->device);
  const int cap = std::max(step_grid_cap(g->device), cg);
  Scratch part(sizeof(double) * (size_t)cap * pw, s);
  auto colmem = std::make_unique<Scratch>();
  ColState st = carve_state(*colmem, pw, s);

  // X = 0; R = P = B = M^T C  (sampling.py:142-149)
  CSC_CUDA(cudaMemsetAsync(Xp, 0, pb, s));
  CSC_CUDA(cudaMemsetAsync(R.get(), 0, pb, s));
  if (n > 0) {
    const int grid = (int)std::min<int64_t>((n * wc + 255) / 256 + 1, 4096);
    k_scatter_rhs<T><<<grid, 256, 0, s>>>(reduced, k, idx, n, c0, wc, pw, R.as<T>());
    CSC_LAUNCHED();
  }
  CSC_CUDA(cudaMemsetAsync(P.get(), 0, pb, s));
  CSC_CUDA(cudaMemsetAsync(Ps.get(), 0, pb, s));
  const int dgrid = (int)std::max<int64_t>(1, std::min<int64_t>((N * pw + 255) / 256, (int64_t)device_props(g->device).sms * 16));
  k_cg_direction<T><<<dgrid, 256, 0, s>>>(P.as<T>(), Ps.as<T>(), R.as<T>(), nullptr, g->dis, N, pw, wc);
  CSC_LAUNCHED();
  k_colsumsq<T><<<cg, 256, 0, s>>>(R.as<T>(), N, pw, wc, part.as<double>());
  CSC_LAUNCHED();
  CSC_CUDA(cudaMemsetAsync(st.nactive, 0, sizeof(int), s));
  k_cg_init<<<wc, 256, 0, s>>>(part.as<double>(), cg, pw, wc, tol, st);
  CSC_LAUNCHED();

  // the current (possibly compacted) panel: its width, columns, buffers and the map
  // from its columns to the caller's panel columns
  int pw_cur = pw, wc_cur = wc;
  T *Xc = Xp, *Rc = R.as<T>(), *Pc = P.as<T>(), *Psc = Ps.as<T>();
  std::unique_ptr<Scratch> own[4];  // compacted X, R, P, Ps
  std::vector<int> hmap(wc);
  for (int c = 0; c < wc; ++c) hmap[c] = c;
  Scratch cmap(sizeof(int) * pw, s), amap(sizeof(int) * pw, s);
  CSC_CUDA(cudaMemcpyAsync(cmap.get(), hmap.data(), sizeof(int) * wc, cudaMemcpyHostToDevice, s));
  const bool compact = g_opt.cg_compact.load() != 0;
  const int min_pw = 32 / (int)sizeof(T);  // narrower rows cost as much per step (one 32-B sector)

  // per-thread pinned staging (cudaMallocHost/cudaFreeHost per call would synchronise the device)
  static thread_local int* h_active = nullptr;
  static thread_local uint8_t* h_flags = nullptr;
  if (!h_active) CSC_CUDA(cudaMallocHost(&h_active, sizeof(int)));
  if (!h_flags) CSC_CUDA(cudaMallocHost(&h_flags, 256));
  int64_t iters = 0;
  CSC_CUDA(cudaMemcpyAsync(h_active, st.nactive, sizeof(int), cudaMemcpyDeviceToHost, s));
  CSC_CUDA(cudaStreamSynchronize(s));
  while (*h_active > 0 && iters < max_iters) {
    EpiExtra ex;
    ex.part = part.as<double>();
    ex.mask = mask;
    ex.gamma = gamma;
    ex.ridge = ridge;
    ex.ap = AP.get();
    const int fgrid = filter_panel<T>(g, hp, nc, Pc, Psc, nullptr, B0.as<T>(), B1.as<T>(), Yacc.as<T>(), pw_cur,
                                      wc_cur, EPI_CGAP, ex, s);
    k_cg_alpha<<<wc_cur, 256, 0, s>>>(part.as<double>(), fgrid, pw_cur, wc_cur, st);
    CSC_LAUNCHED();
    k_cg_update<T><<<cg, 256, 0, s>>>(Xc, Rc, Pc, AP.as<T>(), st.alpha, N, pw_cur, wc_cur, part.as<double>());
    CSC_LAUNCHED();
    ++iters;
    k_cg_beta<<<wc_cur, 256, 0, s>>>(part.as<double>(), cg, pw_cur, wc_cur, iters, st);
    CSC_LAUNCHED();
    k_cg_direction<T><<<dgrid, 256, 0, s>>>(Pc, Psc, Rc, st.beta, g->dis, N, pw_cur, wc_cur);
    CSC_LAUNCHED();
    CSC_CUDA(cudaMemcpyAsync(h_active, st.nactive, sizeof(int), cudaMemcpyDeviceToHost, s));
    CSC_CUDA(cudaStreamSynchronize(s));
    const int nact = *h_active;
    int want = min_pw;
    while (want < nact) want *= 2;
    if (!compact || nact == 0 || iters >= max_iters || want >= pw_cur) continue;
    // ---- compaction: keep the active columns in a panel `want` wide
    CSC_CUDA(cudaMemcpyAsync(h_flags, st.active, (size_t)wc_cur, cudaMemcpyDeviceToHost, s));
    CSC_CUDA(cudaStreamSynchronize(s));
    std::vector<int> act, nmap;
    for (int c = 0; c < wc_cur; ++c)
      if (h_flags[c]) {
        act.push_back(c);
        nmap.push_back(hmap[c]);
      }
    if ((int)act.size() != nact) fail(CSC_ERR_CUDA, "block CG: active-column bookkeeping mismatch");
    // final values of every current column (the kept ones are rewritten at the end)
    k_cg_finish_map<<<1, 128, 0, s>>>(st, wc_cur, iters, cmap.as<int>(), resid, conv, its);
    CSC_LAUNCHED();
    const size_t nb = sizeof(T) * (size_t)N * want;
    std::unique_ptr<Scratch> nxt[4];
    for (auto& b : nxt) b = std::make_unique<Scratch>(nb, s);
    CSC_CUDA(cudaMemcpyAsync(amap.get(), act.data(), sizeof(int) * nact, cudaMemcpyHostToDevice, s));
    const int ggrid = (int)std::max<int64_t>(1, std::min<int64_t>((N * want + 255) / 256,
                                                                   (int64_t)device_props(g->device).sms * 16));
    T* cur[4] = {Xc, Rc, Pc, Psc};
    for (int b = 0; b < 4; ++b) {
      k_gather_cols<T><<<ggrid, 256, 0, s>>>(cur[b], pw_cur, nxt[b]->as<T>(), want, amap.as<int>(), nact, N);
      CSC_LAUNCHED();
    }
    auto colmem_n = std::make_unique<Scratch>();
    ColState stn = carve_state(*colmem_n, want, s);
    k_gather_state<<<1, 128, 0, s>>>(st, stn, amap.as<int>(), nact);
    CSC_LAUNCHED();
    if (Xc != Xp) {  // columns leaving the compacted X go back to the caller's panel
      k_scatter_cols<T><<<ggrid, 256, 0, s>>>(Xc, pw_cur, Xp, pw, cmap.as<int>(), wc_cur, N);
      CSC_LAUNCHED();
    }
    for (int b = 0; b < 4; ++b) own[b] = std::move(nxt[b]);
    Xc = own[0]->as<T>();
    Rc = own[1]->as<T>();
    Pc = own[2]->as<T>();
    Psc = own[3]->as<T>();
    colmem = std::move(colmem_n);
    st = stn;
    CSC_CUDA(cudaMemcpyAsync(st.nactive, h_active, sizeof(int), cudaMemcpyHostToDevice, s));
    hmap = nmap;
    CSC_CUDA(cudaMemcpyAsync(cmap.get(), hmap.data(), sizeof(int) * nact, cudaMemcpyHostToDevice, s));
    CSC_CUDA(cudaStreamSynchronize(s));  // host vectors feeding async copies go out of scope
    pw_cur = want;
    wc_cur = nact;
    if (on_narrow && *on_narrow) {  // first compaction: this panel no longer needs the GPU alone
      (*on_narrow)();
      on_narrow = nullptr;
    }
  }
  k_cg_finish_map<<<1, 128, 0, s>>>(st, wc_cur, iters, cmap.as<int>(), resid, conv, its);
  CSC_LAUNCHED();
  if (Xc != Xp) {
    const int ggrid = (int)std::max<int64_t>(1, std::min<int64_t>((N * wc_cur + 255) / 256,
                                                                   (int64_t)device_props(g->device).sms * 16));
    k_scatter_cols<T><<<ggrid, 256, 0, s>>>(Xc, pw_cur, Xp, pw, cmap.as<int>(), wc_cur, N);
    CSC_LAUNCHED();
  }
  *iters_run = std::max(*iters_run, iters);
}

}  // namespace
}  // namespace csc

namespace csc {
namespace {
// One persistent host thread that runs a narrow remainder panel's CG beside the main
// panels (its pinned per-thread staging in cg_panel is allocated once, like the caller's).
// Leaked on purpose: joining at process exit would race the CUDA runtime's teardown.
class SideWorker {
 public:
  static SideWorker& get() {
    static SideWorker* w = new SideWorker();
    return *w;
  }
  std::future<void> submit(std::function<void()> fn) {
    std::packaged_task<void()> task(std::move(fn));
    std::future<void> fut = task.get_future();
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back(std::move(task));
    }
    cv_.notify_one();
    return fut;
  }

 private:
  SideWorker() : th_([this] { loop(); }) { th_.detach(); }
  void loop() {
    for (;;) {
      std::packaged_task<void()> task;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [this] { return !q_.empty(); });
        task = std::move(q_.front());
        q_.pop_front();
      }
      task();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::packaged_task<void()>> q_;
  std::thread th_;
};
}  // namespace
}  // namespace csc

using namespace csc;

extern "C" int csc_block_cg(const csc_graph* g, const double* hp_coeffs, int ncoeffs, double gamma, double ridge,
                            const int64_t* sample_idx, int64_t n, const double* reduced, int k, double tol,
                            int64_t max_iters, void* X_out, int64_t ldx, int io_dtype, int64_t* iterations,
                            double* residuals, uint8_t* converged, int64_t* iters_run, void* stream) {
  return guard([&] {
    if (!g) fail(CSC_ERR_INVALID, "graph is NULL");
    if (ncoeffs < 1 || !hp_coeffs) fail(CSC_ERR_INVALID, "need high-pass coefficients");
    if (!(gamma > 0)) fail(CSC_ERR_INVALID, "gamma must be positive");
    if (k < 1) fail(CSC_ERR_INVALID, "k must be >= 1");
    if (n < 0 || n > g->n) fail(CSC_ERR_INVALID, "sample count out of range");
    if (n > 0 && (!sample_idx || !reduced)) fail(CSC_ERR_INVALID, "sample arrays are NULL");
    if (max_iters < 0) fail(CSC_ERR_INVALID, "max_iters must be >= 0");
    if (io_dtype != CSC_F64 && io_dtype != CSC_F32) fail(CSC_ERR_INVALID, "io_dtype must be CSC_F64 or CSC_F32");
    if (ldx < k) fail(CSC_ERR_INVALID, "ldx < k");
    if (!X_out && g->n > 0) fail(CSC_ERR_INVALID, "X_out is NULL");
    DeviceGuard dg(g->device);
    ensure_pool(g->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t N = g->n;
    const PanelPlan pp = plan_panels(N, k, g->dtype, g->device, g->nnz);
    const size_t cs = dtype_size(g->dtype);

    DeviceView didx(sample_idx, sizeof(int64_t) * std::max<int64_t>(n, 1), g->device, s);
    DeviceView dred(reduced, sizeof(double) * std::max<int64_t>(n * k, 1), g->device, s);
    Scratch mask(((size_t)N + 4) & ~size_t(3), s), bad(sizeof(int), s);
    CSC_CUDA(cudaMemsetAsync(mask.get(), 0, mask.bytes(), s));
    CSC_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    if (n > 0) {
      k_mask<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(didx.as<int64_t>(), n, N,
                                                                             mask.as<uint8_t>(), bad.as<int>());
      CSC_LAUNCHED();
    }
    int hbad = 0;
    CSC_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    CSC_CUDA(cudaStreamSynchronize(s));
    if (hbad & 1) fail(CSC_ERR_INVALID, "sample index out of range");
    if (hbad & 2) fail(CSC_ERR_INVALID, "sample indices must be distinct");

    DeviceOut oit(iterations, sizeof(int64_t) * k, g->device, s);
    DeviceOut ores(residuals, sizeof(double) * k, g->device, s);
    DeviceOut oconv(converged, (size_t)k, g->device, s);
    Scratch it_s, res_s, conv_s;  // sinks when the caller passes NULL
    int64_t* d_it = oit.as<int64_t>();
    double* d_res = ores.as<double>();
    uint8_t* d_conv = oconv.as<uint8_t>();
    if (!d_it) { it_s.alloc(sizeof(int64_t) * k, s); d_it = it_s.as<int64_t>(); }
    if (!d_res) { res_s.alloc(sizeof(double) * k, s); d_res = res_s.as<double>(); }
    if (!d_conv) { conv_s.alloc(k, s); d_conv = conv_s.as<uint8_t>(); }

    Scratch xp(cs * std::max<int64_t>(pp.total, 1), s);
    int64_t run = 0;
    auto panel = [&](int j, int64_t* runp, cudaStream_t st, const std::function<void()>* on_narrow) {
      if (g->dtype == CSC_F64)
        cg_panel<double>(g, hp_coeffs, ncoeffs, gamma, ridge, mask.as<uint8_t>(), didx.as<int64_t>(), n,
                         dred.as<double>(), k, tol, max_iters, pp.c0[j], pp.pw[j], pp.wc[j],
                         xp.as<double>() + pp.off[j], d_res + pp.c0[j], d_conv + pp.c0[j], d_it + pp.c0[j], runp, st,
                         on_narrow);
      else
        cg_panel<float>(g, hp_coeffs, ncoeffs, gamma, ridge, mask.as<uint8_t>(), didx.as<int64_t>(), n,
                        dred.as<double>(), k, tol, max_iters, pp.c0[j], pp.pw[j], pp.wc[j],
                        xp.as<float>() + pp.off[j], d_res + pp.c0[j], d_conv + pp.c0[j], d_it + pp.c0[j], runp, st,
                        on_narrow);
    };
    // Two panels' CGs run at once where that helps (option cg_overlap: 0 off, 1 auto, 2 no
    // token).  The panels share nothing but read-only inputs, so every result is unchanged.
    //  * A full-width panel holds the "wide" token until its first compaction (its active
    //    columns fit half the width) or its end: two full-width panels of 128/256-B rows
    //    contend for L2 and DRAM (measured C3 +1 %, C5 +40 % when run together), while a
    //    narrower panel -- a remainder (k = 100 -> 32 + 32 + 32 + 4) or a compacted one -- is
    //    bound by row requests and overlaps well (C3 CSC 0.830 -> 0.81 s).
    //  * Panels of 512-B rows (one row per warp, little memory-level parallelism per warp)
    //    whose gather source is <= 4x L2 need no token (C4 k = 250: CG 0.48 -> 0.35 s).
    //  * Gather sources above 4x L2 (C5: 2 GB per 32-wide panel) run one panel at a time.
    const int64_t ovmode = g_opt.cg_overlap.load();
    const bool small_source = (double)N * pp.max_pw * cs <= 4.0 * device_props(g->device).l2_bytes;
    const bool untokened = ovmode == 2 || ((size_t)pp.max_pw * cs == 512 && small_source);
    if (ovmode == 0 || pp.np < 2 || (ovmode == 1 && !small_source)) {  // C5's 2 GB panels: +6 % overlapped
      for (int j = 0; j < pp.np; ++j) panel(j, &run, s, nullptr);
    } else {
      std::vector<int> order;  // narrower panels first, so the side thread starts on one at once
      for (int j = 0; j < pp.np; ++j)
        if (pp.pw[j] < pp.max_pw) order.push_back(j);
      for (int j = 0; j < pp.np; ++j)
        if (pp.pw[j] == pp.max_pw) order.push_back(j);
      std::mutex mu;
      std::condition_variable cv;
      size_t next = 0;
      bool busy = false, abort = false;
      auto worker = [&](cudaStream_t st, int64_t* runp) {
        for (;;) {
          int j = -1;
          bool held = false;
          {
            std::unique_lock<std::mutex> lk(mu);
            if (abort || next >= order.size()) return;
            j = order[next];
            const bool wide = pp.pw[j] == pp.max_pw && !untokened;
            if (wide) {
              cv.wait(lk, [&] { return !busy || abort; });
              if (abort) return;
              busy = held = true;
            }
            ++next;
          }
          const std::function<void()> release = [&] {
            std::lock_guard<std::mutex> lk(mu);
            if (held) {
              busy = held = false;
              cv.notify_all();
            }
          };
          try {
            panel(j, runp, st, held ? &release : nullptr);
          } catch (...) {
            {
              std::lock_guard<std::mutex> lk(mu);
              abort = true;
            }
            release();
            cv.notify_all();
            throw;
          }
          release();
        }
      };
      cudaStream_t ss = nullptr;
      cudaEvent_t ready = nullptr, done = nullptr;
      CSC_CUDA(cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking));
      CSC_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
      CSC_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      CSC_CUDA(cudaEventRecord(ready, s));
      CSC_CUDA(cudaStreamWaitEvent(ss, ready, 0));
      int64_t run_side = 0;
      const int dev = g->device;
      std::future<void> fut = SideWorker::get().submit([&, dev, ss] {
        DeviceGuard sdg(dev);
        worker(ss, &run_side);
      });
      std::exception_ptr err;
      try {
        worker(s, &run);
      } catch (...) {
        err = std::current_exception();
      }
      try {
        fut.get();  // rethrows the side worker's failure
      } catch (...) {
        if (!err) err = std::current_exception();
      }
      cudaEventRecord(done, ss);
      cudaStreamWaitEvent(s, done, 0);
      cudaEventDestroy(ready);
      cudaEventDestroy(done);
      cudaStreamDestroy(ss);
      if (err) std::rethrow_exception(err);
      run = std::max(run, run_side);
    }
    if (N > 0) {
      const bool xdev = is_device_ptr(X_out, g->device);
      const size_t es = dtype_size(io_dtype);
      Scratch xs;
      void* xdst = X_out;
      int64_t xld = ldx;
      if (!xdev) {
        xs.alloc(es * N * k, s);
        xdst = xs.get();
        xld = k;
      }
      unpack_panels(xp.get(), g->dtype, pp, N, xdst, io_dtype, xld, s);
      if (!xdev)
        copy_rows(X_out, ldx, xs.get(), k, N, k, es, cudaMemcpyDeviceToHost, s);
      CSC_CUDA(cudaStreamSynchronize(s));
    }
    oit.finish();
    ores.finish();
    oconv.finish();
    CSC_CUDA(cudaStreamSynchronize(s));
    if (iters_run) *iters_run = run;
  });
}
