// Degree-corrected SBM edges (BASELINE config 4; SURVEY.md §8(d) "C4 (new generator, spec for the
// builder)"): independent Bernoulli edges with P(i~j) = min(1, theta_i theta_j q_{c_i c_j}),
// q = q_intra on the diagonal and q_inter off it, drawn in expected O(N + #E) time.
//
// The reference has no DC-SBM; its SBM generator skips geometrically over the
// candidate pairs of each block pair with one probability per block (sbm.py:83-100).  With
// per-node propensities the probability varies inside a block, so each source node u walks its
// candidates in order of decreasing theta and skips geometrically with the CURRENT bound,
// accepting the landed candidate with probability p_v / p_bound (rejection over geometric
// skipping; Miller & Hagberg 2011, "Efficient generation of networks with given expected
// degrees").  Because the bound never increases along the walk, every pair is accepted with
// exactly min(1, theta_u theta_v q):
//   - intra-community pairs: nodes of each community sorted by theta (descending, ties by
//     index); u = the a-th node walks positions b > a with q_intra;
//   - inter-community pairs: all nodes sorted by theta; u walks positions b > a with q_inter
//     and drops same-community landings (those pairs belong to the intra walk).
// Randomness is counter-based (SplitMix64 keyed by seed, walk and u), so the edge set does not
// depend on the thread count.  Two passes (count, then write at prefix offsets) give the edges
// in walk order; the caller canonicalises (sorts) them.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <thread>
#include <vector>

#include "internal.cuh"

namespace csc {
namespace {

inline uint64_t splitmix64(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// uniform double in (0, 1]: never 0, so log() is finite
inline double uniform_open0(uint64_t& x) { return (double)((splitmix64(x) >> 11) + 1) * 0x1.0p-53; }

struct Walk {
  const int64_t* order;  // node ids sorted by theta descending within the walk's range
  int64_t len;
  double q;
  bool skip_same;  // inter walk: drop pairs inside one community
  uint64_t key;
};

// One source position a of a walk; emit(u, v) for every accepted pair.  Returns the count.
template <class Emit>
int64_t walk_one(const Walk& w, int64_t a, const double* theta, const int32_t* comm, Emit emit) {
  const int64_t u = w.order[a];
  const double tu = theta[u];
  uint64_t st = w.key ^ (0xD1B54A32D192ED03ull * (uint64_t)(a + 1));
  splitmix64(st);
  int64_t b = a + 1, found = 0;
  if (b >= w.len) return 0;
  double p = std::min(1.0, tu * theta[w.order[b]] * w.q);
  while (b < w.len && p > 0.0) {
    if (p < 1.0) {
      const double r = std::floor(std::log(uniform_open0(st)) / std::log1p(-p));
      if (r >= (double)(w.len - b)) break;
      b += (int64_t)r;
    }
    const int64_t v = w.order[b];
    const double pv = std::min(1.0, tu * theta[v] * w.q);
    if (uniform_open0(st) <= pv / p && !(w.skip_same && comm[u] == comm[v])) {
      emit(u, v);
      ++found;
    }
    p = pv;
    ++b;
  }
  return found;
}

}  // namespace
}  // namespace csc

using namespace csc;

extern "C" int csc_dcsbm_edges(int64_t num_nodes, int32_t k, const int64_t* sizes, const double* theta,
                               double q_intra, double q_inter, uint64_t seed, int nthreads, int64_t capacity,
                               int64_t* src, int64_t* dst, int64_t* num_edges) {
  return guard([&] {
    if (num_nodes < 0 || k < 1 || !sizes || !theta || !num_edges)
      fail(CSC_ERR_INVALID, "csc_dcsbm_edges: bad arguments");
    if (!(q_intra >= 0.0) || !(q_inter >= 0.0)) fail(CSC_ERR_INVALID, "csc_dcsbm_edges: negative q");
    std::vector<int32_t> comm(num_nodes);
    std::vector<int64_t> first(k + 1, 0);
    for (int c = 0; c < k; ++c) {
      if (sizes[c] < 0) fail(CSC_ERR_INVALID, "csc_dcsbm_edges: negative community size");
      first[c + 1] = first[c] + sizes[c];
    }
    if (first[k] != num_nodes) fail(CSC_ERR_INVALID, "csc_dcsbm_edges: sizes do not sum to num_nodes");
    for (int64_t i = 0; i < num_nodes; ++i)
      if (!(theta[i] >= 0.0) || !std::isfinite(theta[i]))
        fail(CSC_ERR_INVALID, "csc_dcsbm_edges: propensities must be finite and >= 0");
    for (int c = 0; c < k; ++c)
      for (int64_t i = first[c]; i < first[c + 1]; ++i) comm[i] = c;
    auto by_theta = [&](int64_t x, int64_t y) { return theta[x] > theta[y] || (theta[x] == theta[y] && x < y); };
    // intra order: each community's nodes sorted in place; inter order: all nodes
    std::vector<int64_t> intra(num_nodes), inter(num_nodes);
    std::iota(intra.begin(), intra.end(), 0);
    std::iota(inter.begin(), inter.end(), 0);
    for (int c = 0; c < k; ++c) std::sort(intra.begin() + first[c], intra.begin() + first[c + 1], by_theta);
    std::sort(inter.begin(), inter.end(), by_theta);

    // work items: (walk id, source position); walk 0..k-1 = intra community c, walk k = inter
    std::vector<Walk> walks;
    for (int c = 0; c < k; ++c)
      walks.push_back(Walk{intra.data() + first[c], sizes[c], q_intra, false,
                           seed ^ (0x632BE59BD9B4E019ull * (uint64_t)(c + 1))});
    walks.push_back(Walk{inter.data(), num_nodes, q_inter, true, seed ^ 0x8CB92BA72F3D8DD7ull});
    std::vector<int64_t> item_walk, item_pos;
    item_walk.reserve(2 * num_nodes);
    item_pos.reserve(2 * num_nodes);
    for (size_t wi = 0; wi < walks.size(); ++wi)
      for (int64_t a = 0; a < walks[wi].len; ++a) {
        item_walk.push_back((int64_t)wi);
        item_pos.push_back(a);
      }
    const int64_t items = (int64_t)item_walk.size();
    std::vector<int64_t> cnt(items + 1, 0);
    int T = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
    T = (int)std::min<int64_t>(T, std::max<int64_t>(1, items / 4096 + 1));
    auto run = [&](auto&& body) {
      std::vector<std::thread> pool;
      for (int t = 0; t < T; ++t)
        pool.emplace_back([&, t]() {
          for (int64_t i = t; i < items; i += T) body(i);  // interleaved: heavy sources spread
        });
      for (auto& th : pool) th.join();
    };
    run([&](int64_t i) {
      cnt[i + 1] = walk_one(walks[item_walk[i]], item_pos[i], theta, comm.data(), [](int64_t, int64_t) {});
    });
    std::partial_sum(cnt.begin(), cnt.end(), cnt.begin());
    *num_edges = cnt[items];
    if (cnt[items] > capacity || (!src && cnt[items] > 0) || (!dst && cnt[items] > 0)) return;
    run([&](int64_t i) {
      int64_t o = cnt[i];
      walk_one(walks[item_walk[i]], item_pos[i], theta, comm.data(), [&](int64_t u, int64_t v) {
        src[o] = std::min(u, v);
        dst[o] = std::max(u, v);
        ++o;
      });
    });
  });
}
