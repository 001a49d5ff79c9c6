// K2: the fused Chebyshev-step SpMM and the order-p filter drivers built on it.
//
// Reference: apply_filter (filters.py:140-155) wraps LaplacianOp.apply
// (graph.py:147-155) in the three-term recurrence T_{l+1} = 2(L-I)T_l - T_{l-1},
// Y = sum_l c_l T_l, with L - I = -D^-1/2 W D^-1/2.
//
// Scaled basis.  Every block that is gathered is stored as v~ = D^-1/2 v
// (s = d^-1/2 per row).  Then  s_i (Wn v)_i = d_i^-1 sum_j w_ij v~_j, i.e. the
// recurrence runs on the random-walk operator D^-1 W: one step needs the
// neighbour rows v~_j and, for unit-weight graphs (SBM), nothing per edge but
// the column index -- no per-edge values, no per-edge scale.  The last step
// returns to the symmetric basis: (Wn v)_i = s_i sum_j w_ij v~_j and
// b_i = d_i^{1/2} b~_i.  Isolated nodes (d = 0, where L - I = 0) are fixed up in
// the last step as Y_i = h(1) X_i (T_l(0) = cos(l pi/2)).
//
// One step (one pass over the CSR):
//   mid   out~ = ka d^-1 sum_j w_ij G~_j + ks S~ + kx X~          (scaled -> scaled)
//   last  out  = ka s   sum_j w_ij G~_j + ks d^{1/2} S~ + kx X     (scaled -> symmetric)
//   forward mode also  Y = ky0 Yin + ky d^{1/2} out~               (symmetric accumulator)
// and the last step's value can be reduced in the same pass (epilogues):
//   SUMSQ  sum of squares (eigencount, spectrum.py:86)
//   ROWSQ  per-row sum of squares (feature normalisation, features.py:80)
//   CGAP   AP = mask*P + gamma*(out + ridge*P) and per-column P.AP
//          (_system_apply sampling.py:119-121 + the CG dot at sampling.py:159)
//
// Layout: the N x w block is split into column panels (N x pw, row-major within
// the panel, pw = lanes_per_row * 16B/sizeof(T)).  One node's panel row is one
// contiguous, 32B-sector-aligned segment, so a neighbour gather is a single
// coalesced vector load per lane.  A panel is sized so its gather source can
// stay L2-resident; filters run panel-major (all p steps of panel 0, then
// panel 1, ...), columns being independent (filters.py:140).  The lanes of a
// row load that row's column indices cooperatively and broadcast them with
// warp shuffles, so the load/store unit mostly issues the 16-byte gathers.
//
// Two recurrences are provided:
//   forward   (north-star kernel): T_{l+1} = -2 Wn T_l - T_{l-1};  Y += c_{l+1} T_{l+1}
//             streams per step: gather T_l, read T_{l-1}, write T_{l+1}, read+write Y  (5)
//   Clenshaw  b_l = c_l X - 2 Wn b_{l+1} - b_{l+2};  Y = c_0 X - Wn b_1 - b_2
//             streams per step: gather b_{l+1}, read b_{l+2}, read X, write b_l     (4)
// Both evaluate the same polynomial sum_l c_l T_l(L - I) X with p SpMM passes.
//
// Two step kernels: k_cheb_step (every case: weights, epilogues, forward mode, peer
// stores) and k_cheb_mid, the mid step alone with only that case's state (32 or 40
// registers, more warps or more gathers in flight), used for 16-512-B panel rows whose
// gather source is <= 4x L2 (unit weights, or any weights in fp32); bit-identical results.
#pragma once

#include "internal.cuh"

namespace csc {

enum Epi : int { EPI_NONE = 0, EPI_SUMSQ = 1, EPI_ROWSQ = 2, EPI_CGAP = 3 };

struct StepArgs {
  const int32_t* indptr;
  const int32_t* indices;
  const void* wv;   // edge weights (compute dtype); NULL for unit-weight graphs
  const void* rs;   // per-row (d^-1/2, d^1/2)
  const void* G;    // gathered panel, scaled basis (N x pw); NULL = no SpMM term
  const void* S;    // same-row stream, scaled basis (may alias O)
  const void* X;    // same-row stream: scaled X~ on mid steps, symmetric X on last steps
  const void* Yin;  // forward-mode accumulator input (may alias Y)
  void* O;          // out (scaled on mid steps, symmetric on the last Clenshaw step)
  void* Y;          // forward-mode accumulator output
  void* E;          // CGAP: AP output
  const uint8_t* mask;  // CGAP: sampling mask
  double* part;     // epilogue partials (SUMSQ [grid], ROWSQ [N], CGAP [grid][pw])
  double ka, ks, kx, ky0, ky, gamma, ridge;
  double hz;        // h(1) = sum_l c_l T_l(0): value of the filter on isolated nodes
  int64_t n;
  int wc;        // valid columns in this panel (<= pw)
  int fwd;       // forward-mode accumulate
  int last;      // symmetric-basis output + isolated-node fixup (+ epilogue)
  int hints;     // evict-first hints on streamed operands (set by launch_step)
  int sv;        // panel row stride in 16-B vectors = pw / VEC = lanes per row (set by launch_step)
  int contig;    // contiguous row ranges per warp (set by launch_step)
  int pol;       // output panel stored evict-first (option l2_policy, set by launch_step)
  // row-sharded peer transport (rows.cu): O's rows are also stored into every rank's next
  // gather panel, peers[q] + (peer_row0 + row) * pw, over NVLink -- the all-gather fused
  // into the step.  npeers = 0: off.
  void* const* peers;  // device array of npeers panel pointers
  int npeers;
  int64_t peer_row0;
};

struct PanelPlan {
  int np = 0;
  std::vector<int> pw;      // panel widths (elements)
  std::vector<int> wc;      // valid columns per panel
  std::vector<int> c0;      // first global column of each panel
  std::vector<int64_t> off; // element offset of each panel in the packed buffer
  int64_t total = 0;        // packed elements
  int max_pw = 0;
};

// Panel widths are powers of two (x 16-B vectors); rows rounded to 16 B instead ("tight"
// panels, 224-B rows for C3's d = 56) were measured slower at C3 and removed
// (profiles/r02_ab_tight_panels.txt).
PanelPlan plan_panels(int64_t n, int w, int dtype, int device, int64_t nnz);

// Upper bound of the step kernel's grid (for sizing epilogue partials).
int step_grid_cap(int device);

// Launch one step.  Returns the grid actually used.
template <typename T>
int launch_step(const csc_graph* g, const StepArgs& a, int pw, int epi, cudaStream_t s);

struct EpiExtra {
  double* part = nullptr;
  const uint8_t* mask = nullptr;
  double gamma = 0.0, ridge = 0.0;
  void* ap = nullptr;  // CGAP output panel
};

// Y = sum_{l<nc} c_l T_l(L - I) X on one panel.  X is the symmetric-basis input
// panel, Xs the same panel in the scaled basis (D^-1/2 X); Y the symmetric-basis
// output (NULL for SUMSQ/CGAP).  B0/B1 are N x pw scratch panels; Yacc is needed
// in forward mode when Y is NULL.  Returns the grid of the final (epilogue) step.
template <typename T>
int filter_panel(const csc_graph* g, const double* c, int nc, const T* X, const T* Xs, T* Y, T* B0, T* B1, T* Yacc,
                 int pw, int wc, int epi, const EpiExtra& ex, cudaStream_t s);

// Pack a row-major block (io dtype, leading dim ld) into panels (compute dtype),
// zero-filling pad columns; when `scaled` is non-NULL it also receives the
// panels in the scaled basis (row i times d_i^-1/2).  Unpack is the inverse of
// the symmetric pack over valid columns.
void pack_panels(const void* src, int io_dtype, int64_t ld, void* dst, void* scaled, const csc_graph* g,
                 const PanelPlan& pp, cudaStream_t s);
void unpack_panels(const void* src, int dtype, const PanelPlan& pp, int64_t n, void* dst, int io_dtype, int64_t ld,
                   cudaStream_t s);

// Deterministic fixed-order sum of `count` doubles into out[0] (device).
void reduce_sum(const double* in, int64_t count, double* out, cudaStream_t s);

}  // namespace csc
