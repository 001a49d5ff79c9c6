// K2: the fused Chebyshev-step SpMM and the order-p filter drivers built on it.
//
// Reference: apply_filter (filters.py:140-155) wraps LaplacianOp.apply
// (graph.py:147-155) in the three-term recurrence T_{l+1} = 2(L-I)T_l - T_{l-1},
// Y = sum_l c_l T_l.  Here L - I = -Wn with Wn = D^-1/2 W D^-1/2 stored
// pre-normalized (K1), so one step is one pass over the CSR:
//
//   out[i,:] = ka * sum_j Wn_ij G[j,:]  +  ks * S[i,:]  +  kx * X[i,:]
//   (forward mode also)  Y[i,:] = ky0 * Yin[i,:] + ky * out[i,:]
//
// with the final step's value optionally reduced in the same pass (epilogues):
//   SUMSQ  sum of squares (eigencount, spectrum.py:86)
//   ROWSQ  per-row sum of squares (feature normalisation, features.py:80)
//   CGAP   AP = mask*P + gamma*(out + ridge*P) and per-column P.AP
//          (_system_apply sampling.py:119-121 + the CG dot at sampling.py:159)
//
// Layout: the N x w block is split into column panels (N x pw, row-major within
// the panel, pw = lanes_per_row * 16B/sizeof(T)).  One node's panel row is one
// contiguous, 32B-sector-aligned segment, so a neighbour gather is a single
// coalesced vector load per lane.  A panel is sized to stay L2-resident while it
// is gathered (the gather is the only non-streaming access); everything else is
// streamed with evict-first hints.  Filters run panel-major: all p steps of
// panel 0, then panel 1, ... (columns are independent, filters.py:140).
//
// Two recurrences are provided:
//   forward   (north-star kernel): T_{l+1} = -2 Wn T_l - T_{l-1};  Y += c_{l+1} T_{l+1}
//             streams per step: gather T_l, read T_{l-1}, write T_{l+1}, read+write Y  (5)
//   Clenshaw  b_l = c_l X - 2 Wn b_{l+1} - b_{l+2};  Y = c_0 X - Wn b_1 - b_2
//             streams per step: gather b_{l+1}, read b_{l+2}, read X, write b_l     (4)
// Both evaluate the same polynomial sum_l c_l T_l(L - I) X with p SpMM passes.
#pragma once

#include "internal.cuh"

namespace csc {

enum Epi : int { EPI_NONE = 0, EPI_SUMSQ = 1, EPI_ROWSQ = 2, EPI_CGAP = 3 };

struct StepArgs {
  const int32_t* indptr;
  const int32_t* indices;
  const void* wn;
  const void* G;    // gathered panel (N x pw); NULL = no SpMM term
  const void* S;    // same-row stream (may alias O)
  const void* X;    // same-row stream
  const void* Yin;  // forward-mode accumulator input (may alias Y)
  void* O;          // out
  void* Y;          // forward-mode accumulator output
  void* E;          // CGAP: AP output
  const uint8_t* mask;  // CGAP: sampling mask
  double* part;     // epilogue partials (SUMSQ [grid], ROWSQ [N], CGAP [grid][pw])
  double ka, ks, kx, ky0, ky, gamma, ridge;
  int64_t n;
  int wc;   // valid columns in this panel (<= pw)
  int fwd;  // forward-mode accumulate
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

PanelPlan plan_panels(int64_t n, int w, int dtype, int device);

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

// Y = sum_{l<nc} c_l T_l(L - I) X on one panel (X, Y: N x pw).  B0/B1 are N x pw
// scratch panels; Yacc is needed in forward mode when Y is NULL (SUMSQ/CGAP).
// Returns the grid used by the final (epilogue) step.
template <typename T>
int filter_panel(const csc_graph* g, const double* c, int nc, const T* X, T* Y, T* B0, T* B1, T* Yacc, int pw,
                 int wc, int epi, const EpiExtra& ex, cudaStream_t s);

// Pack a row-major block (io dtype, leading dim ld) into panels (compute dtype),
// zero-filling pad columns; unpack is the inverse over valid columns.
void pack_panels(const void* src, int io_dtype, int64_t ld, void* dst, int dtype, const PanelPlan& pp, int64_t n,
                 cudaStream_t s);
void unpack_panels(const void* src, int dtype, const PanelPlan& pp, int64_t n, void* dst, int io_dtype, int64_t ld,
                   cudaStream_t s);

// Deterministic fixed-order sum of `count` doubles into out[0] (device).
void reduce_sum(const double* in, int64_t count, double* out, cudaStream_t s);
// out[c] = sum_b in[b * stride + c] for c < ncols (fixed order).
void reduce_cols(const double* in, int64_t nblocks, int stride, int ncols, double* out, cudaStream_t s);

}  // namespace csc
