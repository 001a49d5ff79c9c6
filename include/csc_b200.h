/*
 * csc_b200.h — C ABI of the B200-native compressive-spectral-clustering hot path.
 *
 * The reference (`cscluster`, pure Python + scipy) has no C API: its hot path is
 * reached through Python seams.  Each entry point below replaces
 * one of those seams; the reference interface it stands in for is cited as
 * file:line relative to the reference package `pkg/src/cscluster/`.
 *
 * Conventions
 *  - Every call returns an int status: CSC_OK (0) or one of CSC_ERR_*.  The
 *    message of the last failure on the calling thread is csc_last_error().
 *    Python maps CSC_ERR_INVALID -> ValueError, CSC_ERR_GRAPH -> GraphError
 *    (a ValueError subclass, graph.py:19-20), anything else -> RuntimeError.
 *  - Buffers are plain pointers.  Each data pointer may be host memory
 *    (pageable or pinned) or device memory of the graph's device; the library
 *    detects which with cudaPointerGetAttributes and stages host buffers.
 *  - Dense blocks are row-major (one node's columns contiguous) with a leading
 *    dimension `ld` (elements), like the reference's C-contiguous N x w numpy
 *    arrays (spectrum.py:84, features.py:63).  `io_dtype` gives the element type
 *    of those buffers (CSC_F64 / CSC_F32); the arithmetic runs in the graph's
 *    compute dtype.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    stream-ordered; a call returns after its results are in the caller's
 *    buffers for host outputs, and asynchronously for device outputs.
 *  - Graph handles are immutable after creation and may be shared between
 *    threads and streams (LaplacianOp is immutable/reentrant, graph.py:128-134).
 */
#ifndef CSC_B200_H
#define CSC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSC_ABI_VERSION 1

/* status codes */
#define CSC_OK 0
#define CSC_ERR_INVALID 1 /* bad argument / shape  -> ValueError                 */
#define CSC_ERR_GRAPH 2   /* bad edge data         -> GraphError (graph.py:19)    */
#define CSC_ERR_CUDA 3    /* CUDA runtime failure or no device -> RuntimeError    */
#define CSC_ERR_NOMEM 4   /* device allocation failed -> MemoryError              */

/* element / compute types */
#define CSC_F64 0
#define CSC_F32 1

/* build flags */
#define CSC_SELF_LOOPS_ERROR 0 /* build_graph(self_loops="error"), graph.py:115-118 */
#define CSC_SELF_LOOPS_DROP 1  /* build_graph(self_loops="drop"),  graph.py:119-120 */

typedef struct csc_graph csc_graph;
typedef struct csc_comm csc_comm; /* NCCL communicator for row-sharded operators */

#define CSC_UNIQUE_ID_BYTES 128
typedef struct csc_peers csc_peers; /* peer-memory transport for row-sharded operators */
#define CSC_PEER_HANDLE_BYTES 64

/* ---- library ------------------------------------------------------------ */
int csc_abi_version(void);
const char* csc_last_error(void);
/* Number of CUDA kernels this library has launched in the process so far. */
int csc_launch_count(int64_t* out);
/* Tuning knobs (process-wide; not to be changed while calls are in flight):
 *   "panel_width"   columns per panel (0 = auto, degree- and L2-aware)
 *   "recurrence"    0 Clenshaw (4 streams/step, default), 1 forward (5 streams/step)
 *   "cache_hints"   1 evict-first hints on streamed operands, 0 off
 *   "block_threads" threads per CTA (64..256)
 *   "unroll"        neighbour gathers in flight per lane / occupancy: 4 (default: 4 in
 *                   flight, 6 CTAs/SM), 2 (4 in flight, 8 CTAs/SM), 8 (8 in flight, 2 CTAs/SM)
 *   "row_order"     0 interleaved row groups (default), 1 contiguous runs per warp
 *   "lean_mid"      1 (default): lean mid-step kernel for 16- to 512-B panel rows whose
 *                   gather panel is <= 4x L2 (unit weights; weighted graphs in fp32);
 *                   0: always the general step kernel
 *   "pdl"           1 (default): step kernels are launched with programmatic stream
 *                   serialization (their CSR prologue overlaps the previous step's drain); 0 off
 *   "l2_policy"     1 (default): a step's output panel is stored evict-first; 0 write-back
 *   "persistent"    1 (default): step grids of resident CTAs (grid-stride); 0 one CTA per row block
 *   "fast_normalize" 1 (default): vectorised row normaliser for equal-width panels
 *   "h2d_overlap"   1 (default): multi-panel pinned host blocks upload panel by panel,
 *                   overlapping the earlier panels' filters
 *   "l2_budget_pct" L2 share a gathered panel may use (auto panel width)
 *   "l2_persist_pct" >0: persisting-L2 access window on the gathered panel
 *   "cg_compact"    1 (default): block CG moves still-active columns into narrower panels
 *   "cg_overlap"    1 (default): block-CG panels run two at a time (side stream / host thread);
 *                   a full-width panel runs alone until its first compaction (no such limit for
 *                   512-B-row panels with gather sources <= 4x L2); 0 off; 2 no limit
 *   "profile"       1 = time every Chebyshev step launch with CUDA events; 2 = one event
 *                   pair per filter (its step launches run back to back; less intrusive) */
int csc_set_option(const char* key, int64_t value);
int csc_get_option(const char* key, int64_t* value);
/* Profile counters of the Chebyshev step kernels since the last reset:
 * total device ms, launches, algorithmic bytes (SURVEY.md §8d formula applied to
 * the streams each launch touches). */
int csc_profile_read(double* step_ms, int64_t* step_launches, double* step_bytes);
int csc_profile_reset(void);

/* ---- graph (K1) --------------------------------------------------------- */
/* Canonical CSR -> device normalized operator.  Replaces laplacian_op
 * (graph.py:164-169) over a Graph (graph.py:23-55): degrees are fp64 row sums
 * (graph.py:63), d^-1/2 is 0 for zero degree (graph.py:168), and the stored
 * operator is Wn = D^-1/2 W D^-1/2 in the compute dtype.  indptr/indices/weights
 * must already be canonical (sorted, no duplicates, no zeros); they are
 * validated (CSC_ERR_GRAPH otherwise). */
int csc_graph_create(int64_t num_nodes, int64_t nnz, const int32_t* indptr, const int32_t* indices,
                     const double* weights, int dtype, int device, void* stream, csc_graph** out);

/* Edge triples -> canonical CSR on the device, then as csc_graph_create.
 * Replaces build_graph (graph.py:73-125) after its host-side validation:
 * per-direction duplicates summed (graph.py:122-123), W = max(A, A^T)
 * (graph.py:124), sorted columns, explicit zeros dropped (graph.py:60-62). */
int csc_graph_build_coo(int64_t num_nodes, int64_t num_edges, const int64_t* src, const int64_t* dst,
                        const double* weights, int self_loops, int dtype, int device, void* stream,
                        csc_graph** out);

int csc_graph_destroy(csc_graph* g);

/* Sizes of a handle. */
int csc_graph_info(const csc_graph* g, int64_t* num_nodes, int64_t* nnz, int* dtype, int* device);

/* Copy the canonical CSR and degrees back (any pointer may be NULL).  Gives the
 * Graph dataclass fields indptr/indices/weights/degrees (graph.py:31-35) and the
 * operator's d_inv_sqrt (graph.py:137). */
int csc_graph_export(const csc_graph* g, int32_t* indptr, int32_t* indices, double* weights,
                     double* degrees, double* d_inv_sqrt, void* stream);

/* ---- edge-list text I/O (host, multi-threaded) ---------------------------- */
/* Replaces read_edge_list's line loop (graph.py:177-214).  Parses "src dst [weight]" lines,
 * '#' comments and the "# nodes N" header with the reference's classification (universal
 * newlines, ASCII str.strip/split).  Tokens are converted natively only where the value is
 * provably Python's int()/float(); every other line is reported as "complex" (line number,
 * byte range, reserved row slot or -1 for a comment) for the caller to parse with the
 * reference's own rules, so values, row order and errors are the reference's.
 * nthreads <= 0: all hardware threads. */
typedef struct csc_edges csc_edges;
int csc_edgelist_read(const char* path, int nthreads, csc_edges** out);
/* header_nodes: value of the last natively parsed "# nodes N" line (-1: none); header_line:
 * its line number (0: none). */
int csc_edgelist_info(const csc_edges* e, int64_t* num_rows, int64_t* num_complex, int64_t* header_nodes,
                      int64_t* header_line);
/* Rows in file order (src, dst as exact doubles, weight); complex_row[r] = 1 marks a slot
 * reserved for a complex line. */
int csc_edgelist_rows(const csc_edges* e, double* src, double* dst, double* weights, uint8_t* complex_row);
int csc_edgelist_complex(const csc_edges* e, int64_t* line_numbers, int64_t* row_slots, int64_t* byte_offsets,
                         int64_t* byte_lengths);
int csc_edgelist_destroy(csc_edges* e);
/* Replaces write_edge_list (graph.py:215-225): "# nodes N" then "i j repr(w)" per stored
 * entry with i < j in CSR order; repr() is Python's shortest round-trip float format. */
int csc_edgelist_write(const char* path, int64_t num_nodes, const int32_t* indptr, const int32_t* indices,
                       const double* weights, int nthreads);
/* Python repr() of a double as csc_edgelist_write prints it (test hook; cap >= 32). */
int csc_float_repr(double v, char* out, int cap, int* len);

/* ---- operator / filter (K2) --------------------------------------------- */
/* Y = L X for an N x ncols block.  Replaces LaplacianOp.apply (graph.py:147-155). */
int csc_laplacian_apply(const csc_graph* g, const void* X, int64_t ldx, void* Y, int64_t ldy,
                        int ncols, int io_dtype, void* stream);

/* Y = sum_l c_l T_l(L - I) X, l = 0..ncoeffs-1 (ncoeffs = order + 1).
 * Replaces apply_filter (filters.py:140-155). */
int csc_cheb_filter(const csc_graph* g, const double* coeffs, int ncoeffs, const void* X, int64_t ldx,
                    void* Y, int64_t ldy, int ncols, int io_dtype, void* stream);

/* count = sum over all entries of (h(L) R)^2, accumulated in fp64; the filtered
 * block is never written.  Replaces the filter + reduction of eigencount
 * (spectrum.py:81-86). */
int csc_eigencount(const csc_graph* g, const double* coeffs, int ncoeffs, const void* R, int64_t ldr,
                   int ncols, int io_dtype, double* count, void* stream);

/* F = rownormalize(h(L) R).  Rows whose norm is <= 1e-300 are left zero and
 * flagged in zero_flags[N] (uint8, may be NULL); *num_zero receives their count
 * (num_zero NULL: no host synchronisation when F and zero_flags are device buffers).
 * Replaces build_features (features.py:70-93, norm rule at :80-87). */
int csc_build_features(const csc_graph* g, const double* coeffs, int ncoeffs, const void* R, int64_t ldr,
                       int ncols, int io_dtype, void* F, int64_t ldf, uint8_t* zero_flags, int64_t* num_zero,
                       void* stream);

/* Column-sharded features (each rank owns a slice of the signal columns):
 * Y = h(L) R plus rowsq[i] = sum_c Y[i,c]^2 over this slice (fp64, host or
 * device).  After the caller sums rowsq over the slices (NCCL all-reduce),
 * csc_normalize_rows divides by the global row norm with the zero-row rule of
 * features.py:80-87.  One rank with all columns equals csc_build_features. */
int csc_filter_rowsq(const csc_graph* g, const double* coeffs, int ncoeffs, const void* R, int64_t ldr, int ncols,
                     int io_dtype, void* Y, int64_t ldy, double* rowsq, void* stream);
int csc_normalize_rows(const void* Y, int64_t ldy, int64_t num_rows, int ncols, int io_dtype, const double* rowsq,
                       void* F, int64_t ldf, uint8_t* zero_flags, int64_t* num_zero, int device, void* stream);

/* AP = mask * X + gamma * (g(L) X + ridge * X) for an N x ncols block, with the
 * high-pass g given by hp_coeffs and mask[N] a uint8 sampling mask (host or
 * device).  Replaces _system_apply (sampling.py:119-121). */
int csc_system_apply(const csc_graph* g, const double* hp_coeffs, int ncoeffs, double gamma, double ridge,
                     const uint8_t* mask, const void* X, int64_t ldx, void* AP, int64_t ldap, int ncols,
                     int io_dtype, void* stream);

/* ---- sampling / interpolation / assignment (K4-K6) ------------------------ */
/* out[i, :] = F[idx[i], :] for i < n.  Replaces feats.rows[sampling.indices]
 * (pipeline.py:176) and SamplingSet.restrict (sampling.py:52-54). */
int csc_gather_rows(const void* F, int64_t ldf, int64_t num_rows, int ncols, int io_dtype,
                    const int64_t* idx, int64_t n, void* out, int64_t ldo, int device, void* stream);

/* Blocked per-column CG on (M^T M + gamma (g(L) + ridge I)) X = M^T C, with the
 * matched high-pass g given by hp_coeffs.  reduced is n x k row-major fp64 (host
 * or device).  X_out is N x k (io_dtype, leading dim ldx).  Per-column outputs
 * (host or device, may be NULL): iterations (int64[k]), residuals (fp64[k]),
 * converged (uint8[k]); *iters_run receives the number of CG iterations run.
 * Replaces interpolate_all (sampling.py:124-180) with _system_apply
 * (sampling.py:119-121). */
int csc_block_cg(const csc_graph* g, const double* hp_coeffs, int ncoeffs, double gamma, double ridge,
                 const int64_t* sample_idx, int64_t n, const double* reduced, int k, double tol,
                 int64_t max_iters, void* X_out, int64_t ldx, int io_dtype, int64_t* iterations,
                 double* residuals, uint8_t* converged, int64_t* iters_run, void* stream);

/* labels[i] = argmax_j soft[i, j] / ||soft[:, j]|| (ties -> lowest j, zero-norm
 * columns never win); rows that are identically zero fall back to the raw argmax
 * (= 0) and are flagged in fallback[N] (may be NULL); *num_fallback receives
 * their count.  CSC_ERR_INVALID when every column is zero.  Replaces assign
 * (sampling.py:197-220). */
int csc_assign(const void* soft, int64_t ld, int64_t num_rows, int k, int io_dtype, int64_t* labels,
               uint8_t* fallback, int64_t* num_fallback, int device, void* stream);

/* One k-means replicate from given initial centroids: Lloyd iterations with
 * first-minimum labels, mean updates, farthest-point repair of empty clusters and
 * the relative-inertia stop (kmeans.py:64-93).  points n x d and init k x d are
 * row-major fp64 (host or device); labels_out int64[n], centroids_out k x d (may
 * be NULL), *inertia_out / *iters_out as the reference's Labeling fields
 * (kmeans(..., init=...), kmeans.py:110-114). */
int csc_kmeans_lloyd(const double* points, int64_t n, int d, const double* init, int k, int64_t max_iters,
                     double tol, int64_t* labels_out, double* centroids_out, double* inertia_out, int64_t* iters_out,
                     int device, void* stream);

/* `replicates` independent k-means runs, concurrently (one CTA each).  Seeding:
 *   first_index != NULL (host array, as pcg_states): k-means++ (kmeans.py:52-61) -- replicate r's first
 *     centroid is row first_index[r] (the host's rng.integers(q)) and its D^2
 *     draws come from the PCG64 state pcg_states[4r..4r+3] = {state_hi, state_lo,
 *     inc_hi, inc_lo} taken after that draw, with numpy's arithmetic (pairwise
 *     sums, sequential cumsum, searchsorted 'right' of random());
 *   first_index == NULL: init holds replicates x k x d starting centroids.
 * Then Lloyd as csc_kmeans_lloyd.  Outputs per replicate: labels_out
 * [replicates x n], centroids_out [replicates x k x d] (may be NULL),
 * inertia_out / iters_out [replicates], status_out [replicates] (may be NULL):
 * 0 = done, 1 = the D^2 total was not positive during seeding (the reference
 * falls back to rng.integers there, kmeans.py:57-58): rerun that replicate with
 * host seeding.  Replaces the replicate loop of kmeans (kmeans.py:117-124); the
 * caller keeps the first lowest inertia. */
int csc_kmeans_replicates(const double* points, int64_t n, int d, int k, int replicates, const int64_t* first_index,
                          const uint64_t* pcg_states, const double* init, int64_t max_iters, double tol,
                          int64_t* labels_out, double* centroids_out, double* inertia_out, int64_t* iters_out,
                          int32_t* status_out, int device, void* stream);

/* Column-sharded assign: for this rank's columns [col_offset, col_offset + k) of
 * the soft indicators, per row the best normalised value (fp64, -inf if every
 * local column has zero norm), its global column (int64) and whether any local
 * entry is nonzero (uint8).  Ranks merge with the lowest-column tie rule of
 * sampling.py:210-217.  *any_norm receives 1 if some local column is nonzero. */
int csc_assign_partial(const void* soft, int64_t ld, int64_t num_rows, int k, int io_dtype, int64_t col_offset,
                       double* best_val, int64_t* best_col, uint8_t* nonzero, int* any_norm, int device,
                       void* stream);

/* ---- parity RNG --------------------------------------------------------- */
/* numpy's Generator(PCG64).standard_normal reproduced bit for bit on the device
 * (the signal draws of spectrum.py:84 / features.py:63).  Tables: numpy's
 * 256-layer ziggurat (ki uint64, wi, fi fp64), read from the installed numpy by
 * the caller.  csc_numpy_normals writes `count` draws divided by `divisor` to
 * out (fp64, host or device) starting from the 128-bit PCG64 state/increment,
 * and returns in *raw_consumed how many 64-bit outputs the draws used (advance
 * the numpy generator by that much to continue the stream). */
int csc_set_normal_tables(const uint64_t* ki, const double* wi, const double* fi);
int csc_numpy_normals(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t count,
                      double divisor, double* out, int64_t* raw_consumed, int device, void* stream);

/* numpy's 256-layer exponential ziggurat (ke uint64, we, fe fp64), for
 * csc_sbm_edges. */
int csc_set_exponential_tables(const uint64_t* ke, const double* we, const double* fe);

/* Stochastic block model edges on the device, bit-identical to the reference's
 * generator (sbm.py:83-100, 118-155) from the PCG64 state of
 * default_rng(seed).  The npairs community pairs (a <= b, in the reference's
 * order, pairs that draw nothing left out; host arrays) each give: cells (candidate node
 * pairs, > 0), log1m_q = log1p(-q) for its edge probability q in (0, 1/3)
 * (computed by the caller with the C library, as numpy does), batch (the
 * reference's gap batch size), diag (1 for a == b), row_first (first node of
 * a), col_first / col_size (first node and size of b).  Edges are written in
 * the reference's order, each pair once, as src[e] > dst[e] for diagonal pairs
 * and src in a, dst in b otherwise; src/dst are int64 host or device buffers
 * of `capacity` entries.  *num_edges receives the edge count (if it exceeds
 * capacity: CSC_ERR_INVALID, nothing written); *raw_consumed the PCG64
 * outputs used (may be NULL). */
int csc_sbm_edges(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t npairs,
                  const int64_t* cells, const double* log1m_q, const int64_t* batch, const int32_t* diag,
                  const int64_t* row_first, const int64_t* col_first, const int64_t* col_size, int64_t capacity,
                  int64_t* src, int64_t* dst, int64_t* num_edges, int64_t* raw_consumed, int device, void* stream);

/* Degree-corrected SBM edges (BASELINE config 4; the reference has no DC-SBM,
 * SPEC.md:574, so this follows SURVEY.md §8(d)'s spec and stands in for the
 * reference generator sbm.py:118-155 on that config): independent Bernoulli
 * edges P(i~j) = min(1, theta_i theta_j q) with q = q_intra inside a community
 * and q_inter across, drawn in expected O(N + #E) by rejection over geometric
 * skipping along theta-sorted candidates.  Nodes are community-ordered
 * (community c owns sizes[c] consecutive ids); theta: N host doubles.  The
 * edge set depends only on (sizes, theta, q, seed), not on nthreads (<= 0:
 * all cores).  Host-only.  *num_edges receives the edge count; the edges
 * (src < dst, host int64) are written only when it is <= capacity. */
int csc_dcsbm_edges(int64_t num_nodes, int32_t k, const int64_t* sizes, const double* theta, double q_intra,
                    double q_inter, uint64_t seed, int nthreads, int64_t capacity, int64_t* src, int64_t* dst,
                    int64_t* num_edges);

/* ---- row-sharded operator (BASELINE config 5) ------------- */
/* NCCL communicator: rank 0 creates the id, the caller distributes it (e.g. a
 * torch.distributed broadcast), every rank creates its communicator. */
int csc_comm_unique_id(uint8_t* out /* CSC_UNIQUE_ID_BYTES */);
int csc_comm_create(const uint8_t* unique_id, int nranks, int rank, int device, csc_comm** out);
int csc_comm_destroy(csc_comm* comm);

/* Rank `rank`'s row shard of an N-node graph: rows [row_starts[rank],
 * row_starts[rank + 1]) as a CSR (indptr local, starting at 0; indices = global
 * node ids, host arrays).  row_starts (nranks + 1 entries, 0 .. N, non-decreasing)
 * is any contiguous partition -- dist.row_partition balances it by nnz (SURVEY.md
 * §8e).  The gather panel every step reads holds nranks slots of
 * R = max_q (row_starts[q+1] - row_starts[q]) rows, rank q's rows at q R (the
 * all-gather of equal R-row chunks); the shard's column indices are remapped to
 * those panel rows here. */
int csc_graph_create_row_shard(int64_t num_nodes, int nranks, int rank, const int64_t* row_starts, int64_t nnz,
                               const int32_t* indptr, const int32_t* indices, const double* weights, int dtype,
                               int device, void* stream, csc_graph** out);

/* Chebyshev filter on a row-sharded block (X, Y: this rank's rows, device
 * buffers): every step is followed by an ncclAllGather of the step's rows into
 * the full gather panel.  mode 0: Y = h(L) X;  mode 1: *out = sum of squares of
 * this rank's rows of h(L) X (eigencount partial, spectrum.py:86; Y unused);
 * mode 2: Y plus out[i] = row sums of squares (features.py:80; complete per row). */
int csc_cheb_filter_rows(const csc_graph* g, csc_comm* comm, const double* coeffs, int ncoeffs, const void* X,
                         int64_t ldx, void* Y, int64_t ldy, int ncols, int io_dtype, int mode, double* out,
                         void* stream);

/* Every rank's row shard in ONE process on one device, stepped in lockstep with
 * the all-gather done as device copies into the shared gather panel: the
 * single-GPU execution of the multi-rank row-sharded filter (same kernels, same
 * per-rank arguments and panel layout as csc_cheb_filter_rows; ranks that wait on
 * one another cannot share a GPU, so this is how nranks > 1 runs on one device).
 * shards[q] must be rank q's shard; X[q] / Y[q] / out[q] are rank q's blocks and
 * results (modes as csc_cheb_filter_rows). */
int csc_cheb_filter_rows_group(const csc_graph* const* shards, int nshards, const double* coeffs, int ncoeffs,
                               const void* const* X, const int64_t* ldx, void* const* Y, const int64_t* ldy, int ncols,
                               int io_dtype, int mode, double* const* out, void* stream);

/* Peer-memory transport (the all-gather fused into the step kernel over NVLink):
 * csc_peers_create allocates this rank's two gather panels of panel_bytes each
 * (>= R * nranks * csc_panel_row_bytes(...)) plus a flag array, exportable by
 * CUDA IPC; csc_peers_handle writes its CSC_PEER_HANDLE_BYTES handle; every rank
 * distributes its handle (e.g. torch.distributed all_gather_object) and calls
 * csc_peers_attach for every other rank.  A one-rank transport is ready at once. */
int csc_panel_row_bytes(int64_t num_nodes, int ncols, int dtype, int device, int64_t nnz, int64_t* out);
int csc_peers_create(int nranks, int rank, int device, size_t panel_bytes, csc_peers** out);
int csc_peers_handle(const csc_peers* peers, uint8_t* out /* CSC_PEER_HANDLE_BYTES */);
int csc_peers_attach(csc_peers* peers, int peer_rank, const uint8_t* handle);
/* Step boundary through the host instead of the device flag barrier: when fn is set,
 * csc_cheb_filter_rows_peers synchronises its stream after each step (the peer stores have
 * landed) and calls fn(ctx), which must return 0 once every rank has arrived (e.g. a
 * torch.distributed / MPI barrier); non-zero fails the call (CSC_ERR_INVALID).  For ranks
 * that cannot run concurrently -- several processes time-sliced on one GPU, where a kernel
 * spinning on another rank's flag may never see it -- and for checking the IPC mapping and
 * the fused peer stores across processes.  fn = NULL restores the device barrier.  Every
 * rank of a transport must make the same choice. */
typedef int (*csc_host_barrier_fn)(void* ctx);
int csc_peers_set_host_barrier(csc_peers* peers, csc_host_barrier_fn fn, void* ctx);
int csc_peers_destroy(csc_peers* peers);

/* csc_cheb_filter_rows over the peer transport: each mid step's epilogue stores
 * this rank's finished rows into every rank's next gather panel (ping-pong) and
 * a system-scope flag barrier separates steps -- no collective call.  Same modes
 * and results as csc_cheb_filter_rows. */
int csc_cheb_filter_rows_peers(const csc_graph* g, csc_peers* peers, const double* coeffs, int ncoeffs,
                               const void* X, int64_t ldx, void* Y, int64_t ldy, int ncols, int io_dtype, int mode,
                               double* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CSC_B200_H */
