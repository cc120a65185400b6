/* csc_b200.h — C ABI of libcscb200.so, the B200 (sm_100a) CSC hot path.
 *
 * Drop-in boundary for the reference package `cscluster`
 * (/root/reference/pkg/src/cscluster). Every entry point below replaces one
 * reference function (cited as file:line); the Python mirror package
 * `paper_1706_03591_b200` binds them with ctypes, and INTEGRATION.md shows the
 * ctypes stub a cscluster maintainer would add.
 *
 * Conventions
 *  - All functions return an int status: CSC_OK (0) or a CSC_ERR_* code; the
 *    message of the last failure on the calling thread is csc_last_error().
 *  - Pointers named *_dev / device arrays are caller-owned device buffers
 *    (any allocator; the Python side uses torch). The library never frees
 *    caller memory. Pointers documented "host" are plain host memory.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Work is
 *    enqueued asynchronously unless a function is documented to synchronise
 *    (it then says so: it returns a host-side count or scalar).
 *  - Dense blocks (signals, features, centroids) are row-major with a leading
 *    dimension `ld` (elements per row, ld >= d). The filter needs ld*elem_size
 *    to be a multiple of 16 bytes; padding columns must be zero and stay zero.
 *  - Results are deterministic: no floating-point atomics; every reduction
 *    has a fixed order for a given device.
 */
#ifndef CSC_B200_H
#define CSC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSC_OK 0
#define CSC_ERR_ARG 1  /* invalid argument (maps to ValueError) */
#define CSC_ERR_CUDA 2 /* CUDA runtime / launch failure */
#define CSC_ERR_CAPACITY 3 /* caller-supplied buffer too small */

#define CSC_F64 0
#define CSC_F32 1

#define CSC_LAP_NORMALIZED 0
#define CSC_LAP_COMBINATORIAL 1

typedef struct csc_chebop csc_chebop; /* opaque Chebyshev operator plan */

/* ---- library ------------------------------------------------------------ */
int csc_version(void);
const char *csc_last_error(void);
/* number of SMs of the current device (host int) */
int csc_device_info(int *sm_count, int *cc_major, int *cc_minor);

/* ---- graph -> Laplacian (graphs.py:29-76 Graph.degrees/adjacency,
 *      graphs.py:339-362 laplacian) -------------------------------------- */
/* Builds the sorted CSR of the normalized (I - D^-1/2 W D^-1/2, isolated rows
 * empty) or combinatorial (D - W) Laplacian from canonical edges (lo < hi,
 * sorted by lo*n+hi, no duplicates — the Graph invariant), bit-identical to
 * the reference: deg = (sum over lo-edges) + (sum over hi-edges) in edge
 * order, inv = 1/sqrt(deg), off-diagonal -((inv_i*w)*inv_j), diag 1.0.
 * w == NULL means unit weights. indices/vals need capacity 2m+n.
 * SYNCHRONISES: writes *nnz_out and *bound_out (host). deg_dev may be NULL. */
int csc_laplacian_build(int64_t n, int64_t m, const int64_t *lo_dev, const int64_t *hi_dev,
                        const double *w_dev, int variant, int32_t *indptr_dev,
                        int32_t *indices_dev, double *vals_dev, int64_t capacity,
                        double *deg_dev, int64_t *nnz_out, double *bound_out, void *stream);

/* Edge-set delta on canonical codes (code = lo*n + hi, graphs.py:78-80):
 * new = sort((prev \ del) U ins). prev/del/ins must be sorted ascending and
 * duplicate-free; del must be a subset of prev and ins disjoint from
 * prev \ del. new_codes needs capacity m_prev - n_del + n_ins.
 * SYNCHRONISES: writes *m_new_out (host); fails if del is not found in prev. */
int csc_edge_delta(int64_t n, const int64_t *prev_dev, int64_t m_prev, const int64_t *del_dev,
                   int64_t n_del, const int64_t *ins_dev, int64_t n_ins, int64_t *new_dev,
                   int64_t capacity, int64_t *m_new_out, void *stream);
/* Graph canonicalisation (graphs.py:29-54) on device: codes_out = stable
 * ascending sort of min(i,j)*n + max(i,j) (numpy argsort kind="stable"),
 * w_out = weights in that order. flags_host[0..3] = endpoint out of range,
 * self-loop, weight <= 0, duplicate (the sort is skipped if any of the first
 * three is set; the caller raises in that order). SYNCHRONISES. */
int csc_graph_canonicalize(int64_t n, int64_t m, const int64_t *ei_dev, const int64_t *ej_dev,
                           const double *w_dev, int64_t *codes_out_dev, double *w_out_dev,
                           int32_t *flags_host, void *stream);
/* lo = code / n, hi = code % n */
int csc_codes_split(int64_t n, const int64_t *codes_dev, int64_t m, int64_t *lo_dev,
                    int64_t *hi_dev, void *stream);

/* ---- Chebyshev filter (filters.py:155-196) ------------------------------ */
/* Plan for x(L) = I - scale*L (filters.py:172-176, scale = 2/lambda_max):
 * builds M = I - scale*L on device (exact zeros dropped; an isolated row of
 * the normalized L gets M_ii = 1) in the requested dtype, plus the
 * nnz-balanced schedule (rows longer than a threshold are split into
 * fixed-size segments reduced in a fixed order). SYNCHRONISES once. */
int csc_chebop_create(const int32_t *indptr_dev, const int32_t *indices_dev,
                      const double *vals_dev, int64_t n, int64_t nnz, double scale, int dtype,
                      void *stream, csc_chebop **op_out);
int csc_chebop_destroy(csc_chebop *op);
/* host outputs: rows, stored nnz of M, long rows, long-row segments */
int csc_chebop_info(const csc_chebop *op, int64_t *n, int64_t *nnz, int64_t *n_long,
                    int64_t *n_segments);

/* host outputs: *binned = 1 when the plan orders its rows by stored length
 * (skewed degrees, e.g. configs[3]'s Chung-Lu graph: row groups of a warp
 * then gather rows of similar length), and the squared coefficient of
 * variation of M's row lengths the decision used (threshold 1.0; tuning key
 * "row_binning"). Replaces nothing in the reference (SciPy's csr_matvecs,
 * filters.py:176, walks rows in index order); results do not depend on it
 * beyond the fixed per-row accumulation order. */
int csc_chebop_schedule(const csc_chebop *op, int32_t *binned, double *len_cv2);

/* copy the plan's M (CSR) and long-row schedule into caller buffers
 * (sizes from csc_chebop_info; any pointer may be NULL) — for tests/tools */
int csc_chebop_export(const csc_chebop *op, int32_t *indptr_dev, int32_t *indices_dev,
                      void *vals_dev, int32_t *long_rows_dev, int32_t *seg_off_dev, void *stream);

/* out = h(L) x = sum_j coeffs[j] T_j(M) x by the three-term recurrence,
 * running ncoeffs-1 fused SpMM sweeps (each order: gather M*T_j, write
 * T_{j+1} = 2 M T_j - T_{j-1}, accumulate out += c_j T_{j+1}).
 * x, out: n x ld (dtype of the plan); work: 2*n*ld elements of scratch.
 * coeffs_host: ncoeffs >= 2 doubles (host). If sumsq_dev != NULL the last
 * sweep also reduces ||out||_F^2 into sumsq_dev[0] (double, device) — the
 * eigencount of filters.py:190-196 before its scale factor. */
int csc_cheb_filter(const csc_chebop *op, const void *x_dev, int64_t ld, int64_t d,
                    const double *coeffs_host, int32_t ncoeffs, void *out_dev, void *work_dev,
                    double *sumsq_dev, void *stream);

/* csc_cheb_filter (no fused norm) whose result is also copied to host memory:
 * rows of d elements to host_dst, host_pitch bytes apart (pinned memory for an
 * asynchronous copy), on copy_stream. The last order runs as nslices row-range
 * launches on `stream` and each slice's rows are downloaded while the next one
 * computes, so only 1/nslices of the device->host copy is exposed (index-ordered
 * plans without long-row segments and with d within one column chunk; other
 * plans copy once after the last order). Returns after enqueuing: the host rows
 * are valid once copy_stream has completed. Replaces the host side of the
 * reference's apply_filter contract (filters.py:155-187: NumPy in, a new NumPy
 * array out), output bitwise equal to csc_cheb_filter's. */
int csc_cheb_filter_download(const csc_chebop *op, const void *x_dev, int64_t ld, int64_t d,
                             const double *coeffs_host, int32_t ncoeffs, void *out_dev,
                             void *work_dev, void *host_dst, int64_t host_pitch, int32_t nslices,
                             void *copy_stream, void *stream);

/* Chebyshev moments of the block (single-pass eigencount bisection):
 * mu_dev[q] = sum over columns of <x, T_q(M) x>, q = 0 .. 2*m, from one
 * m-order sweep via <T_j,T_j> and <T_{j+1},T_j>. mu_dev: 2m+1 doubles.
 * work: 2*n*ld elements. */
int csc_cheb_moments(const csc_chebop *op, const void *x_dev, int64_t ld, int64_t d, int32_t m,
                     double *mu_dev, void *work_dev, void *stream);
/* Same moments, keeping every order resident for csc_cheb_combine: T_{j+1}
 * is written to block j of keep_dev (m blocks of n*ld elements; fp64 plans).
 * Single-pass bisection without a second sweep series:
 * replaces the final apply_filter at the accepted cutoff (filters.py:176-186). */
int csc_cheb_moments_keep(const csc_chebop *op, const void *x_dev, int64_t ld, int64_t d,
                          int32_t m, double *mu_dev, void *keep_dev, void *stream);
/* out = sum_j c_j T_j from the resident orders of csc_cheb_moments_keep, with
 * the fused sweep's arithmetic (bit-identical to csc_cheb_filter's output for
 * the same coefficients); sumsq_dev (nullable) = ||out||_F^2. fp64. */
int csc_cheb_combine(const void *x_dev, const void *keep_dev, int64_t n, int64_t ld, int64_t d,
                     const double *coeffs_host, int32_t ncoeffs, void *out_dev,
                     double *sumsq_dev, void *stream);

/* Tuning knobs (process-wide; defaults are the measured best):
 *   "chunk_bytes"  row-chunk width per sweep series (default 4096)
 *   "stream_hint"  1: row-local streams use L2 evict_first (default 1)
 *   "vpl"          preferred 16-byte vectors per lane (1, 2, 4): narrower row
 *                  groups, more gathers in flight per lane (default 0 = 2 for rows
 *                  up to 512 B, else 1)
 *   "sweep_g"      force the row-group width (4, 8, 16, 32; default 0 = from
 *                  "vpl")
 *   "row_binning"  row order of plans created afterwards: -1 auto (by the
 *                  row-length CV^2), 0 index order, 1 length order */
int csc_set_tuning(const char *key, int64_t value);

/* Measurement hook: when enabled, every main sweep launch of csc_cheb_filter /
 * csc_cheb_moments is bracketed by CUDA events on its stream (up to 4096
 * launches); csc_sweep_times returns their durations in ms and resets. */
int csc_sweep_timing(int enable);
/* Measurement hook: the kernel instance ("sweep_kernel<f64,G=32,VPL=2,mid,
 * index_order>") and grid of the most recent main sweep launch, so a bench
 * can check that a committed ncu capture was taken of the same launch. */
int csc_sweep_last_launch(char *name_out, int cap, int *grid_out);
int csc_sweep_times(float *ms_host, int max_count, int *count_out);

/* Stream-ordered scratch pool of the current device (diagnostics): bytes
 * reserved now, in use now, and the high-water marks of both. */
int csc_pool_stats(int64_t *out4);
/* rows x width_bytes strided copy (cudaMemcpy2DAsync, direction from the
 * pointers): the column-chunk staging of apply_filter's host pipeline
 * (filters.py apply_filter; reference filters.py:155-178 takes a host matrix). */
int csc_copy2d_async(void *dst, int64_t dpitch, const void *src, int64_t spitch,
                     int64_t width_bytes, int64_t rows, void *stream);

/* sum of squares of a dense n x ld block (dtype) into out_dev[0] (double) and
 * the count of non-finite entries into nonfinite_dev[0] (int64, nullable). */
int csc_sumsq(const void *x_dev, int64_t count, int dtype, double *out_dev,
              int64_t *nonfinite_dev, void *stream);

/* ---- k-means (kmeans.py:54-117), fp64 ---------------------------------- */
/* rownorm[i] = sum_c f[i,c]^2 */
int csc_kmeans_rownorms(const double *f_dev, int64_t n, int64_t d, int64_t ld,
                        double *rownorm_dev, void *stream);
/* labels[i] = first argmin_j max(0, |f_i|^2 - 2 f_i.c_j + |c_j|^2) (kmeans.py:54-61, 96-97);
 * own_d2[i] = that minimum; counts[j] = cluster sizes (int32). c: k x ldc. */
int csc_kmeans_assign(const double *f_dev, const double *rownorm_dev, int64_t n, int64_t d,
                      int64_t ld, const double *c_dev, int64_t ldc, const double *cnorm_dev,
                      int64_t k, int32_t *labels_dev, double *own_d2_dev, int32_t *counts_dev,
                      void *stream);
/* Lloyd plan: scratch for bounds-pruned iterations (n, d, ld, k fixed). */
typedef struct csc_kmeans_plan csc_kmeans_plan;
int csc_kmeans_plan_create(int64_t n, int64_t d, int64_t ld, int64_t k, void *stream,
                           csc_kmeans_plan **out);
int csc_kmeans_plan_destroy(csc_kmeans_plan *plan);
/* rows re-assigned by the last pruned iteration; whether it needed the
 * empty-cluster full pass (host outputs; synchronises) */
int csc_kmeans_plan_stats(const csc_kmeans_plan *plan, int64_t *candidates, int32_t *gated);
/* rows the last screened assignment could not decide (sent to the FP64
 * kernel); 0 without a screen (host output; synchronises) */
int csc_kmeans_plan_screen_stats(const csc_kmeans_plan *plan, int64_t *undecided);
/* One Lloyd iteration (kmeans.py:96-111) on device: assignment (all rows if
 * full != 0, else only rows whose Hamerly bounds cannot exclude a change,
 * recomputed in the reference's GEMM form), empty-cluster repair (exact: a
 * full reassignment precedes it), means by label, counts, and cost2 into
 * cost2_dev[0] via the centroid identity (Q_j - 2 m_j.S_j + n_j |m_j|^2).
 * The first iteration of a run must pass full = 1. cent is updated in place. */
int csc_kmeans_iterate(csc_kmeans_plan *plan, const double *f_dev, const double *rownorm_dev,
                       double *c_dev, int64_t ldc, double *cnorm_dev, int32_t *labels_dev,
                       int32_t *counts_dev, int full, double *cost2_dev, void *stream);
/* A whole Lloyd run of one restart from the seeds in c (kmeans.py:88-117)
 * without host round trips: iteration 1 (full assignment), then a CUDA
 * conditional while-graph of pruned iterations whose last node applies the
 * reference's stop rule (prev - cost2 <= tol * prev, or max_iters) on
 * device. Asynchronous on `stream`; out_dev[0] = cost2 of the last iteration
 * (exact difference form), out_dev[1] = iterations run; history_dev
 * (nullable, max_iters doubles) = per-iteration cost2 (centroid identity).
 * The graph is built once per buffer set and reused. */
int csc_kmeans_run(csc_kmeans_plan *plan, const double *f_dev, const double *rownorm_dev,
                   double *c_dev, int64_t ldc, double *cnorm_dev, int32_t *labels_dev,
                   int32_t *counts_dev, int max_iters, double tol, double *out_dev,
                   double *history_dev, void *stream);
/* Fused Lloyd for small blocks: ALL R restarts of one kmeans() call
 * (kmeans.py:120-144, inner loop _lloyd kmeans.py:88-117) in one cooperative
 * persistent launch, one CTA per SM owning a contiguous row range whose
 * features stay in shared memory; restarts advance in lock step (two grid
 * barriers per iteration: Hamerly-pruned GEMM-form assignment + block
 * partials, then the stop rule and the means). The stop rule uses the exact
 * difference-form cost of kmeans.py:111. Empty clusters are repaired as in
 * kmeans.py:99-108 (exact own distances, first-max reseeding).
 * seeds_dev: R x k x ldc (k-means++ seeds). Outputs (device): labels_dev
 * R x n int32 (each restart's final labels), cost2_dev[R] (final cost2),
 * iters_dev[R] (iterations run). Asynchronous. supported() returns 1 when the
 * shape fits (1 <= k <= 32, d <= 128, R <= 32, max_iters >= 1, the CTA's
 * rows and per-restart bounds within shared memory), else 0 (no error). */
int csc_kmeans_fused_supported(int64_t n, int64_t d, int64_t k, int64_t R, int max_iters);
int csc_kmeans_fused_run(const double *f_dev, const double *rownorm_dev, int64_t n, int64_t d,
                         int64_t ld, int64_t k, int64_t R, const double *seeds_dev, int64_t ldc,
                         int max_iters, double tol, int32_t *labels_dev, double *cost2_dev,
                         int32_t *iters_dev, void *stream);
/* The same fused launch with the k-means++ seeding inside (kmeans.py:64-77):
 * first_idx_host[r] = restart r's integers(n) draw, uniforms_host[r*(k-1)+j-1]
 * = its j-th random() draw (host arrays, the reference's consumption order).
 * Each draw takes searchsorted(cumsum(D^2), u * total) over the rows in
 * order (fixed-order block prefixes), D^2 in the difference form. seeds_dev
 * (nullable, R x k x ldc) receives the seeds; flags_dev[r] (int32) = the first
 * draw whose D^2 mass was 0 (the reference then draws integers(n): the caller
 * must re-seed that restart sequentially and rerun with
 * csc_kmeans_fused_run), else -1. |f|^2 is computed in the kernel with
 * csc_kmeans_rownorms' association. Asynchronous. */
int csc_kmeans_fused_kpp_run(const double *f_dev, int64_t n, int64_t d, int64_t ld, int64_t k,
                             int64_t R, const int64_t *first_idx_host,
                             const double *uniforms_host, int64_t ldc, int max_iters,
                             double tol, int32_t *labels_dev, double *cost2_dev,
                             int32_t *iters_dev, double *seeds_dev, int32_t *flags_dev,
                             void *stream);
/* diagnostics: while trace_dev != NULL, fused runs record CTA 0's
 * %globaltimer (ns) at the phase boundaries of iteration g into
 * trace_dev[g * 16 + slot] (slots 0..5: phase 1 start/end, barrier, phase 2
 * end, barrier, iteration end; 6..10: sub-steps of the first restart's
 * phase 1; 11: its candidate row count), g < iters_cap. */
int csc_kmeans_fused_trace(unsigned long long *trace_dev, int64_t iters_cap);
/* FP32 screen of the Lloyd assignment (csrc/kmeans_screen.cu): the plan's
 * assignments first compute the GEMM-form distances in FP32; a row whose FP32
 * best/second gap exceeds 2 (d+5) 2^-24 (|f| + max|c|)^2 provably has the same
 * FP64 first-argmin and is decided there (Hamerly bounds widened by that
 * error), every other row is recomputed by the FP64 kernels — labels, means
 * and costs are identical to the FP64-only plan. supported(): 1 if (d, k)
 * fit the screen tile. prepare(): f32 = (float)f with row stride ld32
 * (multiple of 4, 16-byte aligned), fn32 = |f32 row|^2 (n floats); call it
 * whenever f changes. set_screen(): the plan uses these buffers from now on
 * (NULL f32 disables); they must stay valid while the plan runs. */
int csc_kmeans_screen_supported(int64_t d, int64_t k);
/* 1 when plans screen (d, k) on the tensor cores (sm_100, k <= 128, d <= 256,
 * the centroid tiles and two ring units within shared memory), else 0 (the
 * FP32 SIMT screen, or FP64 only, then decides). No device work. */
int csc_kmeans_tc_supported(int64_t d, int64_t k);
/* Test hook of the tensor-core (tcgen05 kind::tf32, 3xTF32) screen: e_out
 * (n x roundup(k, 16) fp32, row-major) = |f32_i|^2 - 2 f_i.c_j + |c_j|^2 as
 * the screen computes it, from fp32 features (ld32 % 4 == 0, padding zero),
 * their fp32 norms fn32 and fp64 centroids / norms. */
int csc_kmeans_tc_distances(const void *f32_dev, int64_t n, int64_t d, int64_t ld32,
                            const float *fn32_dev, const double *c_dev, int64_t k, int64_t ldc,
                            const double *cnorm_dev, float *e_out_dev, void *stream);
int csc_kmeans_screen_prepare(const double *f_dev, int64_t n, int64_t d, int64_t ld,
                              float *f32_dev, int64_t ld32, float *fn32_dev, void *stream);
int csc_kmeans_plan_set_screen(csc_kmeans_plan *plan, const float *f32_dev, int64_t ld32,
                               const float *fn32_dev);
/* k-means tuning knobs (performance only; results do not change):
 * "assign_ver" 2|3, "assign_tn" 4|8 (v2 kernel), "assign_tile" 0 (auto) |
 * 1 (small-k kernel) | 88 | 84 | 87 | 48 | 44 | 42 (v3 register tile),
 * "finish_mode" 0|1|2 (fused / fused-256 / split iteration tail),
 * "kpp_staged" 0|1 (batched k-means++ distances: direct row loads / rows
 * staged through shared memory, the default for 16-byte-aligned blocks) */
int csc_kmeans_tuning(const char *key, int64_t value);
/* empty-cluster repair (kmeans.py:99-108): for each empty j ascending, move the
 * row with the largest own_d2 (first max) to j and set its own_d2 to -1.
 * No-op when every count is positive (checked on device; no sync). */
int csc_kmeans_repair(int32_t *labels_dev, double *own_d2_dev, int32_t *counts_dev, int64_t n,
                      int64_t k, void *stream);
/* means by label (kmeans.py:80-85): c = sums / max(count,1), cnorm = |c_j|^2,
 * counts recomputed from labels; deterministic (fixed-order partials). */
int csc_kmeans_update(const double *f_dev, const int32_t *labels_dev, int64_t n, int64_t d,
                      int64_t ld, int64_t k, double *c_dev, int64_t ldc, double *cnorm_dev,
                      int32_t *counts_dev, void *stream);
/* cost2 = sum_i |f_i - c_{label_i}|^2 (kmeans.py:111) into cost2_dev[0] */
int csc_kmeans_cost(const double *f_dev, const int32_t *labels_dev, const double *c_dev,
                    int64_t ldc, int64_t n, int64_t d, int64_t ld, double *cost2_dev,
                    void *stream);
/* k-means++ (kmeans.py:64-77). Rows are split into `nchunks` contiguous
 * chunks (use csc_kmeanspp_nchunks(n)); closest = (first ? d2 : min(closest,
 * d2)) with d2 = |f_i - c_row|^2 (difference form), chunk_sums_dev[b] = the
 * chunk's sum of closest, total_dev[0] (nullable) = their sum in order. */
int csc_kmeanspp_nchunks(int64_t n);
int csc_kmeanspp_dist(const double *f_dev, int64_t n, int64_t d, int64_t ld,
                      const double *c_row_dev, double *closest_dev, int first,
                      double *chunk_sums_dev, int64_t nchunks, double *total_dev,
                      void *stream);
/* D^2 draw for one uniform u: idx = first i with closest_i > 0 and
 * prefix_i > u * total (Generator.choice(n, p=closest/total) ==
 * searchsorted(cumsum(p), u, 'right')). If fixed_idx >= 0 it is used instead
 * (the reference's rng.integers(n) paths). Copies row idx of f into
 * c_row_dev and writes idx to idx_dev[0] (int64). */
int csc_kmeanspp_pick(const double *f_dev, int64_t n, int64_t d, int64_t ld,
                      const double *closest_dev, const double *chunk_sums_dev,
                      int64_t nchunks, double u, int64_t fixed_idx, double *c_row_dev,
                      int64_t *idx_dev, void *stream);

/* Batched k-means++ for R <= 16 restarts in one pass per centroid index.
 * first_idx_host[r] = the restart's integers(n) draw; uniforms_host[r*(k-1)+j-1]
 * = its j-th random() draw (host arrays). Writes cent[r*k*ldc + j*ldc + c]
 * (device, R x k x ldc). flags_dev[r] (int32, device) = first j whose D^2
 * mass was 0 (the reference then draws integers(n): the caller must replay
 * that restart on the sequential path), else -1. */
int csc_kmeanspp_batch(const double *f_dev, int64_t n, int64_t d, int64_t ld, int64_t R, int64_t k,
                       const int64_t *first_idx_host, const double *uniforms_host, double *cent_dev,
                       int64_t ldc, int32_t *flags_dev, void *stream);

/* ---- probe signals (signals.py:16-37) ---------------------------------- */
/* out[i*ld + col0 + c] = 0.0 + sigma * z_c[i], z_c = numpy's
 * Generator(PCG64).standard_normal stream from the column's initial PCG64
 * state states_host[4c..4c+3] = (state lo, state hi, inc lo, inc hi) (host).
 * Chunk-parallel ziggurat with verified chunk boundaries; bad_host[c] = 1
 * marks a column the caller must regenerate on the host (boundary
 * disagreement or too few draws; not expected in practice). Bit-identical
 * to numpy except that tail samples (|z| > 3.65) go through the device
 * log1p/exp, which may round the last bit differently. SYNCHRONISES. */
/* numpy SeedSequence -> PCG64 seeding on the host (signals.py:34-37 builds
 * default_rng(child) per column): states_out[4c..4c+3] = (state lo, state hi,
 * inc lo, inc hi) of PCG64(child c) for the children first_child .. + d - 1 of
 * the SeedSequence with the given run entropy and spawn key (little-endian
 * uint32 words, as numpy coerces them) and pool size. No device work. */
int csc_seed_states(const uint32_t *run_entropy, int64_t n_run, const uint32_t *key_prefix,
                    int64_t n_key, int64_t first_child, int64_t d, int32_t pool_size,
                    uint64_t *states_out);
int csc_normal_columns(const uint64_t *states_host, int64_t ncols, int64_t n, double sigma,
                       double *out_dev, int64_t ld, int64_t col0, int32_t *bad_host, void *stream);
/* The same without synchronising: the flags go to bad_dev (ncols int32,
 * device) for the caller to read at its next synchronisation. */
int csc_normal_columns_async(const uint64_t *states_host, int64_t ncols, int64_t n, double sigma,
                             double *out_dev, int64_t ld, int64_t col0, int32_t *bad_dev,
                             void *stream);

/* ---- dense helpers ------------------------------------------------------ */
/* dst[:, j] = src[:, cols[j]] for j < ncols (row-major, f64), the Theta
 * assembly of dynamic.py:163-168. cols_dev: int64. */
int csc_gather_columns(const double *src_dev, int64_t n, int64_t ld_src, const int64_t *cols_dev,
                       int64_t ncols, double *dst_dev, int64_t ld_dst, int64_t dst_col0,
                       void *stream);

/* ---- O(m) synthetic graph generators on device ------------
 * Replace the reference's O(n^2) samplers for n in the millions:
 * sbm_generate (graphs.py:194-221), perturb_edges (graphs.py:236-273, with
 * _absent_pairs graphs.py:228-233) and perturb_nodes (graphs.py:276-319).
 * Equal in distribution, not stream-identical: Philox-4x32-10 keyed by
 * `seed`, deterministic for a seed. Blocks are nblocks near-equal contiguous
 * node ranges (sizes[:n % nblocks] one larger), as SbmParams uses. Outputs
 * are sorted, duplicate-free canonical codes lo*n+hi. All SYNCHRONISE. */
/* planted partition: pair_counts (host, nblocks*(nblocks+1)/2, pairs (a, b)
 * with a <= b in row-major order) edges per block pair — the caller's
 * Binomial(pairs of (a, b), q) draws — each a uniform distinct subset of the
 * pair's node pairs. codes_out capacity >= sum of the counts. */
int csc_gen_planted_partition(int64_t n, int32_t nblocks, const int64_t *pair_counts, uint64_t seed,
                              int64_t *codes_out_dev, int64_t capacity, int64_t *m_out,
                              void *stream);
/* Chung-Lu / degree-corrected SBM: m_draw edge draws, each a block pair
 * from pair_cum_host (nblocks^2 doubles, inclusive cumulative weights, index
 * a*nblocks+b) and endpoints from cum_theta_dev (n doubles, per-block
 * inclusive cumulative theta); self-loops and repeats dropped. */
int csc_gen_chung_lu(int64_t n, int32_t nblocks, const double *cum_theta_dev,
                     const double *pair_cum_host, int64_t m_draw, uint64_t seed,
                     int64_t *codes_out_dev, int64_t capacity, int64_t *m_out, void *stream);
/* edge churn (perturb_edges semantics): `count` present edges deleted
 * uniformly, `count` absent pairs inserted in proportion to q1 (same label)
 * / q2 (different labels) without replacement; pairs in both lists dropped
 * from both. labels_dev: n int32 in [0, nblocks). del/ins capacity >= count. */
int csc_gen_edge_churn(int64_t n, const int64_t *codes_dev, int64_t m, const int32_t *labels_dev,
                       int32_t nblocks, double q1, double q2, int64_t count, uint64_t seed,
                       int64_t *del_out_dev, int64_t *n_del, int64_t *ins_out_dev, int64_t *n_ins,
                       void *stream);
/* node switch (perturb_nodes semantics): `count` distinct nodes move to a
 * uniformly drawn other label (labels_dev updated in place), every edge at a
 * moved node is deleted, every pair with a moved endpoint is drawn once with
 * q1 / q2 under the new labels; pairs in both lists dropped from both.
 * del capacity >= m; CSC_ERR_CAPACITY if insertions exceed ins_capacity. */
int csc_gen_node_switch(int64_t n, const int64_t *codes_dev, int64_t m, int32_t *labels_dev,
                        int32_t nblocks, double q1, double q2, int64_t count, uint64_t seed,
                        int64_t *del_out_dev, int64_t *n_del, int64_t *ins_out_dev,
                        int64_t ins_capacity, int64_t *n_ins, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CSC_B200_H */
