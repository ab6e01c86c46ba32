/*
 * ftk_b200.h -- C ABI of the B200-native FT K-means Lloyd hot path.
 *
 * Plain C types only: device pointers (void*, int64_t*), sizes and a
 * cudaStream_t passed as void*.  Every entry point returns an int status:
 *   FTK_OK (0), FTK_OVERFLOW (1, detection-event ring overflowed -- the
 *   reference's _checked_range return value, abft.py:315-316), or a negative
 *   error (ftk_last_error() has the message).  Kernels never raise; the host
 *   layer maps statuses to the reference's exception types.
 *
 * Reference interface each entry point replaces (ftkmeans 0.1.0, numba):
 *   ftk_row_sq_norms      <- _kernels._row_sq_norms            (_kernels.py:106-114)
 *   ftk_assign            <- _kernels._assign_range            (_kernels.py:432-475)
 *                            driven by gemm.fused_assign       (gemm.py:88-141)
 *   ftk_checked_assign    <- _kernels._checked_range(materialize=0)
 *                                                              (_kernels.py:479-612)
 *                            driven by abft._checked_run       (abft.py:247-341)
 *   ftk_gemm              <- _kernels._gemm_range / _checked_range(materialize=1)
 *                                                              (_kernels.py:409-428, 608-609)
 *   ftk_update_sums       <- the bincount loop of kmeans.update_step
 *                                                              (kmeans.py:167-189)
 *   ftk_update_finalize   <- means + empty detection           (kmeans.py:191-197)
 *   ftk_pairwise_sum      <- float(np.sum(sq_dists))           (kmeans.py:275, 307)
 *   ftk_movement          <- the np.linalg.norm movement test  (kmeans.py:289-293)
 * All device memory is caller-owned except the scratch a context caches.
 */
#ifndef FTK_B200_H
#define FTK_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FTK_OK 0
#define FTK_OVERFLOW 1
#define FTK_ERR_CUDA (-1)
#define FTK_ERR_ARG (-2)
#define FTK_ERR_UNSUPPORTED (-3)

#define FTK_F32 0
#define FTK_F64 1

/* Assign-kernel variants (ftk_assign / ftk_checked_assign `variant`). */
#define FTK_VARIANT_AUTO 0
#define FTK_VARIANT_EXACT 1  /* SIMT, reference evaluation order, bit-exact   */
#define FTK_VARIANT_TC 2     /* tcgen05 tf32 screen + certified exact refine  */
/* Forced kernel families (variants.py VariantTable; the reference's
 * TuneTable/select, tuner.py:230-351, chooses a CPU tile instead).  Each is
 * bit-exact like every other variant; a family that does not apply to the
 * dtype is FTK_ERR_ARG, a shape it cannot take FTK_ERR_UNSUPPORTED. */
#define FTK_VARIANT_TC_PAIR 3    /* CTA-pair tcgen05 screen (tc_pair.cu; f64: tc64.cu) */
#define FTK_VARIANT_TC_NARROW 4  /* f32: streamed-X narrow screen (tc_narrow.cu) */
#define FTK_VARIANT_F64_DMMA 5   /* f64: DMMA screen (dscreen.cu)               */
#define FTK_VARIANT_F64_DFMA 6   /* f64: DFMA SIMT screen (dscreen.cu)          */

/* Scheduled injections for one kernel call: the eight arrays of
 * FaultHook.kernel_arrays (faults.py:261-277), as DEVICE pointers.  Entries
 * address logical tiles of the fault grid (bm x bn), like the reference. */
typedef struct ftk_injection {
    int64_t n;
    const int64_t *bi, *bj, *ei, *ej, *bit;
    int64_t *applied;  /* out: 1 when the flip landed on a live cell     */
    double *before;    /* out: accumulator value before the flip (f64)   */
    double *after;     /* out: after                                     */
    /* optional: live count on the device. When set, n is the capacity of the
     * arrays and the launches never read the count on the host, so a checked
     * assignment with scheduled flips can be captured in a CUDA graph and
     * replayed with a new schedule copied into the same arrays. */
    const int64_t *n_dev;
} ftk_injection;

/* Detection-event ring (abft.py:281-294): rec is cap x 7 int64
 * (iteration, tile_i, tile_j, kind, loc_i, loc_j, interval), delta is cap
 * doubles, count a single int64 that may exceed cap (overflow). */
typedef struct ftk_events {
    int64_t cap;
    int64_t *rec;
    double *delta;
    int64_t *count;
} ftk_events;

typedef struct ftk_ctx ftk_ctx;

const char *ftk_last_error(void);
int ftk_version(void);
/* Number of kernels this library launched since load (for launch accounting). */
int64_t ftk_launch_count(void);
/* Account n kernels replayed from a CUDA graph captured from this library's
 * launches (the replay itself bypasses the launch sites). */
void ftk_add_launches(int64_t n);

ftk_ctx *ftk_ctx_create(int device);
void ftk_ctx_destroy(ftk_ctx *ctx);

/* Per-row screening bounds of an fp32 matrix, info: m x 4 floats per row
 * (sum x^2, sum (x - tf32(x))^2, max |x|, 0), any summation order (they only
 * feed upper bounds).  Used by the tensor-core assignment certificate. */
int ftk_row_info(ftk_ctx *ctx, const float *x, int64_t m, int64_t d, float *info, void *stream);

/* Register precomputed row bounds (ftk_row_info) for the data matrix x of a
 * fit: assignment calls with exactly this (x, m, d) read them instead of
 * recomputing them from x every call.  The caller guarantees x is not
 * modified while registered; pass x = NULL to unregister.  The reference has
 * no counterpart (its kernels recompute nothing across calls). */
int ftk_ctx_set_rows(ftk_ctx *ctx, const void *x, int64_t m, int64_t d, const float *info);
/* Float64 data screened on the tf32 tensor cores (tc64.cu): x32 (m x d fp32,
 * caller-allocated) receives fp32(x), info the row bounds measured against
 * the float64 rows (|x|^2, |x - tf32(fp32(x))|^2, max|x|, 0).  Registering
 * them (ftk_ctx_set_rows64) lets every float64 assignment of the fit reuse
 * the copy; unregistered calls convert per call.  Replaces nothing in the
 * reference (its float64 kernel, _kernels.py:432-475, has no screen). */
int ftk_row_info64(ftk_ctx *ctx, const double *x, int64_t m, int64_t d, float *x32, float *info,
                   void *stream);
int ftk_ctx_set_rows64(ftk_ctx *ctx, const double *x, int64_t m, int64_t d, const float *x32,
                       const float *info);
/* Label hint for the next assignments on this context: labels (m int32,
 * device) of the previous Lloyd iteration.  The narrow screen (d > 256,
 * k + 4 <= 256) computes the exact reference value of the hinted centroid
 * while X streams through shared memory, so rows whose label is unchanged
 * need no second read of X.  Only a speed hint: any content (even out of
 * range) gives the same results.  Used while m matches; NULL clears it.  The
 * caller keeps the buffer alive while it is set.  No reference counterpart. */
int ftk_ctx_set_label_hint(ftk_ctx *ctx, const int32_t *labels, int64_t m);

/* Context options.  FTK_OPT_INJ_REPLAY (default 1): the logical row blocks
 * carrying scheduled flips are replayed by the exact checked kernel after a
 * screened checked assignment, so their detection events are the reference's
 * own.  0 (validation of the in-kernel correction): the screen's own
 * detect/locate/correct result stands and it records an event for every
 * detection (narrow screen). */
#define FTK_OPT_INJ_REPLAY 1
int ftk_ctx_set_option(ftk_ctx *ctx, int option, int64_t value);

/* Number of scratch (re)allocations on this context so far: a CUDA graph
 * captured from this context's launches is stale once it changes. */
int64_t ftk_ctx_generation(ftk_ctx *ctx);

/* k-means++ D^2 seeding (replaces the numpy body of kmeans.init_centroids,
 * kmeans.py:86-103).  ftk_kpp_d2 / ftk_kpp_update: d2[i] = sum_f (x[i,f] -
 * x[pick,f])^2 in float64 with numpy's pairwise association over the feature
 * axis (any d), then np.minimum with the previous d2 unless `first`.  The
 * pick is `host_pick` when >= 0, else read from *pick_dev; picks[c] records
 * it (picks may be NULL). */
int ftk_kpp_d2(ftk_ctx *ctx, int dtype, const void *x, int64_t m, int64_t d, int64_t pick,
               int first, double *d2, void *stream);
int ftk_kpp_update(ftk_ctx *ctx, int dtype, const void *x, int64_t m, int64_t d, int64_t host_pick,
                   const int64_t *pick_dev, int first, double *d2, int64_t *picks, int64_t c,
                   void *stream);
/* *pick_dev = min(searchsorted(cumsum(d2), r, side="right"), m - 1) with
 * numpy's SEQUENTIAL float64 cumsum, bit-exact: a parallel scan classifies
 * every prefix against r under a rigorous rounding bound; if any prefix is
 * within the bound of r, one thread replays the sequential cumsum (and
 * *n_replays is incremented).  r = Generator.random() * d2.sum() from the
 * host, as in the reference.  No host synchronisation. */
int ftk_kpp_search(ftk_ctx *ctx, const double *d2, int64_t m, double r, int64_t *pick_dev,
                   uint64_t *n_replays, void *stream);

/* out[i] = left-to-right sum of x[i,j]^2 in the data dtype. */
int ftk_row_sq_norms(ftk_ctx *ctx, int dtype, const void *x, int64_t m, int64_t n, void *out,
                     void *stream);

/* Fused nearest-centroid assignment.  x: m x d, y: k x d (row-major, dtype),
 * ynorms: k (dtype).  out_idx: m int32 labels, out_val: m dtype values of
 * yn[j] - 2 x.y at the winner -- bit-identical to the reference for every
 * variant.  (bm, bn) is the logical fault-tile geometry (TileConfig.block)
 * that `inj` addresses; inj may be NULL.  xnorm (m floats, sqrt of the row
 * norms rounded up) is only read by the TC variant; pass NULL to have the
 * library compute it. */
int ftk_assign(ftk_ctx *ctx, int dtype, int variant, const void *x, const void *y,
               const void *ynorms, int64_t m, int64_t k, int64_t d, int64_t bm, int64_t bn,
               int64_t bk, int32_t *out_idx, void *out_val, const ftk_injection *inj,
               void *stream);

/* Checksum-protected assignment over logical (bm, bn, bk) tiles.  Detection,
 * location, correction and the event record follow _checked_range exactly
 * (tolerance delta_rel * max(1, amax_x * amax_y) * k_acc + abs_tol, float64
 * checksums).  Returns FTK_OVERFLOW when *ev->count ends above ev->cap
 * (requires a stream sync; pass sync_check = 1 to perform it). */
int ftk_checked_assign(ftk_ctx *ctx, int dtype, int variant, const void *x, const void *y,
                       const void *ynorms, int64_t m, int64_t k, int64_t d, int64_t bm,
                       int64_t bn, int64_t bk, double delta_rel, double abs_tol,
                       int64_t iteration, int32_t *out_idx, void *out_val,
                       const ftk_injection *inj, ftk_events *ev, void *stream);

/* Materialised x @ y.T (m x k, dtype), unprotected (ev == NULL) or checked. */
int ftk_gemm(ftk_ctx *ctx, int dtype, const void *x, const void *y, int64_t m, int64_t k,
             int64_t d, int64_t bm, int64_t bn, int64_t bk, double delta_rel, double abs_tol,
             int64_t iteration, void *out, const ftk_injection *inj, ftk_events *ev,
             void *stream);

/* Per-cluster sums in float64 with the reference's accumulation order
 * (ascending sample index per cluster) and int64 counts.  sums_b / counts_b
 * (nullable) receive an independent duplicate accumulation (DMR).
 * labels are int32 in [0, k). */
int ftk_update_sums(ftk_ctx *ctx, int dtype, const void *x, const int32_t *labels, int64_t m,
                    int64_t d, int64_t k, double *sums_a, int64_t *counts_a, double *sums_b,
                    int64_t *counts_b, void *stream);

/* Bitwise comparison of the two DMR accumulations; *out_mismatch (device
 * int32) is set to 1 if any word differs, else 0. */
int ftk_dmr_compare(ftk_ctx *ctx, const double *sums_a, const int64_t *counts_a,
                    const double *sums_b, const int64_t *counts_b, int64_t k, int64_t d,
                    int32_t *out_mismatch, void *stream);

/* centroids[j] = dtype(sums[j] / counts[j]) for non-empty clusters, 0 for
 * empty ones; *n_empty (device int32) = number of empty clusters. */
int ftk_update_finalize(ftk_ctx *ctx, int dtype, const double *sums, const int64_t *counts,
                        int64_t k, int64_t d, void *centroids, int32_t *n_empty, void *stream);

/* Empty-cluster reseed (kmeans.py:197-206): successive farthest points by
 * sq_dists (first maximum wins), written into centroids rows of the empty
 * clusters in ascending cluster order.  sq_dists is modified (-inf marks). */
int ftk_reseed_empty(ftk_ctx *ctx, int dtype, const void *x, int64_t m, int64_t d,
                     const int64_t *counts, int64_t k, double *sq_dists, void *centroids,
                     void *stream);

/* sq[i] = double(min_dists[i]) + x_sq[i];  *out = numpy pairwise sum of sq. */
int ftk_sq_dists(ftk_ctx *ctx, int dtype, const void *min_dists, const double *x_sq, int64_t m,
                 double *sq, void *stream);
int ftk_pairwise_sum(ftk_ctx *ctx, const double *a, int64_t n, double *out, void *stream);

/* *moved = max_j ||new_j - old_j|| / (||old_j|| + eps), float64, with numpy's
 * pairwise row reduction (np.linalg.norm(axis=1)). */
int ftk_movement(ftk_ctx *ctx, int dtype, const void *new_c, const void *old_c, int64_t k,
                 int64_t d, double eps, double *moved, void *stream);

/* *out = 1 if a[0:m] == b[0:m] (int32 labels), else 0 (device int32). */
int ftk_labels_equal(ftk_ctx *ctx, const int32_t *a, const int32_t *b, int64_t m, int32_t *out,
                     void *stream);

/* out[i] = sum_f (x[i,f] - cent64[labels[i], f])^2 in float64 with numpy's
 * pairwise association (the update_step fallback when sq_dists is not
 * supplied, kmeans.py:199-201). */
int ftk_own_sq_dists(ftk_ctx *ctx, int dtype, const void *x, const int32_t *labels,
                     const double *cent64, int64_t m, int64_t d, double *out, void *stream);

/* XOR bit `bit` of element (i, j) of a float64 k x d device array
 * (update-accumulator fault site, faults.py:295-324 applied on device). */
int ftk_flip_f64(ftk_ctx *ctx, double *a, int64_t d, int64_t i, int64_t j, int64_t bit,
                 double *before_after, void *stream);

/* Diagnostics: out[0] = rows the last TC-variant assignment could not certify
 * with the 1xTF32 screen, out[1] = rows the 3xTF32 re-screen still could not
 * certify (resolved by the exact kernel). */
int ftk_tc_fallback_rows(ftk_ctx *ctx, int64_t *out, void *stream);

/* Upload `nbytes` from PAGEABLE host memory (e.g. a numpy array) to device
 * memory at pinned-copy speed: parallel host copies into page-locked staging
 * buffers overlapped with the DMA.  Returns when the host source may be
 * reused; `stream` is ordered behind the upload (no device synchronisation).
 * Replaces the reference's implicit numpy residency (its kernels read the
 * caller's array in place, gemm.py:108-131). */
int ftk_h2d(ftk_ctx *ctx, void *dst, const void *src, int64_t nbytes, void *stream);

/* Diagnostics: cumulative count of rows whose tensor-core / DMMA row
 * checksum failed (every screened checked assignment on this context since
 * the last reset; *out = 0 before the first).  reset != 0 zeroes it after
 * the read.  Synchronises `stream`. */
int ftk_abft_flags_total(ftk_ctx *ctx, int64_t *out, int reset, void *stream);

/* Diagnostics: device time (CUDA events on the launching stream) of the
 * last tensor-core screen launch (the CTA-pair pass-1 kernel), in ms; -1 if
 * the last TC assignment did not use it. */
int ftk_tc_last_kernel_ms(ftk_ctx *ctx, float *ms);

/* Validation hook for the screening error model: runs the TC assignment
 * (split = 0: 1xTF32 pass then 3xTF32 on ties; split = 1: 3xTF32 on every
 * row) and also materialises the raw tensor-core dot products of the screen
 * into raw (m x k fp32, row-major). */
int ftk_tc_raw_dots(ftk_ctx *ctx, int split, const float *x, const float *y, const float *ynorms,
                    int64_t m, int64_t k, int64_t d, float *raw, int32_t *out_idx,
                    float *out_val, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* FTK_B200_H */
