/*
 * ftk_oracle.c -- CPU restatement of the reference's Lloyd hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the checker or as the
 * timed CPU baseline.  The product path (paper_2408_01391_b200) never calls it.
 *
 * Reference: ftkmeans 0.1.0 (/root/reference/pkg/src/ftkmeans), a numba CPU
 * package.  Every function below restates one reference routine with the same
 * floating-point evaluation order, so results are bit-identical to it:
 *
 *   - products and sums are separate IEEE roundings (numba emits vmul+vadd,
 *     no FMA; SURVEY.md Appendix B probe 2).  Build with -ffp-contract=off.
 *   - dot products accumulate k ascending from 0.0 (_kernels.py:44-70 with
 *     _zero_tile 74-77: per output element the k loop is sequential across
 *     k-blocks and within them).
 *   - the distance expression is  yn[j] - (acc + acc)  in the data dtype and
 *     the argmin is the first strict minimum in ascending j, starting from
 *     (+inf, 0) (_kernels.py:88-102, 450-452).
 *   - update sums are numpy.bincount(labels, weights=x[:, f]): float64,
 *     ascending sample order (kmeans.py:167-171).
 *   - numpy's pairwise summation for float64 add.reduce (inertia, kmeans.py:275
 *     and 307; row norms in np.linalg.norm, kmeans.py:289-292).
 *
 * Pinned against the reference by tests/golden/ (see tests/golden/make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MAXT 256

/* ---------------------------------------------------------------- norms -- */
/* _kernels.py:106-114 : s = x0*x0; s += xj*xj  (dtype, left to right) */
void ftko_row_sq_norms_f32(const float *x, int64_t m, int64_t n, float *out) {
    for (int64_t i = 0; i < m; ++i) {
        const float *r = x + i * n;
        float s = r[0] * r[0];
        for (int64_t j = 1; j < n; ++j) {
            float p = r[j] * r[j];
            s = s + p;
        }
        out[i] = s;
    }
}

void ftko_row_sq_norms_f64(const double *x, int64_t m, int64_t n, double *out) {
    for (int64_t i = 0; i < m; ++i) {
        const double *r = x + i * n;
        double s = r[0] * r[0];
        for (int64_t j = 1; j < n; ++j) {
            double p = r[j] * r[j];
            s = s + p;
        }
        out[i] = s;
    }
}

/* --------------------------------------------------------------- assign -- */
/* Fused distance + argmin (_kernels.py:432-475 with _accum_panel 44-70 and
 * _argmin_merge 88-102).  The column-blocked loop nest below only exists so
 * the compiler vectorises the j loop (like numba does); the per-element
 * evaluation order is exactly the reference's. */
#define OBN 64

typedef struct {
    const void *x, *y, *yn;
    int64_t m, k, d, lo, hi;
    int64_t *idx;
    void *val;
} assign_job;

static void *assign_f32_worker(void *arg) {
    assign_job *J = (assign_job *)arg;
    const float *x = J->x, *y = J->y, *yn = J->yn;
    int64_t k = J->k, d = J->d;
    float *bt = malloc(sizeof(float) * d * OBN);
    float acc[OBN];
    for (int64_t j0 = 0; j0 < k; j0 += OBN) {
        int64_t nj = k - j0 < OBN ? k - j0 : OBN;
        for (int64_t kk = 0; kk < d; ++kk)
            for (int64_t j = 0; j < nj; ++j) bt[kk * OBN + j] = y[(j0 + j) * d + kk];
        for (int64_t i = J->lo; i < J->hi; ++i) {
            const float *xr = x + i * d;
            for (int64_t j = 0; j < OBN; ++j) acc[j] = 0.0f;
            for (int64_t kk = 0; kk < d; ++kk) {
                float xv = xr[kk];
                const float *br = bt + kk * OBN;
                for (int64_t j = 0; j < OBN; ++j) {
                    float p = xv * br[j];
                    acc[j] = acc[j] + p;
                }
            }
            float bv = j0 == 0 ? INFINITY : ((float *)J->val)[i];
            int64_t bj = j0 == 0 ? 0 : J->idx[i];
            for (int64_t j = 0; j < nj; ++j) {
                float dd = yn[j0 + j] - (acc[j] + acc[j]);
                int64_t gj = j0 + j;
                if (dd < bv || (dd == bv && gj < bj)) { bv = dd; bj = gj; }
            }
            ((float *)J->val)[i] = bv;
            J->idx[i] = bj;
        }
    }
    free(bt);
    return NULL;
}

static void *assign_f64_worker(void *arg) {
    assign_job *J = (assign_job *)arg;
    const double *x = J->x, *y = J->y, *yn = J->yn;
    int64_t k = J->k, d = J->d;
    double *bt = malloc(sizeof(double) * d * OBN);
    double acc[OBN];
    for (int64_t j0 = 0; j0 < k; j0 += OBN) {
        int64_t nj = k - j0 < OBN ? k - j0 : OBN;
        for (int64_t kk = 0; kk < d; ++kk)
            for (int64_t j = 0; j < nj; ++j) bt[kk * OBN + j] = y[(j0 + j) * d + kk];
        for (int64_t i = J->lo; i < J->hi; ++i) {
            const double *xr = x + i * d;
            for (int64_t j = 0; j < OBN; ++j) acc[j] = 0.0;
            for (int64_t kk = 0; kk < d; ++kk) {
                double xv = xr[kk];
                const double *br = bt + kk * OBN;
                for (int64_t j = 0; j < OBN; ++j) {
                    double p = xv * br[j];
                    acc[j] = acc[j] + p;
                }
            }
            double bv = j0 == 0 ? INFINITY : ((double *)J->val)[i];
            int64_t bj = j0 == 0 ? 0 : J->idx[i];
            for (int64_t j = 0; j < nj; ++j) {
                double dd = yn[j0 + j] - (acc[j] + acc[j]);
                int64_t gj = j0 + j;
                if (dd < bv || (dd == bv && gj < bj)) { bv = dd; bj = gj; }
            }
            ((double *)J->val)[i] = bv;
            J->idx[i] = bj;
        }
    }
    free(bt);
    return NULL;
}

static void run_rows(void *(*fn)(void *), assign_job base, int threads) {
    if (threads < 1) threads = 1;
    if (threads > MAXT) threads = MAXT;
    if (base.m < threads) threads = base.m > 0 ? (int)base.m : 1;
    pthread_t th[MAXT];
    assign_job jobs[MAXT];
    int64_t step = (base.m + threads - 1) / threads;
    int n = 0;
    for (int64_t lo = 0; lo < base.m; lo += step, ++n) {
        jobs[n] = base;
        jobs[n].lo = lo;
        jobs[n].hi = lo + step < base.m ? lo + step : base.m;
    }
    if (n == 1) { fn(&jobs[0]); return; }
    for (int t = 0; t < n; ++t) pthread_create(&th[t], NULL, fn, &jobs[t]);
    for (int t = 0; t < n; ++t) pthread_join(th[t], NULL);
}

void ftko_assign_f32(const float *x, const float *y, const float *yn, int64_t m, int64_t k,
                     int64_t d, int64_t *idx, float *val, int threads) {
    assign_job J = {x, y, yn, m, k, d, 0, m, idx, val};
    run_rows(assign_f32_worker, J, threads);
}

void ftko_assign_f64(const double *x, const double *y, const double *yn, int64_t m, int64_t k,
                     int64_t d, int64_t *idx, double *val, int threads) {
    assign_job J = {x, y, yn, m, k, d, 0, m, idx, val};
    run_rows(assign_f64_worker, J, threads);
}

/* ------------------------------------------------------- checked assign -- */
/* The reference's checksum-protected fused assignment, DETECTION ONLY
 * (_kernels.py:479-612 with _encode_c1_amax 158-180, _apply_col_refs 128-137,
 * _tile_colsums 183-202 and _block_absmax 117-125): per logical tile
 * (bm x bn) and k-interval (bk) the e1 column references
 * ref1[j] += sum_k (e1' X_blk)[k] * C[j][k] (f64) are compared with the
 * column sums of the accumulator tile (4-row pre-reduction in the data
 * dtype, then f64) under tol = delta_rel * max(1, amax_X * amax_C) * k_acc
 * + abs_tol.  The accumulators and the argmin are the unprotected ones
 * (bit-identical labels), so this is the reference's fault-free ABFT cost;
 * violations are only counted (no flips are injected on this path, and
 * _diagnose is not restated), and the caller raises if any occur. */
typedef struct {
    const void *x, *y, *yn;
    int64_t m, k, d, bm, bn, bk, lo, hi;  /* lo/hi: row BLOCKS */
    double delta_rel, abs_tol;
    const double *cmax;  /* per column block: max |C| */
    int64_t *idx;
    void *val;
    int64_t viol;
} chk_job;

#define DEFINE_CHECKED(T, NAME)                                                              \
static void *NAME(void *arg) {                                                               \
    chk_job *J = (chk_job *)arg;                                                             \
    const T *x = J->x, *y = J->y, *yn = J->yn;                                               \
    const int64_t k = J->k, d = J->d, bm = J->bm, bn = J->bn, bk = J->bk;                    \
    const int64_t nbk = (d + bk - 1) / bk;                                                   \
    T *bt = malloc(sizeof(T) * d * OBN);                                                     \
    T *acc = malloc(sizeof(T) * bm * OBN);                                                   \
    double *c1 = malloc(sizeof(double) * nbk * bk);                                          \
    double ref1[OBN], s1[OBN];                                                               \
    T p[OBN];                                                                                \
    for (int64_t bi = J->lo; bi < J->hi; ++bi) {                                             \
        const int64_t i0 = bi * bm, mi = J->m - i0 < bm ? J->m - i0 : bm;                    \
        double amax = 0.0;                                                                   \
        for (int64_t q = 0; q < nbk * bk; ++q) c1[q] = 0.0;                                  \
        for (int64_t i = 0; i < mi; ++i)                                                     \
            for (int64_t f = 0; f < d; ++f) {                                                \
                const double v = (double)x[(i0 + i) * d + f];                                \
                c1[f] += v;                                                                  \
                const double av = v < 0.0 ? -v : v;                                          \
                if (av > amax) amax = av;                                                    \
            }                                                                                \
        for (int64_t i = 0; i < mi; ++i) {                                                   \
            ((T *)J->val)[i0 + i] = (T)INFINITY;                                             \
            J->idx[i0 + i] = 0;                                                              \
        }                                                                                    \
        for (int64_t j0 = 0; j0 < k; j0 += bn) {                                             \
            const int64_t nj = k - j0 < bn ? k - j0 : bn;                                    \
            double scale = amax * J->cmax[j0 / bn];                                          \
            if (scale < 1.0) scale = 1.0;                                                    \
            const double tol_base = J->delta_rel * scale;                                    \
            for (int64_t s0 = j0; s0 < j0 + nj; s0 += OBN) {                                 \
                const int64_t sn = j0 + nj - s0 < OBN ? j0 + nj - s0 : OBN;                  \
                for (int64_t f = 0; f < d; ++f)                                              \
                    for (int64_t j = 0; j < OBN; ++j)                                        \
                        bt[f * OBN + j] = j < sn ? y[(s0 + j) * d + f] : (T)0;               \
                for (int64_t q = 0; q < mi * OBN; ++q) acc[q] = (T)0;                        \
                for (int64_t j = 0; j < OBN; ++j) ref1[j] = 0.0;                             \
                for (int64_t t = 0; t < nbk; ++t) {                                          \
                    const int64_t k0 = t * bk, kk = d - k0 < bk ? d - k0 : bk;               \
                    for (int64_t i = 0; i < mi; ++i) {                                       \
                        const T *xr = x + (i0 + i) * d;                                      \
                        T *ar = acc + i * OBN;                                               \
                        for (int64_t f = k0; f < k0 + kk; ++f) {                             \
                            const T xv = xr[f];                                              \
                            const T *br = bt + f * OBN;                                      \
                            for (int64_t j = 0; j < OBN; ++j) {                              \
                                T pr = xv * br[j];                                           \
                                ar[j] = ar[j] + pr;                                          \
                            }                                                                \
                        }                                                                    \
                    }                                                                        \
                    for (int64_t f = k0; f < k0 + kk; ++f) {                                 \
                        const double w1 = c1[f];                                             \
                        for (int64_t j = 0; j < OBN; ++j) ref1[j] += w1 * (double)bt[f * OBN + j]; \
                    }                                                                        \
                    for (int64_t j = 0; j < OBN; ++j) s1[j] = 0.0;                           \
                    int64_t i = 0;                                                           \
                    for (; i + 4 <= mi; i += 4) {                                            \
                        for (int64_t j = 0; j < OBN; ++j)                                    \
                            p[j] = (acc[i * OBN + j] + acc[(i + 1) * OBN + j]) +             \
                                   (acc[(i + 2) * OBN + j] + acc[(i + 3) * OBN + j]);        \
                        for (int64_t j = 0; j < OBN; ++j) s1[j] += (double)p[j];             \
                    }                                                                        \
                    for (; i < mi; ++i)                                                      \
                        for (int64_t j = 0; j < OBN; ++j) s1[j] += (double)acc[i * OBN + j]; \
                    const int64_t kacc = (t + 1) * bk < d ? (t + 1) * bk : d;                \
                    const double tol = tol_base * (double)kacc + J->abs_tol;                 \
                    for (int64_t j = 0; j < sn; ++j)                                         \
                        if (!(fabs(s1[j] - ref1[j]) <= tol)) J->viol += 1;                   \
                }                                                                            \
                for (int64_t i = 0; i < mi; ++i) {                                           \
                    T bv = ((T *)J->val)[i0 + i];                                            \
                    int64_t bj = J->idx[i0 + i];                                             \
                    for (int64_t j = 0; j < sn; ++j) {                                       \
                        const T a = acc[i * OBN + j];                                        \
                        const T dd = yn[s0 + j] - (a + a);                                   \
                        if (dd < bv || (dd == bv && s0 + j < bj)) { bv = dd; bj = s0 + j; }  \
                    }                                                                        \
                    ((T *)J->val)[i0 + i] = bv;                                              \
                    J->idx[i0 + i] = bj;                                                     \
                }                                                                            \
            }                                                                                \
        }                                                                                    \
    }                                                                                        \
    free(bt); free(acc); free(c1);                                                           \
    return NULL;                                                                             \
}

DEFINE_CHECKED(float, checked_f32_worker)
DEFINE_CHECKED(double, checked_f64_worker)

static int64_t run_checked(int is64, const void *x, const void *y, const void *yn, int64_t m,
                           int64_t k, int64_t d, int64_t bm, int64_t bn, int64_t bk,
                           double delta_rel, double abs_tol, int64_t *idx, void *val, int threads) {
    const int64_t nbi = (m + bm - 1) / bm, nbj = (k + bn - 1) / bn;
    double *cmax = calloc((size_t)(nbj > 0 ? nbj : 1), sizeof(double));
    for (int64_t j = 0; j < k; ++j)
        for (int64_t f = 0; f < d; ++f) {
            double v = is64 ? ((const double *)y)[j * d + f] : (double)((const float *)y)[j * d + f];
            v = v < 0.0 ? -v : v;
            if (v > cmax[j / bn]) cmax[j / bn] = v;
        }
    if (threads < 1) threads = 1;
    if (threads > MAXT) threads = MAXT;
    if (nbi < threads) threads = nbi > 0 ? (int)nbi : 1;
    pthread_t th[MAXT];
    chk_job jobs[MAXT];
    const int64_t step = (nbi + threads - 1) / threads;
    int n = 0;
    for (int64_t lo = 0; lo < nbi; lo += step, ++n) {
        chk_job J = {x, y, yn, m, k, d, bm, bn, bk, lo, lo + step < nbi ? lo + step : nbi,
                     delta_rel, abs_tol, cmax, idx, val, 0};
        jobs[n] = J;
    }
    void *(*fn)(void *) = is64 ? checked_f64_worker : checked_f32_worker;
    for (int t = 0; t < n; ++t) pthread_create(&th[t], NULL, fn, &jobs[t]);
    int64_t viol = 0;
    for (int t = 0; t < n; ++t) {
        pthread_join(th[t], NULL);
        viol += jobs[t].viol;
    }
    free(cmax);
    return viol;
}

int64_t ftko_checked_assign(int is64, const void *x, const void *y, const void *yn, int64_t m,
                            int64_t k, int64_t d, int64_t bm, int64_t bn, int64_t bk,
                            double delta_rel, double abs_tol, int64_t *idx, void *val, int threads) {
    return run_checked(is64, x, y, yn, m, k, d, bm, bn, bk, delta_rel, abs_tol, idx, val, threads);
}

/* Exact accumulator value acc[i][j] (the quantity the reference's fault hook
 * flips, _kernels.py:462-474). */
float ftko_dot_f32(const float *a, const float *b, int64_t d) {
    float s = 0.0f;
    for (int64_t k = 0; k < d; ++k) { float p = a[k] * b[k]; s = s + p; }
    return s;
}
double ftko_dot_f64(const double *a, const double *b, int64_t d) {
    double s = 0.0;
    for (int64_t k = 0; k < d; ++k) { double p = a[k] * b[k]; s = s + p; }
    return s;
}

/* --------------------------------------------------------------- update -- */
/* kmeans.py:167-171: sums[:, f] = bincount(labels, weights=x[:, f]) (f64,
 * ascending sample order); counts = bincount(labels).  Features are
 * independent, so threads split the feature range. */
typedef struct {
    const void *x;
    const int64_t *lab;
    int64_t m, d, k, f0, f1;
    double *sums;
    int is64;
} upd_job;

static void *update_worker(void *arg) {
    upd_job *J = (upd_job *)arg;
    for (int64_t i = 0; i < J->m; ++i) {
        double *row = J->sums + J->lab[i] * J->d;
        if (J->is64) {
            const double *xr = (const double *)J->x + i * J->d;
            for (int64_t f = J->f0; f < J->f1; ++f) row[f] = row[f] + xr[f];
        } else {
            const float *xr = (const float *)J->x + i * J->d;
            for (int64_t f = J->f0; f < J->f1; ++f) row[f] = row[f] + (double)xr[f];
        }
    }
    return NULL;
}

void ftko_update_sums(int is64, const void *x, const int64_t *labels, int64_t m, int64_t d,
                      int64_t k, double *sums, int64_t *counts, int threads) {
    memset(sums, 0, sizeof(double) * k * d);
    memset(counts, 0, sizeof(int64_t) * k);
    for (int64_t i = 0; i < m; ++i) counts[labels[i]] += 1;
    if (threads < 1) threads = 1;
    if (threads > MAXT) threads = MAXT;
    if (threads > d) threads = (int)d;
    pthread_t th[MAXT];
    upd_job jobs[MAXT];
    int64_t step = (d + threads - 1) / threads;
    int n = 0;
    for (int64_t f0 = 0; f0 < d; f0 += step, ++n) {
        upd_job J = {x, labels, m, d, k, f0, f0 + step < d ? f0 + step : d, sums, is64};
        jobs[n] = J;
    }
    if (n == 1) { update_worker(&jobs[0]); return; }
    for (int t = 0; t < n; ++t) pthread_create(&th[t], NULL, update_worker, &jobs[t]);
    for (int t = 0; t < n; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------- pairwise sum -- */
/* numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
 * pairwise_sum for DOUBLE; block size 128, 8 accumulators), as used by
 * float(sq_dists.sum()) in kmeans.py:275/307 and by np.linalg.norm. */
static double pairwise_strided(const double *a, int64_t n, int64_t stride) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i * stride];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j * stride];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[(i + j) * stride];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i * stride];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_strided(a, n2, stride) + pairwise_strided(a + n2 * stride, n - n2, stride);
}

double ftko_pairwise_sum(const double *a, int64_t n) { return pairwise_strided(a, n, 1); }

/* np.linalg.norm(a, axis=1) for a C-contiguous (rows, cols) f64 array:
 * sqrt(add.reduce(a*a, axis=1)) with a pairwise reduce along each row. */
void ftko_row_norms_pairwise(const double *a, int64_t rows, int64_t cols, double *out) {
    double *sq = malloc(sizeof(double) * (cols > 0 ? cols : 1));
    for (int64_t i = 0; i < rows; ++i) {
        for (int64_t j = 0; j < cols; ++j) sq[j] = a[i * cols + j] * a[i * cols + j];
        out[i] = sqrt(pairwise_strided(sq, cols, 1));
    }
    free(sq);
}
