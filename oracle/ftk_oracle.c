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
