// dscreen.cu -- float64 screened assignment (sm_100a, DFMA pipe).
//
// The reference evaluates every float64 distance as a sequential chain of
// separately rounded products and sums (_kernels.py:44-102, no FMA).  This
// path screens all K distances with fused multiply-adds -- one DFMA per MAC,
// half the instructions of the exact chain -- from a register-tiled SIMT
// GEMM with the row argmin fused into its epilogue, certifies the screened
// argmin with a rigorous error bound, and recomputes the winner's distance
// in the reference's order.  Rows the bound cannot certify (exact or
// near-exact ties, ~1e-14 relative) are resolved by the exact kernel.
//
//   |s_j - ref_j| <= A + B |s_j|,  A = 2 (3D + 2) 2^-53 |x| cmax (1 + 2^-20)
//   (FMA chain and the reference's mul+add chain, each <= (D+1) u sum|x c|),
//   B = 2^-34 (column index packed in the low 16 mantissa bits + roundings).
//
// Tile: 64 rows x 128 centroids per step, 256 threads, each thread a 4 x 8
// accumulator block (rows ty + 16 r, columns tx + 16 c), k staged through
// shared memory in chunks of 8 with register prefetch of the next chunk.
// ABFT (checked mode): the epilogue also sums each row's accumulators over
// all K; the refine compares the sum with x . (sum_j c_j) (tolerance of the
// reference's relative threshold) and sends failing rows to the exact path.

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "tc_pair.cuh"

namespace ftk {

constexpr int DS_BM = 64, DS_BN = 128, DS_KC = 8, DS_THREADS = 256;

struct DsParams {
    const double *x, *y, *yn;
    int64_t m, k, d;
    const double *cmax2;  // max_j |c_j|^2 (device scalar)
    int32_t *out_idx;
    double *out_val;
    int32_t *fb_rows;
    unsigned *fb_count;
    // checked mode
    const double *csum;   // d: sum_j c_j
    const double *camax;  // max |c|
    double tau_coef, tau_abs;
    unsigned *abft_count;
};

__device__ __forceinline__ double pack_idx(double v, uint32_t j) {
    const unsigned long long u = (static_cast<unsigned long long>(__double_as_longlong(v)) &
                                  ~0xFFFFull) | j;
    return __longlong_as_double(static_cast<long long>(u));
}

template <bool CHK>
__global__ void __launch_bounds__(DS_THREADS, 2) dscreen_kernel(DsParams P) {
    __shared__ double As[2][DS_KC][DS_BM];
    __shared__ double Bs[2][DS_KC][DS_BN];
    __shared__ double yns[DS_BN];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t nrt = (P.m + DS_BM - 1) / DS_BM;
    const int64_t nct = (P.k + DS_BN - 1) / DS_BN;
    const int nkc = int((P.d + DS_KC - 1) / DS_KC);
    for (int64_t rt = blockIdx.x; rt < nrt; rt += gridDim.x) {
        const int64_t r0 = rt * DS_BM;
        double m1[4], m2[4], rs[4];
        int t1[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            m1[i] = INFINITY;
            m2[i] = INFINITY;
            rs[i] = 0.0;
            t1[i] = 0;
        }
        for (int64_t ct = 0; ct < nct; ++ct) {
            const int64_t c0 = ct * DS_BN;
            double acc[4][8];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[i][c] = 0.0;
            // global -> register prefetch of one k-chunk: A 64x8 (2 per
            // thread), B 128x8 (4 per thread); element e -> (row e/8, k e%8)
            double pa[2], pb[4];
            auto fetch = [&](int kc) {
                const int64_t k0 = int64_t(kc) * DS_KC;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int e = tid + q * DS_THREADS, rr = e >> 3, kk = e & 7;
                    const int64_t row = r0 + rr, kcol = k0 + kk;
                    pa[q] = (row < P.m && kcol < P.d) ? __ldg(P.x + row * P.d + kcol) : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int e = tid + q * DS_THREADS, cc = e >> 3, kk = e & 7;
                    const int64_t col = c0 + cc, kcol = k0 + kk;
                    pb[q] = (col < P.k && kcol < P.d) ? __ldg(P.y + col * P.d + kcol) : 0.0;
                }
            };
            auto stash = [&](int buf) {
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int e = tid + q * DS_THREADS;
                    As[buf][e & 7][e >> 3] = pa[q];
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int e = tid + q * DS_THREADS;
                    Bs[buf][e & 7][e >> 3] = pb[q];
                }
            };
            if (tid < DS_BN) yns[tid] = (c0 + tid < P.k) ? P.yn[c0 + tid] : INFINITY;
            fetch(0);
            stash(0);
            __syncthreads();
            for (int kc = 0; kc < nkc; ++kc) {
                const int buf = kc & 1;
                if (kc + 1 < nkc) fetch(kc + 1);
#pragma unroll
                for (int kk = 0; kk < DS_KC; ++kk) {
                    double a[4], b[8];
#pragma unroll
                    for (int i = 0; i < 4; ++i) a[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
                    for (int c = 0; c < 8; ++c) b[c] = Bs[buf][kk][tx + 16 * c];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int c = 0; c < 8; ++c) acc[i][c] = fma(a[i], b[c], acc[i][c]);
                }
                if (kc + 1 < nkc) stash(buf ^ 1);
                __syncthreads();
            }
            // epilogue: screened values, per-row top-2 over this thread's 8
            // columns, then across the 16 threads of the row group
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                double a1 = INFINITY, a2 = INFINITY, ssum = 0.0;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int col = tx + 16 * c;
                    if (CHK && c0 + col < P.k) ssum += acc[i][c];
                    const double s = pack_idx(fma(-2.0, acc[i][c], yns[col]), uint32_t(col));
                    const double hi = fmax(a1, s);
                    a1 = fmin(a1, s);
                    a2 = fmin(a2, hi);
                }
#pragma unroll
                for (int off = 1; off < 16; off <<= 1) {
                    const double o1 = __shfl_xor_sync(0xffffffffu, a1, off);
                    const double o2 = __shfl_xor_sync(0xffffffffu, a2, off);
                    const double hi = fmax(a1, o1);
                    a1 = fmin(a1, o1);
                    a2 = fmin(fmin(a2, o2), hi);
                    if (CHK) ssum += __shfl_xor_sync(0xffffffffu, ssum, off);
                }
                const double hi = fmax(m1[i], a1);
                if (a1 < m1[i]) t1[i] = int(ct);
                m1[i] = fmin(m1[i], a1);
                m2[i] = fmin(fmin(m2[i], a2), hi);
                if (CHK) rs[i] += ssum;
            }
            __syncthreads();  // yns / As / Bs reuse by the next column tile
        }
        // refine: thread tx < 4 of row group ty takes row ty + 16 tx
        if (tx < 4) {
            double mm1 = m1[0], mm2 = m2[0], rsum = rs[0];
            int tt = t1[0];
#pragma unroll
            for (int i = 1; i < 4; ++i)
                if (tx == i) {
                    mm1 = m1[i];
                    mm2 = m2[i];
                    rsum = rs[i];
                    tt = t1[i];
                }
            const int64_t row = r0 + ty + 16 * tx;
            if (row < P.m) {
                bool ok = false;
                double dval = 0.0;
                int j = 0;
                if (mm1 < INFINITY) {
                    j = tt * DS_BN + int(static_cast<unsigned long long>(__double_as_longlong(mm1)) & 0xFFFFull);
                    const double *xr = P.x + row * P.d;
                    const double *cr = P.y + int64_t(j) * P.d;
                    double acc = 0.0, xx = 0.0, rref = 0.0, amax = 0.0;
                    for (int64_t f = 0; f < P.d; ++f) {
                        const double xv = __ldg(xr + f);
                        acc = __dadd_rn(acc, __dmul_rn(xv, __ldg(cr + f)));
                        xx = fma(xv, xv, xx);
                        if (CHK) {
                            rref = fma(xv, __ldg(P.csum + f), rref);
                            amax = fmax(amax, fabs(xv));
                        }
                    }
                    dval = __dsub_rn(P.yn[j], __dadd_rn(acc, acc));
                    const double xn = sqrt(xx * (1.0 + 0x1p-20));
                    const double cm = sqrt(*P.cmax2 * (1.0 + 0x1p-20));
                    const double A = 2.0 * (3.0 * double(P.d) + 2.0) * 0x1p-53 * xn * cm * (1.0 + 0x1p-20);
                    bool bad = false;
                    if (CHK) {
                        // reference tolerance + float64 evaluation error of both
                        // sides: <= (2D + K) u K |x| cmax
                        const double tau = P.tau_coef * fmax(1.0, amax * *P.camax) + P.tau_abs +
                                           2.0 * (2.0 * double(P.d) + double(P.k)) * 0x1p-53 *
                                               double(P.k) * xn * cm;
                        bad = !(fabs(rsum - rref) <= tau);
                        if (bad) atomicAdd(P.abft_count, 1u);
                    }
                    ok = !bad && isfinite(dval) && xn * cm < 1e300 &&
                         (mm2 - A - 0x1p-34 * (fabs(mm2) + fabs(mm1)) > dval);
                }
                if (ok) {
                    P.out_idx[row] = j;
                    P.out_val[row] = dval;
                } else {
                    P.fb_rows[atomicAdd(P.fb_count, 1u)] = int32_t(row);
                }
            }
        }
        __syncthreads();
    }
}

// max_j |c_j|^2 from the exact norms; checked mode: sum_j c_j and max |c|
__global__ void dprep_kernel(const double *y, const double *yn, int64_t k, int64_t d, int chk,
                             double *out /* [0] cmax2, [1] camax, [2..] csum */) {
    const int64_t f = int64_t(blockIdx.x) - 1;  // block 0: norms; block 1+f: feature f
    double s = 0.0, mx = 0.0;
    if (f < 0) {
        for (int64_t j = threadIdx.x; j < k; j += blockDim.x) s = fmax(s, yn[j]);
    } else {
        for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
            const double v = y[j * d + f];
            s += v;
            mx = fmax(mx, fabs(v));
        }
    }
    __shared__ double sh[2][32];
    for (int off = 16; off; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, s, off);
        s = f < 0 ? fmax(s, o) : s + o;
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    }
    if ((threadIdx.x & 31) == 0) {
        sh[0][threadIdx.x >> 5] = s;
        sh[1][threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = f < 0 ? 0.0 : 0.0, m = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) {
            t = f < 0 ? fmax(t, sh[0][w]) : t + sh[0][w];
            m = fmax(m, sh[1][w]);
        }
        if (f < 0) {
            out[0] = t;
        } else {
            out[2 + f] = t;
            // max |c| over features: order-free maximum via integer atomics
            atomicMax(reinterpret_cast<unsigned long long *>(out + 1),
                      static_cast<unsigned long long>(__double_as_longlong(m)));
        }
    }
    (void)chk;
}

__global__ void dgather_rows_kernel(const double *x, int64_t d, const int32_t *rows,
                                    const unsigned *count, double *g) {
    const int64_t n = int64_t(*count) * d;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x)
        g[e] = x[int64_t(rows[e / d]) * d + e % d];
}

__global__ void dscatter_rows_kernel(const int32_t *rows, const unsigned *count, const int32_t *idx,
                                     const double *val, int32_t *out_idx, double *out_val) {
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < *count;
         q += int64_t(gridDim.x) * blockDim.x) {
        out_idx[rows[q]] = idx[q];
        out_val[rows[q]] = val[q];
    }
}

int exact_run(ftk_ctx *, int, const void *, const void *, const void *, int64_t, int64_t, int64_t,
              int64_t, int64_t, int64_t, int32_t *, void *, void *, bool, double, double, int64_t,
              const ftk_injection *, ftk_events *, cudaStream_t);

static unsigned g_ds_last[2] = {0, 0};

int dscreen_run(ftk_ctx *ctx, const double *x, const double *y, const double *yn, int64_t m,
                int64_t k, int64_t d, int32_t *out_idx, double *out_val, const TcFt *ft,
                cudaStream_t st) {
    if (m <= 0) return FTK_OK;
    if (k >= 65536 || m >= (int64_t(1) << 31)) {
        set_error("dscreen: unsupported shape");
        return FTK_ERR_UNSUPPORTED;
    }
    const size_t need = sizeof(double) * size_t(d + 8) + sizeof(int32_t) * size_t(m + 1) + 64;
    char *buf = static_cast<char *>(scratch(ctx, SLOT_DS, need, st));
    if (!buf) return FTK_ERR_CUDA;
    double *prep = reinterpret_cast<double *>(buf);
    unsigned *cnt = reinterpret_cast<unsigned *>(prep + d + 4);  // [0] fallback, [1] abft
    int32_t *fb = reinterpret_cast<int32_t *>(prep + d + 6);
    FTK_CUDA(cudaMemsetAsync(prep, 0, sizeof(double) * size_t(d + 6), st));
    dprep_kernel<<<unsigned(1 + (ft ? d : 0)), 256, 0, st>>>(y, yn, k, d, ft ? 1 : 0, prep);
    FTK_LAUNCHED("dprep_kernel");
    DsParams P{};
    P.x = x; P.y = y; P.yn = yn; P.m = m; P.k = k; P.d = d;
    P.cmax2 = prep;
    P.out_idx = out_idx;
    P.out_val = out_val;
    P.fb_rows = fb;
    P.fb_count = cnt;
    if (ft) {
        P.csum = prep + 2;
        P.camax = prep + 1;
        P.tau_coef = ft->delta_rel * double(d) * std::sqrt(double(k) / 32.0);
        P.tau_abs = ft->abs_tol;
        P.abft_count = cnt + 1;
    }
    const int64_t nrt = (m + DS_BM - 1) / DS_BM;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const unsigned grid = unsigned(std::min<int64_t>(nrt, int64_t(nsm) * 2));
    if (ft) dscreen_kernel<true><<<grid, DS_THREADS, 0, st>>>(P);
    else dscreen_kernel<false><<<grid, DS_THREADS, 0, st>>>(P);
    FTK_LAUNCHED("dscreen_kernel");
    unsigned h[2] = {0, 0};
    FTK_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
    FTK_CUDA(cudaStreamSynchronize(st));
    g_ds_last[0] = h[0];
    g_ds_last[1] = h[1];
    if (h[0] > 0) {
        // exact resolution of the uncertified rows
        const unsigned n = h[0];
        double *g = static_cast<double *>(scratch(ctx, SLOT_DS_G, sizeof(double) * (size_t(n) * (d + 1)) + sizeof(int32_t) * n + 64, st));
        if (!g) return FTK_ERR_CUDA;
        double *gv = g + size_t(n) * d;
        int32_t *gi = reinterpret_cast<int32_t *>(gv + n);
        dgather_rows_kernel<<<148 * 4, 256, 0, st>>>(x, d, fb, cnt, g);
        FTK_LAUNCHED("dgather_rows_kernel");
        int rc = exact_run(ctx, FTK_F64, g, y, yn, n, k, d, 8, 256, 16, gi, gv, nullptr, false, 0.0,
                           0.0, 0, nullptr, nullptr, st);
        if (rc) return rc;
        dscatter_rows_kernel<<<148, 256, 0, st>>>(fb, cnt, gi, gv, out_idx, out_val);
        FTK_LAUNCHED("dscatter_rows_kernel");
    }
    if (ft && ft->inj && ft->inj->n > 0)
        return emulate_injected_blocks<double>(ctx, x, y, yn, m, k, d, *ft, out_idx, out_val, st);
    return FTK_OK;
}

int dscreen_last(unsigned *out) {
    out[0] = g_ds_last[0];
    out[1] = g_ds_last[1];
    return FTK_OK;
}

}  // namespace ftk
