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
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "tc_pair.cuh"

namespace ftk {

constexpr int DS_RM = 8;  // rows per thread (rows ty + 16 i)
constexpr int DS_BM = 16 * DS_RM, DS_BN = 128, DS_KC = 8, DS_THREADS = 256, DS_STAGES = 4;

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
    unsigned long long *abft_total;
};

__device__ __forceinline__ void cp_async8_zfill(void *dst, const void *src, bool ok) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(src),
                 "r"(ok ? 8 : 0)
                 : "memory");
}

__device__ __forceinline__ double pack_idx(double v, uint32_t j) {
    const unsigned long long u = (static_cast<unsigned long long>(__double_as_longlong(v)) &
                                  ~0xFFFFull) | j;
    return __longlong_as_double(static_cast<long long>(u));
}

// Exact refine + certificate of one row (shared by the DFMA and DMMA screens):
// the reference's value for the screened winner, the ABFT row check, and
// either the outputs or a fallback-list entry.
template <bool CHK>
__device__ __forceinline__ void ds_refine_row(const DsParams &P, int64_t row, double mm1,
                                              double mm2, double rsum, int tt, int bn) {
    if (row < P.m) {
        bool ok = false;
        double dval = 0.0;
        int j = 0;
        if (mm1 < INFINITY) {
            j = tt * bn + int(static_cast<unsigned long long>(__double_as_longlong(mm1)) & 0xFFFFull);
            const double *xr = P.x + row * P.d;
            const double *cr = P.y + int64_t(j) * P.d;
            double acc = 0.0, xx = 0.0, rref = 0.0, amax = 0.0;
            // 8 features per step: the loads of a step are issued together,
            // then folded in the reference's order
            int64_t f = 0;
            for (; f + 8 <= P.d; f += 8) {
                double xv[8], cv[8], sv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    xv[u] = __ldg(xr + f + u);
                    cv[u] = __ldg(cr + f + u);
                    if (CHK) sv[u] = __ldg(P.csum + f + u);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    acc = __dadd_rn(acc, __dmul_rn(xv[u], cv[u]));
                    xx = fma(xv[u], xv[u], xx);
                    if (CHK) {
                        rref = fma(xv[u], sv[u], rref);
                        amax = fmax(amax, fabs(xv[u]));
                    }
                }
            }
            for (; f < P.d; ++f) {
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
                if (bad) {
                    atomicAdd(P.abft_count, 1u);
                    if (P.abft_total) atomicAdd(P.abft_total, 1ull);
                }
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

template <bool CHK>
__global__ void __launch_bounds__(DS_THREADS, 1) dscreen_kernel(DsParams P) {
    // cp.async multistage ring: DS_STAGES k-chunks of A (64 x 8) and B (128 x 8)
    extern __shared__ __align__(16) double ds_smem[];
    double(*As)[DS_KC][DS_BM] = reinterpret_cast<double(*)[DS_KC][DS_BM]>(ds_smem);
    double(*Bs)[DS_KC][DS_BN] =
        reinterpret_cast<double(*)[DS_KC][DS_BN]>(ds_smem + DS_STAGES * DS_KC * DS_BM);
    double *yns = ds_smem + DS_STAGES * DS_KC * (DS_BM + DS_BN);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t nrt = (P.m + DS_BM - 1) / DS_BM;
    const int64_t nct = (P.k + DS_BN - 1) / DS_BN;
    const int nkc = int((P.d + DS_KC - 1) / DS_KC);
    for (int64_t rt = blockIdx.x; rt < nrt; rt += gridDim.x) {
        const int64_t r0 = rt * DS_BM;
        double m1[DS_RM], m2[DS_RM], rs[DS_RM];
        int t1[DS_RM];
#pragma unroll
        for (int i = 0; i < DS_RM; ++i) {
            m1[i] = INFINITY;
            m2[i] = INFINITY;
            rs[i] = 0.0;
            t1[i] = 0;
        }
        for (int64_t ct = 0; ct < nct; ++ct) {
            const int64_t c0 = ct * DS_BN;
            double acc[DS_RM][8];
#pragma unroll
            for (int i = 0; i < DS_RM; ++i)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[i][c] = 0.0;
            // cp.async of one k-chunk into ring slot `buf`: A 64x8 (2 per
            // thread), B 128x8 (4 per thread); element e -> (row e/8, k e%8),
            // stored k-major (transposed); out-of-range elements zero-filled
            auto issue = [&](int kc) {
                const int buf = kc % DS_STAGES;
                const int64_t k0 = int64_t(kc) * DS_KC;
                if (kc < nkc) {
#pragma unroll
                    for (int q = 0; q < DS_BM * DS_KC / DS_THREADS; ++q) {
                        const int e = tid + q * DS_THREADS, rr = e >> 3, kk = e & 7;
                        const int64_t row = r0 + rr, kcol = k0 + kk;
                        const bool ok = row < P.m && kcol < P.d;
                        cp_async8_zfill(&As[buf][kk][rr], ok ? P.x + row * P.d + kcol : P.x, ok);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int e = tid + q * DS_THREADS, cc = e >> 3, kk = e & 7;
                        const int64_t col = c0 + cc, kcol = k0 + kk;
                        const bool ok = col < P.k && kcol < P.d;
                        cp_async8_zfill(&Bs[buf][kk][cc], ok ? P.y + col * P.d + kcol : P.y, ok);
                    }
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            if (tid < DS_BN) yns[tid] = (c0 + tid < P.k) ? P.yn[c0 + tid] : INFINITY;
#pragma unroll
            for (int q = 0; q < DS_STAGES - 1; ++q) issue(q);
            for (int kc = 0; kc < nkc; ++kc) {
                asm volatile("cp.async.wait_group %0;" ::"n"(DS_STAGES - 2) : "memory");
                __syncthreads();  // chunk kc landed for everyone; slot (kc-1) is free
                issue(kc + DS_STAGES - 1);
                const int buf = kc % DS_STAGES;
#pragma unroll
                for (int kk = 0; kk < DS_KC; ++kk) {
                    double a[DS_RM], b[8];
#pragma unroll
                    for (int i = 0; i < DS_RM; ++i) a[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
                    for (int c = 0; c < 8; ++c) b[c] = Bs[buf][kk][tx + 16 * c];
#pragma unroll
                    for (int i = 0; i < DS_RM; ++i)
#pragma unroll
                        for (int c = 0; c < 8; ++c) acc[i][c] = fma(a[i], b[c], acc[i][c]);
                }
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            // epilogue: screened values, per-row top-2 over this thread's 8
            // columns, then across the 16 threads of the row group
#pragma unroll
            for (int i = 0; i < DS_RM; ++i) {
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
        // refine: thread tx < DS_RM of row group ty takes row ty + 16 tx
        if (tx < DS_RM) {
            double mm1 = m1[0], mm2 = m2[0], rsum = rs[0];
            int tt = t1[0];
#pragma unroll
            for (int i = 1; i < DS_RM; ++i)
                if (tx == i) {
                    mm1 = m1[i];
                    mm2 = m2[i];
                    rsum = rs[i];
                    tt = t1[i];
                }
            ds_refine_row<CHK>(P, r0 + ty + 16 * tx, mm1, mm2, rsum, tt, DS_BN);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ DMMA screen --
// Same screen / certify / refine scheme on the float64 tensor cores
// (mma.sync.m16n8k4.f64 -> DMMA): CTA tile 128 rows x 128 centroids, 8 warps
// of 64 x 32 (4 x 4 m16n8 tiles), k streamed in chunks of 8 through a
// cp.async ring.  A fragment: rows gid, gid + 8, column tig; B fragment:
// row tig, column gid; accumulators: rows gid / gid + 8, columns 2 tig, +1.
// The DMMA accumulates each product into the sum without intermediate
// rounding of the product (like DFMA), so the DFMA error bound holds.
// MT = m16 tiles per warp: 4 -> 128-row CTA tiles (255 registers, one CTA
// per SM); 2 -> 64-row tiles, <= 128 registers and a 3-stage ring, so two
// CTAs share an SM and one's refine / epilogue overlaps the other's DMMAs.
constexpr int DM_BN = 128, DM_KC = 16, DM_PB = DM_BN + 4;  // padded k-rows: conflict-free fragments
template <int MT> struct DmGeom {
    static constexpr int BM = 32 * MT, PA = BM + 4, STAGES = MT == 4 ? 4 : 3, MINB = MT == 4 ? 1 : 2;
    static constexpr size_t smem() {
        return sizeof(double) * (size_t(STAGES) * DM_KC * (PA + DM_PB) + DM_BN + 4 * BM * 3) +
               sizeof(int) * 4 * BM;
    }
};

__device__ __forceinline__ void dmma16x8x4(double (&c)[4], double a0, double a1, double b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ void top2_d(double s, double &t1, double &t2) {
    const double hi = fmax(t1, s);
    t1 = fmin(t1, s);
    t2 = fmin(t2, hi);
}

template <bool CHK, int MT>
__global__ void __launch_bounds__(256, DmGeom<MT>::MINB) dmma_screen_kernel(DsParams P) {
    constexpr int DM_BM = DmGeom<MT>::BM, DM_PA = DmGeom<MT>::PA, DM_STAGES = DmGeom<MT>::STAGES;
    constexpr int NR = 2 * MT;  // accumulator rows per thread (mt, half)
    extern __shared__ __align__(16) double dm_smem[];
    double(*As)[DM_KC][DM_PA] = reinterpret_cast<double(*)[DM_KC][DM_PA]>(dm_smem);
    double(*Bs)[DM_KC][DM_PB] =
        reinterpret_cast<double(*)[DM_KC][DM_PB]>(dm_smem + DM_STAGES * DM_KC * DM_PA);
    double *yns = dm_smem + DM_STAGES * DM_KC * (DM_PA + DM_PB);
    double *red = yns + DM_BN;  // [4 wn][128 rows][3]: m1, m2, rsum
    int *redt = reinterpret_cast<int *>(red + 4 * DM_BM * 3);  // [4 wn][128 rows] tile of m1
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int wm = warp & 1, wn = warp >> 1;
    const int64_t nrt = (P.m + DM_BM - 1) / DM_BM;
    const int64_t nct = (P.k + DM_BN - 1) / DM_BN;
    const int nkc = int((P.d + DM_KC - 1) / DM_KC);
    for (int64_t rt = blockIdx.x; rt < nrt; rt += gridDim.x) {
        const int64_t r0 = rt * DM_BM;
        // running per-row state for this thread's 8 rows (mt, half)
        double m1[NR], m2[NR], rs[NR];
        int t1[NR];
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            m1[i] = INFINITY;
            m2[i] = INFINITY;
            rs[i] = 0.0;
            t1[i] = 0;
        }
        for (int64_t ct = 0; ct < nct; ++ct) {
            const int64_t c0 = ct * DM_BN;
            double acc[MT][4][4];
#pragma unroll
            for (int a = 0; a < MT; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b)
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[a][b][q] = 0.0;
            auto issue = [&](int kc) {
                const int buf = kc % DM_STAGES;
                const int64_t k0 = int64_t(kc) * DM_KC;
                if (kc < nkc) {
#pragma unroll
                    for (int q = 0; q < DM_BM * DM_KC / 256; ++q) {
                        const int e = tid + q * 256, rr = e / DM_KC, kk = e % DM_KC;
                        const int64_t row = r0 + rr, kcol = k0 + kk;
                        const bool ok = row < P.m && kcol < P.d;
                        cp_async8_zfill(&As[buf][kk][rr], ok ? P.x + row * P.d + kcol : P.x, ok);
                    }
#pragma unroll
                    for (int q = 0; q < DM_BN * DM_KC / 256; ++q) {
                        const int e = tid + q * 256, cc = e / DM_KC, kk = e % DM_KC;
                        const int64_t col = c0 + cc, kcol = k0 + kk;
                        const bool ok = col < P.k && kcol < P.d;
                        cp_async8_zfill(&Bs[buf][kk][cc], ok ? P.y + col * P.d + kcol : P.y, ok);
                    }
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            if (tid < DM_BN) yns[tid] = (c0 + tid < P.k) ? P.yn[c0 + tid] : INFINITY;
#pragma unroll
            for (int q = 0; q < DM_STAGES - 1; ++q) issue(q);
            for (int kc = 0; kc < nkc; ++kc) {
                asm volatile("cp.async.wait_group %0;" ::"n"(DM_STAGES - 2) : "memory");
                __syncthreads();
                issue(kc + DM_STAGES - 1);
                const int buf = kc % DM_STAGES;
#pragma unroll
                for (int ks = 0; ks < DM_KC / 4; ++ks) {
                    const int kr = ks * 4 + tig;
                    double a0[MT], a1[MT], b0[4];
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        a0[mt] = As[buf][kr][wm * (16 * MT) + mt * 16 + gid];
                        a1[mt] = As[buf][kr][wm * (16 * MT) + mt * 16 + gid + 8];
                    }
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) b0[nt] = Bs[buf][kr][wn * 32 + nt * 8 + gid];
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) dmma16x8x4(acc[mt][nt], a0[mt], a1[mt], b0[nt]);
                }
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            // epilogue: per row, top-2 over this thread's 8 columns, then over
            // the 4 lanes (tig) sharing the row -> the warp's 32-column strip
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double a1v = INFINITY, a2v = INFINITY, ssum = 0.0;
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int col = wn * 32 + nt * 8 + 2 * tig + e;
                            const double v = acc[mt][nt][2 * h + e];
                            if (CHK && c0 + col < P.k) ssum += v;
                            top2_d(pack_idx(fma(-2.0, v, yns[col]), uint32_t(col)), a1v, a2v);
                        }
#pragma unroll
                    for (int off = 1; off < 4; off <<= 1) {
                        const double o1 = __shfl_xor_sync(0xffffffffu, a1v, off);
                        const double o2 = __shfl_xor_sync(0xffffffffu, a2v, off);
                        const double hi = fmax(a1v, o1);
                        a1v = fmin(a1v, o1);
                        a2v = fmin(fmin(a2v, o2), hi);
                        if (CHK) ssum += __shfl_xor_sync(0xffffffffu, ssum, off);
                    }
                    const int i = mt * 2 + h;
                    const double hi = fmax(m1[i], a1v);
                    if (a1v < m1[i]) t1[i] = int(ct);
                    m1[i] = fmin(m1[i], a1v);
                    m2[i] = fmin(fmin(m2[i], a2v), hi);
                    if (CHK) rs[i] += ssum;
                }
            __syncthreads();  // yns / ring reuse by the next column tile
        }
        // merge the 4 column-strip warps of every row through shared memory
        if (tig == 0) {
#pragma unroll
            for (int i = 0; i < NR; ++i) {
                const int rr = wm * (16 * MT) + (i >> 1) * 16 + gid + (i & 1) * 8;
                double *q = red + (wn * DM_BM + rr) * 3;
                q[0] = m1[i];
                q[1] = m2[i];
                q[2] = rs[i];
                redt[wn * DM_BM + rr] = t1[i];
            }
        }
        __syncthreads();
        if (tid < DM_BM) {
            double mm1 = INFINITY, mm2 = INFINITY, rsum = 0.0;
            int tt = 0;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const double *q = red + (w * DM_BM + tid) * 3;
                const double hi = fmax(mm1, q[0]);
                // tie on the packed value: same column strip position in different
                // strips cannot tie (the packed column differs)
                if (q[0] < mm1) tt = redt[w * DM_BM + tid];
                mm1 = fmin(mm1, q[0]);
                mm2 = fmin(fmin(mm2, q[1]), hi);
                rsum += q[2];
            }
            ds_refine_row<CHK>(P, r0 + tid, mm1, mm2, rsum, tt, DM_BN);
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
        P.abft_total = abft_total_ptr(ctx, st);
    }
    const int64_t nrt = (m + DS_BM - 1) / DS_BM;
    int nsm = 148;
    nsm = current_sm_count();
    const unsigned grid = unsigned(std::min<int64_t>(nrt, int64_t(nsm)));
    const char *se = getenv("FTK_F64_SIMT");
    if (ctx->family == 4 || (ctx->family != 3 && se && atoi(se))) {  // DFMA SIMT screen
        const size_t smem = sizeof(double) * (DS_STAGES * DS_KC * (DS_BM + DS_BN) + DS_BN);
        auto kern = ft ? dscreen_kernel<true> : dscreen_kernel<false>;
        FTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<grid, DS_THREADS, smem, st>>>(P);
    } else {
        const char *mte = getenv("FTK_DMMA_MT");  // A/B knob: 4 = one 128-row CTA per SM
        const bool big = mte && atoi(mte) == 4;
        const int bm = big ? DmGeom<4>::BM : DmGeom<2>::BM;
        const size_t smem = big ? DmGeom<4>::smem() : DmGeom<2>::smem();
        const int64_t nrt2 = (m + bm - 1) / bm;
        const int per_sm = big ? 1 : 2;
        const unsigned grid2 = unsigned(std::min<int64_t>(nrt2, int64_t(nsm) * per_sm));
        auto kern = big ? (ft ? dmma_screen_kernel<true, 4> : dmma_screen_kernel<false, 4>)
                        : (ft ? dmma_screen_kernel<true, 2> : dmma_screen_kernel<false, 2>);
        FTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<grid2, 256, smem, st>>>(P);
    }
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
