// exact.cu -- SIMT assignment / GEMM kernels that evaluate every accumulator
// in the reference's exact floating-point order (sm_100a).
//
// Compiled with --fmad=false: every product and sum is a separate IEEE
// rounding, k ascending from 0.0, exactly like the reference's numba tile
// kernels (_kernels.py:44-70; no FMA, SURVEY.md App. B probe 2).  One CTA owns
// one LOGICAL row block (TileConfig.block rows) and sweeps every logical
// column block, so the fault grid, tile-local coordinates, checksum tolerance
// and event records are the reference's own (_kernels.py:479-612).  Thread
// (r, j) owns column j of the tile and TM consecutive rows, which makes the
// e1 column checksum of _checked_range a per-thread quantity.
//
// This is the parity path: labels, min_dists, corrected values, events and
// deltas are bit-identical to the reference.  It also serves rows the tensor
// core screen cannot certify (tc.cu).

#include <cfloat>

#include <algorithm>

#include "common.cuh"

namespace ftk {

constexpr int KC = 16;  // k-chunk staged in shared memory per step

struct ExactParams {
    const void *x, *y, *yn;
    int64_t m, k, d, bm, bn, bk;
    int64_t prow;  // physical rows per CTA (== bm in checked mode)
    int pb;  // physical tile width (live columns of a logical column block)
    int32_t *out_idx;
    void *out_val;
    void *out_mat;  // materialise x @ y.T when non-null
    // checked mode
    double delta_rel, abs_tol;
    int64_t iteration;
    const double *bmax;  // per logical column block: max |y| over its rows
    // injection (faults.py:261-277 arrays, device)
    int64_t n_inj;
    const int64_t *n_inj_dev;  // live count on the device (n_inj = capacity), or null
    const int64_t *m_dev;      // live rows on the device (m = capacity), or null
    const int64_t *ibi, *ibj, *iei, *iej, *ibit;
    int64_t *iapplied;
    double *ibefore, *iafter;
    // column-split grid (gridDim.y > 1): per-(row, split) argmin partials,
    // merged by exact_split_merge_kernel
    void *part_v;
    int32_t *part_j;
    // events (abft.py:281-294)
    int64_t ev_cap;
    int64_t *ev_rec;
    double *ev_delta;
    unsigned long long *ev_count;
};

struct SmemLayout {
    size_t xs, cs, c1, tile, diag, red, total;
};

template <typename T>
__host__ __device__ static SmemLayout smem_layout(int64_t bm, int pb, int64_t bk, bool checked, bool mat) {
    SmemLayout L{};
    size_t off = 0;
#define take(bytes) (off += (((bytes) + 15) & ~size_t(15)), off - (((bytes) + 15) & ~size_t(15)))
    L.xs = take(sizeof(T) * KC * bm);
    L.cs = take(sizeof(T) * pb * (KC + 1));
    L.c1 = take(sizeof(double) * KC);
    L.tile = (checked || mat) ? take(sizeof(T) * bm * (pb + 1)) : 0;
    // diag: s1 ref1 s2 ref2 (pb each), t1 t2 r1 r2 (bm each), rs1 rs2 c2 (bk each), ints
    L.diag = checked ? take(sizeof(double) * (4 * pb + 4 * bm + 3 * bk) + 64) : 0;
    size_t red = (sizeof(T) + sizeof(int32_t)) * bm * ((pb + 31) / 32 + 1) + 64;
    L.red = take(red > 512 ? red : 512);
#undef take
    L.total = off;
    return L;
}

// ------------------------------------------------------ block reductions --
__device__ __forceinline__ int block_sum_int(int v, int *sh) {
    __syncthreads();
    if (threadIdx.x == 0) *sh = 0;
    __syncthreads();
    if (v) atomicAdd(sh, v);
    __syncthreads();
    int r = *sh;
    __syncthreads();
    return r;
}

// ------------------------------------------------ diagnose (rare path) --
// Restates _diagnose (_kernels.py:321-405) and _recheck (298-317) with the
// block cooperating where the reference's loops are independent and a
// single thread where they are sequential.  `tile` holds the tile in dtype,
// row stride ts.  Returns kind (0 corrected, 1 uncorrectable) via smem ints.
template <typename T>
__device__ void diagnose(const ExactParams &P, T *tile, int ts, double *s1, double *ref1,
                         double *s2, double *ref2, double *t1, double *t2, double *r1,
                         double *r2, double *rs1, double *rs2, double *c2, int *ints,
                         int64_t i0, int mi, int64_t j0, int nj, int64_t t_last, double tol,
                         double *out_delta, T *Xs, T *Cs, int64_t xs_stride) {
    const T *a = static_cast<const T *>(P.x);
    const T *b = static_cast<const T *>(P.y);
    const int64_t kdim = P.d;
    const int64_t bk = P.bk;
    const int tid = threadIdx.x, nth = blockDim.x;

    // _tile_colsums_w / _tile_rowsums
    for (int j = tid; j < nj; j += nth) {
        double s = 0.0;
        for (int i = 0; i < mi; ++i) s = add_rn(s, mul_rn(double(i + 1), double(tile[i * ts + j])));
        s2[j] = s;
    }
    for (int i = tid; i < mi; i += nth) {
        double a1 = 0.0, a2 = 0.0;
        for (int j = 0; j < nj; ++j) {
            double v = double(tile[i * ts + j]);
            a1 = add_rn(a1, v);
            a2 = add_rn(a2, mul_rn(double(j + 1), v));
        }
        t1[i] = a1;
        t2[i] = a2;
        r1[i] = 0.0;
        r2[i] = 0.0;
    }
    for (int j = tid; j < nj; j += nth) ref2[j] = 0.0;
    __syncthreads();
    // _row_refs_replay and _col_ref2_replay, interval by interval
    for (int64_t tt = 0; tt <= t_last; ++tt) {
        int64_t k0 = tt * bk;
        int kk = int(bk < kdim - k0 ? bk : kdim - k0);
        // the interval's operand panels, staged in the (now idle) k-chunk
        // buffers: the sequential sums below then read shared memory instead
        // of strided global loads (same values, same order)
        const bool staged = kk <= KC;
        if (staged) {
            __syncthreads();
            for (int e = tid; e < mi * kk; e += nth) {
                const int i = e / kk, k = e % kk;
                Xs[k * xs_stride + i] = a[(i0 + i) * kdim + k0 + k];
            }
            for (int e = tid; e < nj * kk; e += nth) {
                const int j = e / kk, k = e % kk;
                Cs[j * (KC + 1) + k] = b[(j0 + j) * kdim + k0 + k];
            }
            __syncthreads();
        }
        auto A_ = [&](int i, int k) {
            return double(staged ? Xs[k * xs_stride + i] : a[(i0 + i) * kdim + k0 + k]);
        };
        auto B_ = [&](int j, int k) {
            return double(staged ? Cs[j * (KC + 1) + k] : b[(j0 + j) * kdim + k0 + k]);
        };
        for (int k = tid; k < kk; k += nth) {
            double a1 = 0.0, a2 = 0.0;
            for (int j = 0; j < nj; ++j) {
                double v = B_(j, k);
                a1 = add_rn(a1, v);
                a2 = add_rn(a2, mul_rn(double(j + 1), v));
            }
            rs1[k] = a1;
            rs2[k] = a2;
            double c = 0.0;
            for (int i = 0; i < mi; ++i) c = add_rn(c, mul_rn(double(i + 1), A_(i, k)));
            c2[k] = c;
        }
        __syncthreads();
        for (int i = tid; i < mi; i += nth) {
            double a1 = 0.0, a2 = 0.0;
            for (int k = 0; k < kk; ++k) {
                double v = A_(i, k);
                a1 = add_rn(a1, mul_rn(v, rs1[k]));
                a2 = add_rn(a2, mul_rn(v, rs2[k]));
            }
            r1[i] = add_rn(r1[i], a1);
            r2[i] = add_rn(r2[i], a2);
        }
        for (int j = tid; j < nj; j += nth) {
            double s = ref2[j];
            for (int k = 0; k < kk; ++k) s = add_rn(s, mul_rn(c2[k], B_(j, k)));
            ref2[j] = s;
        }
        __syncthreads();
    }
    // _count_viol on columns and rows: count + first index
    if (tid == 0) {
        ints[0] = 0; ints[1] = 0x7fffffff; ints[2] = 0; ints[3] = 0x7fffffff;
    }
    __syncthreads();
    for (int j = tid; j < nj; j += nth) {
        double dd = s1[j] - ref1[j];
        if (!(fabs(dd) <= tol)) { atomicAdd(&ints[0], 1); atomicMin(&ints[1], j); }
    }
    for (int i = tid; i < mi; i += nth) {
        double dd = t1[i] - r1[i];
        if (!(fabs(dd) <= tol)) { atomicAdd(&ints[2], 1); atomicMin(&ints[3], i); }
    }
    __syncthreads();
    // scalar decision logic (thread 0), result in ints[4..6]
    if (tid == 0) {
        int ncv = ints[0], jhat = ncv ? ints[1] : -1;
        int nrv = ints[2], ihat = nrv ? ints[3] : -1;
        int kind = -1;
        double delta = 0.0;
        auto saturate = [](double v) {
            if (isnan(v)) return DBL_MAX;
            if (v > DBL_MAX) return DBL_MAX;
            if (v < -DBL_MAX) return -DBL_MAX;
            return v;
        };
        if (ncv == 1 && nrv == 0) {
            double dq1 = s1[jhat] - ref1[jhat];
            double dq2 = s2[jhat] - ref2[jhat];
            if (isfinite(dq1) && isfinite(dq2) && dq1 != 0.0) {
                double q = floor(dq2 / dq1 + 0.5);
                long long ri = (q >= -9.0e18 && q <= 9.0e18) ? (long long)q : LLONG_MIN;
                if (ri >= 1 && ri <= mi) { ihat = int(ri - 1); nrv = 1; }
            }
        }
        if (ncv != 1 || nrv != 1) {
            double dd = jhat >= 0 ? s1[jhat] - ref1[jhat] : 0.0;
            kind = 1;
            delta = saturate(dd);
        } else {
            double dc1 = s1[jhat] - ref1[jhat];
            double dc2 = s2[jhat] - ref2[jhat];
            double dr1 = t1[ihat] - r1[ihat];
            double dr2 = t2[ihat] - r2[ihat];
            if (isfinite(dc1) && isfinite(dc2) && isfinite(dr1) && isfinite(dr2)) {
                double lim = 0.05 * fabs(dc1);
                if (!(fabs(dc1 - dr1) <= (tol > lim ? tol : lim))) {
                    kind = 1;
                    delta = saturate(dc1);
                } else if (fabs(dc1) > 32.0 * tol) {
                    double qi = dc2 / dc1, qj = dr2 / dr1;
                    double fi = floor(qi + 0.5), fj = floor(qj + 0.5);
                    long long ri = (fi >= -9.0e18 && fi <= 9.0e18) ? (long long)fi : LLONG_MIN;
                    long long rj = (fj >= -9.0e18 && fj <= 9.0e18) ? (long long)fj : LLONG_MIN;
                    if (fabs(qi - double(ri)) > 0.05 || fabs(qj - double(rj)) > 0.05 || ri < 1 ||
                        ri > mi || rj < 1 || rj > nj || ri - 1 != ihat || rj - 1 != jhat) {
                        kind = 1;
                        delta = saturate(dc1);
                    }
                }
                if (kind < 0) delta = dc1;
            } else {
                delta = saturate(dc1);
            }
            if (kind < 0) {
                // acc[ihat, jhat] = ref1[jhat] - sum_{i != ihat} acc[i, jhat]
                double other = 0.0;
                for (int i = 0; i < mi; ++i)
                    if (i != ihat) other = add_rn(other, double(tile[i * ts + jhat]));
                tile[ihat * ts + jhat] = T(ref1[jhat] - other);
                kind = 2;  // pending recheck
            }
        }
        ints[4] = kind;
        ints[5] = ihat;
        ints[6] = jhat;
        *out_delta = delta;
        ints[7] = 0;  // recheck failures
    }
    __syncthreads();
    if (ints[4] == 2) {
        // _recheck: all four checksums of the corrected tile
        for (int j = tid; j < nj; j += nth) {
            double s = 0.0;
            int i = 0;
            for (; i + 4 <= mi; i += 4) {
                T p = add_rn(add_rn(tile[i * ts + j], tile[(i + 1) * ts + j]),
                             add_rn(tile[(i + 2) * ts + j], tile[(i + 3) * ts + j]));
                s = add_rn(s, double(p));
            }
            for (; i < mi; ++i) s = add_rn(s, double(tile[i * ts + j]));
            double w = 0.0;
            for (int ii = 0; ii < mi; ++ii)
                w = add_rn(w, mul_rn(double(ii + 1), double(tile[ii * ts + j])));
            if (!(fabs(s - ref1[j]) <= tol)) atomicAdd(&ints[7], 1);
            if (!(fabs(w - ref2[j]) <= tol * nj)) atomicAdd(&ints[7], 1);
        }
        for (int i = tid; i < mi; i += nth) {
            double a1 = 0.0, a2 = 0.0;
            for (int j = 0; j < nj; ++j) {
                double v = double(tile[i * ts + j]);
                a1 = add_rn(a1, v);
                a2 = add_rn(a2, mul_rn(double(j + 1), v));
            }
            if (!(fabs(a1 - r1[i]) <= tol)) atomicAdd(&ints[7], 1);
            if (!(fabs(a2 - r2[i]) <= tol * mi)) atomicAdd(&ints[7], 1);
        }
        __syncthreads();
        if (tid == 0) ints[4] = ints[7] ? 1 : 0;
        __syncthreads();
    }
}

// ------------------------------------------------------------ kernel --
__host__ __device__ constexpr int exact_max_threads(int tm) {
    return tm <= 4 ? 1024 : (tm == 8 ? 512 : 256);
}

template <typename T, int TM, bool CHECKED>
__global__ void __launch_bounds__(exact_max_threads(TM)) exact_tile_kernel(ExactParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int pb = P.pb;
    const int64_t bm = P.prow, lbm = P.bm, bn = P.bn, kdim = P.d;  // bm: physical rows
    const SmemLayout L = smem_layout<T>(bm, pb, P.bk, CHECKED, P.out_mat != nullptr);
    T *Xs = reinterpret_cast<T *>(smem + L.xs);
    T *Cs = reinterpret_cast<T *>(smem + L.cs);
    double *c1s = reinterpret_cast<double *>(smem + L.c1);
    T *tile = reinterpret_cast<T *>(smem + L.tile);
    const int ts = pb + 1;

    const T *x = static_cast<const T *>(P.x);
    const T *y = static_cast<const T *>(P.y);
    const T *yn = static_cast<const T *>(P.yn);

    const int tid = threadIdx.x, nth = blockDim.x;
    const int jl = tid % pb;   // column within the tile
    const int r = tid / pb;    // row group (r >= bm / TM: padding thread)
    const bool real_row_group = r * TM < bm;
    const int64_t bi = blockIdx.x;
    const int64_t i0 = bi * bm;
    const int64_t m_all = P.m_dev ? *P.m_dev : P.m;
    if (i0 >= m_all) return;  // device row count: whole CTA idle (before any barrier)
    const int mi = int(bm < m_all - i0 ? bm : m_all - i0);
    const int64_t n_inj = P.n_inj_dev ? (*P.n_inj_dev < P.n_inj ? *P.n_inj_dev : P.n_inj) : P.n_inj;
    const int64_t nbj = (P.k + bn - 1) / bn;
    const int64_t nbk = (kdim + P.bk - 1) / P.bk;

    T bestv[TM];
    int32_t bestj[TM];
#pragma unroll
    for (int t = 0; t < TM; ++t) {
        bestv[t] = T(INFINITY);
        bestj[t] = 0;
    }

    // checked-mode per-row-block quantity: amax over the row block (all D)
    double amax_a = 0.0;
    if (CHECKED) {
        double am = 0.0;
        for (int64_t e = tid; e < int64_t(mi) * kdim; e += nth) {
            double v = double(x[i0 * kdim + e]);
            double av = v < 0.0 ? -v : v;
            am = av > am ? av : am;
        }
        // block max
        for (int off = 16; off; off >>= 1) {
            double o = __shfl_xor_sync(0xffffffffu, am, off);
            am = o > am ? o : am;
        }
        double *red = reinterpret_cast<double *>(smem + L.red);
        __syncthreads();
        if ((tid & 31) == 0) red[tid >> 5] = am;
        __syncthreads();
        if (tid == 0) {
            double mm = 0.0;
            for (int w = 0; w < (nth + 31) / 32; ++w) mm = red[w] > mm ? red[w] : mm;
            red[0] = mm;
        }
        __syncthreads();
        amax_a = red[0];
        __syncthreads();
    }

    for (int64_t bj = blockIdx.y; bj < nbj; bj += gridDim.y) {
        const int64_t j0 = bj * bn;
        const int nj = int(bn < P.k - j0 ? bn : P.k - j0);
        const bool live_col = jl < nj;
        T acc[TM];
#pragma unroll
        for (int t = 0; t < TM; ++t) acc[t] = T(0);
        double ref1 = 0.0;

        for (int64_t k0 = 0; k0 < kdim; k0 += KC) {
            const int kc = int(KC < kdim - k0 ? KC : kdim - k0);
            __syncthreads();
            // stage X tile (transposed, k-major) and the centroid panel
            for (int e = tid; e < mi * KC; e += nth) {
                int i = e / KC, kk = e % KC;
                Xs[kk * bm + i] = kk < kc ? x[(i0 + i) * kdim + k0 + kk] : T(0);
            }
            for (int e = tid; e < pb * KC; e += nth) {
                int j = e / KC, kk = e % KC;
                Cs[j * (KC + 1) + kk] = (j < nj && kk < kc) ? y[(j0 + j) * kdim + k0 + kk] : T(0);
            }
            __syncthreads();
            if (CHECKED) {
                // e1 column encoding of the row block (_encode_c1_amax)
                for (int kk = tid; kk < kc; kk += nth) {
                    double s = 0.0;
                    for (int i = 0; i < mi; ++i) s = add_rn(s, double(Xs[kk * bm + i]));
                    c1s[kk] = s;
                }
                __syncthreads();
            }
            const T *xr = Xs + r * TM;
            const T *cr = Cs + jl * (KC + 1);
            for (int kk = 0; kk < (real_row_group ? kc : 0); ++kk) {  // padding threads: no reads
                const T cv = cr[kk];
                const T *xk = xr + kk * bm;
#pragma unroll
                for (int t = 0; t < TM; ++t) acc[t] = add_rn(acc[t], mul_rn(xk[t], cv));
                if (CHECKED) ref1 = add_rn(ref1, mul_rn(c1s[kk], double(cv)));
            }
        }

        // scheduled flips on the accumulator after the last k-interval
        // (_kernels.py:462-474 / 568-583)
        if (n_inj > 0 && live_col) {
            for (int64_t q = 0; q < n_inj; ++q) {
                if (P.ibj[q] != bj) continue;
                int64_t ei = P.iei[q], ej = P.iej[q];
                // logical tile (bi, bj) cell (ei, ej) -> global row; live cells only
                int64_t grow = P.ibi[q] * lbm + ei;
                if (ej != jl || ej >= nj || ei >= lbm || grow >= m_all) continue;
                int64_t lrow = grow - i0;  // row within this CTA
                if (lrow < 0 || lrow >= mi) continue;
#pragma unroll
                for (int t = 0; t < TM; ++t) {
                    if (r * TM + t == lrow) {
                        T before = acc[t];
                        T after = flip_bit(before, P.ibit[q]);
                        acc[t] = after;
                        P.iapplied[q] = 1;
                        P.ibefore[q] = double(before);
                        P.iafter[q] = double(after);
                    }
                }
            }
        }

        if (CHECKED || P.out_mat) {
            __syncthreads();
#pragma unroll
            for (int t = 0; t < TM; ++t)
                if (r * TM + t < mi) tile[(r * TM + t) * ts + jl] = acc[t];
            __syncthreads();
        }

        if (CHECKED) {
            double *dg = reinterpret_cast<double *>(smem + L.diag);
            double *s1 = dg, *rf1 = dg + pb, *s2 = dg + 2 * pb, *rf2 = dg + 3 * pb;
            double *t1 = dg + 4 * pb, *t2 = t1 + bm, *r1 = t2 + bm, *r2 = r1 + bm;
            double *rs1 = r2 + bm, *rs2 = rs1 + P.bk, *c2 = rs2 + P.bk;
            int *ints = reinterpret_cast<int *>(c2 + P.bk);
            double scale = amax_a * P.bmax[bj];
            if (scale < 1.0) scale = 1.0;
            const double tol_base = P.delta_rel * scale;
            const double tol = tol_base * double(kdim) + P.abs_tol;
            int viol = 0;
            if (r == 0 && live_col) {
                // _tile_colsums: 4-row pre-reduce in dtype, then float64
                double s = 0.0;
                int i = 0;
                for (; i + 4 <= mi; i += 4) {
                    T p = add_rn(add_rn(tile[i * ts + jl], tile[(i + 1) * ts + jl]),
                                 add_rn(tile[(i + 2) * ts + jl], tile[(i + 3) * ts + jl]));
                    s = add_rn(s, double(p));
                }
                for (; i < mi; ++i) s = add_rn(s, double(tile[i * ts + jl]));
                s1[jl] = s;
                rf1[jl] = ref1;
                viol = !(fabs(s - ref1) <= tol);
            }
            int nviol = block_sum_int(viol, ints + 8);
            if (nviol) {
                double delta = 0.0;
                diagnose<T>(P, tile, ts, s1, rf1, s2, rf2, t1, t2, r1, r2, rs1, rs2, c2, ints,
                            i0, mi, j0, nj, nbk - 1, tol, &delta, Xs, Cs, bm);
                if (tid == 0) {
                    unsigned long long c = atomicAdd(P.ev_count, 1ull);
                    if (int64_t(c) < P.ev_cap) {
                        int64_t *rec = P.ev_rec + c * 7;
                        rec[0] = P.iteration;
                        rec[1] = bi;
                        rec[2] = bj;
                        rec[3] = ints[4];
                        rec[4] = ints[5];
                        rec[5] = ints[6];
                        rec[6] = nbk - 1;
                        P.ev_delta[c] = delta;
                    }
                }
                __syncthreads();
            }
            // reload (possibly corrected) values
#pragma unroll
            for (int t = 0; t < TM; ++t)
                if (r * TM + t < mi) acc[t] = tile[(r * TM + t) * ts + jl];
        }

        if (P.out_mat) {
            T *out = static_cast<T *>(P.out_mat);
            for (int e = tid; e < mi * nj; e += nth) {
                int i = e / nj, j = e % nj;
                out[(i0 + i) * P.k + j0 + j] = tile[i * ts + j];
            }
        } else if (live_col) {
            const T ynj = yn[j0 + jl];
            const int32_t gj = int32_t(j0 + jl);
#pragma unroll
            for (int t = 0; t < TM; ++t) {
                T dd = sub_rn(ynj, add_rn(acc[t], acc[t]));
                argmin_merge(bestv[t], bestj[t], dd, gj);
            }
        }
    }

    if (P.out_mat) return;
    // cross-thread reduction of the per-thread running minima over the pb
    // threads that share each row (order-independent: a min over a total order)
    const int seg = pb < 32 ? pb : 32;
#pragma unroll
    for (int t = 0; t < TM; ++t) {
        for (int off = seg / 2; off; off >>= 1) {
            T ov = __shfl_xor_sync(0xffffffffu, bestv[t], off);
            int32_t oj = __shfl_xor_sync(0xffffffffu, bestj[t], off);
            argmin_merge(bestv[t], bestj[t], ov, oj);
        }
    }
    const int nw = (pb + 31) / 32;
    T *rv = reinterpret_cast<T *>(smem + L.red);
    int32_t *rj = reinterpret_cast<int32_t *>(rv + bm * nw);
    __syncthreads();
    if (jl % seg == 0 && real_row_group) {
        const int w = jl / 32;
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            rv[(r * TM + t) * nw + w] = bestv[t];
            rj[(r * TM + t) * nw + w] = bestj[t];
        }
    }
    __syncthreads();
    for (int i = tid; i < mi; i += nth) {
        T bv = T(INFINITY);
        int32_t bj = 0;
        for (int w = 0; w < nw; ++w) argmin_merge(bv, bj, rv[i * nw + w], rj[i * nw + w]);
        if (gridDim.y > 1) {
            const int64_t q = (i0 + i) * gridDim.y + blockIdx.y;
            static_cast<T *>(P.part_v)[q] = bv;
            P.part_j[q] = bj;
        } else {
            P.out_idx[i0 + i] = bj;
            static_cast<T *>(P.out_val)[i0 + i] = bv;
        }
    }
}

// Merge of the column-split partials: the same total order (value, then
// index; NaN never wins) as the in-CTA reduction, so the split is invisible.
template <typename T>
__global__ void exact_split_merge_kernel(const T *pv, const int32_t *pj, int gy, int64_t m,
                                         const int64_t *m_dev, int32_t *out_idx, T *out_val) {
    const int64_t mm = m_dev ? *m_dev : m;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < mm;
         i += int64_t(gridDim.x) * blockDim.x) {
        T bv = T(INFINITY);
        int32_t bj = 0;
        for (int s = 0; s < gy; ++s) argmin_merge(bv, bj, pv[i * gy + s], pj[i * gy + s]);
        out_idx[i] = bj;
        out_val[i] = bv;
    }
}

// bmax[bj] = max |y| over the rows of logical column block bj (_block_absmax)
template <typename T>
__global__ void block_absmax_kernel(const T *y, int64_t k, int64_t d, int64_t bn, double *bmax) {
    // grid (column blocks, slices): each CTA takes a slice of its block's
    // rows; the maximum of non-negative doubles is order-free, so the slices
    // merge with an integer atomicMax on the bit pattern (bmax pre-zeroed)
    int64_t bj = blockIdx.x;
    int64_t j0 = bj * bn;
    int64_t nj = bn < k - j0 ? bn : k - j0;
    const int64_t n = nj * d, per = (n + gridDim.y - 1) / gridDim.y;
    const int64_t e0 = int64_t(blockIdx.y) * per, e1 = e0 + per < n ? e0 + per : n;
    double m = 0.0;
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        double v = fabs(double(y[j0 * d + e]));
        m = v > m ? v : m;
    }
    for (int off = 16; off; off >>= 1) {
        double o = __shfl_xor_sync(0xffffffffu, m, off);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0 && m > 0.0)
        atomicMax(reinterpret_cast<unsigned long long *>(bmax + bj),
                  static_cast<unsigned long long>(__double_as_longlong(m)));
}

// _row_sq_norms: s = x0*x0; s += xj*xj, left to right in dtype
template <typename T>
__global__ void row_sq_norms_kernel(const T *x, int64_t m, int64_t n, T *out) {
    // 32 rows per block; columns staged 32 at a time through shared memory
    // (128 threads, 8 independent coalesced loads each), then each row is
    // folded left to right by its own thread: s = x0*x0; s += xj*xj
    constexpr int R = 32, C = 32;
    __shared__ T tile[R][C + 1];
    const int64_t r0 = int64_t(blockIdx.x) * R;
    const int64_t rows = m - r0 < R ? m - r0 : R;
    T s = T(0);
    for (int64_t c0 = 0; c0 < n; c0 += C) {
        const int cols = int(n - c0 < C ? n - c0 : C);
        __syncthreads();
        T v[R * C / 128];
#pragma unroll
        for (int q = 0; q < R * C / 128; ++q) {
            const int e = threadIdx.x + q * 128, rr = e / C, cc = e % C;
            v[q] = (rr < rows && cc < cols) ? x[(r0 + rr) * n + c0 + cc] : T(0);
        }
#pragma unroll
        for (int q = 0; q < R * C / 128; ++q) {
            const int e = threadIdx.x + q * 128;
            tile[e / C][e % C] = v[q];
        }
        __syncthreads();
        if (threadIdx.x < rows) {
            for (int cc = 0; cc < cols; ++cc) {
                const T w = tile[threadIdx.x][cc];
                s = (c0 == 0 && cc == 0) ? mul_rn(w, w) : add_rn(s, mul_rn(w, w));
            }
        }
    }
    if (threadIdx.x < rows) out[r0 + threadIdx.x] = s;
}

// ------------------------------------------------------------ launch --
template <typename T, int TM, bool CHECKED>
static int launch_tm(const ExactParams &P, int threads, size_t smem, cudaStream_t st) {
    auto kern = exact_tile_kernel<T, TM, CHECKED>;
    if (smem > 48 * 1024)
        FTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem)));
    int64_t nbi = (P.m + P.prow - 1) / P.prow;
    // few row blocks (replayed injected blocks, small inputs): split the
    // logical column blocks over gridDim.y so more SMs share the pass
    const int64_t nbj = (P.k + P.bn - 1) / P.bn;
    int gy = 1;
    if (P.part_v && !P.out_mat && nbj > 1 && nbi < 2 * 148)
        gy = int(std::min<int64_t>(std::min<int64_t>(nbj, (2 * 148 + nbi - 1) / nbi), 64));
    kern<<<dim3(unsigned(nbi), unsigned(gy)), dim3(threads), smem, st>>>(P);
    FTK_LAUNCHED("exact_tile_kernel");
    if (gy > 1) {
        exact_split_merge_kernel<T><<<unsigned(std::min<int64_t>((P.m + 255) / 256, 148 * 8)), 256, 0, st>>>(
            static_cast<const T *>(P.part_v), P.part_j, gy, P.m, P.m_dev, P.out_idx,
            static_cast<T *>(P.out_val));
        FTK_LAUNCHED("exact_split_merge_kernel");
    }
    return FTK_OK;
}

template <typename T, bool CHECKED>
static int launch_exact(ExactParams P, cudaStream_t st) {
    // Physical CTA rows: the whole logical row block when checksums need it
    // (checked / materialised-checked), otherwise split large logical blocks
    // into independent row slabs (unprotected rows do not interact).
    const bool f64 = sizeof(T) == 8;
    const int tm_cap = f64 ? 32 : 64;
    const bool mat = P.out_mat != nullptr;
    int64_t prow = P.bm;
    int tm = 0, threads = 0;
    for (;;) {
        tm = int(prow < (f64 ? 16 : 32) ? prow : (f64 ? 16 : 32));
        auto nthreads = [&](int t) { return int((P.pb * (prow / t) + 31) / 32 * 32); };
        while (nthreads(tm) < 128 && tm > 4) tm /= 2;
        while (nthreads(tm) > exact_max_threads(tm) && tm < tm_cap && tm < prow) tm *= 2;
        threads = nthreads(tm);  // whole warps; padding threads own no rows
        SmemLayout L = smem_layout<T>(prow, P.pb, P.bk, CHECKED, mat);
        bool fits = threads <= exact_max_threads(tm) && L.total <= 227 * 1024;
        if (fits) break;
        if (CHECKED || prow <= 1) {
            set_error("logical tile too large for the exact checked kernel");
            return FTK_ERR_UNSUPPORTED;
        }
        prow /= 2;
    }
    P.prow = prow;
    SmemLayout L = smem_layout<T>(prow, P.pb, P.bk, CHECKED, mat);
    switch (tm) {
        case 1: return launch_tm<T, 1, CHECKED>(P, threads, L.total, st);
        case 2: return launch_tm<T, 2, CHECKED>(P, threads, L.total, st);
        case 4: return launch_tm<T, 4, CHECKED>(P, threads, L.total, st);
        case 8: return launch_tm<T, 8, CHECKED>(P, threads, L.total, st);
        case 16: return launch_tm<T, 16, CHECKED>(P, threads, L.total, st);
        case 32: return launch_tm<T, 32, CHECKED>(P, threads, L.total, st);
        case 64: return launch_tm<T, 64, CHECKED>(P, threads, L.total, st);
    }
    set_error("bad tile geometry");
    return FTK_ERR_ARG;
}

int exact_run_m(ftk_ctx *ctx, int dtype, const void *x, const void *y, const void *yn, int64_t m,
                int64_t k, int64_t d, int64_t bm, int64_t bn, int64_t bk, int32_t *out_idx,
                void *out_val, void *out_mat, bool checked, double delta_rel, double abs_tol,
                int64_t iteration, const ftk_injection *inj, ftk_events *ev, cudaStream_t st,
                const int64_t *m_dev) {
    if (m <= 0) return FTK_OK;
    if (bm < 1 || bn < 1 || bk < 1 || d < 1) {
        set_error("bad tile/shape");
        return FTK_ERR_ARG;
    }
    ExactParams P{};
    P.x = x; P.y = y; P.yn = yn;
    P.m = m; P.k = k; P.d = d; P.bm = bm; P.bn = bn; P.bk = bk;
    int64_t live = bn < k ? bn : k;
    if (live < 1) live = 1;
    int64_t pb = 1;
    while (pb < live) pb *= 2;
    P.pb = int(pb);
    P.out_idx = out_idx; P.out_val = out_val; P.out_mat = out_mat;
    P.m_dev = m_dev;
    if (!out_mat && k > bn && m <= 2 * 148 * bm) {  // room for the column-split partials
        const size_t per = sizeof(double) + sizeof(int32_t);
        const int64_t nbj = (k + bn - 1) / bn;
        const int64_t splits = nbj < 64 ? nbj : 64;
        char *pb = static_cast<char *>(scratch(ctx, SLOT_EXACT_SPLIT, size_t(m) * splits * per + 64, st));
        if (!pb) return FTK_ERR_CUDA;
        P.part_v = pb;
        P.part_j = reinterpret_cast<int32_t *>(pb + size_t(m) * splits * sizeof(double));
    }
    P.delta_rel = delta_rel; P.abs_tol = abs_tol; P.iteration = iteration;
    if (inj && inj->n > 0) {
        P.n_inj = inj->n;
        P.n_inj_dev = inj->n_dev;
        P.ibi = inj->bi; P.ibj = inj->bj; P.iei = inj->ei; P.iej = inj->ej; P.ibit = inj->bit;
        P.iapplied = inj->applied; P.ibefore = inj->before; P.iafter = inj->after;
    }
    if (checked) {
        if (!ev) {
            set_error("checked mode needs an event ring");
            return FTK_ERR_ARG;
        }
        P.ev_cap = ev->cap; P.ev_rec = ev->rec; P.ev_delta = ev->delta;
        P.ev_count = reinterpret_cast<unsigned long long *>(ev->count);
        int64_t nbj = (k + bn - 1) / bn;
        double *bmax = static_cast<double *>(scratch(ctx, SLOT_BMAX, sizeof(double) * (nbj + 1), st));
        if (!bmax) return FTK_ERR_CUDA;
        if (nbj > 0) {
            FTK_CUDA(cudaMemsetAsync(bmax, 0, sizeof(double) * nbj, st));
            const int64_t per_block = std::min<int64_t>(bn, k) * d;
            const unsigned sl = unsigned(std::max<int64_t>(1, std::min<int64_t>(64, per_block / 4096)));
            if (dtype == FTK_F32)
                block_absmax_kernel<float><<<dim3(unsigned(nbj), sl), 256, 0, st>>>(
                    static_cast<const float *>(y), k, d, bn, bmax);
            else
                block_absmax_kernel<double><<<dim3(unsigned(nbj), sl), 256, 0, st>>>(
                    static_cast<const double *>(y), k, d, bn, bmax);
            FTK_LAUNCHED("block_absmax_kernel");
        }
        P.bmax = bmax;
    }
    if (dtype == FTK_F32)
        return checked ? launch_exact<float, true>(P, st) : launch_exact<float, false>(P, st);
    return checked ? launch_exact<double, true>(P, st) : launch_exact<double, false>(P, st);
}

int exact_run(ftk_ctx *ctx, int dtype, const void *x, const void *y, const void *yn, int64_t m,
              int64_t k, int64_t d, int64_t bm, int64_t bn, int64_t bk, int32_t *out_idx,
              void *out_val, void *out_mat, bool checked, double delta_rel, double abs_tol,
              int64_t iteration, const ftk_injection *inj, ftk_events *ev, cudaStream_t st) {
    return exact_run_m(ctx, dtype, x, y, yn, m, k, d, bm, bn, bk, out_idx, out_val, out_mat, checked,
                       delta_rel, abs_tol, iteration, inj, ev, st, nullptr);
}

int row_sq_norms_run(int dtype, const void *x, int64_t m, int64_t n, void *out, cudaStream_t st) {
    if (m <= 0) return FTK_OK;
    unsigned grid = unsigned((m + 31) / 32);
    if (dtype == FTK_F32)
        row_sq_norms_kernel<float><<<grid, 128, 0, st>>>(static_cast<const float *>(x), m, n,
                                                         static_cast<float *>(out));
    else
        row_sq_norms_kernel<double><<<grid, 128, 0, st>>>(static_cast<const double *>(x), m, n,
                                                          static_cast<double *>(out));
    FTK_LAUNCHED("row_sq_norms_kernel");
    return FTK_OK;
}

}  // namespace ftk
