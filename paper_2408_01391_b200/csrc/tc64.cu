// tc64.cu -- float64 assignment screened on the tf32 tensor cores.
//
// The reference evaluates float64 distances as sequential chains of
// separately rounded products and sums (_kernels.py:44-102).  Its labels only
// depend on those values through the row argmin, and Gaussian-blob data keep
// the argmin gap many orders above tf32 screening error, so the float64 path
// need not run at FP64 tensor rate (DMMA: ~36 TF/s on a B200) to be
// bit-exact: it is screened by the same CTA-pair tcgen05 kind::tf32 kernel as
// float32 data (tc_pair.cu, ~500+ TF/s) and certified in float64.
//
//   1. X32 = fp32(X) once per fit (registered with ftk_ctx_set_rows64) with
//      per-row bounds computed against the float64 rows: ||x||^2,
//      ||x - tf32(fp32(x))||^2, max|x|.  C32 / yn32 per call, with
//      max_j ||c_j||^2 and max_j ||c_j - tf32(fp32(c_j))||^2.
//   2. Screen (tc_pair.cu, F64 mode): s_j = yn32_j - 2 acc_j (fp32 TMEM).
//      |s_j - ref_j| <= A + B|s_j| with the float32 path's A plus the fp32
//      rounding of the float64 norms (2^-23 cmax^2) and the reference's own
//      float64 chain error (2 (D+2) 2^-53 |x| cmax).  Per row the kernel
//      records (j1, T = m2 - A - B|m2| - 2^-21(|m1|+|m2|)) -- and, checked,
//      verifies the row checksum against x~ . sum_j c~_j as in float32.
//   3. Refine (tc64_refine_kernel): d1 = yn_j1 - (acc + acc), acc the
//      reference's float64 chain; d1 < T proves j1 is the reference's strict
//      argmin and d1 its min_dist bits.
//   4. Rows no certificate covers (near ties, checksum flags, non-finite) go
//      to the DMMA screen (dscreen.cu), whose own leftovers go exact.
// Scheduled flips are replayed by the exact checked kernel over their logical
// row blocks (reference-identical records), like the DMMA path.

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tc_pair.cuh"

namespace ftk {

int make_tc_map(CUtensorMap *map, const float *base, int64_t rows, int64_t cols, uint32_t box_rows);
int make_f64_map(CUtensorMap *map, const double *base, int64_t rows, int64_t cols, uint32_t box_rows);
int prep_csum_run(ftk_ctx *ctx, int slot, const float *y, int64_t k, int64_t d, int nkb, int trunc,
                  float **csum, float **camax, cudaStream_t st, float **csumw);
int dscreen_run(ftk_ctx *ctx, const double *x, const double *y, const double *yn, int64_t m,
                int64_t k, int64_t d, int32_t *out_idx, double *out_val, const TcFt *ft,
                cudaStream_t st);

constexpr int T64_KB = 32;

// fp32 upper bound of a non-negative double
__device__ __forceinline__ float up32(double v) { return __double2float_ru(v * (1.0 + 0x1p-40)); }

// X32 = fp32(X) and the per-row screening bounds: one warp per group of 4
// rows, all four rows' loads in flight together (HBM-bound, one pass).
__global__ void row_info64_kernel(const double *x, int64_t m, int64_t d, float *x32, float4 *info) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i0 = w0 * 4; i0 < m; i0 += nw * 4) {
        double xx[4] = {0.0, 0.0, 0.0, 0.0}, ee[4] = {0.0, 0.0, 0.0, 0.0}, am[4] = {0.0, 0.0, 0.0, 0.0};
        for (int64_t f = lane; f < d; f += 32) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = i0 + u < m ? __ldcs(x + (i0 + u) * d + f) : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float v32 = __double2float_rn(v[u]);
                if (i0 + u < m) x32[(i0 + u) * d + f] = v32;
                const double r = v[u] - double(tf32_trunc(v32));
                xx[u] = fma(v[u], v[u], xx[u]);
                ee[u] = fma(r, r, ee[u]);
                am[u] = fmax(am[u], fabs(v[u]));
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            for (int off = 16; off; off >>= 1) {
                xx[u] += __shfl_xor_sync(0xffffffffu, xx[u], off);
                ee[u] += __shfl_xor_sync(0xffffffffu, ee[u], off);
                am[u] = fmax(am[u], __shfl_xor_sync(0xffffffffu, am[u], off));
            }
            if (lane == u && i0 + u < m) info[i0 + u] = make_float4(up32(xx[u]), up32(ee[u]), up32(am[u]), 0.0f);
        }
    }
}

// C32 = fp32(C), yn32 = fp32(yn); bounds[0] >= max_j yn_j, bounds[1] >=
// max_j ||c_j - tf32(fp32(c_j))||^2 (zeroed by the caller; non-negative
// floats order like their bit patterns).
__global__ void tc64_prep_kernel(const double *y, const double *yn, int64_t k, int64_t d, float *y32,
                                 float *yn32, float *bounds) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    float mx = 0.0f, me = 0.0f;
    for (int64_t j = w0; j < k; j += nw) {
        double e = 0.0;
        for (int64_t f = lane; f < d; f += 32) {
            const double v = y[j * d + f];
            const float v32 = __double2float_rn(v);
            y32[j * d + f] = v32;
            const double r = v - double(tf32_trunc(v32));
            e = fma(r, r, e);
        }
        for (int off = 16; off; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
        me = fmaxf(me, up32(e));
        mx = fmaxf(mx, up32(fabs(yn[j])));
        if (lane == 0) yn32[j] = __double2float_rn(yn[j]);
    }
    if (lane == 0) {
        atomicMax(reinterpret_cast<int *>(bounds), __float_as_int(mx));
        atomicMax(reinterpret_cast<int *>(bounds + 1), __float_as_int(me));
    }
}

// Outputs of one row's float64 certificate (both refine kernels): certified
// rows write the reference's (j1, d1); the rest are appended to fb with the
// pass-2 candidate threshold thr = d1 + A + 2(B + 2^-20)(|d1| + A) (screen
// units, rounded up): a centroid can beat d1 only if its screened value is
// <= thr.  Rows with no usable screen (j1 < 0, non-finite d1) get -inf.
__device__ __forceinline__ void t64_finish(int64_t row, int64_t m, int j, float T, double acc,
                                           const double *yn, const float *a64, int32_t *out_idx,
                                           double *out_val, int32_t *fb, unsigned *fb_count,
                                           float *fb_thr) {
    const int lane = threadIdx.x & 31;
    bool need = false;
    float thr = -INFINITY;
    if (row < m) {
        bool ok = false;
        double dval = 0.0;
        if (j >= 0) {
            dval = __dsub_rn(__ldg(yn + j), __dadd_rn(acc, acc));
            ok = isfinite(dval) && double(T) > dval;
        }
        if (ok) {
            out_idx[row] = j;
            out_val[row] = dval;
        } else if (j >= 0 && isfinite(dval) && a64) {
            const double A = double(__ldg(a64 + row));
            if (A >= 0.0) {
                double t = dval + A + 2.0 * (double((0x1p-14 + 0x1p-22) * 1.01) + 0x1p-20) * (fabs(dval) + A);
                t += fabs(t) * 0x1p-20;
                thr = __double2float_ru(t);
            }
        }
        need = !ok;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, need);
    if (bal) {
        unsigned b0 = 0;
        if (lane == 0) b0 = atomicAdd(fb_count, unsigned(__popc(bal)));
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (need) {
            const unsigned pos = b0 + __popc(bal & ((1u << lane) - 1u));
            fb[pos] = int32_t(row);
            if (fb_thr) fb_thr[pos] = thr;
        }
    }
}

// Certify each screened row in float64: the reference's chain for the
// winner, d1 < T.  One warp per 32-row tile, one lane per row; X streams in
// 32-feature chunks: 16-byte coalesced loads (two rows per instruction) are
// transposed through shared memory so each lane runs its row's sequential
// chain, with its winner's centroid chunk (L2-resident) loaded alongside.
// Uncertified rows are appended (warp-aggregated) to fb.
constexpr int R64_WARPS = 4, R64_LD = 34;  // row stride in doubles (16-byte aligned rows)
__global__ void __launch_bounds__(32 * R64_WARPS) tc64_refine_kernel(
    const double *x, const double *y, const double *yn, int64_t m, int64_t d, const int2 *rec,
    const float *a64, int32_t *out_idx, double *out_val, int32_t *fb, unsigned *fb_count, float *fb_thr) {
    __shared__ __align__(16) double sx[R64_WARPS][32 * R64_LD];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *s = sx[w];
    const int64_t ntile = (m + 31) / 32;
    for (int64_t tile = int64_t(blockIdx.x) * R64_WARPS + w; tile < ntile;
         tile += int64_t(gridDim.x) * R64_WARPS) {
        const int64_t r0 = tile * 32, row = r0 + lane;
        const int2 r = row < m ? rec[row] : make_int2(-1, 0);
        const int j = r.x;
        const double *cr = y + int64_t(j < 0 ? 0 : j) * d;
        double acc = 0.0;
        const int half = lane >> 4, q = lane & 15;  // x loads: row 2i + half, features 2q, 2q+1
        for (int64_t f0 = 0; f0 < d; f0 += 32) {
            const int fw = int(d - f0 < 32 ? d - f0 : 32);
            double2 xv[16], cv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int64_t rr = r0 + 2 * i + half;
                xv[i] = (rr < m && 2 * q < fw) ? __ldcs(reinterpret_cast<const double2 *>(x + rr * d + f0) + q)
                                               : make_double2(0.0, 0.0);
                cv[i] = (j >= 0 && 2 * i < fw) ? __ldg(reinterpret_cast<const double2 *>(cr + f0) + i)
                                               : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int i = 0; i < 16; ++i)
                *reinterpret_cast<double2 *>(s + (2 * i + half) * R64_LD + 2 * q) = xv[i];
            __syncwarp();
            const double *sr = s + lane * R64_LD;
            if (fw == 32) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    acc = __dadd_rn(acc, __dmul_rn(sr[2 * i], cv[i].x));
                    acc = __dadd_rn(acc, __dmul_rn(sr[2 * i + 1], cv[i].y));
                }
            } else {
                for (int f = 0; f < fw; ++f) acc = __dadd_rn(acc, __dmul_rn(sr[f], __ldg(cr + f0 + f)));
            }
            __syncwarp();  // the tile buffer is refilled by the next chunk
        }
        t64_finish(row, m, j, __int_as_float(r.y), acc, yn, a64, out_idx, out_val, fb, fb_count, fb_thr);
    }
}

// TMA-fed variant: a producer warp streams 32-row tiles of X (all d
// features, 16-double x 32-row boxes with 128-byte swizzle) into one
// shared-memory slot per consumer warp; four consumer warps take the tiles
// round-robin, one lane per row running its winner's float64 chain from the
// swizzled tile (16-byte reads, 4 wavefronts per warp) with the centroid chunk
// from L2.  The copy engine, not a warp's outstanding loads, keeps X in flight.
constexpr int RT_CONS = 4;  // consumer warps
struct RtGeom {
    int nbox;       // 16-double boxes per row (ceil(d / 16))
    int stages;     // ring depth
    size_t stage;   // bytes per stage (nbox * 4 KB)
};
// CT: the centroids live in shared memory for the whole kernel (K*D*8 <= 128
// KB, d % 16 == 0), 16-byte chunks XOR-swizzled by (row & 7) within each
// 128-byte group: the per-lane centroid reads (32 different rows per warp)
// cost a few shared-memory wavefronts instead of 32 L1 wavefronts each -- the
// gathers from L2 saturated the L1 (ncu: L1/TEX 97 %, DRAM 49 %).  One CTA
// per SM then, with NC = 6 consumer slots beside the table.
constexpr int RT_CONS_CT = 6;
constexpr int64_t RT_CT_MAX_BYTES = 128 * 1024;

template <int NC, bool CT>
__global__ void __launch_bounds__(32 * (NC + 1)) tc64_refine_tma_kernel(
    const __grid_constant__ CUtensorMap tmx, const double *y, const double *yn, int64_t m, int64_t d,
    int nbox, const int2 *rec, const float *a64, int32_t *out_idx, double *out_val, int32_t *fb,
    unsigned *fb_count, float *fb_thr, int64_t k) {
    extern __shared__ __align__(1024) unsigned char rt_raw[];
    unsigned char *smem = rt_raw + ((1024u - (smem_u32(rt_raw) & 1023u)) & 1023u);
    constexpr int stages = NC;  // slot w belongs to consumer w
    const size_t stage_bytes = size_t(nbox) * 4096;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + size_t(stages) * stage_bytes);
    uint64_t *empty = full + stages;
    unsigned char *ctab = smem + size_t(stages) * stage_bytes + 128;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntile = (m + 31) / 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    if (CT) {
        const int64_t cpr = d / 2;  // 16-byte chunks per centroid row
        const double2 *y2 = reinterpret_cast<const double2 *>(y);
        for (int64_t e = threadIdx.x; e < k * cpr; e += blockDim.x) {
            const int64_t j = e / cpr, c = e % cpr;
            const int64_t cs = (c & ~int64_t(7)) | ((c ^ j) & 7);
            *reinterpret_cast<double2 *>(ctab + (j * cpr + cs) * 16) = __ldg(y2 + e);
        }
    }
    __syncthreads();
    if (warp == NC) {
        // ----------------------------------------------------- producer --
        if (lane == 0) {
            prefetch_tmap(&tmx);
            int q = 0;
            for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x, ++q) {
                const int s = q % stages;
                mbar_wait(&empty[s], (uint32_t(q / stages) & 1u) ^ 1u);
                mbar_expect_tx(&full[s], uint32_t(stage_bytes));
                for (int b = 0; b < nbox; ++b)
                    tma_load_2d(smem + size_t(s) * stage_bytes + size_t(b) * 4096, &tmx, &full[s], b * 16,
                                int(tile * 32));
            }
        }
        return;
    }
    // ------------------------------------------------------- consumers --
    int q = warp;
    for (int64_t tile = int64_t(blockIdx.x) + int64_t(warp) * gridDim.x; tile < ntile;
         tile += int64_t(gridDim.x) * NC, q += NC) {
        const int s = q % stages;
        const int64_t row = tile * 32 + lane;
        const int2 r = row < m ? rec[row] : make_int2(-1, 0);
        const int j = r.x;
        const double *cr = y + int64_t(j < 0 ? 0 : j) * d;
        const unsigned char *crs = ctab + size_t(j < 0 ? 0 : j) * size_t(d) * 8;
        const int jsw = (j < 0 ? 0 : j) & 7;
        double cv[16];
        auto c_chunk = [&](int f0, int u) -> double2 {  // features f0 + 2u, f0 + 2u + 1 (f0 % 16 == 0)
            if (CT) return *reinterpret_cast<const double2 *>(crs + size_t(f0) * 8 + ((u ^ jsw) << 4));
            return __ldg(reinterpret_cast<const double2 *>(cr + f0) + u);
        };
        auto load_c = [&](int f0) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const bool ok = j >= 0 && f0 + 2 * u + 1 < d;
                const double2 c2 = ok ? c_chunk(f0, u) : make_double2(0.0, 0.0);
                cv[2 * u] = c2.x;
                cv[2 * u + 1] = c2.y;
            }
        };
        load_c(0);  // the first chunk's centroid values travel while the tile lands
        mbar_wait(&full[s], uint32_t(q / stages) & 1u);
        const unsigned char *tb = smem + size_t(s) * stage_bytes + lane * 128;
        const int sw = lane & 7;
        double acc = 0.0;
        for (int b = 0; b < nbox; ++b) {
            const int f0 = b * 16;
            double cn[16];
            const bool more = b + 1 < nbox;
            if (more) {  // next chunk's centroid values in flight during this chunk's chain
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const bool ok = j >= 0 && f0 + 16 + 2 * u + 1 < d;
                    const double2 c2 = ok ? c_chunk(f0 + 16, u) : make_double2(0.0, 0.0);
                    cn[2 * u] = c2.x;
                    cn[2 * u + 1] = c2.y;
                }
            }
            const unsigned char *bx = tb + size_t(b) * 4096;
            if (f0 + 16 <= d) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double2 xv = *reinterpret_cast<const double2 *>(bx + ((u ^ sw) << 4));
                    acc = __dadd_rn(acc, __dmul_rn(xv.x, cv[2 * u]));
                    acc = __dadd_rn(acc, __dmul_rn(xv.y, cv[2 * u + 1]));
                }
            } else {
                for (int f = f0; f < d; ++f) {
                    const int fc = f - f0;
                    const double xv = *reinterpret_cast<const double *>(bx + (((fc >> 1) ^ sw) << 4) + (fc & 1) * 8);
                    acc = __dadd_rn(acc, __dmul_rn(xv, __ldg(cr + f)));
                }
            }
            if (more) {
#pragma unroll
                for (int u = 0; u < 16; ++u) cv[u] = cn[u];
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        t64_finish(row, m, j, __int_as_float(r.y), acc, yn, a64, out_idx, out_val, fb, fb_count, fb_thr);
    }
}

__global__ void tc64_gather_kernel(const double *x, int64_t d, const int32_t *rows, const unsigned *count,
                                   double *g) {
    const int64_t n = int64_t(*count) * d;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x)
        g[e] = x[int64_t(rows[e / d]) * d + e % d];
}

__global__ void tc64_scatter_kernel(const int32_t *rows, const unsigned *count, const int32_t *idx,
                                    const double *val, int32_t *out_idx, double *out_val) {
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < *count;
         q += int64_t(gridDim.x) * blockDim.x) {
        out_idx[rows[q]] = idx[q];
        out_val[rows[q]] = val[q];
    }
}

// ---------------------------------------------- pass 2 (candidates) -----
// The rows the float64 certificate left open: their fp32 rows are re-screened
// (CTA-pair COLLECT mode) against their own threshold, and every centroid
// that can still beat the row's exact d1 is evaluated in float64 in the
// reference's order; the row's result is the smallest value, then the
// smallest index (the reference's first strict minimum).
__device__ __forceinline__ unsigned long long ord64(double v) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v));
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord64(unsigned long long k) {
    const unsigned long long u = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double(static_cast<long long>(u));
}

__global__ void t64p2_gather_kernel(const float *x32, int64_t d, const int32_t *rows, const unsigned *count,
                                    float *g, unsigned *row_cnt, unsigned long long *key, int32_t *kidx) {
    const unsigned n = *count;
    const int64_t tot = int64_t(n) * d;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t q = e / d, f = e % d;
        g[e] = x32[int64_t(rows[q]) * d + f];
        if (f == 0) {
            row_cnt[q] = 0u;
            key[q] = ~0ull;
            kidx[q] = 0x7FFFFFFF;
        }
    }
}

// one thread per candidate (gathered row q, centroid j): the exact value
__global__ void t64p2_value_kernel(const double *x, const double *y, const double *yn, int64_t d,
                                   const int32_t *rows, const int2 *cand, const unsigned *count, unsigned cap,
                                   const unsigned *row_cnt, unsigned row_cap, double *cval,
                                   unsigned long long *key) {
    const unsigned n = min(*count, cap);
    for (unsigned c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        const int2 e = cand[c];
        if (row_cnt[e.x] > row_cap) continue;
        const double *xr = x + int64_t(rows[e.x]) * d;
        const double *cr = y + int64_t(e.y) * d;
        double acc = 0.0;
        int64_t f = 0;
        if ((d & 1) == 0) {
            const double2 *x2 = reinterpret_cast<const double2 *>(xr);
            const double2 *c2 = reinterpret_cast<const double2 *>(cr);
            for (; f < d / 2; ++f) {
                const double2 a = __ldg(x2 + f), b = __ldg(c2 + f);
                acc = __dadd_rn(acc, __dmul_rn(a.x, b.x));
                acc = __dadd_rn(acc, __dmul_rn(a.y, b.y));
            }
        } else {
            for (; f < d; ++f) acc = __dadd_rn(acc, __dmul_rn(__ldg(xr + f), __ldg(cr + f)));
        }
        const double v = __dsub_rn(__ldg(yn + e.y), __dadd_rn(acc, acc));
        cval[c] = v;
        if (v < INFINITY) atomicMin(key + e.x, ord64(v));
    }
}

// the smallest index among the candidates holding the row's minimum
__global__ void t64p2_index_kernel(const int2 *cand, const unsigned *count, unsigned cap, const unsigned *row_cnt,
                                   unsigned row_cap, const double *cval, const unsigned long long *key,
                                   int32_t *kidx) {
    const unsigned n = min(*count, cap);
    for (unsigned c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        const int2 e = cand[c];
        if (row_cnt[e.x] > row_cap) continue;
        const double v = cval[c];
        if (v < INFINITY && ord64(v) == key[e.x]) atomicMin(kidx + e.x, e.y);
    }
}

// resolved rows write their outputs; the rest (no screen, too many
// candidates, list overflow) go on to the DMMA screen
__global__ void t64p2_finalize_kernel(const int32_t *rows, const unsigned *n_rows, const unsigned *row_cnt,
                                      unsigned row_cap, const unsigned *count, unsigned cap,
                                      const unsigned long long *key, const int32_t *kidx, int32_t *out_idx,
                                      double *out_val, int32_t *rows2, unsigned *n2) {
    const unsigned n = *n_rows;
    const bool over = *count > cap;
    for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int32_t row = rows[q];
        if (over || row_cnt[q] > row_cap || key[q] == ~0ull) {
            rows2[atomicAdd(n2, 1u)] = row;
            continue;
        }
        out_idx[row] = kidx[q];
        out_val[row] = unord64(key[q]);
    }
}

bool tc64_supported(int64_t m, int64_t k, int64_t d) {
    return m >= 1 && k >= 1 && k < 65536 && d >= 4 && d <= 256 && d % 4 == 0 &&
           m < (int64_t(1) << 31);
}

int row_info64_run(const double *x, int64_t m, int64_t d, float *x32, float *info, cudaStream_t st) {
    if (m == 0) return FTK_OK;
    const int64_t blocks = std::min<int64_t>((m + 31) / 32, 148 * 8);
    row_info64_kernel<<<unsigned(blocks), 256, 0, st>>>(x, m, d, x32, reinterpret_cast<float4 *>(info));
    FTK_LAUNCHED("row_info64_kernel");
    return FTK_OK;
}

static unsigned g_t64_last[2] = {0, 0};

int tc64_assign_run(ftk_ctx *ctx, const double *x, const double *y, const double *yn, int64_t m,
                    int64_t k, int64_t d, int32_t *out_idx, double *out_val, const TcFt *ft,
                    cudaStream_t st) {
    if (!tc64_supported(m, k, d)) {
        set_error("tc64: unsupported shape (d % 4 == 0, d <= 256, k < 65536)");
        return FTK_ERR_UNSUPPORTED;
    }
    // X32 and row bounds: the fit's registered copy, else converted here
    const float *x32;
    const float4 *info;
    if (ctx->rows_x == x && ctx->rows_x32 && ctx->rows_m == m && ctx->rows_d == d && ctx->rows_info) {
        x32 = ctx->rows_x32;
        info = reinterpret_cast<const float4 *>(ctx->rows_info);
    } else {
        char *b = static_cast<char *>(scratch(ctx, SLOT_TC64_X, sizeof(float) * size_t(m) * (d + 4) + 256, st));
        if (!b) return FTK_ERR_CUDA;
        float *xs = reinterpret_cast<float *>(b);
        float *inf = reinterpret_cast<float *>(b + ((sizeof(float) * size_t(m) * d + 255) & ~size_t(255)));
        int rc = row_info64_run(x, m, d, xs, inf, st);
        if (rc) return rc;
        x32 = xs;
        info = reinterpret_cast<const float4 *>(inf);
    }
    const size_t cbytes = (sizeof(float) * size_t(k) * d + 255) & ~size_t(255);
    char *cb = static_cast<char *>(scratch(ctx, SLOT_TC64_C, cbytes + sizeof(float) * size_t(k) + 512, st));
    if (!cb) return FTK_ERR_CUDA;
    float *c32 = reinterpret_cast<float *>(cb);
    float *yn32 = reinterpret_cast<float *>(cb + cbytes);
    float *bounds = yn32 + ((k + 63) & ~int64_t(63));  // [0] cmax2, [1] ecmax2, then counters
    unsigned *cnt = reinterpret_cast<unsigned *>(bounds + 8);  // [0] uncertified, [2] abft, [4] corrected, [5] flags
    FTK_CUDA(cudaMemsetAsync(bounds, 0, 64, st));
    tc64_prep_kernel<<<unsigned(std::min<int64_t>((k + 7) / 8, 296)), 256, 0, st>>>(y, yn, k, d, c32, yn32,
                                                                                     bounds);
    FTK_LAUNCHED("tc64_prep_kernel");
    char *rb = static_cast<char *>(scratch(ctx, SLOT_TC64_REC, sizeof(int2) * size_t(m) + sizeof(int32_t) * size_t(m + 1) +
                                                                   2 * sizeof(float) * size_t(m + 1) + 64, st));
    if (!rb) return FTK_ERR_CUDA;
    int2 *rec = reinterpret_cast<int2 *>(rb);
    int32_t *fb = reinterpret_cast<int32_t *>(rec + m);
    float *a64 = reinterpret_cast<float *>(fb + (m + 1));   // per-row screen bound
    float *fb_thr = a64 + (m + 1);                          // per uncertified row: pass-2 threshold
    const bool p2 = !getenv("FTK_T64_NO_P2");

    const int nkb = int((d + T64_KB - 1) / T64_KB);
    PairParams Q{};
    Q.x = x32; Q.y = c32; Q.yn = yn32; Q.m = m; Q.k = k; Q.d = d;
    // tf32 accumulation (the float32 path's term) + the reference's float64 chain
    Q.a_coef = float(3.0 * double(d) * 0x1p-24 + 2.0 * (double(d) + 2.0) * 0x1p-53);
    Q.b_coef = float((0x1p-14 + 0x1p-22) * 1.01);
    Q.a_abs = 0x1p-23f;  // x cmax^2: fp32 rounding of the float64 norms
    Q.cmax2 = bounds;
    Q.ecmax2 = bounds + 1;
    Q.out_idx = out_idx;
    Q.out_val = nullptr;
    Q.fb_rows = fb;
    Q.fb_count = cnt;
    Q.rowinfo = info;
    Q.rec64 = rec;
    Q.a64 = p2 ? a64 : nullptr;
    if (const char *e = getenv("FTK_TC_DEBUG")) Q.dbg = atoi(e);  // timing probe (results invalid)
    constexpr unsigned kFlagCap = 4096;
    double4 *flag_rec = nullptr;
    float *csum = nullptr, *camax = nullptr, *csumw = nullptr;
    if (ft) {
        int rc = prep_csum_run(ctx, SLOT_TC_CSUM1, c32, k, d, nkb, 1, &csum, &camax, st, &csumw);
        if (rc) return rc;
        flag_rec = static_cast<double4 *>(scratch(ctx, SLOT_PAIR_FLAG, sizeof(double4) * kFlagCap, st));
        if (!flag_rec) return FTK_ERR_CUDA;
        Q.csum = csum;
        Q.camax = camax;
        Q.tau_coef = float(ft->delta_rel * double(d) * std::sqrt(double(k) / 32.0));
        Q.tau_abs = float(ft->abs_tol);
        Q.abft_count = cnt + 2;
        Q.abft_total = abft_total_ptr(ctx, st);
        Q.flag_rec = flag_rec;
        Q.flag_count = cnt + 5;
        Q.flag_cap = kFlagCap;
    }
    CUtensorMap mx, mc;
    int rc = make_tc_map(&mx, x32, m, d, 128);
    if (!rc) rc = make_tc_map(&mc, c32, k, d, PAIR_BN / 2);
    if (rc) return rc;
    if ((rc = pair_screen_launch(mx, mc, Q, ft != nullptr, st))) return rc;
    {
        const int nbox = int((d + 15) / 16);
        const size_t stage = size_t(nbox) * 4096;
        const size_t ring = size_t(RT_CONS) * stage;  // one slot per consumer warp
        CUtensorMap tx;
        const bool tma = ring <= 200 * 1024 && !getenv("FTK_T64_REFINE_LDG") && !make_f64_map(&tx, x, m, d, 32);
        const int64_t ct_bytes = k * d * 8;
        const char *cte = getenv("FTK_T64_CTAB");  // A/B knob: 0 = centroids gathered from L2
        const size_t ct_smem = size_t(RT_CONS_CT) * stage + 128 + size_t(ct_bytes) + 1024;
        const bool ctab = tma && d % 16 == 0 && ct_bytes <= RT_CT_MAX_BYTES && ct_smem <= 227 * 1024 &&
                          !(cte && atoi(cte) == 0) && (reinterpret_cast<uintptr_t>(y) & 15) == 0;
        const int64_t ntile = (m + 31) / 32;
        if (ctab) {
            const size_t smem = ct_smem;
            auto kern = tc64_refine_tma_kernel<RT_CONS_CT, true>;
            FTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            kern<<<unsigned(std::min<int64_t>(ntile, int64_t(current_sm_count()))), 32 * (RT_CONS_CT + 1), smem, st>>>(
                tx, y, yn, m, d, nbox, rec, p2 ? a64 : nullptr, out_idx, out_val, fb, cnt, p2 ? fb_thr : nullptr, k);
            FTK_LAUNCHED("tc64_refine_tma_kernel");
        } else if (tma) {
            const int per_sm = int(std::min<size_t>(3, (200 * 1024) / ring));  // CTAs per SM
            const size_t smem = ring + 128 + 1024;
            auto kern = tc64_refine_tma_kernel<RT_CONS, false>;
            FTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            kern<<<unsigned(std::min<int64_t>(ntile, int64_t(current_sm_count()) * per_sm)), 32 * (RT_CONS + 1), smem,
                   st>>>(tx, y, yn, m, d, nbox, rec, p2 ? a64 : nullptr, out_idx, out_val, fb, cnt,
                         p2 ? fb_thr : nullptr, k);
            FTK_LAUNCHED("tc64_refine_tma_kernel");
        } else {
            tc64_refine_kernel<<<unsigned(std::min<int64_t>((m + 32 * R64_WARPS - 1) / (32 * R64_WARPS), 148 * 6)),
                                 32 * R64_WARPS, 0, st>>>(x, y, yn, m, d, rec, p2 ? a64 : nullptr, out_idx,
                                                          out_val, fb, cnt, p2 ? fb_thr : nullptr);
            FTK_LAUNCHED("tc64_refine_kernel");
        }
    }
    if (ft) {
        // location + event records of the checksum-flagged rows (the DMMA pass
        // below re-resolves them: the correction)
        FlagEvents F{};
        F.x = x32; F.d = d; F.k = k;
        F.csumw = csumw; F.camax = camax;
        F.rec = flag_rec; F.count = cnt + 5; F.cap = kFlagCap;
        F.inj_col = nullptr;
        F.events_for_scheduled = 1;
        if (ft->ev) F.ev = *ft->ev;
        F.iteration = ft->iteration;
        F.bm = ft->bm;
        F.bn = ft->bn;
        F.interval = ft->bk > 0 ? (d + ft->bk - 1) / ft->bk - 1 : 0;
        F.corrected = cnt + 4;
        if ((rc = abft_flag_events_run(F, st))) return rc;
    }
    unsigned h[3] = {0, 0, 0};
    FTK_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
    FTK_CUDA(cudaStreamSynchronize(st));
    g_t64_last[0] = h[0];
    g_t64_last[1] = h[2];
    ctx->stat_dev[0] = ctx->stat_dev[1] = ctx->stat_dev[2] = nullptr;
    ctx->last_fb[0] = h[0];
    ctx->last_fb[1] = 0;
    ctx->last_fb[2] = h[2];
    int32_t *dm_rows = fb;        // rows for the DMMA screen
    const unsigned *dm_cnt = cnt;
    unsigned n_dm = h[0];
    if (h[0] > 0 && p2) {
        // pass 2: COLLECT re-screen of the uncertified rows' fp32 copies, float64
        // evaluation of every candidate that can still beat the row's d1
        const unsigned n1 = h[0];
        const unsigned row_cap = 256;
        const unsigned cap = unsigned(std::min<int64_t>(int64_t(n1) * 16 + 65536, int64_t(1) << 30));
        const size_t gbytes = (sizeof(float) * size_t(n1) * d + 255) & ~size_t(255);
        const size_t need = gbytes + sizeof(int2) * cap + sizeof(double) * cap + 8 * size_t(n1) +
                            4 * size_t(n1) * 3 + 256;
        char *b2 = static_cast<char *>(scratch(ctx, SLOT_TC64_P2, need, st));
        if (!b2) return FTK_ERR_CUDA;
        float *g32 = reinterpret_cast<float *>(b2);
        int2 *cand = reinterpret_cast<int2 *>(b2 + gbytes);
        double *cval = reinterpret_cast<double *>(cand + cap);
        unsigned long long *key = reinterpret_cast<unsigned long long *>(cval + cap);
        int32_t *kidx = reinterpret_cast<int32_t *>(key + n1);
        unsigned *row_cnt = reinterpret_cast<unsigned *>(kidx + n1);
        int32_t *rows2 = reinterpret_cast<int32_t *>(row_cnt + n1);
        unsigned *cc = cnt + 8;  // [0] candidates, [1] rows for the DMMA screen
        FTK_CUDA(cudaMemsetAsync(cc, 0, 2 * sizeof(unsigned), st));
        t64p2_gather_kernel<<<148 * 4, 256, 0, st>>>(x32, d, fb, cnt, g32, row_cnt, key, kidx);
        FTK_LAUNCHED("t64p2_gather_kernel");
        CUtensorMap mg, mc2;
        if ((rc = make_tc_map(&mg, g32, n1, d, 128)) || (rc = make_tc_map(&mc2, c32, k, d, PAIR_BN / 2)))
            return rc;
        PairParams R{};
        R.x = g32; R.y = c32; R.yn = yn32; R.m = n1; R.k = k; R.d = d;
        R.cmax2 = bounds;
        R.ecmax2 = bounds + 1;
        R.thr = fb_thr;
        R.cand = cand;
        R.cand_count = cc;
        R.cand_cap = cap;
        R.row_cnt = row_cnt;
        if ((rc = pair_screen_launch(mg, mc2, R, false, st))) return rc;
        t64p2_value_kernel<<<148 * 8, 256, 0, st>>>(x, y, yn, d, fb, cand, cc, cap, row_cnt, row_cap, cval, key);
        FTK_LAUNCHED("t64p2_value_kernel");
        t64p2_index_kernel<<<148 * 4, 256, 0, st>>>(cand, cc, cap, row_cnt, row_cap, cval, key, kidx);
        FTK_LAUNCHED("t64p2_index_kernel");
        t64p2_finalize_kernel<<<148, 256, 0, st>>>(fb, cnt, row_cnt, row_cap, cc, cap, key, kidx, out_idx, out_val,
                                                   rows2, cc + 1);
        FTK_LAUNCHED("t64p2_finalize_kernel");
        unsigned h2 = 0;
        FTK_CUDA(cudaMemcpyAsync(&h2, cc + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        FTK_CUDA(cudaStreamSynchronize(st));
        dm_rows = rows2;
        dm_cnt = cc + 1;
        n_dm = h2;
        ctx->last_fb[1] = h2;
    }
    if (n_dm > 0) {
        // rows left: the DMMA screen (checked like the pass) over the gathered rows
        const unsigned n = n_dm;
        const size_t gb = (sizeof(double) * size_t(n) * d + 255) & ~size_t(255);
        char *g = static_cast<char *>(scratch(ctx, SLOT_TC64_G, gb + (sizeof(double) + sizeof(int32_t)) * size_t(n) + 64, st));
        if (!g) return FTK_ERR_CUDA;
        double *gx = reinterpret_cast<double *>(g);
        double *gv = reinterpret_cast<double *>(g + gb);
        int32_t *gi = reinterpret_cast<int32_t *>(gv + n);
        tc64_gather_kernel<<<148 * 4, 256, 0, st>>>(x, d, dm_rows, dm_cnt, gx);
        FTK_LAUNCHED("tc64_gather_kernel");
        TcFt ft2{};
        if (ft) {
            ft2 = *ft;
            ft2.inj = nullptr;
            ft2.ev = nullptr;
        }
        const int fam = ctx->family;
        ctx->family = 3;  // DMMA for the leftovers
        rc = dscreen_run(ctx, gx, y, yn, n, k, d, gi, gv, ft ? &ft2 : nullptr, st);
        ctx->family = fam;
        if (rc) return rc;
        tc64_scatter_kernel<<<148, 256, 0, st>>>(dm_rows, dm_cnt, gi, gv, out_idx, out_val);
        FTK_LAUNCHED("tc64_scatter_kernel");
    }
    if (ft && ft->inj && ft->inj->n > 0)
        return emulate_injected_blocks<double>(ctx, x, y, yn, m, k, d, *ft, out_idx, out_val, st);
    return FTK_OK;
}

int tc64_last(unsigned *out) {
    out[0] = g_t64_last[0];
    out[1] = g_t64_last[1];
    return FTK_OK;
}

}  // namespace ftk
