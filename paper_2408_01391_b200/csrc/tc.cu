// tc.cu -- tensor-core screened assignment with certified exact refinement
// (sm_100a: TMA + mbarrier pipeline, tcgen05.mma kind::tf32 into TMEM,
// tcgen05.ld epilogue).
//
// The reference's labels and min_dists are functions of its exact fp32
// evaluation order (_kernels.py:44-102).  This path reproduces them bit for
// bit without evaluating every distance exactly:
//
//   1. SCREEN  (tensor cores): s_ij = yn_j - 2 <x_i, c_j>, fp32 TMEM
//      accumulators.  Pass 1 uses 1xTF32 (operands truncated to 10 mantissa
//      bits).  The epilogue keeps per row the two smallest screened values
//      (index packed in the low mantissa bits of the minimum): the N x K
//      distance matrix never leaves the SM.
//   2. CERTIFY: |s_ij - d_ij^ref| <= A_i + B |s_ij|, with
//        pass 1: A_i = 2 ||x_i|| cmax (2^-9 + 2^-20 + 3 D 2^-24)
//        pass 2: A_i = 2 ||x_i|| cmax (3 2^-20 + 7 D 2^-24)
//      (operand truncation, fp32 tensor-core accumulation <= 2^-23 per add,
//      and the reference's own sequential rounding) and B = 2^-15 + 2^-22
//      (index packing, final roundings).  If m2 - m1 > 2 A_i + B (|m1|+|m2|)
//      the reference's strict argmin is provably the screened winner.
//   3. REFINE  (SIMT, exact order): acc = sum_k fl(x_ik c_jk), k ascending;
//      min_dist = yn_j - (acc + acc), for the winner only, from the X tile
//      already resident in shared memory.
//   4. Rows pass 1 cannot certify are gathered and re-screened with 3xTF32
//      (x = x_hi + x_lo, c = c_hi + c_lo; hi*hi + hi*lo + lo*hi), whose bound
//      is ~2^9 tighter; rows that still tie are resolved by the exact SIMT
//      kernel (exact.cu).  Every row therefore carries the reference's bits.
//
// Roles per CTA (6 warps): w0 TMA producer, w1 TMEM allocator + MMA issuer
// (one elected thread), w2..w5 epilogue (one accumulator row per thread; warp
// w reads TMEM lanes 32*(w%4)..+31).  The X tile (128 rows x D) is loaded
// once and stays resident; centroid k-blocks stream through a ring; two TMEM
// accumulators let the MMA of centroid tile t+1 overlap the epilogue of t.

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tc_pair.cuh"

namespace ftk {

constexpr int TC_BM = 128;       // rows per CTA (UMMA M)
constexpr int TC_KB = 32;        // fp32 elements per 128-byte swizzle row
constexpr int TC_THREADS = 192;  // 6 warps
constexpr int TC_MAX_D = 256;    // resident-A limit
constexpr int TC_SX_MAX_D = 8192;  // streamed-X pair screen (any k)

struct TcParams {
    const float *x;      // rows x d  (exact values; pass 2: the gathered rows)
    const float *y;      // k x d
    const float *yn;     // k         (exact fp32 squared norms, reference order)
    int64_t m, k, d;
    int nkb;             // ceil(d / 32)
    int ntiles;          // ceil(k / BN)
    int stages;
    int abufs;           // resident X tile buffers (2: next tile prefetched)
    float a_coef;        // see header
    float b_coef;
    const float *cmax2;  // device scalar: upper bound of max_j ||c_j||^2
    const float *ecmax2; // device scalar: upper bound of max_j ||c_j - tf32(c_j)||^2
    const int32_t *rows; // pass 2: row r of the tile is global row rows[r]
    int32_t *out_idx;
    float *out_val;
    int32_t *fb_rows;    // uncertified rows (global indices)
    unsigned *fb_count;
    float *raw;          // debug: materialise the raw screened dot products
    int dbg;             // debug bit 1: skip the screening math (pipeline timing only)
    // FT mode (CHK kernels): per-N-tile row checksums verified in the epilogue
    const float *csum;   // nkb*32: checksum centroid sum_j c~_j over all K centroids
    const float *camax;  // scalar: max |c|
    float tau_coef;      // delta_rel * D * sqrt(K / 32): reference tolerance, K-column checksum
    float tau_abs;
    const int32_t *inj_col;    // per row: injected column (-1: none)
    const float *inj_before;   // exact accumulator value before the flip
    const float *inj_after;    // after the flip
    unsigned *abft_count;      // rows whose checksum failed (diagnostics)
    unsigned long long *abft_total;  // cumulative (ftk_abft_flags_total)
};

// ------------------------------------------------------------- kernel ----
// ABFT reference for row r of the resident X tile and centroid tile t:
// x~ . sum_j c~_j (x~ = tf32(x) in the 1xTF32 pass, x itself in the 3xTF32 one)
template <bool SPLIT>
__device__ __forceinline__ double row_checksum(const unsigned char *rowA, const float *csum, int t,
                                              int nkb, int r) {
    const float4 *cs4 = reinterpret_cast<const float4 *>(csum) + int64_t(t) * nkb * 8;
    double rr = 0.0;  // float64: the reference side must be well below the tolerance
    for (int kb = 0; kb < nkb; ++kb)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 xv = *reinterpret_cast<const float4 *>(rowA + uint32_t(kb) * TC_BM * 128 +
                                                                ((q ^ (r & 7)) << 4));
            const float4 sv = __ldg(cs4 + kb * 8 + q);
            rr = fma(double(SPLIT ? xv.x : tf32_trunc(xv.x)), double(sv.x), rr);
            rr = fma(double(SPLIT ? xv.y : tf32_trunc(xv.y)), double(sv.y), rr);
            rr = fma(double(SPLIT ? xv.z : tf32_trunc(xv.z)), double(sv.z), rr);
            rr = fma(double(SPLIT ? xv.w : tf32_trunc(xv.w)), double(sv.w), rr);
        }
    return rr;
}

template <int BN, bool SPLIT, bool CHK>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_screen_kernel(const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ CUtensorMap tmXl,
                     const __grid_constant__ CUtensorMap tmC,
                     const __grid_constant__ CUtensorMap tmCl, TcParams P) {
    // Persistent: CTA b handles row tiles b, b + grid, ...; the X tile is
    // double-buffered when it fits so the next tile streams in while this
    // tile's last epilogue / refinement runs.
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // align to 1024 B by pointer arithmetic on the __shared__ array itself so
    // the compiler keeps the shared address space (LDS/STS, not generic LD/ST)
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int NOP = SPLIT ? 2 : 1;             // hi (+ lo) operand copies
    constexpr uint32_t IDX_MASK = BN > 128 ? 0xFFu : 0x7Fu;
    const int nkb = P.nkb, S = P.stages, NA = P.abufs;
    const uint32_t A_KB_BYTES = TC_BM * 128;       // one k-block of X
    const uint32_t A_BYTES = A_KB_BYTES * nkb * NOP;
    const uint32_t B_BYTES = BN * 128;             // one k-block of C
    unsigned char *sA = smem;                      // NA x [NOP x nkb x 16 KB] (hi first)
    unsigned char *sB = sA + size_t(NA) * A_BYTES; // S x NOP x B_BYTES
    uint64_t *bars = reinterpret_cast<uint64_t *>(sB + size_t(S) * NOP * B_BYTES);
    uint64_t *full = bars, *empty = bars + S;
    uint64_t *a_full = bars + 2 * S, *a_empty = a_full + 2;
    uint64_t *t_full = a_full + 4, *t_empty = a_full + 6;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(a_full + 8);
    float *yn_s = reinterpret_cast<float *>(a_full + 10);  // [2][BN] centroid norms

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntm = (P.m + TC_BM - 1) / TC_BM;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmX);
        prefetch_tmap(&tmC);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&a_full[a], 1);
            mbar_init(&a_empty[a], 4);
            mbar_init(&t_full[a], 1);
            mbar_init(&t_empty[a], 4);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 2 * BN);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int64_t tile = blockIdx.x; tile < ntm; tile += gridDim.x, ++it) {
                const int ab = it % NA;
                const uint32_t ause = uint32_t(it / NA) & 1;
                mbar_wait(&a_empty[ab], ause ^ 1);
                unsigned char *a_dst = sA + size_t(ab) * A_BYTES;
                const int row0 = int(tile * TC_BM);
                mbar_expect_tx(&a_full[ab], A_BYTES);
                for (int kb = 0; kb < nkb; ++kb) {
                    tma_load_2d(a_dst + size_t(kb) * A_KB_BYTES, &tmX, &a_full[ab], kb * TC_KB, row0);
                    if (SPLIT)
                        tma_load_2d(a_dst + size_t(nkb + kb) * A_KB_BYTES, &tmXl, &a_full[ab],
                                    kb * TC_KB, row0);
                }
                for (int t = 0; t < P.ntiles; ++t) {
                    for (int kb = 0; kb < nkb; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        mbar_expect_tx(&full[stage], B_BYTES * NOP);
                        unsigned char *dst = sB + size_t(stage) * NOP * B_BYTES;
                        tma_load_2d(dst, &tmC, &full[stage], kb * TC_KB, t * BN);
                        if (SPLIT)
                            tma_load_2d(dst + B_BYTES, &tmCl, &full[stage], kb * TC_KB, t * BN);
                        if (++stage == S) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(TC_BM, BN);
            const uint32_t b_base = smem_u32(sB);
            int stage = 0;
            uint32_t phase = 0;
            uint32_t g = 0;  // global accumulator-tile counter (TMEM buffer ring)
            int it = 0;
            for (int64_t tile = blockIdx.x; tile < ntm; tile += gridDim.x, ++it) {
                const int ab = it % NA;
                mbar_wait(&a_full[ab], uint32_t(it / NA) & 1);
                const uint32_t a_base = smem_u32(sA) + uint32_t(ab) * A_BYTES;
                const uint32_t a_lo = a_base + uint32_t(nkb) * A_KB_BYTES;
                for (int t = 0; t < P.ntiles; ++t, ++g) {
                    const int buf = g & 1;
                    mbar_wait(&t_empty[buf], ((g >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem + uint32_t(buf * BN);
                    for (int kb = 0; kb < nkb; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint32_t bs = b_base + uint32_t(stage) * NOP * B_BYTES;
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {  // 4 x (K = 8 tf32) per 128-byte row
                            const uint32_t ao = uint32_t(kb) * A_KB_BYTES + kk * 32;
                            const uint64_t ah = smem_desc(a_base + ao);
                            const uint64_t bh = smem_desc(bs + kk * 32);
                            mma_tf32(d_tmem, ah, bh, idesc, (kb | kk) != 0);
                            if (SPLIT) {
                                mma_tf32(d_tmem, ah, smem_desc(bs + B_BYTES + kk * 32), idesc, 1);
                                mma_tf32(d_tmem, smem_desc(a_lo + ao), bh, idesc, 1);
                            }
                        }
                        mma_commit(&empty[stage]);
                        if (++stage == S) { stage = 0; phase ^= 1; }
                    }
                    mma_commit(&t_full[buf]);
                }
            }
        }
    } else {
        // ---------------------------------------------------- epilogue --
        const int quad = warp & 3;              // TMEM lane group this warp may access
        const int r = quad * 32 + lane;         // accumulator row within the tile
        const uint32_t lane_base = uint32_t(quad * 32) << 16;
        const int et = threadIdx.x - 64;        // 0..127 among the epilogue threads
        uint32_t g = 0;
        int it = 0;
        for (int64_t tile = blockIdx.x; tile < ntm; tile += gridDim.x, ++it) {
            const int ab = it % NA;
            const int64_t grow = tile * TC_BM + r;  // row within this pass
            float m1 = INFINITY, m2 = INFINITY;
            int tile1 = 0;
            bool abft_bad = false;
            float amax_i = 0.0f;
            double rref = 0.0;
            double rsum = 0.0;  // row checksum over all centroid tiles
            int inj_c = -1;
            float inj_b = 0.0f, inj_a = 0.0f;
            const unsigned char *rowA = sA + size_t(ab) * A_BYTES + uint32_t(r) * 128;
            if (CHK) {
                if (grow < P.m && P.inj_col) {
                    inj_c = P.inj_col[grow];
                    if (inj_c >= 0) {
                        inj_b = P.inj_before[grow];
                        inj_a = P.inj_after[grow];
                    }
                }
                mbar_wait(&a_full[ab], uint32_t(it / NA) & 1);  // the X tile is resident
                for (int kb = 0; kb < nkb; ++kb)
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float4 xv = *reinterpret_cast<const float4 *>(
                            rowA + uint32_t(kb) * A_KB_BYTES + ((q ^ (r & 7)) << 4));
                        amax_i = fmaxf(amax_i, fmaxf(fmaxf(fabsf(xv.x), fabsf(xv.y)),
                                                     fmaxf(fabsf(xv.z), fabsf(xv.w))));
                    }
                // the row's checksum reference x~ . sum_j c~_j, computed while the
                // tensor core works on the first centroid tile
                rref = row_checksum<SPLIT>(rowA, P.csum, 0, nkb, r);
            }
            // centroid norms of tile t live in yn_s[t & 1]: each epilogue thread
            // stages BN/128 values per tile, prefetched one tile ahead (named
            // barrier 1 synchronises the 128 epilogue threads only)
            for (int e = et; e < BN; e += 128) yn_s[e] = e < P.k ? __ldg(P.yn + e) : 0.0f;
            asm volatile("bar.sync 1, 128;" ::: "memory");
            for (int t = 0; t < P.ntiles; ++t, ++g) {
                const int buf = g & 1;
                const int ybuf = t & 1;
                const int64_t c0 = int64_t(t) * BN;
                float yn_next[(BN + 127) / 128];
#pragma unroll
                for (int q = 0; q < (BN + 127) / 128; ++q) {
                    const int e = et + q * 128;
                    const int64_t cn = c0 + BN + e;
                    yn_next[q] = (e < BN && cn < P.k) ? __ldg(P.yn + cn) : 0.0f;
                }
                const float *ynt = yn_s + ybuf * BN;
                mbar_wait(&t_full[buf], (g >> 1) & 1);
                tc_fence_after();
                float t1 = INFINITY, t2 = INFINITY, tsum = 0.0f;
                const int live = int(P.k - c0 < BN ? P.k - c0 : BN);
                const uint32_t tbase = tmem + lane_base + uint32_t(buf * BN);
                // software-pipelined TMEM drain: chunk ch+1 in flight while ch is screened
                uint32_t va[32], vb[32];
                tmem_ld32_issue(tbase, va);
                tmem_ld_wait(va);
#pragma unroll
                for (int ch = 0; ch < ((P.dbg & 1) ? 0 : BN / 32); ch += 2) {
                    if (ch + 1 < BN / 32) tmem_ld32_issue(tbase + uint32_t((ch + 1) * 32), vb);
                    if (P.raw && grow < P.m)
#pragma unroll
                        for (int e = 0; e < 32; ++e)  // static indices: va stays in registers
                            if (ch * 32 + e < live)
                                P.raw[grow * P.k + c0 + ch * 32 + e] = __uint_as_float(va[e]);
                    if (CHK && inj_c >= int(c0) + ch * 32 && inj_c < int(c0) + ch * 32 + 32)
                        inject_into(va, inj_c - int(c0) - ch * 32, inj_b, inj_a);
                    screen_chunk<CHK>(va, ynt + ch * 32, ch * 32, live - ch * 32, IDX_MASK, t1, t2,
                                      tsum);
                    if (ch + 1 < BN / 32) {
                        tmem_ld_wait(vb);
                        if (ch + 2 < BN / 32) tmem_ld32_issue(tbase + uint32_t((ch + 2) * 32), va);
                        if (P.raw && grow < P.m)
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if ((ch + 1) * 32 + e < live)
                                    P.raw[grow * P.k + c0 + (ch + 1) * 32 + e] =
                                        __uint_as_float(vb[e]);
                        if (CHK && inj_c >= int(c0) + (ch + 1) * 32 &&
                            inj_c < int(c0) + (ch + 1) * 32 + 32)
                            inject_into(vb, inj_c - int(c0) - (ch + 1) * 32, inj_b, inj_a);
                        screen_chunk<CHK>(vb, ynt + (ch + 1) * 32, (ch + 1) * 32,
                                          live - (ch + 1) * 32, IDX_MASK, t1, t2, tsum);
                        if (ch + 2 < BN / 32) tmem_ld_wait(va);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&t_empty[buf]);
                // stage the next tile's norms (that buffer was last read two
                // tiles ago, before the previous barrier)
#pragma unroll
                for (int q = 0; q < (BN + 127) / 128; ++q)
                    if (et + q * 128 < BN) yn_s[(ybuf ^ 1) * BN + et + q * 128] = yn_next[q];
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (CHK) rsum += double(tsum);
                if (CHK && t == P.ntiles - 1 && grow < P.m && !(P.dbg & 1)) {
                    // ABFT: the row checksum of all K accumulators against
                    // x~ . (sum_j c~_j), evaluated on the CUDA cores
                    const float tau = P.tau_coef * fmaxf(1.0f, amax_i * *P.camax) + P.tau_abs;
                    if (!(fabs(rsum - rref) <= double(tau))) abft_bad = true;
                }
                // merge the tile's top-2 into the running top-2
                const float hi = fmaxf(m1, t1);
                if (t1 < m1) tile1 = t;
                m1 = fminf(m1, t1);
                m2 = fminf(fminf(m2, t2), hi);
            }

            if (grow < P.m) {
                const int j = tile1 * BN + int(__float_as_uint(m1) & IDX_MASK);
                const int64_t orow = P.rows ? int64_t(P.rows[grow]) : grow;
                // one pass over the resident X row: ||x||^2, the truncation
                // residual, and the exact sequential dot product with the
                // screened winner (fetched 32 floats at a time so the L2 round
                // trips overlap).  Chunk q of row r sits at chunk position
                // q ^ (r & 7) of the 128-byte swizzled row; the hi tile holds
                // the full fp32 x (the MMA truncates it).
                const unsigned char *sAt = sA + size_t(ab) * A_BYTES;
                const float4 *cj4 = reinterpret_cast<const float4 *>(P.y + int64_t(j) * P.d);
                float acc = 0.0f, xx = 0.0f, ee = 0.0f;
                for (int kb = 0; kb < nkb; ++kb) {
                    const int k0 = kb * TC_KB;
                    float4 cv[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        cv[q] = (k0 + 4 * q < P.d) ? __ldg(cj4 + (k0 >> 2) + q)
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                    const unsigned char *rowp = sAt + uint32_t(kb) * A_KB_BYTES + uint32_t(r) * 128;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (k0 + 4 * q < P.d) {
                            const float4 xv =
                                *reinterpret_cast<const float4 *>(rowp + ((q ^ (r & 7)) << 4));
                            acc = __fadd_rn(acc, __fmul_rn(xv.x, cv[q].x));
                            acc = __fadd_rn(acc, __fmul_rn(xv.y, cv[q].y));
                            acc = __fadd_rn(acc, __fmul_rn(xv.z, cv[q].z));
                            acc = __fadd_rn(acc, __fmul_rn(xv.w, cv[q].w));
                            xx = fmaf(xv.x, xv.x, xx);
                            xx = fmaf(xv.y, xv.y, xx);
                            xx = fmaf(xv.z, xv.z, xx);
                            xx = fmaf(xv.w, xv.w, xx);
                            if (!SPLIT) {  // truncation residual ||x - tf32(x)||^2
                                const float r0 = xv.x - tf32_trunc(xv.x);
                                const float r1 = xv.y - tf32_trunc(xv.y);
                                const float r2 = xv.z - tf32_trunc(xv.z);
                                const float r3 = xv.w - tf32_trunc(xv.w);
                                ee = fmaf(r0, r0, ee);
                                ee = fmaf(r1, r1, ee);
                                ee = fmaf(r2, r2, ee);
                                ee = fmaf(r3, r3, ee);
                            }
                        }
                    }
                }
                const float xn = sqrtf(xx * (1.0f + 0x1p-10f));
                const float cm = sqrtf(*P.cmax2 * (1.0f + 0x1p-10f));  // yn: rounded sum
                // pass 1: |x.c - x~.c~| <= ||x - x~|| cmax + ||x|| max_j ||c_j - c~_j||
                // (Cauchy-Schwarz on the actual truncation residuals) plus the
                // accumulation terms; pass 2: the worst-case 3xTF32 coefficient.
                const float A = SPLIT ? P.a_coef * xn * cm
                                      : 2.0f * (1.0f + 0x1p-10f) *
                                            (sqrtf(ee * (1.0f + 0x1p-10f)) * cm +
                                             xn * sqrtf(*P.ecmax2 * (1.0f + 0x1p-10f)) +
                                             P.a_coef * xn * cm);
                const float gap_need = 2.0f * A + P.b_coef * (fabsf(m1) + fabsf(m2));
                if (CHK && abft_bad) {
                    atomicAdd(P.abft_count, 1u);
                    if (P.abft_total) atomicAdd(P.abft_total, 1ull);
                }
                if (m2 - m1 > gap_need && m1 < INFINITY && !abft_bad) {
                    P.out_idx[orow] = j;
                    P.out_val[orow] = __fsub_rn(P.yn[j], __fadd_rn(acc, acc));
                } else {
                    const unsigned slot = atomicAdd(P.fb_count, 1u);
                    P.fb_rows[slot] = int32_t(orow);
                }
            }
            // this X buffer may be refilled once every epilogue warp is done with it
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_empty[ab]);
        }
    }

    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 2 * BN);
    }
}

// --------------------------------------------------------- small kernels --
// Per-row bounds for the screen certificate (one warp per row, any order).
__global__ void row_info_kernel(const float *x, int64_t m, int64_t d, float4 *info) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = w0; i < m; i += nw) {
        float xx = 0.0f, ee = 0.0f, am = 0.0f;
        for (int64_t f = lane; f < d; f += 32) {
            const float v = x[i * d + f];
            const float r = v - tf32_trunc(v);
            xx = fmaf(v, v, xx);
            ee = fmaf(r, r, ee);
            am = fmaxf(am, fabsf(v));
        }
        for (int off = 16; off; off >>= 1) {
            xx += __shfl_xor_sync(0xffffffffu, xx, off);
            ee += __shfl_xor_sync(0xffffffffu, ee, off);
            am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, off));
        }
        if (lane == 0) info[i] = make_float4(xx, ee, am, 0.0f);
    }
}

int row_info_run(const float *x, int64_t m, int64_t d, float *info, cudaStream_t st) {
    if (m == 0) return FTK_OK;
    const int64_t blocks = std::min<int64_t>((m + 7) / 8, 148 * 16);
    row_info_kernel<<<unsigned(blocks), 256, 0, st>>>(x, m, d, reinterpret_cast<float4 *>(info));
    FTK_LAUNCHED("row_info_kernel");
    return FTK_OK;
}

// Upper bounds of max_j ||c_j||^2 (from the exact fp32 norms) and of
// max_j ||c_j - tf32(c_j)||^2: one warp per centroid row, float maxima via
// integer atomicMax (non-negative floats order like their bit patterns).
// bounds[0..1] must be zeroed; the consumer inflates them for rounding.
__global__ void tc_prep_kernel(const float *y, const float *yn, int64_t k, int64_t d,
                               float *bounds) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    float m = 0.0f, e = 0.0f;
    for (int64_t j = w0; j < k; j += nw) {
        float s = 0.0f;
        for (int64_t f = lane; f < d; f += 32) {
            const float v = y[j * d + f];
            const float r = v - tf32_trunc(v);
            s = fmaf(r, r, s);
        }
        for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        e = fmaxf(e, s);
        m = fmaxf(m, yn[j]);
    }
    if (lane == 0) {
        atomicMax(reinterpret_cast<int *>(bounds), __float_as_int(m));
        atomicMax(reinterpret_cast<int *>(bounds + 1), __float_as_int(e));
    }
}

// FT mode: checksum centroid sum_j tf32(c_j) (float64 sum in a fixed tree
// order, then fp32) zero-padded to nkb*32 features, and max |c| (one block
// per feature; the last block to finish folds the per-feature maxima).
// ABFT checksum centroids: csum[f] = sum_j c~_jf and csumw[f] = sum_j (j/128
// + 1) c~_jf in float64, fmax[f] = max_j |c_jf|.  Grid (feature blocks of 32,
// CSUM_SLICES row slices), coalesced; per-slice partials, then the last CTA
// adds the slices in order (fixed association: deterministic tolerances) and
// writes camax = (max |c|, -, |csum|^2, |csumw|^2).
constexpr int CSUM_SLICES = 16;
__global__ void tile_csum_kernel(const float *y, int64_t k, int64_t d, int nkb, int trunc,
                                 float *csum, float *camax, float *fmax, unsigned *done,
                                 float *csumw, double *part) {
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;  // 8 row groups
    const int64_t nf = int64_t(nkb) * 32;
    const int64_t f = int64_t(blockIdx.x) * 32 + lane;
    const int64_t per = (k + CSUM_SLICES - 1) / CSUM_SLICES;
    const int64_t j0 = int64_t(blockIdx.y) * per, j1 = j0 + per < k ? j0 + per : k;
    double s = 0.0, sw = 0.0;
    float am = 0.0f;
    if (f < d)
        for (int64_t j = j0 + g; j < j1; j += 8) {
            const float v = y[j * d + f];
            const double tv = double(trunc ? tf32_trunc(v) : v);  // 3xTF32 pass: ~exact operands
            s += tv;
            sw += double(j / 128 + 1) * tv;  // location weight of column j's 128-column group
            am = fmaxf(am, fabsf(v));
        }
    __shared__ double sh[8][32], shw[8][32];
    __shared__ float shm[8][32];
    __shared__ unsigned s_last;
    sh[g][lane] = s;
    shw[g][lane] = sw;
    shm[g][lane] = am;
    __syncthreads();
    if (g == 0) {
        double t = 0.0, tw = 0.0;
        float m = 0.0f;
        for (int q = 0; q < 8; ++q) {
            t += sh[q][lane];
            tw += shw[q][lane];
            m = fmaxf(m, shm[q][lane]);
        }
        double *ps = part + (int64_t(blockIdx.y) * nf + f) * 3;
        ps[0] = t;
        ps[1] = tw;
        ps[2] = double(m);
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x * gridDim.y - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    float n2 = 0.0f, w2 = 0.0f, gm = 0.0f;
    for (int64_t ff = threadIdx.x; ff < nf; ff += blockDim.x) {
        double t = 0.0, tw = 0.0, m = 0.0;
        for (int sl = 0; sl < CSUM_SLICES; ++sl) {
            const double *ps = part + (int64_t(sl) * nf + ff) * 3;
            t += ps[0];
            tw += ps[1];
            m = ps[2] > m ? ps[2] : m;
        }
        csum[ff] = float(t);
        csumw[ff] = float(tw);
        fmax[ff] = float(m);
        n2 = fmaf(float(t), float(t), n2);
        w2 = fmaf(float(tw), float(tw), w2);
        gm = fmaxf(gm, float(m));
    }
    __shared__ float rn[256], rw[256], rm[256];
    rn[threadIdx.x] = n2;
    rw[threadIdx.x] = w2;
    rm[threadIdx.x] = gm;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (int(threadIdx.x) < o) {
            rn[threadIdx.x] += rn[threadIdx.x + o];
            rw[threadIdx.x] += rw[threadIdx.x + o];
            rm[threadIdx.x] = fmaxf(rm[threadIdx.x], rm[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        camax[0] = rm[0];
        camax[2] = rn[0];  // |csum|^2 (bounds the fp32 reference error)
        camax[3] = rw[0];  // |csumw|^2
        *done = 0;
    }
}
__global__ void inj_rows_kernel(const float *x, const float *y, int64_t m, int64_t k, int64_t d,
                                int64_t bm, int64_t bn, ftk_injection inj, int32_t *inj_col,
                                float *inj_before, float *inj_after) {
    const int64_t n = inj.n_dev ? (*inj.n_dev < inj.n ? *inj.n_dev : inj.n) : inj.n;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += int64_t(gridDim.x) * blockDim.x) {
        const int64_t ei = inj.ei[q], ej = inj.ej[q];
        const int64_t row = inj.bi[q] * bm + ei, col = inj.bj[q] * bn + ej;
        if (ei >= bm || ej >= bn || row >= m || col >= k) continue;
        float acc = 0.0f;
        for (int64_t f = 0; f < d; ++f) acc = __fadd_rn(acc, __fmul_rn(x[row * d + f], y[col * d + f]));
        inj_col[row] = int32_t(col);
        inj_before[row] = acc;
        inj_after[row] = flip_bit(acc, inj.bit[q]);
    }
}

__global__ void remap_events_kernel(int64_t *rec, const int64_t *count, int64_t cap,
                                    const int64_t *blocks) {
    const int64_t n = *count < cap ? *count : cap;
    for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n;
         c += int64_t(gridDim.x) * blockDim.x)
        rec[c * 7 + 1] = blocks[rec[c * 7 + 1]];
}

__global__ void remap_inj_kernel(const int64_t *bi, int64_t n, const int64_t *blk_of, int64_t nb,
                                 int64_t *bi_out) {
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += int64_t(gridDim.x) * blockDim.x) {
        int64_t pos = -1;
        for (int64_t b = 0; b < nb; ++b)
            if (blk_of[b] == bi[q]) pos = b;
        bi_out[q] = pos < 0 ? int64_t(1) << 40 : pos;  // unmatched -> never applies
    }
}

// Device-count injections (ftk_injection.n_dev): the sorted distinct logical
// row blocks that carry a flip, each flip's compact block index, and
// nb_rows = {blocks, compact rows} -- what emulate_injected_blocks derives on
// the host, computed without a host round trip.  One CTA, O(n^2) over the
// (small) schedule of one pass, dynamic smem 9 bytes per capacity entry.
// Also clears the applied/before/after outputs.
__global__ void inj_blocks_kernel(ftk_injection inj, int64_t nbi, int64_t m, int64_t bm,
                                  int64_t *blocks, int64_t *bi_out, int64_t *nb_rows) {
    extern __shared__ int64_t sbi[];
    __shared__ int s_nb;
    const int64_t n = *inj.n_dev < inj.n ? *inj.n_dev : inj.n;
    unsigned char *first = reinterpret_cast<unsigned char *>(sbi + inj.n);
    if (threadIdx.x == 0) s_nb = 0;
    for (int64_t q = threadIdx.x; q < inj.n; q += blockDim.x) {
        const int64_t v = q < n ? inj.bi[q] : -1;
        sbi[q] = (v >= 0 && v < nbi) ? v : -1;
        inj.applied[q] = 0;
        inj.before[q] = 0.0;
        inj.after[q] = 0.0;
    }
    __syncthreads();
    for (int64_t q = threadIdx.x; q < n; q += blockDim.x) {
        bool f = sbi[q] >= 0;
        for (int64_t p = 0; p < q && f; ++p) f = sbi[p] != sbi[q];
        first[q] = f;
    }
    __syncthreads();
    for (int64_t q = threadIdx.x; q < n; q += blockDim.x) {
        const int64_t v = sbi[q];
        if (v < 0) {
            bi_out[q] = int64_t(1) << 40;  // never applies
            continue;
        }
        int64_t rank = 0;  // distinct valid blocks below v
        for (int64_t p = 0; p < n; ++p) rank += (first[p] && sbi[p] < v);
        bi_out[q] = rank;
        if (first[q]) {
            blocks[rank] = v;
            atomicAdd(&s_nb, 1);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int64_t nb = s_nb;
        nb_rows[0] = nb;
        // the (possibly partial) last row block sorts last in the compact set
        nb_rows[1] = nb == 0 ? 0
                     : (blocks[nb - 1] == nbi - 1 ? (nb - 1) * bm + (m - (nbi - 1) * bm) : nb * bm);
    }
}

// gather rows [blocks[b]*bm, +bm) (clipped to m) into a compact buffer
template <typename T>
__global__ void gather_blocks_kernel(const T *x, int64_t m, int64_t d, int64_t bm,
                                     const int64_t *blocks, int64_t nb, T *g,
                                     const int64_t *nb_dev = nullptr) {
    const int64_t n = (nb_dev ? *nb_dev : nb) * bm * d;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / d, f = e % d;
        const int64_t row = blocks[r / bm] * bm + r % bm;
        if (row < m) g[e] = x[row * d + f];
    }
}

template <typename T>
__global__ void scatter_blocks_kernel(const int32_t *idx, const T *val, int64_t m, int64_t bm,
                                      const int64_t *blocks, int64_t nb, int32_t *out_idx,
                                      T *out_val, const int64_t *nb_dev = nullptr) {
    if (nb_dev) nb = *nb_dev;
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < nb * bm;
         r += int64_t(gridDim.x) * blockDim.x) {
        const int64_t row = blocks[r / bm] * bm + r % bm;
        if (row < m) {
            out_idx[row] = idx[r];
            out_val[row] = val[r];
        }
    }
}

// lo[i] = v[i] - trunc_tf32(v[i]) (exact in fp32)
__global__ void split_lo_kernel(const float *v, int64_t n, float *lo) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        lo[i] = __fsub_rn(v[i], tf32_trunc(v[i]));
}

// Gather listed rows: g = x[rows], g_lo = g - trunc(g)  (count on device)
__global__ void gather_rows_kernel(const float *x, int64_t d, const int32_t *rows,
                                   const unsigned *count, float *g, float *g_lo) {
    const int64_t n = int64_t(*count) * d;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t q = e / d, f = e % d;
        const float v = x[int64_t(rows[q]) * d + f];
        g[e] = v;
        if (g_lo) g_lo[e] = __fsub_rn(v, tf32_trunc(v));
    }
}

template <typename T>
__global__ void scatter_rows_kernel(const int32_t *rows, const unsigned *count,
                                    const int32_t *idx, const T *val, int32_t *out_idx,
                                    T *out_val) {
    const unsigned n = *count;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += int64_t(gridDim.x) * blockDim.x) {
        out_idx[rows[q]] = idx[q];
        out_val[rows[q]] = val[q];
    }
}

// ------------------------------------------------------------- host ------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                    const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    });
    return fn;
}

static int make_map(CUtensorMap *map, const float *base, int64_t rows, int64_t cols,
                    uint32_t box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return FTK_ERR_CUDA;
    }
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows < 1 ? 1 : rows)};
    cuuint64_t strides[1] = {cuuint64_t(cols) * sizeof(float)};
    cuuint32_t box[2] = {TC_KB, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
        return FTK_ERR_CUDA;
    }
    return FTK_OK;
}

int make_tc_map(CUtensorMap *map, const float *base, int64_t rows, int64_t cols, uint32_t box_rows) {
    return make_map(map, base, rows, cols, box_rows);
}

// float64 rows, box = 16 doubles (one 128-byte swizzle row) x box_rows, 128B swizzle
int make_f64_map(CUtensorMap *map, const double *base, int64_t rows, int64_t cols, uint32_t box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return FTK_ERR_CUDA;
    }
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows < 1 ? 1 : rows)};
    cuuint64_t strides[1] = {cuuint64_t(cols) * sizeof(double)};
    cuuint32_t box[2] = {16, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (f64) failed (" + std::to_string(int(r)) + ")");
        return FTK_ERR_CUDA;
    }
    return FTK_OK;
}

// Unswizzled 2-D map with an arbitrary box (cols * 4 bytes a multiple of 16).
int make_plain_map(CUtensorMap *map, const float *base, int64_t rows, int64_t cols,
                   uint32_t box_cols, uint32_t box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return FTK_ERR_CUDA;
    }
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows < 1 ? 1 : rows)};
    cuuint64_t strides[1] = {cuuint64_t(cols) * sizeof(float)};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (plain) failed (" + std::to_string(int(r)) + ")");
        return FTK_ERR_CUDA;
    }
    return FTK_OK;
}

template <int BN, bool SPLIT, bool CHK>
static int launch_screen(TcParams P, const CUtensorMap &mx, const CUtensorMap &mxl,
                         const CUtensorMap &mc, const CUtensorMap &mcl, cudaStream_t st) {
    constexpr int NOP = SPLIT ? 2 : 1;
    const size_t a_bytes = size_t(P.nkb) * TC_BM * 128 * NOP;
    const size_t b_bytes = size_t(BN) * 128 * NOP;
    const size_t extra = 1024 + 256 + 2 * BN * sizeof(float);  // align slack, barriers, norms
    const size_t cap = 227 * 1024;
    // one persistent CTA per SM (TMEM: 2 x BN columns); prefer a double-
    // buffered X tile with >= 3 centroid stages, else a single buffer
    int abufs = 2;
    if (extra + 2 * a_bytes + 3 * b_bytes > cap) abufs = 1;
    if (const char *e = getenv("FTK_TC_ABUFS")) abufs = atoi(e) == 1 ? 1 : abufs;  // tuning
    int stages = int((cap - extra - abufs * a_bytes) / b_bytes);
    if (stages > 8) stages = 8;
    if (const char *e = getenv("FTK_TC_STAGES")) stages = atoi(e) < stages ? atoi(e) : stages;
    if (stages < 2) {
        set_error("tc: tile exceeds shared memory");
        return FTK_ERR_UNSUPPORTED;
    }
    P.stages = stages;
    P.abufs = abufs;
    const size_t smem = extra + abufs * a_bytes + size_t(stages) * b_bytes;
    const int64_t ntm = (P.m + TC_BM - 1) / TC_BM;
    if (ntm == 0) return FTK_OK;
    int nsm = 148;
    nsm = current_sm_count();
    const int64_t grid = ntm < nsm ? ntm : nsm;
    auto kern = tc_screen_kernel<BN, SPLIT, CHK>;
    FTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<dim3(unsigned(grid)), dim3(TC_THREADS), smem, st>>>(mx, mxl, mc, mcl, P);
    FTK_LAUNCHED("tc_screen_kernel");
    return FTK_OK;
}

template <bool SPLIT>
static int screen(int bn, const TcParams &P, const CUtensorMap &mx, const CUtensorMap &mxl,
                  const CUtensorMap &mc, const CUtensorMap &mcl, cudaStream_t st) {
    if (P.csum) {
        switch (bn) {
            case 32: return launch_screen<32, SPLIT, true>(P, mx, mxl, mc, mcl, st);
            case 64: return launch_screen<64, SPLIT, true>(P, mx, mxl, mc, mcl, st);
            case 128: return launch_screen<128, SPLIT, true>(P, mx, mxl, mc, mcl, st);
            default: return launch_screen<256, SPLIT, true>(P, mx, mxl, mc, mcl, st);
        }
    }
    switch (bn) {
        case 32: return launch_screen<32, SPLIT, false>(P, mx, mxl, mc, mcl, st);
        case 64: return launch_screen<64, SPLIT, false>(P, mx, mxl, mc, mcl, st);
        case 128: return launch_screen<128, SPLIT, false>(P, mx, mxl, mc, mcl, st);
        default: return launch_screen<256, SPLIT, false>(P, mx, mxl, mc, mcl, st);
    }
}

int tc_supported(int dtype, int64_t m, int64_t k, int64_t d) {
    // d > 256: the CTA-pair screen with X streamed through its stages (one
    // column tile, k <= 256) -- experimental, FTK_TC_SX=1: its exact refine
    // reads X rows from global memory and is latency-bound (c3 D=512 K=16:
    // pass 1 2.0 ms, 0.49 ms without the refine), no faster than the exact
    // kernel yet.  The resident-X kernels stop at 256.
    // d > 256: the streamed-X narrow screen (tc_narrow.cu, k + 4 <= 256) or
    // the CTA-pair screen with X streamed through its stages (any k)
    return dtype == FTK_F32 && d >= 4 && d % 4 == 0 &&
           (d <= TC_SX_MAX_D || narrow_supported(k, d, true)) && k >= 1 && m >= 1 &&
           m < (int64_t(1) << 31) && k < (int64_t(1) << 24);
}

// exact.cu: the tiled exact kernel (used on gathered tie rows)
int exact_run(ftk_ctx *, int, const void *, const void *, const void *, int64_t, int64_t, int64_t,
              int64_t, int64_t, int64_t, int32_t *, void *, void *, bool, double, double, int64_t,
              const ftk_injection *, ftk_events *, cudaStream_t);


  // pass-1 / pass-2 uncertified, TC ABFT flags


// FT mode helpers: checksum centroids for a given N tiling
static int prep_csum(ftk_ctx *ctx, int slot, const float *y, int64_t k, int64_t d, int nkb,
                     int trunc, float **csum, float **camax, cudaStream_t st,
                     float **csumw = nullptr) {
    const int64_t nf = int64_t(nkb) * 32;
    float *buf = static_cast<float *>(
        scratch(ctx, slot, sizeof(float) * (3 * nf + 64) + sizeof(double) * 3 * CSUM_SLICES * nf + 64, st));
    if (!buf) return FTK_ERR_CUDA;
    double *part = reinterpret_cast<double *>(buf + 3 * nf + 64);
    *csum = buf;
    *camax = buf + nf;  // [0] max|c|, [1] counter, [2] |csum|^2, [3] |csumw|^2
    float *fmax = buf + nf + 32;
    float *cw = buf + 2 * nf + 32;  // 16-byte aligned (nf % 32 == 0)
    if (csumw) *csumw = cw;
    unsigned *done = reinterpret_cast<unsigned *>(buf + nf + 1);
    FTK_CUDA(cudaMemsetAsync(done, 0, sizeof(unsigned), st));
    tile_csum_kernel<<<dim3(unsigned(nkb), CSUM_SLICES), 256, 0, st>>>(y, k, d, nkb, trunc, *csum, *camax,
                                                                     fmax, done, cw, part);
    FTK_LAUNCHED("tile_csum_kernel");
    return FTK_OK;
}

int prep_csum_run(ftk_ctx *ctx, int slot, const float *y, int64_t k, int64_t d, int nkb, int trunc,
                  float **csum, float **camax, cudaStream_t st, float **csumw) {
    return prep_csum(ctx, slot, y, k, d, nkb, trunc, csum, camax, st, csumw);
}

// Reference-identical handling of scheduled flips: the logical row blocks
// that carry an injection are recomputed by the exact checked kernel (the
// reference's detection / location / correction / events, bit for bit) and
// overwrite the TC results for those rows.
int exact_run_m(ftk_ctx *, int, const void *, const void *, const void *, int64_t, int64_t,
                int64_t, int64_t, int64_t, int64_t, int32_t *, void *, void *, bool, double, double,
                int64_t, const ftk_injection *, ftk_events *, cudaStream_t, const int64_t *);

// The same with the schedule's count on the device (ftk_injection.n_dev): no
// host round trip, so the pass stays capturable in a CUDA graph.  Buffers are
// sized for the capacity inj.n; the kernels read the live block / row counts.
template <typename T>
static int emulate_injected_blocks_dev(ftk_ctx *ctx, const T *xf, const T *yf, const T *ynf,
                                       int64_t m, int64_t k, int64_t d, const TcFt &ft,
                                       int32_t *out_idx, T *outv, cudaStream_t st) {
    const ftk_injection &inj = *ft.inj;
    const int64_t cap = inj.n;
    if (cap > 4096) {
        set_error("device-count injection: capacity above 4096 flips per pass");
        return FTK_ERR_ARG;
    }
    const int64_t nbi = (m + ft.bm - 1) / ft.bm;
    const int64_t nbc = cap < nbi ? cap : nbi;  // at most this many distinct row blocks
    const size_t need = sizeof(int64_t) * (nbc + cap + 8) +
                        sizeof(T) * (nbc * ft.bm * d + 2 * nbc * ft.bm) + 256;
    char *buf = static_cast<char *>(scratch(ctx, SLOT_INJ, need, st));
    if (!buf) return FTK_ERR_CUDA;
    int64_t *d_blocks = reinterpret_cast<int64_t *>(buf);
    int64_t *d_bi = d_blocks + nbc;
    int64_t *nb_rows = d_bi + cap;  // {distinct blocks, compact rows}
    T *g = reinterpret_cast<T *>(nb_rows + 8);
    T *gv = g + nbc * ft.bm * d;
    int32_t *gi = reinterpret_cast<int32_t *>(gv + nbc * ft.bm);
    inj_blocks_kernel<<<1, 256, size_t(cap) * 9 + 16, st>>>(inj, nbi, m, ft.bm, d_blocks, d_bi,
                                                            nb_rows);
    FTK_LAUNCHED("inj_blocks_kernel");
    gather_blocks_kernel<T><<<148, 256, 0, st>>>(xf, m, d, ft.bm, d_blocks, nbc, g, nb_rows);
    FTK_LAUNCHED("gather_blocks_kernel");
    ftk_injection rin = inj;
    rin.bi = d_bi;
    int rc = exact_run_m(ctx, sizeof(T) == 4 ? FTK_F32 : FTK_F64, g, yf, ynf, nbc * ft.bm, k, d,
                         ft.bm, ft.bn, ft.bk, gi, gv, nullptr, true, ft.delta_rel, ft.abs_tol,
                         ft.iteration, &rin, ft.ev, st, nb_rows + 1);
    if (rc) return rc;
    remap_events_kernel<<<1, 256, 0, st>>>(ft.ev->rec, ft.ev->count, ft.ev->cap, d_blocks);
    FTK_LAUNCHED("remap_events_kernel");
    scatter_blocks_kernel<T><<<148, 256, 0, st>>>(gi, gv, m, ft.bm, d_blocks, nbc, out_idx, outv,
                                                  nb_rows);
    FTK_LAUNCHED("scatter_blocks_kernel");
    return FTK_OK;
}

template <typename T>
int emulate_injected_blocks(ftk_ctx *ctx, const T *xf, const T *yf, const T *ynf, int64_t m,
                            int64_t k, int64_t d, const TcFt &ft, int32_t *out_idx, T *outv,
                            cudaStream_t st) {
    const ftk_injection &inj = *ft.inj;
    if (inj.n_dev)
        return emulate_injected_blocks_dev<T>(ctx, xf, yf, ynf, m, k, d, ft, out_idx, outv, st);
    std::vector<int64_t> bi(inj.n);
    FTK_CUDA(cudaMemcpyAsync(bi.data(), inj.bi, sizeof(int64_t) * inj.n, cudaMemcpyDeviceToHost, st));
    FTK_CUDA(cudaStreamSynchronize(st));
    const int64_t nbi = (m + ft.bm - 1) / ft.bm;
    std::vector<int64_t> blocks;
    for (int64_t v : bi)
        if (v >= 0 && v < nbi) blocks.push_back(v);
    std::sort(blocks.begin(), blocks.end());
    blocks.erase(std::unique(blocks.begin(), blocks.end()), blocks.end());
    if (blocks.empty()) return FTK_OK;
    // the (possibly partial) last row block must stay last in the compact set
    const int64_t nb = int64_t(blocks.size());
    const int64_t rows_c = (blocks.back() == nbi - 1) ? (nb - 1) * ft.bm + (m - (nbi - 1) * ft.bm)
                                                      : nb * ft.bm;
    const size_t need = sizeof(int64_t) * (2 * nb + 2 * inj.n + 8) +
                        sizeof(T) * (nb * ft.bm * d + 2 * nb * ft.bm) + 256;
    char *buf = static_cast<char *>(scratch(ctx, SLOT_INJ, need, st));
    if (!buf) return FTK_ERR_CUDA;
    int64_t *d_blocks = reinterpret_cast<int64_t *>(buf);
    int64_t *d_bi = d_blocks + nb;
    T *g = reinterpret_cast<T *>(d_bi + inj.n + 2);
    T *gv = g + nb * ft.bm * d;
    int32_t *gi = reinterpret_cast<int32_t *>(gv + nb * ft.bm);
    FTK_CUDA(cudaMemcpyAsync(d_blocks, blocks.data(), sizeof(int64_t) * nb, cudaMemcpyHostToDevice, st));
    remap_inj_kernel<<<1, 256, 0, st>>>(inj.bi, inj.n, d_blocks, nb, d_bi);
    FTK_LAUNCHED("remap_inj_kernel");
    gather_blocks_kernel<T><<<148, 256, 0, st>>>(xf, m, d, ft.bm, d_blocks, nb, g);
    FTK_LAUNCHED("gather_blocks_kernel");
    ftk_injection rin = inj;
    rin.bi = d_bi;
    int rc = exact_run(ctx, sizeof(T) == 4 ? FTK_F32 : FTK_F64, g, yf, ynf, rows_c, k, d, ft.bm,
                       ft.bn, ft.bk, gi, gv, nullptr,
                       true, ft.delta_rel, ft.abs_tol, ft.iteration, &rin, ft.ev, st);
    if (rc) return rc;
    remap_events_kernel<<<1, 256, 0, st>>>(ft.ev->rec, ft.ev->count, ft.ev->cap, d_blocks);
    FTK_LAUNCHED("remap_events_kernel");
    scatter_blocks_kernel<T><<<148, 256, 0, st>>>(gi, gv, m, ft.bm, d_blocks, nb, out_idx, outv);
    FTK_LAUNCHED("scatter_blocks_kernel");
    FTK_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope
    return FTK_OK;
}

int tc_assign_run(ftk_ctx *ctx, int dtype, const void *x, const void *y, const void *yn,
                  int64_t m, int64_t k, int64_t d, int32_t *out_idx, void *out_val,
                  cudaStream_t st, float *raw, int split_only, const TcFt *ft) {
    if (!tc_supported(dtype, m, k, d) || (ctx->family == 1 && d > TC_SX_MAX_D) ||
        (ctx->family == 2 && !narrow_supported(k, d, ft != nullptr))) {
        set_error("tc variant: unsupported shape/dtype");
        return FTK_ERR_UNSUPPORTED;
    }
    const float *xf = static_cast<const float *>(x), *yf = static_cast<const float *>(y);
    const float *ynf = static_cast<const float *>(yn);
    float *outv = static_cast<float *>(out_val);
    int bn = k > 128 ? 256 : (k > 64 ? 128 : (k > 32 ? 64 : 32));
    if (const char *e = getenv("FTK_TC_BN")) {  // tuning knob
        const int want = atoi(e);
        if ((want == 128 || want == 64 || want == 32) && want < bn) bn = want;
    }
    const int bn2 = k > 64 ? 128 : (k > 32 ? 64 : 32);  // pass 2: hi+lo operands
    float *misc = static_cast<float *>(scratch(ctx, SLOT_TC_MISC, 256, st));
    int32_t *rows1 = static_cast<int32_t *>(scratch(ctx, SLOT_TC_ROWS, sizeof(int32_t) * 2 * (m + 1), st));
    float *c_lo = static_cast<float *>(scratch(ctx, SLOT_TC_B, sizeof(float) * k * d, st));
    if (!misc || !rows1 || !c_lo) return FTK_ERR_CUDA;
    int32_t *rows2 = rows1 + (m + 1);
    unsigned *cnt = reinterpret_cast<unsigned *>(misc + 8);  // [0] pass-1, [1] pass-2, [2] abft
    FTK_CUDA(cudaMemsetAsync(misc, 0, 64, st));  // bounds + counters
    tc_prep_kernel<<<unsigned((k + 7) / 8 < 296 ? (k + 7) / 8 : 296), 256, 0, st>>>(yf, ynf, k, d,
                                                                                misc);
    FTK_LAUNCHED("tc_prep_kernel");

    TcParams P{};
    P.x = xf; P.y = yf; P.yn = ynf;
    P.m = m; P.k = k; P.d = d;
    P.nkb = int((d + TC_KB - 1) / TC_KB);
    P.b_coef = float((0x1p-14 + 0x1p-22) * 1.01);  // <= 255-ulp index packing + roundings
    P.cmax2 = misc;
    P.ecmax2 = misc + 1;
    P.out_idx = out_idx;
    P.out_val = outv;
    P.raw = raw;
    if (const char *e = getenv("FTK_TC_DEBUG")) P.dbg = atoi(e);  // pipeline-timing probe
    float *csum1 = nullptr, *camax1 = nullptr, *csum2 = nullptr, *camax2 = nullptr, *csumw1 = nullptr;
    if (ft) {
        int rc0 = prep_csum(ctx, SLOT_TC_CSUM1, yf, k, d, P.nkb, 1, &csum1, &camax1, st, &csumw1);
        if (rc0) return rc0;  // the 3xTF32 checksum centroid is built by the single-CTA pass 2
        P.tau_abs = float(ft->abs_tol);
        P.abft_count = cnt + 2;
        P.abft_total = abft_total_ptr(ctx, st);
        if (ft->inj && ft->inj->n > 0) {
            int32_t *ic = static_cast<int32_t *>(scratch(ctx, SLOT_TC_INJROWS, sizeof(float) * 3 * (m + 1), st));
            if (!ic) return FTK_ERR_CUDA;
            float *ib = reinterpret_cast<float *>(ic + (m + 1));
            float *ia = ib + (m + 1);
            FTK_CUDA(cudaMemsetAsync(ic, 0xFF, sizeof(int32_t) * m, st));  // -1: no flip
            inj_rows_kernel<<<1, 128, 0, st>>>(xf, yf, m, k, d, ft->bm, ft->bn, *ft->inj, ic, ib, ia);
            FTK_LAUNCHED("inj_rows_kernel");
            P.inj_col = ic;
            P.inj_before = ib;
            P.inj_after = ia;
        }
    }
    {
        const char *sx = getenv("FTK_TC_SX");
        // auto: wide rows go to the narrow screen when it can take k (the
        // variant table measures the rest; FTK_TC_SX=1 forces the pair screen)
        const bool narrow = ctx->family == 2 ||
                            (ctx->family == 0 && d > TC_MAX_D && !(sx && atoi(sx) == 1) &&
                             narrow_supported(k, d, ft != nullptr));
        if (!split_only && raw == nullptr && narrow && narrow_supported(k, d, ft != nullptr)) {
            // wide rows, few centroids: the streamed-X narrow screen
            NarrowIn in{};
            in.x = xf; in.y = yf; in.yn = ynf; in.m = m; in.k = k; in.d = d;
            in.out_idx = out_idx; in.out_val = outv;
            in.cmax2 = P.cmax2; in.ecmax2 = P.ecmax2;
            in.fb_rows = rows1; in.cnt = cnt; in.ft = ft;
            in.inj_col = P.inj_col; in.inj_before = P.inj_before; in.inj_after = P.inj_after;
            int rcn = narrow_assign_run(ctx, in, st);
            if (rcn) return rcn;
            if (ft && ft->inj && ft->inj->n > 0 && ctx->inj_replay)
                return emulate_injected_blocks(ctx, xf, yf, ynf, m, k, d, *ft, out_idx, outv, st);
            return FTK_OK;
        }
    }
    CUtensorMap mx, mc;
    constexpr unsigned kFlagCap = 4096;  // flagged rows recorded per pass (beyond: no event)
    double4 *flag_rec = nullptr;
    float *pair_fb_thr = nullptr;
    unsigned long long *pair_fb_seed = nullptr;
    int rc = make_map(&mc, yf, k, d, uint32_t(bn));
    if (rc) return rc;
    unsigned n1 = unsigned(m);
    const int32_t *pass2_rows = nullptr;
    if (!split_only) {
        // ---------------- pass 1: 1xTF32 over every row
        rc = make_map(&mx, xf, m, d, TC_BM);
        if (rc) return rc;
        P.ntiles = int((k + bn - 1) / bn);
        P.a_coef = float(3.0 * double(d) * 0x1p-24);  // accumulation terms (tight bound)
        P.fb_rows = rows1;
        P.fb_count = cnt;
        if (ft) {
            P.csum = csum1;
            P.camax = camax1;
            P.tau_coef = float(ft->delta_rel * double(d) * sqrt(double(k) / 32.0));
        }
        const char *pe = getenv("FTK_TC_PAIR");
        if (!(pe && atoi(pe) == 0) && d <= TC_SX_MAX_D && raw == nullptr) {
            // CTA-pair kernel (tc_pair.cu): M = 256 per cluster, half the L2 traffic
            CUtensorMap mc128;
            if ((rc = make_map(&mc128, yf, k, d, PAIR_BN / 2))) return rc;
            PairParams Q{};
            Q.x = xf; Q.y = yf; Q.yn = ynf; Q.m = m; Q.k = k; Q.d = d;
            Q.a_coef = P.a_coef; Q.b_coef = P.b_coef; Q.cmax2 = P.cmax2; Q.ecmax2 = P.ecmax2;
            Q.out_idx = out_idx; Q.out_val = outv; Q.fb_rows = rows1; Q.fb_count = cnt;
            Q.csum = P.csum; Q.camax = P.camax; Q.tau_coef = P.tau_coef; Q.tau_abs = P.tau_abs;
            Q.inj_col = P.inj_col; Q.inj_before = P.inj_before; Q.inj_after = P.inj_after;
            Q.hint = (ctx->hint && ctx->hint_m == m && !getenv("FTK_PAIR_NOHINT")) ? ctx->hint : nullptr;
            Q.abft_count = P.abft_count;
            Q.abft_total = P.abft_total;
            if (ft) {
                flag_rec = static_cast<double4 *>(scratch(ctx, SLOT_PAIR_FLAG, sizeof(double4) * kFlagCap, st));
                if (!flag_rec) return FTK_ERR_CUDA;
                Q.flag_rec = flag_rec;
                Q.flag_count = cnt + 5;
                Q.flag_cap = kFlagCap;
            }
            Q.dbg = P.dbg;
            if (ctx->rows_info && ctx->rows_x == x && ctx->rows_m == m && ctx->rows_d == d)
                Q.rowinfo = reinterpret_cast<const float4 *>(ctx->rows_info);
            {
                char *fb = static_cast<char *>(scratch(ctx, SLOT_PAIR_FB, (sizeof(float) + 8) * size_t(m + 1) + 64, st));
                if (!fb) return FTK_ERR_CUDA;
                Q.fb_seed = reinterpret_cast<unsigned long long *>(fb);
                Q.fb_thr = reinterpret_cast<float *>(fb + 8 * size_t(m + 1));
                pair_fb_thr = Q.fb_thr;
                pair_fb_seed = Q.fb_seed;
            }
            static long long *dclk = nullptr;  // FTK_PAIR_CLK=1: role timing printed to stderr
            const char *ce = getenv("FTK_PAIR_CLK");
            if (ce && atoi(ce)) {
                if (!dclk) cudaMalloc(&dclk, 10 * sizeof(long long));
                cudaMemsetAsync(dclk, 0, 10 * sizeof(long long), st);
                Q.clk = dclk;
            }
            if (!ctx->time_ev[0]) {  // pass-1 kernel timing
                cudaEventCreate(&ctx->time_ev[0]);
                cudaEventCreate(&ctx->time_ev[1]);
            }
            cudaEvent_t ev0 = ctx->time_ev[0], ev1 = ctx->time_ev[1];
            cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
            cudaStreamIsCapturing(st, &cap);
            const bool timed = cap == cudaStreamCaptureStatusNone;  // no timing inside graphs
            if (timed) cudaEventRecord(ev0, st);
            rc = pair_screen_launch(mx, mc128, Q, ft != nullptr, st);
            if (timed) {
                cudaEventRecord(ev1, st);
            }
            ctx->last_path = 1;
            if (Q.clk) {
                long long h[10];
                cudaMemcpyAsync(h, Q.clk, sizeof(h), cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                fprintf(stderr, "pair clk: screen busy %.0f wait %.0f per tile (%lld tiles); "
                        "mma wait t_empty %.0f full %.0f a_full %.0f per tile\n",
                        double(h[0]) / h[5], double(h[1]) / h[5], h[5], 2.0 * h[2] / h[5],
                        2.0 * h[3] / h[5], 2.0 * h[4] / h[5]);
                const double nrt = double(h[5]) / (P.ntiles > 0 ? double((k + 255) / 256) : 1.0);
                fprintf(stderr, "pair clk per row tile: refine wait %.0f busy %.0f (loop %.0f, post %.0f)\n", h[6] / nrt, h[7] / nrt, h[8] / nrt, h[9] / nrt);
            }
        } else {
            if (d > TC_MAX_D) {
                set_error("tc variant: d > 256 needs the CTA-pair screen");
                return FTK_ERR_UNSUPPORTED;
            }
            rc = screen<false>(bn, P, mx, mx, mc, mc, st);
            ctx->last_path = 0;
        }
        if (rc) return rc;
        if (ctx->last_path == 1) {
            // ---------------- pass 2, device-driven (no host synchronisation):
            // the rows pass 1 left uncertified (device count) are gathered and
            // re-screened by the CTA-pair kernel in COLLECT mode; every
            // centroid whose screened value can still beat the row's exact d1
            // is evaluated exactly; rows with too many candidates (or beyond
            // the pass-2 capacity) are resolved by exact_rows_kernel
            // rows pass 2 can take (the rest go to the exact row kernel): an
            // eighth of the rows, or 64 MB of gathered rows when D is small
            const unsigned cap_rows = unsigned(std::min<int64_t>(
                m, std::max<int64_t>(std::max<int64_t>(65536, m / 8), (int64_t(64) << 20) / (4 * d))));
            const unsigned row_cap = 256;
            const unsigned cap = unsigned(std::min<int64_t>(int64_t(cap_rows) * 16 + 65536, int64_t(1) << 30));
            const size_t gbytes = (sizeof(float) * size_t(cap_rows) * d + 255) & ~size_t(255);
            const size_t need = gbytes + sizeof(int2) * cap + 8 * size_t(cap_rows) + 4 * size_t(cap_rows) + 256;
            char *buf = static_cast<char *>(scratch(ctx, SLOT_PAIR_CAND, need, st));
            if (!buf) return FTK_ERR_CUDA;
            float *g = reinterpret_cast<float *>(buf);
            int2 *cand = reinterpret_cast<int2 *>(buf + gbytes);
            unsigned long long *key = reinterpret_cast<unsigned long long *>(cand + cap);
            unsigned *row_cnt = reinterpret_cast<unsigned *>(key + cap_rows);
            unsigned *ccount = row_cnt + cap_rows;  // [0] candidates, [1] rows for the exact kernel
            FTK_CUDA(cudaMemsetAsync(ccount, 0, 2 * sizeof(unsigned), st));
            if ((rc = pass2_gather_run(xf, d, rows1, cnt, cap_rows, pair_fb_seed, g, key, row_cnt, st)))
                return rc;
            CUtensorMap mg, mc64;
            if ((rc = make_map(&mg, g, cap_rows, d, TC_BM)) ||
                (rc = make_map(&mc64, yf, k, d, PAIR_BN / 2)))
                return rc;
            PairParams Q{};
            Q.x = g; Q.y = yf; Q.yn = ynf; Q.m = cap_rows; Q.k = k; Q.d = d;
            Q.m_dev = cnt;
            Q.cmax2 = P.cmax2; Q.ecmax2 = P.ecmax2;
            Q.thr = pair_fb_thr;
            Q.cand = cand;
            Q.cand_count = ccount;
            Q.cand_cap = cap;
            Q.row_cnt = row_cnt;
            if ((rc = pair_screen_launch(mg, mc64, Q, false, st))) return rc;
            if ((rc = pair_candidates_run(g, yf, ynf, d, cand, ccount, cap, row_cnt, row_cap, key,
                                          rows1, cnt, cap_rows, out_idx, outv, rows2, ccount + 1, st)))
                return rc;
            if ((rc = exact_rows_run(xf, yf, ynf, k, d, rows2, ccount + 1, out_idx, outv, st))) return rc;
            if (getenv("FTK_TC_P2_DEBUG")) {  // diagnostics: pass-2 rows and candidates
                unsigned h[3] = {0, 0, 0};
                cudaMemcpyAsync(h, cnt, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
                cudaMemcpyAsync(h + 1, ccount, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                fprintf(stderr, "pass 2: %u rows, %u candidates, %u rows to the exact kernel\n", h[0], h[1], h[2]);
            }
            ctx->stat_dev[0] = cnt;          // read lazily by tc_last_fallback
            ctx->stat_dev[1] = ccount + 1;
            ctx->stat_dev[2] = ft ? cnt + 2 : nullptr;
            if (ft) {
                // location + event records of the flagged rows (pass 2 has
                // re-resolved them: the correction)
                FlagEvents F{};
                F.x = xf; F.d = d; F.k = k;
                F.csumw = csumw1; F.camax = camax1;
                F.rec = flag_rec; F.count = cnt + 5; F.cap = kFlagCap;
                F.inj_col = P.inj_col;
                F.events_for_scheduled = ctx->inj_replay ? 0 : 1;
                if (ft->ev) F.ev = *ft->ev;
                F.iteration = ft->iteration;
                F.bm = ft->bm;
                F.bn = ft->bn;
                F.interval = ft->bk > 0 ? (d + ft->bk - 1) / ft->bk - 1 : 0;
                F.corrected = cnt + 4;
                if ((rc = abft_flag_events_run(F, st))) return rc;
            }
            if (ft && ft->inj && ft->inj->n > 0 && ctx->inj_replay)
                return emulate_injected_blocks(ctx, xf, yf, ynf, m, k, d, *ft, out_idx, outv, st);
            return FTK_OK;
        }
        FTK_CUDA(cudaMemcpyAsync(&n1, cnt, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        FTK_CUDA(cudaStreamSynchronize(st));
        pass2_rows = rows1;
    }
    ctx->stat_dev[0] = ctx->stat_dev[1] = ctx->stat_dev[2] = nullptr;
    ctx->last_fb[0] = n1;
    ctx->last_fb[1] = 0;
    if (n1 > 0) {
        // ---------------- pass 2: 3xTF32 over the gathered uncertified rows
        float *g = static_cast<float *>(scratch(ctx, SLOT_TC_A, sizeof(float) * 2 * size_t(n1) * d + 64, st));
        if (!g) return FTK_ERR_CUDA;
        float *g_lo = g + size_t(n1) * d;
        if (split_only) {
            // identity row list for a direct 3xTF32 call (testing / forced mode)
            std::vector<int32_t> ids(m);
            for (int64_t i = 0; i < m; ++i) ids[i] = int32_t(i);
            FTK_CUDA(cudaMemcpyAsync(rows1, ids.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
            FTK_CUDA(cudaMemcpyAsync(cnt, &n1, sizeof(unsigned), cudaMemcpyHostToDevice, st));
            FTK_CUDA(cudaStreamSynchronize(st));
            pass2_rows = rows1;
        }
        gather_rows_kernel<<<148 * 8, 256, 0, st>>>(xf, d, pass2_rows, cnt, g, g_lo);
        FTK_LAUNCHED("gather_rows_kernel");
        split_lo_kernel<<<148 * 4, 256, 0, st>>>(yf, k * d, c_lo);
        FTK_LAUNCHED("split_lo_kernel");
        CUtensorMap mg, mgl, mc2, mcl2;
        if ((rc = make_map(&mg, g, n1, d, TC_BM)) || (rc = make_map(&mgl, g_lo, n1, d, TC_BM)) ||
            (rc = make_map(&mc2, yf, k, d, uint32_t(bn2))) ||
            (rc = make_map(&mcl2, c_lo, k, d, uint32_t(bn2))))
            return rc;
        TcParams Q = P;
        Q.x = g;
        Q.m = n1;
        Q.ntiles = int((k + bn2 - 1) / bn2);
        Q.a_coef = float(2.0 * (3.0 * 0x1p-20 + 7.0 * double(d) * 0x1p-24) * (1.0 + 0x1p-10));
        Q.rows = pass2_rows;
        Q.fb_rows = rows2;
        Q.fb_count = cnt + 1;
        Q.raw = split_only ? raw : nullptr;
        Q.inj_col = nullptr;  // pass-1 flips do not recur in the re-screen
        if (ft) {
            if ((rc = prep_csum(ctx, SLOT_TC_CSUM2, yf, k, d, P.nkb, 0, &csum2, &camax2, st))) return rc;
            Q.csum = csum2;
            Q.camax = camax2;
            Q.tau_coef = float(ft->delta_rel * double(d) * sqrt(double(k) / 32.0));
        }
        rc = screen<true>(bn2, Q, mg, mgl, mc2, mcl2, st);
        unsigned n2 = 0;
        unsigned *cnt2 = cnt + 1;
        if (rc == FTK_ERR_UNSUPPORTED) {
            // hi+lo X tile does not fit (large D): every pass-1 tie goes exact
            rows2 = const_cast<int32_t *>(pass2_rows);
            n2 = n1;
            cnt2 = cnt;
            rc = FTK_OK;
        } else {
            if (rc) return rc;
            FTK_CUDA(cudaMemcpyAsync(&n2, cnt2, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
            FTK_CUDA(cudaStreamSynchronize(st));
        }
        ctx->last_fb[1] = n2;
        if (n2 > 0) {
            // ---------------- exact resolution of the remaining ties (tiled SIMT kernel)
            gather_rows_kernel<<<148 * 4, 256, 0, st>>>(xf, d, rows2, cnt2, g, nullptr);
            FTK_LAUNCHED("gather_rows_kernel");
            int32_t *idx2 = reinterpret_cast<int32_t *>(g_lo);
            float *val2 = g_lo + n2;
            // 8-row slabs: few rows, so spread them over many CTAs
            rc = exact_run(ctx, FTK_F32, g, yf, ynf, n2, k, d, 8, 256, 16, idx2, val2, nullptr,
                           false, 0.0, 0.0, 0, nullptr, nullptr, st);
            if (rc) return rc;
            scatter_rows_kernel<float><<<148, 256, 0, st>>>(rows2, cnt2, idx2, val2, out_idx, outv);
            FTK_LAUNCHED("scatter_rows_kernel");
        }
    }
    if (ft) {
        unsigned nab = 0;
        FTK_CUDA(cudaMemcpyAsync(&nab, cnt + 2, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        FTK_CUDA(cudaStreamSynchronize(st));
        ctx->last_fb[2] = nab;
        if (ft->inj && ft->inj->n > 0)
            return emulate_injected_blocks(ctx, xf, yf, ynf, m, k, d, *ft, out_idx, outv, st);
    }
    return FTK_OK;
}

int tc_checked_run(ftk_ctx *ctx, int dtype, const void *x, const void *y, const void *yn,
                   int64_t m, int64_t k, int64_t d, int64_t bm, int64_t bn, int64_t bk,
                   double delta_rel, double abs_tol, int64_t iteration, int32_t *out_idx,
                   void *out_val, const ftk_injection *inj, ftk_events *ev, cudaStream_t st) {
    TcFt ft{delta_rel, abs_tol, bm, bn, bk, iteration, inj, ev};
    return tc_assign_run(ctx, dtype, x, y, yn, m, k, d, out_idx, out_val, st, nullptr, 0, &ft);
}

template int emulate_injected_blocks<double>(ftk_ctx *, const double *, const double *,
                                             const double *, int64_t, int64_t, int64_t,
                                             const TcFt &, int32_t *, double *, cudaStream_t);

// Device time of the last CTA-pair pass-1 launch (ms), -1 if none.
float tc_last_pass1_ms(ftk_ctx *ctx) {
    if (!ctx->time_ev[0] || (ctx->last_path != 1 && ctx->last_path != 2)) return -1.0f;
    float ms = -1.0f;
    if (cudaEventSynchronize(ctx->time_ev[1]) != cudaSuccess) return -1.0f;
    cudaEventElapsedTime(&ms, ctx->time_ev[0], ctx->time_ev[1]);
    return ms;
}

int tc_last_fallback(ftk_ctx *ctx, unsigned *out, cudaStream_t st) {
    if (ctx->stat_dev[0]) {  // device-driven pass 2: counters still on the device
        FTK_CUDA(cudaStreamSynchronize(st));
        for (int q = 0; q < 3; ++q) {
            ctx->last_fb[q] = 0;
            if (ctx->stat_dev[q])
                FTK_CUDA(cudaMemcpy(&ctx->last_fb[q], ctx->stat_dev[q], sizeof(unsigned), cudaMemcpyDeviceToHost));
        }
    }
    out[0] = ctx->last_fb[0];
    out[1] = ctx->last_fb[1];
    out[2] = ctx->last_fb[2];
    return FTK_OK;
}

}  // namespace ftk
