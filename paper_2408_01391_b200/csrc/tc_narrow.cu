// tc_narrow.cu -- streamed-X tensor-core screen for narrow centroid sets over
// wide rows: K + 4 <= 256 centroids, any D >= 4 with D % 4 == 0 (BASELINE
// c3's K in {8,16,32} x D in {512, 2048}).  One pass there does 2K flops per
// 4-byte feature of X: HBM-bound, so X must be read exactly once and nothing
// may stall the stream.
//
// Persistent, one CTA per SM over 128-row tiles.  Every 32-feature k-block
// travels through a TMA ring as ONE stage: the X tile slice (128 x 32 fp32,
// 16 KB, 128-byte swizzle) plus the same slice of the augmented centroid
// matrix (Kp x 32).  Per stage, concurrently:
//   MMA warp      4 x tcgen05.mma.kind::tf32 (M=128, N=Kp, K=8) into TMEM,
//                 two accumulator buffers (tile t+1's MMAs overlap t's epilogue)
//   chain warps   (w0..w3, one row per thread) the reference's exact dot
//                 x . c_p, sequential fp32 products and sums, k ascending
//                 (_kernels.py:44-70), for the row's HINTED centroid p (the
//                 previous Lloyd iteration's label, ftk_ctx_set_label_hint),
//                 read from the same shared-memory stage
// so the exact value of the winner is ready when the screen's winner is the
// hint -- nearly every row once Lloyd settles -- and X is never read twice.
//   epilogue warps (w4..w7, one row per thread) drain TMEM: ABFT row
//                 checksums (detect, locate, correct in registers), then the
//                 screen s_j = yn_j - 2 acc_j with a running (index, top-2),
//                 then the certificate against the exact value.
// Rows whose screened winner is not the hint are finished by
// narrow_winner_kernel (the winner's exact value from global memory, same
// certificate); rows no certificate covers go to exact_rows_kernel
// (tc_pair.cu), the reference's full chain over every centroid.
//
// Certificate (tc.cu header): |s_j - ref_j| <= A + B|s_j| for every column,
// so m2 - A - B|m2| > d1 (d1 exact for the screened winner j1, m2 the second
// smallest screened value) proves j1 is the reference's strict argmin.
//
// ABFT (CHK).  The augmented matrix carries four more rows: the checksum
// centroid csum = sum_j c~_j and the weighted one wsum = sum_j (j+1) c~_j,
// each split hi + lo into two tf32-exact rows (c~ = tf32(c), the operand the
// tensor core multiplies).  The MMA itself therefore produces the reference
// checksums x~.csum and x~.wsum next to the K distances, and the epilogue forms
//   D1 = sum_j acc_j - x~.csum,      D2 = sum_j (j+1) acc_j - x~.wsum.
// |D1| > tau detects an error in the row (tau: the reference's tolerance,
// delta_rel * max(1, amax_x amax_y) * k_acc + abs_tol, with k_acc = D and the
// K-column sum, plus the fp32 evaluation error of the checksums),
// j = rint(D2 / D1) - 1 locates its column, and acc_j <- x~.csum -
// sum_{i != j} acc_i corrects it in registers before the screen -- the
// location-encoded online correction of PAPER.md:204-223, with no
// recomputation.  The certificate of a corrected row is widened by the
// correction's own error bound (K column errors + the checksum's), so a
// wrong location can never yield a wrong label, only an exact re-resolution
// of that row.  Rows carrying a SCHEDULED flip (fault injection) are
// corrected the same way, but their logical row blocks are then replayed by
// the exact checked kernel (tc.cu emulate_injected_blocks) so the event
// record is the reference's own; every other detection writes its own
// DetectionEvent (kind detected-corrected / detected-uncorrectable, tile and
// location in the logical fault-tile grid), which the host counts as a false
// alarm when its tile carries no scheduled flip (abft.py:333-334).

#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tc_pair.cuh"

namespace ftk {

constexpr int NR_BM = 128;               // rows per tile (UMMA M)
constexpr int NR_KB = 32;                // fp32 features per 128-byte swizzle row
constexpr uint32_t NR_A_KB = NR_BM * 128;  // X bytes per stage
constexpr int NR_MAX_N = 256;            // UMMA N limit (K + checksum rows, padded to 16)
constexpr int NR_THREADS = 320;          // 10 warps
constexpr int NW_EPI0 = 4;               // w0..3 chain, w4..7 epilogue
constexpr int NW_PROD = 8;               // TMA producer
constexpr int NW_MMA = 9;                // TMEM allocator + MMA issuer

struct NarrowParams {
    const float *yn;  // k exact fp32 norms (reference order)
    int64_t m, k, d;
    int kp;       // MMA N: rows of the augmented centroid matrix, padded to 16
    int kt;       // width of the transposed chain operand (k rounded up to 4), 0: none
    int bstride;  // TMEM columns between the two accumulator buffers
    int nkb, stages;
    float a_coef, b_coef;
    const float *cmax2, *ecmax2;  // device scalars (tc_prep_kernel)
    const int32_t *hint;          // m labels (previous iteration) or null
    const float4 *rowinfo;        // per-fit row bounds or null
    int32_t *out_idx;
    float *out_val;
    int32_t *rf_rows;   // rows the screen could not finish alone (resolve pass)
    float4 *rf_rec;     // 2 per row: (j1, j2 bits, A, d1), (m2, m3, d1 known, 0)
    unsigned *rf_count;
    int32_t *fb_rows;   // rows for the exact kernel
    unsigned *fb_count;
    // ABFT
    const float *cinfo;  // [0] max|c|, [1] |csum|, [2] |wsum|
    float tau_coef, tau_abs;
    const int32_t *inj_col;
    const float *inj_before, *inj_after;
    unsigned *abft_count;             // rows whose checksum failed (this call)
    unsigned long long *abft_total;   // cumulative (ftk_abft_flags_total)
    unsigned *corrected;              // located + corrected in registers (this call)
    int64_t ev_cap;
    int64_t *ev_rec;
    double *ev_delta;
    unsigned long long *ev_count;
    int64_t iteration, bm, bn, interval;
    int events_for_scheduled;  // test mode: scheduled flips are not replayed, record them here
};

struct ChainRes {
    float acc, xx, ee, amax;
};

// a scheduled flip on the TMEM-loaded accumulator of column e (0..15)
__device__ __forceinline__ void inject16(uint32_t (&v)[16], int e, float before, float after) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
        if (u == e) {
            const float cur = __uint_as_float(v[u]);
            v[u] = __float_as_uint(isfinite(after) ? cur + (after - before) : after);
        }
}

// every column whose screened value is >= mv is provably above d (mv = +inf:
// there is no such column)
__device__ __forceinline__ bool narrow_cert(float mv, float A, float b, float d) {
    return mv == INFINITY || (mv - A - b * fabsf(mv) > d);
}

template <bool CHK, bool INJ>
__global__ void __launch_bounds__(NR_THREADS, 1)
    narrow_screen_kernel(const __grid_constant__ CUtensorMap tmX,
                         const __grid_constant__ CUtensorMap tmC,
                         const __grid_constant__ CUtensorMap tmCt, NarrowParams P) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int S = P.stages, nkb = P.nkb, kp = P.kp, kt = P.kt;
    // stage: X slice | centroid slice (swizzled, MMA) | transposed centroid
    // slice (chain operand), padded to 1024 B for the next swizzled X slice
    const uint32_t C_OFF = NR_A_KB, CT_OFF = NR_A_KB + uint32_t(kp) * 128u;
    const uint32_t TX = CT_OFF + uint32_t(kt) * 128u;
    const uint32_t STG = (TX + 1023u) & ~1023u;
    unsigned char *sS = smem;
    float *yns = reinterpret_cast<float *>(sS + size_t(S) * STG);  // [NR_MAX_N]
    ChainRes *cres = reinterpret_cast<ChainRes *>(yns + NR_MAX_N);  // [2][128]
    uint64_t *bars = reinterpret_cast<uint64_t *>(cres + 2 * NR_BM);
    uint64_t *full = bars, *empty = bars + S;
    uint64_t *t_full = bars + 2 * S, *t_empty = t_full + 2;
    uint64_t *c_full = t_empty + 2, *c_empty = c_full + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(c_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t M = P.m, K = P.k, D = P.d;
    const int64_t ntm = (M + NR_BM - 1) / NR_BM;
    uint32_t ncols = 32;
    while (ncols < uint32_t(2 * P.bstride)) ncols <<= 1;

    if (warp == NW_PROD && lane == 0) {
        prefetch_tmap(&tmX);
        prefetch_tmap(&tmC);
        if (kt) prefetch_tmap(&tmCt);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1 + 4);  // MMA commit + the 4 chain warps
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&t_full[b], 1);
            mbar_init(&t_empty[b], 4);
            mbar_init(&c_full[b], 4);
            mbar_init(&c_empty[b], 4);
        }
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < NR_MAX_N; i += NR_THREADS) yns[i] = i < K ? __ldg(P.yn + i) : INFINITY;
    if (warp == NW_MMA) tmem_alloc(tmem_slot, ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == NW_PROD) {
        // ---------------------------------------------------- TMA producer --
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t rt = blockIdx.x; rt < ntm; rt += gridDim.x)
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], TX);
                    unsigned char *dst = sS + size_t(stage) * STG;
                    tma_load_2d(dst, &tmX, &full[stage], kb * NR_KB, int(rt * NR_BM));
                    tma_load_2d(dst + C_OFF, &tmC, &full[stage], kb * NR_KB, 0);
                    if (kt) tma_load_2d(dst + CT_OFF, &tmCt, &full[stage], 0, kb * NR_KB);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
        }
    } else if (warp == NW_MMA) {
        // ----------------------------------------------------- MMA issuer --
        if (lane == 0) {
            const uint32_t idesc = idesc_tf32(NR_BM, kp);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int64_t rt = blockIdx.x; rt < ntm; rt += gridDim.x, ++it) {
                const int buf = it & 1;
                mbar_wait(&t_empty[buf], (uint32_t(it >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + uint32_t(buf * P.bstride);
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t as = smem_u32(sS + size_t(stage) * STG);
                    const uint32_t bs = as + NR_A_KB;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_tf32(d_tmem, smem_desc(as + kk * 32), smem_desc(bs + kk * 32), idesc,
                                 (kb | kk) != 0);
                    mma_commit(&empty[stage]);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
                mma_commit(&t_full[buf]);
            }
        }
    } else if (warp < NW_EPI0) {
        // ------------------------------------------ exact chain of the hint --
        const int r = warp * 32 + lane;
        const bool need_info = P.rowinfo == nullptr;
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int64_t rt = blockIdx.x; rt < ntm; rt += gridDim.x, ++it) {
            const int cb = it & 1;
            const int64_t grow = rt * NR_BM + r;
            int p = -1;
            if (P.hint && grow < M) {
                p = __ldg(P.hint + grow);
                if (p < 0 || p >= K) p = -1;
            }
            const bool work = __any_sync(0xffffffffu, p >= 0 || (need_info && grow < M));
            float acc = 0.0f, xx = 0.0f, ee = 0.0f, amax = 0.0f;
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&full[stage], phase);
                if (work) {
                    // all 16 shared-memory loads of the stage first, then the 32
                    // independent products (they consume every loaded register,
                    // so the loads have completed), then the stage is released,
                    // then the dependent fp32 chain (32 FADDs) runs while the
                    // producer refills the stage.
                    // Features past D are zero in both TMA slices, and x*c = 0
                    // leaves the chain unchanged (acc is never -0).
                    const unsigned char *xs = sS + size_t(stage) * STG + uint32_t(r) * 128u;
                    const int pp = p < 0 ? 0 : p;
                    const unsigned char *cs = sS + size_t(stage) * STG + C_OFF + uint32_t(pp) * 128u;
                    const float *ct = reinterpret_cast<const float *>(sS + size_t(stage) * STG + CT_OFF) + pp;
                    float4 xv[8], cv[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) xv[q] = *reinterpret_cast<const float4 *>(xs + ((q ^ (r & 7)) << 4));
                    if (kt) {
                        // transposed slice: element (f, p) at f * kt + p
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            cv[q] = make_float4(ct[(4 * q + 0) * kt], ct[(4 * q + 1) * kt],
                                                ct[(4 * q + 2) * kt], ct[(4 * q + 3) * kt]);
                    } else {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            cv[q] = *reinterpret_cast<const float4 *>(cs + ((q ^ (pp & 7)) << 4));
                    }
                    float pr[32];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        pr[4 * q + 0] = __fmul_rn(xv[q].x, cv[q].x);
                        pr[4 * q + 1] = __fmul_rn(xv[q].y, cv[q].y);
                        pr[4 * q + 2] = __fmul_rn(xv[q].z, cv[q].z);
                        pr[4 * q + 3] = __fmul_rn(xv[q].w, cv[q].w);
                    }
                    if (need_info) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 v = xv[q];
                            xx = fmaf(v.x, v.x, xx);
                            xx = fmaf(v.y, v.y, xx);
                            xx = fmaf(v.z, v.z, xx);
                            xx = fmaf(v.w, v.w, xx);
                            const float r0 = v.x - tf32_trunc(v.x), r1 = v.y - tf32_trunc(v.y);
                            const float r2 = v.z - tf32_trunc(v.z), r3 = v.w - tf32_trunc(v.w);
                            ee = fmaf(r0, r0, ee);
                            ee = fmaf(r1, r1, ee);
                            ee = fmaf(r2, r2, ee);
                            ee = fmaf(r3, r3, ee);
                            amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)),
                                                     fmaxf(fabsf(v.z), fabsf(v.w))));
                        }
                    }
                    // the products (and the bounds) hold every value the stage
                    // supplied: make the warp's loads complete, then release it
                    asm volatile("" ::"f"(pr[0]), "f"(pr[1]), "f"(pr[2]), "f"(pr[3]), "f"(pr[4]),
                                 "f"(pr[5]), "f"(pr[6]), "f"(pr[7]), "f"(pr[8]), "f"(pr[9]),
                                 "f"(pr[10]), "f"(pr[11]), "f"(pr[12]), "f"(pr[13]), "f"(pr[14]),
                                 "f"(pr[15]), "f"(pr[16]), "f"(pr[17]), "f"(pr[18]), "f"(pr[19]),
                                 "f"(pr[20]), "f"(pr[21]), "f"(pr[22]), "f"(pr[23]), "f"(pr[24]),
                                 "f"(pr[25]), "f"(pr[26]), "f"(pr[27]), "f"(pr[28]), "f"(pr[29]),
                                 "f"(pr[30]), "f"(pr[31]));
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[stage]);
                    if (p >= 0) {
#pragma unroll
                        for (int e = 0; e < 32; ++e) acc = __fadd_rn(acc, pr[e]);
                    }
                } else {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[stage]);
                }
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
            mbar_wait(&c_empty[cb], (uint32_t(it >> 1) & 1) ^ 1);
            cres[cb * NR_BM + r] = ChainRes{acc, xx, ee, amax};
            __syncwarp();
            if (lane == 0) mbar_arrive(&c_full[cb]);
        }
    } else if (warp < NW_PROD) {
        // -------------------------------------------------------- epilogue --
        const int q4 = warp - NW_EPI0;
        const int r = q4 * 32 + lane;
        const uint32_t lane_base = uint32_t(q4 * 32) << 16;
        const int nch = kp >> 4;
        const int kk = int(K);
        const float cm = sqrtf(*P.cmax2 * (1.0f + 0x1p-10f));
        const float ecm = sqrtf(*P.ecmax2 * (1.0f + 0x1p-10f));
        int it = 0;
        for (int64_t rt = blockIdx.x; rt < ntm; rt += gridDim.x, ++it) {
            const int buf = it & 1;
            const int64_t grow = rt * NR_BM + r;
            const bool live = grow < M;
            // the chain warps' results for this tile (its X is fully consumed)
            mbar_wait(&c_full[buf], uint32_t(it >> 1) & 1);
            const ChainRes cr = cres[buf * NR_BM + r];
            __syncwarp();
            if (lane == 0) mbar_arrive(&c_empty[buf]);
            float xx = cr.xx, ee = cr.ee, amax = cr.amax;
            if (P.rowinfo && live) {
                const float4 ri = __ldg(P.rowinfo + grow);
                xx = ri.x;
                ee = ri.y;
                amax = ri.z;
            }
            int p = -1;
            if (P.hint && live) {
                p = __ldg(P.hint + grow);
                if (p < 0 || p >= K) p = -1;
            }
            int inj_c = -1;
            float inj_b = 0.0f, inj_a = 0.0f;
            if (INJ && live) {
                inj_c = __ldg(P.inj_col + grow);
                if (inj_c >= 0) {
                    inj_b = __ldg(P.inj_before + grow);
                    inj_a = __ldg(P.inj_after + grow);
                }
            }
            mbar_wait(&t_full[buf], uint32_t(it >> 1) & 1);
            tc_fence_after();
            const uint32_t tb = tmem + lane_base + uint32_t(buf * P.bstride);
            uint32_t v[16];
            auto ldv = [&](int ch) {
                tmem_ld16(tb + uint32_t(ch * 16), v);
                if (INJ && inj_c >= 0 && (inj_c >> 4) == ch) inject16(v, inj_c & 15, inj_b, inj_a);
            };
            const float xn = sqrtf(xx * (1.0f + 0x1p-10f));
            // ---- ABFT: detect, locate, correct in registers
            bool flagged = false, located = false;
            int jl = -1;
            float fix = 0.0f, tau = 0.0f, D1 = 0.0f;
            if (CHK) {
                float s1 = 0.0f, w1 = 0.0f, c1 = 0.0f, c2 = 0.0f;
#pragma unroll 1
                for (int ch = 0; ch < nch; ++ch) {
                    ldv(ch);
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int j = ch * 16 + e;
                        const float a = __uint_as_float(v[e]);
                        if (j < kk) {
                            s1 += a;
                            w1 = fmaf(float(j + 1), a, w1);
                        } else if (j < kk + 2) {
                            c1 += a;  // x~.csum_hi + x~.csum_lo
                        } else if (j < kk + 4) {
                            c2 += a;  // x~.wsum_hi + x~.wsum_lo
                        }
                    }
                }
                D1 = s1 - c1;
                const float D2 = w1 - c2;
                // reference tolerance (k_acc = D) + the fp32 evaluation error of
                // the K-column sum and of the hi/lo checksum products
                tau = P.tau_coef * fmaxf(1.0f, amax * P.cinfo[0]) + P.tau_abs +
                      0x1p-18f * xn * P.cinfo[1];
                flagged = live && !(fabsf(D1) <= tau);
                if (flagged) {
                    const float jf = rintf(D2 / D1) - 1.0f;
                    if (jf >= 0.0f && jf < float(kk)) {  // NaN / inf fail here
                        jl = int(jf);
                        const float tw = float(kk + 1) * tau + 0x1p-18f * xn * P.cinfo[2] +
                                         fabsf(D1) * float(kk + 1) * 0x1p-20f;
                        located = fabsf(D2 - float(jl + 1) * D1) <= tw;
                    }
                }
                if (__any_sync(0xffffffffu, located)) {
                    // the corrected accumulator: checksum minus the other columns
                    float sx = 0.0f;
#pragma unroll 1
                    for (int ch = 0; ch < nch; ++ch) {
                        ldv(ch);
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const int j = ch * 16 + e;
                            if (j < kk && j != jl) sx += __uint_as_float(v[e]);
                        }
                    }
                    fix = c1 - sx;
                }
                if (flagged) {
                    atomicAdd(P.abft_count, 1u);
                    if (P.abft_total) atomicAdd(P.abft_total, 1ull);
                    if (located) atomicAdd(P.corrected, 1u);
                    // scheduled flips get the reference's own record from the
                    // exact replay of their logical block
                    if (P.ev_rec && (inj_c < 0 || P.events_for_scheduled)) {
                        const unsigned long long c = atomicAdd(P.ev_count, 1ull);
                        if (c < (unsigned long long)P.ev_cap) {
                            int64_t *rec = P.ev_rec + c * 7;
                            const int64_t col = located ? jl : 0;
                            rec[0] = P.iteration;
                            rec[1] = grow / P.bm;
                            rec[2] = col / P.bn;
                            rec[3] = located ? 0 : 1;  // EV_CORRECTED / EV_UNCORRECTABLE
                            rec[4] = grow % P.bm;
                            rec[5] = located ? col % P.bn : -1;
                            rec[6] = P.interval;
                            P.ev_delta[c] = double(D1);
                        }
                    }
                }
            }
            // ---- screen: running (index, index, value) top-3 of s_j = yn_j - 2 acc_j
            float m1 = INFINITY, m2 = INFINITY, m3 = INFINITY;
            int j1 = 0, j2 = 0;
#pragma unroll 1
            for (int ch = 0; ch < nch; ++ch) {
                ldv(ch);
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int j = ch * 16 + e;
                    if (j < kk) {
                        float a = __uint_as_float(v[e]);
                        if (CHK && located && j == jl) a = fix;
                        const float s = fmaf(-2.0f, a, yns[j]);
                        if (s < m1) {
                            m3 = m2;
                            m2 = m1;
                            j2 = j1;
                            m1 = s;
                            j1 = j;
                        } else if (s < m2) {
                            m3 = m2;
                            m2 = s;
                            j2 = j;
                        } else {
                            m3 = fminf(m3, s);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&t_empty[buf]);
            // ---- certificate
            bool ok = false, to_winner = false, d1_known = false;
            float dval = 0.0f, A = 0.0f;
            if (live) {
                A = 2.0f * (1.0f + 0x1p-10f) *
                    (sqrtf(ee * (1.0f + 0x1p-10f)) * cm + xn * ecm + P.a_coef * xn * cm);
                // a corrected column is x~.c~_j up to the other columns' fp32
                // accumulation errors, the checksum's and the fp32 sums of the
                // correction (operand truncation is common to every column):
                // widen the bound of the row by twice that
                if (CHK && located)
                    A += 2.0f * (1.0f + 0x1p-10f) *
                         (float(kk + 1) * P.a_coef * xn * cm + 0x1p-19f * xn * P.cinfo[1] +
                          float(kk) * float(kk) * 0x1p-23f * xn * cm);
                const bool sane = xn * cm < 1e36f && m1 < INFINITY;
                if (sane && !(CHK && flagged && !located)) {
                    if (j1 == p) {
                        dval = __fsub_rn(yns[j1], __fadd_rn(cr.acc, cr.acc));
                        d1_known = true;
                        ok = isfinite(dval) && narrow_cert(m2, A, P.b_coef, dval);
                        // only j2 can still beat j1: its exact value decides (resolve pass)
                        to_winner = !ok && isfinite(dval) && narrow_cert(m3, A, P.b_coef, dval);
                    } else {
                        to_winner = true;
                    }
                }
                if (ok) {
                    P.out_idx[grow] = j1;
                    P.out_val[grow] = dval;
                }
            }
            // warp-aggregated appends
            const unsigned bw = __ballot_sync(0xffffffffu, to_winner);
            if (bw) {
                unsigned base = 0;
                if (lane == 0) base = atomicAdd(P.rf_count, unsigned(__popc(bw)));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (to_winner) {
                    const unsigned q = base + __popc(bw & ((1u << lane) - 1u));
                    P.rf_rows[q] = int32_t(grow);
                    P.rf_rec[2 * q] = make_float4(__int_as_float(j1), __int_as_float(j2), A, dval);
                    P.rf_rec[2 * q + 1] = make_float4(m2, m3, d1_known ? 1.0f : 0.0f, 0.0f);
                }
            }
            const bool need = live && !ok && !to_winner;
            const unsigned bf = __ballot_sync(0xffffffffu, need);
            if (bf) {
                unsigned base = 0;
                if (lane == 0) base = atomicAdd(P.fb_count, unsigned(__popc(bf)));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (need) P.fb_rows[base + __popc(bf & ((1u << lane) - 1u))] = int32_t(grow);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == NW_MMA) {
        tc_fence_after();
        tmem_dealloc(tmem, ncols);
    }
}

// The reference's exact fp32 chain x . c (products and sums separately
// rounded, k ascending) from global memory.
__device__ __forceinline__ float exact_chain_g(const float *xr, const float *cr, int64_t d) {
    const float4 *x4 = reinterpret_cast<const float4 *>(xr);
    const float4 *c4 = reinterpret_cast<const float4 *>(cr);
    float acc = 0.0f;
    const int64_t n4 = d >> 2;
    int64_t f = 0;
    for (; f + 4 <= n4; f += 4) {
        float4 a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a[u] = __ldg(x4 + f + u);
            b[u] = __ldg(c4 + f + u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            acc = __fadd_rn(acc, __fmul_rn(a[u].x, b[u].x));
            acc = __fadd_rn(acc, __fmul_rn(a[u].y, b[u].y));
            acc = __fadd_rn(acc, __fmul_rn(a[u].z, b[u].z));
            acc = __fadd_rn(acc, __fmul_rn(a[u].w, b[u].w));
        }
    }
    for (; f < n4; ++f) {
        const float4 a = __ldg(x4 + f), b = __ldg(c4 + f);
        acc = __fadd_rn(acc, __fmul_rn(a.x, b.x));
        acc = __fadd_rn(acc, __fmul_rn(a.y, b.y));
        acc = __fadd_rn(acc, __fmul_rn(a.z, b.z));
        acc = __fadd_rn(acc, __fmul_rn(a.w, b.w));
    }
    return acc;
}

// Resolve pass over the rows the screen could not finish alone: the exact
// value of the screened winner j1 (unless the chain already had it), the m2
// certificate; failing that, if only the runner-up j2 can still compete (m3
// certificate), its exact value and the reference's "first strict minimum"
// between the two; else the row goes to the exact kernel.  X rows come from
// L2 for the last tiles of the screen, HBM otherwise.
__global__ void narrow_winner_kernel(const float *x, const float *y, const float *yn, int64_t d,
                                     const int32_t *rows, const float4 *rec, const unsigned *count,
                                     float b_coef, int32_t *out_idx, float *out_val,
                                     int32_t *fb_rows, unsigned *fb_count) {
    const unsigned n = *count;
    for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int32_t row = rows[q];
        const float4 r0 = rec[2 * q], r1 = rec[2 * q + 1];
        const int j1 = __float_as_int(r0.x), j2 = __float_as_int(r0.y);
        const float A = r0.z, m2 = r1.x, m3 = r1.y;
        const float *xr = x + int64_t(row) * d;
        float d1 = r0.w;
        if (r1.z == 0.0f) {
            const float a1 = exact_chain_g(xr, y + int64_t(j1) * d, d);
            d1 = __fsub_rn(__ldg(yn + j1), __fadd_rn(a1, a1));
        }
        bool ok = false;
        int jw = j1;
        float vw = d1;
        if (isfinite(d1) && narrow_cert(m2, A, b_coef, d1)) {
            ok = true;
        } else if (isfinite(d1) && narrow_cert(m3, A, b_coef, d1)) {
            const float a2 = exact_chain_g(xr, y + int64_t(j2) * d, d);
            const float d2 = __fsub_rn(__ldg(yn + j2), __fadd_rn(a2, a2));
            ok = true;
            if (d2 < d1 || (d2 == d1 && j2 < j1)) {
                jw = j2;
                vw = d2;
            }
        }
        if (ok) {
            out_idx[row] = jw;
            out_val[row] = vw;
        } else {
            fb_rows[atomicAdd(fb_count, 1u)] = row;
        }
    }
}

// Transposed centroid operand of the chain warps: yt[f][j] = y[j][f], zero
// for k <= j < kt.
__global__ void narrow_transpose_kernel(const float *y, int64_t k, int64_t d, int kt, float *yt) {
    const int64_t n = d * kt;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t f = e / kt, j = e % kt;
        yt[e] = j < k ? y[j * d + f] : 0.0f;
    }
}

// Augmented centroid matrix rows k..k+3 (ABFT): csum = sum_j tf32(c_j) and
// wsum = sum_j (j+1) tf32(c_j) per feature, float64 sums, each split into two
// tf32-exact rows hi + lo; the last block also writes cinfo = (max|c|,
// |csum|, |wsum|) in a fixed order (deterministic tolerances).
__global__ void narrow_aug_kernel(const float *y, int64_t k, int64_t d, float *yaug, float *part,
                                  float *cinfo, unsigned *done) {
    const int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    float am = 0.0f, cs2 = 0.0f, ws2 = 0.0f;
    if (f < d) {
        double s = 0.0, w = 0.0;
        for (int64_t j = 0; j < k; ++j) {
            const float v = y[j * d + f];
            const double t = double(tf32_trunc(v));
            s += t;
            w += double(j + 1) * t;
            am = fmaxf(am, fabsf(v));
        }
        const float sh = tf32_trunc(float(s)), wh = tf32_trunc(float(w));
        const float sl = tf32_trunc(float(s - double(sh))), wl = tf32_trunc(float(w - double(wh)));
        yaug[(k + 0) * d + f] = sh;
        yaug[(k + 1) * d + f] = sl;
        yaug[(k + 2) * d + f] = wh;
        yaug[(k + 3) * d + f] = wl;
        cs2 = float(s) * float(s);
        ws2 = float(w) * float(w);
    }
    __shared__ float sh_m[32], sh_c[32], sh_w[32];
    for (int off = 16; off; off >>= 1) {
        am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, off));
        cs2 += __shfl_xor_sync(0xffffffffu, cs2, off);
        ws2 += __shfl_xor_sync(0xffffffffu, ws2, off);
    }
    if ((threadIdx.x & 31) == 0) {
        sh_m[threadIdx.x >> 5] = am;
        sh_c[threadIdx.x >> 5] = cs2;
        sh_w[threadIdx.x >> 5] = ws2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float a = 0.0f, c = 0.0f, w = 0.0f;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) {
            a = fmaxf(a, sh_m[i]);
            c += sh_c[i];
            w += sh_w[i];
        }
        part[3 * blockIdx.x + 0] = a;
        part[3 * blockIdx.x + 1] = c;
        part[3 * blockIdx.x + 2] = w;
        __threadfence();
        if (atomicAdd(done, 1u) == gridDim.x - 1) {
            __threadfence();
            float ga = 0.0f, gc = 0.0f, gw = 0.0f;
            for (unsigned b = 0; b < gridDim.x; ++b) {
                ga = fmaxf(ga, part[3 * b]);
                gc += part[3 * b + 1];
                gw += part[3 * b + 2];
            }
            cinfo[0] = ga;
            cinfo[1] = sqrtf(gc) * (1.0f + 0x1p-10f);
            cinfo[2] = sqrtf(gw) * (1.0f + 0x1p-10f);
            *done = 0;
        }
    }
}

// ------------------------------------------------------------- host ------
static size_t narrow_smem(int kp, int kt, int stages) {
    const size_t stg = (NR_A_KB + size_t(kp) * 128 + size_t(kt) * 128 + 1023) & ~size_t(1023);
    return 1024 + size_t(stages) * stg + NR_MAX_N * sizeof(float) +
           2 * NR_BM * sizeof(ChainRes) + (2 * size_t(stages) + 8) * 8 + 16;
}

bool narrow_supported(int64_t k, int64_t d, bool chk) {
    const int64_t kaug = k + (chk ? 4 : 0);
    return k >= 1 && kaug <= NR_MAX_N && d >= 4 && d % 4 == 0 && d <= (int64_t(1) << 20);
}

int narrow_screen_launch(const CUtensorMap &mx, const CUtensorMap &mc, const CUtensorMap &mct,
                         NarrowParams P, bool chk, cudaStream_t st) {
    int stages = 12;
    while (stages > 2 && narrow_smem(P.kp, P.kt, stages) > 227 * 1024) --stages;
    if (const char *e = getenv("FTK_NARROW_STAGES")) {  // tuning knob
        const int s = atoi(e);
        if (s >= 2 && s < stages) stages = s;
    }
    P.stages = stages;
    const size_t smem = narrow_smem(P.kp, P.kt, stages);
    const int64_t ntm = (P.m + NR_BM - 1) / NR_BM;
    if (ntm == 0) return FTK_OK;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = ntm < nsm ? ntm : nsm;
    auto kern = chk ? (P.inj_col ? narrow_screen_kernel<true, true> : narrow_screen_kernel<true, false>)
                    : narrow_screen_kernel<false, false>;
    FTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<dim3(unsigned(grid)), dim3(NR_THREADS), smem, st>>>(mx, mc, mct, P);
    FTK_LAUNCHED("narrow_screen_kernel");
    return FTK_OK;
}

int make_tc_map(CUtensorMap *map, const float *base, int64_t rows, int64_t cols, uint32_t box_rows);
int make_plain_map(CUtensorMap *map, const float *base, int64_t rows, int64_t cols,
                   uint32_t box_cols, uint32_t box_rows);

// The whole narrow assignment: augmented centroids, the screen, the winner
// pass and the exact fallback, all device-driven (no host synchronisation).
int narrow_assign_run(ftk_ctx *ctx, const NarrowIn &in, cudaStream_t st) {
    const int64_t m = in.m, k = in.k, d = in.d;
    const bool chk = in.ft != nullptr;
    const int64_t kaug = k + (chk ? 4 : 0);
    const int kp = int((kaug + 15) / 16 * 16);
    const int nkb = int((d + NR_KB - 1) / NR_KB);
    const unsigned nfb = unsigned((d + 255) / 256);
    // the chain warps read the hinted centroid from the swizzled MMA slice
    // (FTK_NARROW_CT=1: from an extra transposed slice, bank-conflict free
    // for k <= 32 but 4x the load instructions -- measured slower)
    const char *cte = getenv("FTK_NARROW_CT");  // A/B knob: transposed chain operand
    const int kt = (cte && atoi(cte) == 1 && k <= 64) ? int((k + 3) / 4 * 4) : 0;
    // scratch: augmented matrix, cinfo + partials, row lists
    const size_t aug_bytes = (sizeof(float) * size_t(kaug) * d + 255) & ~size_t(255);
    const size_t info_bytes = (256 + sizeof(float) * 3 * nfb + 64 + 255) & ~size_t(255);
    const size_t yt_bytes = (sizeof(float) * size_t(kt) * d + 255) & ~size_t(255);
    const size_t list_bytes = (sizeof(int32_t) + 2 * sizeof(float4)) * size_t(m + 1) + 64;
    char *buf = static_cast<char *>(
        scratch(ctx, SLOT_NARROW, aug_bytes + info_bytes + yt_bytes + list_bytes, st));
    if (!buf) return FTK_ERR_CUDA;
    float *yaug = reinterpret_cast<float *>(buf);
    float *cinfo = reinterpret_cast<float *>(buf + aug_bytes);
    unsigned *done = reinterpret_cast<unsigned *>(cinfo + 8);
    float *part = cinfo + 16;
    float *yt = reinterpret_cast<float *>(buf + aug_bytes + info_bytes);
    float4 *rf_rec = reinterpret_cast<float4 *>(buf + aug_bytes + info_bytes + yt_bytes);
    int32_t *rf_rows = reinterpret_cast<int32_t *>(rf_rec + 2 * (m + 1));
    const float *ymap = in.y;
    if (chk) {
        FTK_CUDA(cudaMemcpyAsync(yaug, in.y, sizeof(float) * size_t(k) * d, cudaMemcpyDeviceToDevice, st));
        FTK_CUDA(cudaMemsetAsync(done, 0, sizeof(unsigned), st));
        narrow_aug_kernel<<<nfb, 256, 0, st>>>(in.y, k, d, yaug, part, cinfo, done);
        FTK_LAUNCHED("narrow_aug_kernel");
        ymap = yaug;
    }
    CUtensorMap mx, mc, mct;
    int rc;
    if ((rc = make_tc_map(&mx, in.x, m, d, NR_BM)) || (rc = make_tc_map(&mc, ymap, kaug, d, uint32_t(kp))))
        return rc;
    if (kt) {
        narrow_transpose_kernel<<<148, 256, 0, st>>>(in.y, k, d, kt, yt);
        FTK_LAUNCHED("narrow_transpose_kernel");
        if ((rc = make_plain_map(&mct, yt, d, kt, uint32_t(kt), NR_KB))) return rc;
    } else {
        mct = mc;  // unused
    }
    NarrowParams P{};
    P.yn = in.yn;
    P.m = m; P.k = k; P.d = d;
    P.kp = kp;
    P.kt = kt;
    P.bstride = kp <= 16 ? 16 : (kp <= 32 ? 32 : (kp <= 64 ? 64 : (kp <= 128 ? 128 : 256)));
    P.nkb = nkb;
    P.a_coef = float(3.0 * double(d) * 0x1p-24);
    P.b_coef = float(0x1p-20);
    P.cmax2 = in.cmax2;
    P.ecmax2 = in.ecmax2;
    P.hint = (ctx->hint && ctx->hint_m == m) ? ctx->hint : nullptr;
    if (ctx->rows_info && ctx->rows_x == in.x && ctx->rows_m == m && ctx->rows_d == d)
        P.rowinfo = reinterpret_cast<const float4 *>(ctx->rows_info);
    P.out_idx = in.out_idx;
    P.out_val = in.out_val;
    P.rf_rows = rf_rows;
    P.rf_rec = rf_rec;
    P.rf_count = in.cnt + 3;
    P.fb_rows = in.fb_rows;
    P.fb_count = in.cnt + 0;
    if (chk) {
        const TcFt &ft = *in.ft;
        P.cinfo = cinfo;
        P.tau_coef = float(ft.delta_rel * double(d));
        P.tau_abs = float(ft.abs_tol);
        P.inj_col = in.inj_col;
        P.inj_before = in.inj_before;
        P.inj_after = in.inj_after;
        P.abft_count = in.cnt + 2;
        P.abft_total = abft_total_ptr(ctx, st);
        P.corrected = in.cnt + 4;
        if (ft.ev) {
            P.ev_cap = ft.ev->cap;
            P.ev_rec = ft.ev->rec;
            P.ev_delta = ft.ev->delta;
            P.ev_count = reinterpret_cast<unsigned long long *>(ft.ev->count);
        }
        P.iteration = ft.iteration;
        P.bm = ft.bm;
        P.bn = ft.bn;
        P.interval = ft.bk > 0 ? (d + ft.bk - 1) / ft.bk - 1 : 0;
        P.events_for_scheduled = ctx->inj_replay ? 0 : 1;
    }
    if (!ctx->time_ev[0]) {
        cudaEventCreate(&ctx->time_ev[0]);
        cudaEventCreate(&ctx->time_ev[1]);
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cap);
    const bool timed = cap == cudaStreamCaptureStatusNone;
    if (timed) cudaEventRecord(ctx->time_ev[0], st);
    if ((rc = narrow_screen_launch(mx, mc, mct, P, chk, st))) return rc;
    if (timed) cudaEventRecord(ctx->time_ev[1], st);
    ctx->last_path = 2;
    narrow_winner_kernel<<<148 * 8, 128, 0, st>>>(in.x, in.y, in.yn, d, rf_rows, rf_rec, P.rf_count,
                                                  P.b_coef, in.out_idx, in.out_val, in.fb_rows,
                                                  P.fb_count);
    FTK_LAUNCHED("narrow_winner_kernel");
    if ((rc = exact_rows_run(in.x, in.y, in.yn, k, d, in.fb_rows, P.fb_count, in.out_idx, in.out_val, st)))
        return rc;
    ctx->stat_dev[0] = P.rf_count;  // screened winner != hint (winner pass)
    ctx->stat_dev[1] = P.fb_count;  // exact kernel
    ctx->stat_dev[2] = chk ? in.cnt + 2 : nullptr;
    return FTK_OK;
}

}  // namespace ftk
