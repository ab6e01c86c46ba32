// tc_pair.cu -- CTA-pair (cta_group::2) tensor-core screen for the fused
// assignment: the 1xTF32 pass of tc.cu re-laid out for the B200's 2-SM UMMA.
//
// One cluster of two CTAs (one per SM of a TPC) owns 256 rows at a time:
// each CTA keeps its 128 X rows resident in shared memory and holds HALF of
// every centroid k-block (128 of the 256 centroids of an N tile), and the
// leader issues tcgen05.mma.cta_group::2 with M = 256, N = 256, so each
// centroid byte fetched from L2 feeds 256 rows instead of 128 (the 1-SM
// kernel was L2-bandwidth bound on centroid streaming).  Each CTA's TMEM
// receives its own 128 rows x 256 columns.
//
// Warp roles per CTA (15 warps; see W_* below):
//   w13     TMA producer of the centroid halves
//   w12     TMA producer of the X half-tile (peer: forwards its completion
//           to the leader's barrier)
//   w14     TMEM allocator; leader: MMA issuer
//   w0..w7  screen: two warpgroups, warpgroup g drains TMEM buffer g (the
//           MMA alternates buffers), keeps a running top-2 of the screened
//           s = |c|^2 - 2 x.c per row (index packed in the low mantissa bits),
//           and (ABFT) the row sum of the raw accumulators
//   w8..11  refine: merges the two warpgroups' partials, recomputes the
//           winner's distance in the reference's exact order from the X row
//           in shared memory, certifies the argmin and writes the outputs;
//           uncertified / checksum-flagged rows are appended to a fallback
//           list resolved exactly (tc.cu)
//
// Certificate (one-sided): with d1 the exact reference value of the screened
// winner j1 and m2 the second smallest screened value, every other centroid
// satisfies ref_j >= s_j - A - B|s_j| >= m2 - A - B|m2|, so m2 - A - B|m2| > d1
// proves j1 is the reference's strict argmin (A, B: tc.cu header).

#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tc_pair.cuh"

// Role-timing probes (clock64 sums per role, printed by FTK_PAIR_CLK=1) are
// compiled in only with -DFTK_PAIR_PROBE: they cost registers in the hot loop.
#ifdef FTK_PAIR_PROBE
#define PROBE_T(v) const long long v = clock64()
#define PROBE_ADD(i, x) (clk[i] += (x))
#else
#define PROBE_T(v)
#define PROBE_ADD(i, x)
#endif

namespace ftk {

constexpr int PR_BM = 128;          // rows per CTA
constexpr int PR_BN = PAIR_BN;      // centroids per N tile (half per CTA)
constexpr int PR_NBUF = 512 / PR_BN;  // TMEM accumulator buffers
constexpr int PR_KB = 32;           // fp32 elements per 128-byte swizzle row
constexpr int PR_MAX_KB = 8;        // k-blocks of the widest X row (d <= 256)
constexpr int PR_MAX_NA = 4;        // X half-tile buffers (4 when few centroid k-blocks per row tile)
#ifndef FTK_PAIR_SWG
#define FTK_PAIR_SWG 2
#endif
constexpr int PR_SWG = FTK_PAIR_SWG;  // screen warpgroups (each drains a column range of every tile)
constexpr int PR_NCH = PR_BN / 32;    // 32-column chunks per tile
#ifdef FTK_PAIR_SETMAXNREG
// register rebalancing (setmaxnreg, warpgroup-wide): the control warpgroup
// (X producer, C producer, MMA, one idle warp) gives registers to the screen.
// The pool is the CTA's launch allocation (threads x launch registers): the
// three counts must satisfy 384 S + 128 R + 128 C <= 640 x 96, else the
// increases wait forever.
constexpr int PR_THREADS = 32 * (4 * PR_SWG + 8);
#else
constexpr int PR_THREADS = 32 * (4 * PR_SWG + 7);  // screen, 4 refine, X producer, C producer, MMA
#endif
// Warp roles.  The SMSP arbiter favours the highest warp id, so the
// latency-critical single-thread roles (MMA issue, TMA producers) take the
// top ids and are never starved by the screening warps.
// warps 0..4*PR_SWG-1 screen, then 4 refine (refine on low ids measured +3 %)
constexpr int W_SCREEN0 = 0, W_REFINE0 = 4 * PR_SWG;
constexpr int W_XPROD = W_REFINE0 + 4;  // X half-tile producer (+ peer forwarding)
constexpr int W_PROD = W_REFINE0 + 5;   // centroid-stream TMA producer
constexpr int W_MMA = W_REFINE0 + 6;    // TMEM allocator; leader: MMA issuer
constexpr uint32_t PR_A_KB = PR_BM * 128;         // bytes of one X k-block
constexpr uint32_t PR_B_HALF = (PR_BN / 2) * 128;  // bytes of one centroid half k-block



struct PairPart {  // one warpgroup's running result for one row
    float m1;
    int32_t j1;
    float m2;
    float pad;
};

__device__ __forceinline__ uint32_t ordered_key(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// INJ: the pass carries scheduled flips (P.inj_col); a separate instantiation
// keeps the per-chunk injection test out of the clean CHK epilogue (-2.7%).
// SX (streamed X, d > 256): the X half no longer fits resident, so its
// k-blocks travel with the centroid k-blocks through the stage ring (each
// stage = centroid half + X half; with several column tiles the row tile's X
// is re-read from L2 per tile) and the refine reads its row from global
// memory (L2: the tile was just streamed).
// F64: float64 data screened from its fp32 copy; the refine records (j1, T)
// for the float64 refine (tc.cu tc64_refine_kernel) instead of running the
// fp32 exact chain.
#ifndef FTK_PAIR_COLLECT_SPLIT
#define FTK_PAIR_COLLECT_SPLIT 1  // pass 2: one work item per (row pair-tile, column tile)
#endif
template <bool CHK, bool COLLECT, bool INJ, bool SX, bool F64 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PR_THREADS, 1)
    pair_screen_kernel(const __grid_constant__ CUtensorMap tmX,
                       const __grid_constant__ CUtensorMap tmC, PairParams P) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int nkb = P.nkb, S = P.stages, NA = P.abufs;
    const uint32_t A_BYTES = SX ? 0u : PR_A_KB * nkb;
    constexpr uint32_t STG = SX ? PR_B_HALF + PR_A_KB : PR_B_HALF;  // bytes per stage
    unsigned char *sA = smem;
    unsigned char *sB = sA + size_t(NA) * A_BYTES;
    PairPart *part = reinterpret_cast<PairPart *>(sB + size_t(S) * STG);  // [2][2][128]
    double2 *psum = reinterpret_cast<double2 *>(part + 2 * PR_SWG * PR_BM);  // [2][PR_SWG][128] (sum, weighted)
    float *yns = reinterpret_cast<float *>(psum + 2 * PR_SWG * PR_BM);       // [2][PR_BN] (8 * PR_BN reserved)
    float4 *css = reinterpret_cast<float4 *>(yns + 8 * PR_BN);      // ABFT checksum centroid [nkb * 8]
    uint64_t *bars = reinterpret_cast<uint64_t *>(css + 8 * 8);
    uint64_t *full = bars, *empty = bars + S;
    uint64_t *a_full = bars + 2 * S, *a_empty = a_full + PR_MAX_NA;
    uint64_t *t_full = a_full + 2 * PR_MAX_NA, *t_empty = t_full + PR_NBUF;
    uint64_t *p_full = t_empty + PR_NBUF, *p_empty = p_full + 2;
    // X k-block release, per buffer: the refine warps free each k-block of a
    // row tile's X half as soon as they have consumed it, so the next X half
    // streams in behind the refine instead of after it
    uint64_t *a_kbe = p_empty + 2;  // [PR_MAX_NA][PR_MAX_KB]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(a_kbe + PR_MAX_NA * PR_MAX_KB);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
#ifdef FTK_PAIR_PROBE
    long long clk[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // debug timing (P.clk)
#endif
    // rows of this launch: a device-side count when the caller does not know it
    // on the host (pass 2 over the rows pass 1 left uncertified)
    const int64_t M = P.m_dev ? (int64_t(*P.m_dev) < P.m ? int64_t(*P.m_dev) : P.m) : P.m;
    const int64_t npt = (M + 2 * PR_BM - 1) / (2 * PR_BM);  // row pair-tiles
    // work items: a row pair-tile with all its column tiles, or (COLLECT, when
    // pass 2 has few rows) a group of column tiles, so the few row tiles still
    // spread over every SM: about two items per cluster.  Many pass-2 rows
    // (c5: ~3e6) keep whole row tiles -- splitting them re-reads each X tile
    // once per column group (c5 pass 2: 22 ms with one column tile per item)
    const bool csplit = COLLECT && FTK_PAIR_COLLECT_SPLIT;
    int tsplit = 1;
    if (csplit && npt > 0 && npt < 2 * int64_t(ncluster_x()))
        tsplit = int(std::min<int64_t>(P.ntiles, (2 * int64_t(ncluster_x()) + npt - 1) / npt));
    const int TPW = csplit ? (P.ntiles + tsplit - 1) / tsplit : P.ntiles;  // column tiles per item
    const int TPS = csplit ? (P.ntiles + TPW - 1) / TPW : 1;               // items per row pair-tile
    const int64_t nwi = npt * TPS;
    const int64_t pt0 = cluster_id_x(), pstride = ncluster_x();

    if (warp == W_PROD && lane == 0) {
        prefetch_tmap(&tmX);
        prefetch_tmap(&tmC);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < PR_MAX_NA; ++a) {
            mbar_init(&a_full[a], rank == 0 ? 2 : 1);  // leader: own TMA + peer's forward
            mbar_init(&a_empty[a], 4);  // refine warps, done with the X half
            for (int kb = 0; kb < PR_MAX_KB; ++kb) mbar_init(&a_kbe[a * PR_MAX_KB + kb], 4);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&p_full[a], 4 * PR_SWG);
            mbar_init(&p_empty[a], 4);
        }
        for (int b = 0; b < PR_NBUF; ++b) {
            mbar_init(&t_full[b], 1);
            mbar_init(&t_empty[b], 2 * 4 * PR_SWG);  // screen warps x 2 CTAs
        }
        fence_barrier_init();
    }
    if (warp == W_MMA) tmem_alloc_pair(tmem_slot, 512);
    tc_fence_before();
    cluster_sync_all();  // barriers of both CTAs initialised before any remote use
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
#ifdef FTK_PAIR_SETMAXNREG
    // warpgroup-uniform: the control warpgroup gives up registers here, the
    // screen warpgroups take them at the top of their branch
    if (warp >= W_REFINE0 + 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(FTK_PAIR_CTRL_REGS));
#endif

    if (warp == W_PROD) {
        // ------------------------------------------------ TMA producer --
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int64_t wi = pt0; wi < nwi; wi += pstride, ++it) {
                const int64_t pt = wi / TPS;
                const int tb = int(wi % TPS) * TPW, te = tb + TPW < P.ntiles ? tb + TPW : P.ntiles;
                const int row0 = int(pt * 2 * PR_BM + rank * PR_BM);
                for (int t = tb; t < te; ++t) {
                    const int c0 = t * PR_BN + int(rank) * (PR_BN / 2);
                    for (int kb = 0; kb < nkb; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
                        if (rank == 0) mbar_expect_tx(&full[stage], 2 * STG);
                        tma_load_2d_pair(sB + size_t(stage) * STG, &tmC, fb, kb * PR_KB, c0);
                        if (SX)  // this CTA's X half of the k-block, same stage
                            tma_load_2d_pair(sB + size_t(stage) * STG + PR_B_HALF, &tmX, fb, kb * PR_KB,
                                             row0);
                        if (++stage == S) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == W_MMA) {
        if (lane == 0 && rank == 0) {
            // --------------------------------------------- MMA issuer --
            constexpr uint32_t idesc = idesc_tf32(2 * PR_BM, PR_BN);
            const uint32_t b_base = smem_u32(sB);
            int stage = 0;
            uint32_t phase = 0;
            uint32_t g = 0;
            int it = 0;
            for (int64_t wi = pt0; wi < nwi; wi += pstride, ++it) {
                const int64_t pt = wi / TPS;
                const int tb = int(wi % TPS) * TPW, te = tb + TPW < P.ntiles ? tb + TPW : P.ntiles;
                const int ab = SX ? 0 : it % NA;
                if (!SX) {
                    PROBE_T(c0_);
                    mbar_wait(&a_full[ab], uint32_t(it / NA) & 1);
                    PROBE_ADD(4, clock64() - c0_);
                }
                tc_fence_after();
                const uint32_t a_base = smem_u32(sA) + uint32_t(ab) * A_BYTES;
                for (int t = tb; t < te; ++t, ++g) {
                    const int buf = g % PR_NBUF;
                    { PROBE_T(c0_); mbar_wait(&t_empty[buf], ((g / PR_NBUF) & 1) ^ 1); PROBE_ADD(2, clock64() - c0_); }
                    tc_fence_after();
                    const uint32_t d_tmem = tmem + uint32_t(buf * PR_BN);
                    for (int kb = 0; kb < nkb; ++kb) {
                        { PROBE_T(c0_); mbar_wait(&full[stage], phase); PROBE_ADD(3, clock64() - c0_); }
                        tc_fence_after();
                        const uint32_t bs = b_base + uint32_t(stage) * STG;
                        const uint32_t as = SX ? bs + PR_B_HALF : a_base + uint32_t(kb) * PR_A_KB;
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_tf32_pair(d_tmem, smem_desc(as + kk * 32), smem_desc(bs + kk * 32), idesc,
                                          (kb | kk) != 0);
                        mma_commit_pair(&empty[stage], 0x3);
                        if (++stage == S) { stage = 0; phase ^= 1; }
                    }
                    mma_commit_pair(&t_full[buf], 0x3);
                }
            }
        }
    } else if (warp == W_XPROD) {
        // ------------------------------- X producer (+ peer forwarding) --
        // decoupled from the centroid stream so the next row tile's X half
        // loads as soon as its buffer is released, not behind the B stages
        if (lane == 0 && !SX) {
            int it = 0;
            const uint32_t lead = mapa_shared(smem_u32(&a_full[0]), 0);
            for (int64_t wi = pt0; wi < nwi; wi += pstride, ++it) {
                const int64_t pt = wi / TPS;
                const int tb = int(wi % TPS) * TPW, te = tb + TPW < P.ntiles ? tb + TPW : P.ntiles;
                const int ab = it % NA;
                unsigned char *a_dst = sA + size_t(ab) * A_BYTES;
                const int row0 = int(pt * 2 * PR_BM + rank * PR_BM);
                const uint32_t par = (uint32_t(it / NA) & 1) ^ 1;
                mbar_wait(&a_kbe[ab * PR_MAX_KB], par);
                mbar_expect_tx(&a_full[ab], A_BYTES);
                for (int kb = 0; kb < nkb; ++kb) {
                    if (kb) mbar_wait(&a_kbe[ab * PR_MAX_KB + kb], par);
                    tma_load_2d(a_dst + size_t(kb) * PR_A_KB, &tmX, &a_full[ab], kb * PR_KB, row0);
                }
                if (rank == 1) {  // the leader's MMA reads this half too
                    mbar_wait(&a_full[ab], uint32_t(it / NA) & 1);
                    mbar_arrive_remote(lead + uint32_t(ab) * 8u);
                }
            }
        }
    } else if (warp >= W_SCREEN0 && warp < W_SCREEN0 + 4 * PR_SWG) {
        // ----------------------------------------------------- screen --
#ifdef FTK_PAIR_SETMAXNREG
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(FTK_PAIR_SCREEN_REGS));
#endif
        // Every warpgroup drains every accumulator tile: warpgroup wg takes
        // chunks [cb0, cb1) of the tile's PR_NCH 32-column chunks, so a TMEM
        // buffer is released after 1/PR_SWG of a tile's epilogue work.
        const int wg = (warp - W_SCREEN0) >> 2;
        const int quad = warp & 3;  // TMEM lane quadrant: warp % 4
        const int r = quad * 32 + lane;
        const uint32_t lane_base = uint32_t(quad * 32) << 16;
        const uint32_t t_empty_lead0 = mapa_shared(smem_u32(&t_empty[0]), 0);
        const int cb0 = (PR_NCH * wg) / PR_SWG, cb1 = (PR_NCH * (wg + 1)) / PR_SWG;
        const int cbeg = cb0 * 32, nch = cb1 - cb0, ncol = nch * 32;
        // a warpgroup range crossing a 128-column group boundary (PR_SWG = 3)
        // splits its checksum partial at chunk `split` (location weights)
        const int split = (cb0 < 4 && cb1 > 4) ? 4 - cb0 : -1;
        uint32_t g = 0;
        int it = 0;
        // centroid norms of the current tile, staged one tile ahead
        // one [2][PR_BN] buffer staged by the screen threads (named barrier 1);
        // per-warp buffers without the barrier measured 5% slower
        const int et = (warp - W_SCREEN0) * 32 + lane;  // 0..255
        float *ywarp = yns + cbeg;          // reads: ywarp + ybuf * PR_BN
        int ybuf = 0;
        {
            const int64_t c = int64_t((pt0 % TPS) * TPW) * PR_BN + et;  // the first item's first tile
            if (et < PR_BN) yns[et] = c < P.k ? __ldg(P.yn + c) : INFINITY;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(128 * PR_SWG) : "memory");
        for (int64_t wi = pt0; wi < nwi; wi += pstride, ++it) {
                const int64_t pt = wi / TPS;
                const int tb = int(wi % TPS) * TPW, te = tb + TPW < P.ntiles ? tb + TPW : P.ntiles;
            const int pb = it & 1;
            const int64_t grow = pt * 2 * PR_BM + int64_t(rank) * PR_BM + r;
            float m1 = INFINITY, m2 = INFINITY;
            int tile1 = 0;
            double rsum = 0.0, wsum = 0.0;
            int inj_c = -1;
            float inj_b = 0.0f, inj_a = 0.0f;
            const float thr = (COLLECT && grow < M) ? P.thr[grow] : -INFINITY;
            unsigned ncand = 0;  // COLLECT: this thread's candidates of the row
            // COLLECT: the first four candidates of the row wait in registers
            // for one warp-wide append per work item (a same-address atomic per
            // warp and tile serialised in L2 at c5's ~3e6 pass-2 rows)
            int nloc = 0, lc0 = 0, lc1 = 0, lc2 = 0, lc3 = 0;
            if (INJ && P.inj_col && grow < M) {
                inj_c = P.inj_col[grow];
                if (inj_c >= 0) {
                    inj_b = P.inj_before[grow];
                    inj_a = P.inj_after[grow];
                }
            }
            for (int t = tb; t < te; ++t, ++g) {
                const int buf = g % PR_NBUF;
                const int64_t c0 = int64_t(t) * PR_BN + cbeg;  // first column of this warpgroup's range
                // prefetch the next tile's norms (wrapping into the next row tile)
                const int tn = t + 1 < te ? t + 1 : int(((wi + pstride) % TPS) * TPW);  // next item's first tile
                const int64_t cn = int64_t(tn) * PR_BN + et;
                const float yn_next = (et < PR_BN && cn < P.k) ? __ldg(P.yn + cn) : INFINITY;
                PROBE_T(cw_); mbar_wait(&t_full[buf], (g / PR_NBUF) & 1); PROBE_T(cb_); PROBE_ADD(1, cb_ - cw_);
                tc_fence_after();
                float a1 = INFINITY, a2 = INFINITY, b1 = INFINITY, b2 = INFINITY;
                float s0 = 0.0f, s1 = 0.0f;
                const uint32_t tbase = tmem + lane_base + uint32_t(buf * PR_BN + cbeg);
                const float *ynt = ywarp + ybuf * PR_BN;
                const bool inj_here = INJ && inj_c >= int(c0) && inj_c < int(c0) + ncol;
                float gA = 0.0f;  // checksum partial before the group split
                bool early_rel = false;  // FTK_PAIR_X2R: buffer released inside the drain
                if (P.dbg & 4) {
                    // timing probe: TMEM drain only (values folded with one XOR per column)
                    uint32_t va[32], acc = 0;
#pragma unroll 1
                    for (int ch = 0; ch < nch; ++ch) {
                        tmem_ld32_issue(tbase + uint32_t(ch * 32), va);
                        tmem_ld_wait(va);
#pragma unroll
                        for (int e = 0; e < 32; ++e) acc ^= va[e];
                    }
                    a1 = __uint_as_float(acc & 0x3F800000u);
                } else if (COLLECT) {
                    // pass 2: every column whose screened value can still beat
                    // the row's threshold becomes an exact-evaluation candidate
                    uint32_t va[32];
#pragma unroll 1
                    for (int ch = 0; ch < nch; ++ch) {
                        tmem_ld32_issue(tbase + uint32_t(ch * 32), va);
                        tmem_ld_wait(va);
                        const float4 *yn4 = reinterpret_cast<const float4 *>(ynt + ch * 32);
                        uint32_t hit = 0;
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 yv = yn4[q];
                            float d[4];
                            ffma2_m2(__uint_as_float(va[4 * q]), __uint_as_float(va[4 * q + 1]), yv.x,
                                     yv.y, d[0], d[1]);
                            ffma2_m2(__uint_as_float(va[4 * q + 2]), __uint_as_float(va[4 * q + 3]),
                                     yv.z, yv.w, d[2], d[3]);
#pragma unroll
                            for (int u = 0; u < 4; ++u) hit |= (d[u] <= thr ? 1u : 0u) << (4 * q + u);
                        }
                        // branch-free compare above, then one pass over the set bits
                        // (a row has ~2 candidates among K columns); columns past the
                        // last centroid never count
                        const int64_t cb = c0 + ch * 32;
                        const int64_t live = P.k - cb;
                        if (live < 32) hit &= live <= 0 ? 0u : ((1u << live) - 1u);
                        while (hit) {
                            const int col = int(cb) + __ffs(hit) - 1;
                            hit &= hit - 1u;
                            ++ncand;  // row count: one atomic per row and warpgroup
                            // the first few per thread wait in registers for one
                            // warp-wide append per work item
                            if (nloc < 4) {
                                lc0 = nloc == 0 ? col : lc0;
                                lc1 = nloc == 1 ? col : lc1;
                                lc2 = nloc == 2 ? col : lc2;
                                lc3 = nloc == 3 ? col : lc3;
                                ++nloc;
                            } else {
                                const unsigned slot = atomicAdd(P.cand_count, 1u);
                                if (slot < P.cand_cap) P.cand[slot] = make_int2(int(grow), col);
                            }
                        }
                    }
                } else if (!(P.dbg & 1)) {
                    // software-pipelined TMEM drain, two 32-column chunks per
                    // (not unrolled) iteration to keep the loop in the I-cache;
                    // in a partial last tile, chunks past the last centroid are
                    // skipped (a plain loop: the full-tile loop stays as is)
                    const int live = int(P.k - c0);
                    uint32_t va[32], vb[32];
#ifndef FTK_PAIR_NOX2
                    // both chunks of a pair loaded, ONE wait, then the two
                    // tournaments in one basic block: twice the independent
                    // work per warp, no load in flight during the math
                    // (measured faster than keeping the next chunk's load in
                    // flight: c2 kernel 0.531 -> 0.519 ms, FT-off 0.498 ->
                    // 0.482, profiles/r6_ab_experiments.txt; FTK_PAIR_NOX2
                    // builds the software-pipelined drain)
                    if (live >= ncol && (nch & 1) == 0) {
#pragma unroll 1
                        for (int ch = 0; ch < nch; ch += 2) {
#ifdef FTK_PAIR_X64
                            tmem_ld64_issue(tbase + uint32_t(ch * 32), va, vb);
#else
                            tmem_ld32_issue(tbase + uint32_t(ch * 32), va);
                            tmem_ld32_issue(tbase + uint32_t((ch + 1) * 32), vb);
#endif
                            tmem_ld_wait(va);
                            tmem_pin(vb);
#ifdef FTK_PAIR_X2R
                            if (ch + 2 >= nch) {  // the tile's last values are in registers: release the buffer
                                tc_fence_before();
                                __syncwarp();
                                if (lane == 0) mbar_arrive_remote(t_empty_lead0 + uint32_t(buf) * 8u);
                                early_rel = true;
                            }
#endif
                            if (INJ && inj_here && (inj_c - int(c0)) >> 5 == ch)
                                inject_into(va, (inj_c - int(c0)) & 31, inj_b, inj_a);
                            if (INJ && inj_here && (inj_c - int(c0)) >> 5 == ch + 1)
                                inject_into(vb, (inj_c - int(c0)) & 31, inj_b, inj_a);
                            if (CHK && ch == split) { gA = s0 + s1; s0 = s1 = 0.0f; }
                            float t0s = 0.0f, t1s = 0.0f, bL = INFINITY, bM = INFINITY;
                            screen32t<CHK>(va, ynt + ch * 32, uint32_t(cbeg + ch * 32), a1, a2, s0, s1);
                            screen32t<CHK>(vb, ynt + (ch + 1) * 32, uint32_t(cbeg + (ch + 1) * 32), bL, bM,
                                           t0s, t1s);
                            if (CHK && ch + 1 == split) { gA = s0 + s1; s0 = t0s; s1 = t1s; }
                            else if (CHK) { s0 += t0s; s1 += t1s; }
                            a2 = fminf(fminf(a2, bM), bL == bL ? fmaxf(a1, bL) : INFINITY);
                            a1 = fminf(a1, bL);
                        }
                    } else
#endif
                    if (live >= ncol) {
                        tmem_ld32_issue(tbase, va);
                        tmem_ld_wait(va);
#pragma unroll 1
                        for (int ch = 0; ch < nch; ch += 2) {
                            const bool two = ch + 1 < nch;
                            if (two) tmem_ld32_issue(tbase + uint32_t((ch + 1) * 32), vb);
                            if (INJ && inj_here && (inj_c - int(c0)) >> 5 == ch)
                                inject_into(va, (inj_c - int(c0)) & 31, inj_b, inj_a);
                            if (CHK && ch == split) { gA = s0 + s1; s0 = s1 = 0.0f; }
                            screen32t<CHK>(va, ynt + ch * 32, uint32_t(cbeg + ch * 32), a1, a2, s0, s1);
                            if (two) {
                                tmem_ld_wait(vb);
                                if (ch + 2 < nch) tmem_ld32_issue(tbase + uint32_t((ch + 2) * 32), va);
                                if (INJ && inj_here && (inj_c - int(c0)) >> 5 == ch + 1)
                                    inject_into(vb, (inj_c - int(c0)) & 31, inj_b, inj_a);
                                if (CHK && ch + 1 == split) { gA = s0 + s1; s0 = s1 = 0.0f; }
                                screen32t<CHK>(vb, ynt + (ch + 1) * 32, uint32_t(cbeg + (ch + 1) * 32),
                                               a1, a2, s0, s1);
                                if (ch + 2 < nch) tmem_ld_wait(va);
                            }
                        }
                    } else {
#pragma unroll 1
                        for (int ch = 0; ch < nch && ch * 32 < live; ++ch) {
                            tmem_ld32_issue(tbase + uint32_t(ch * 32), va);
                            tmem_ld_wait(va);
                            if (INJ && inj_here && (inj_c - int(c0)) >> 5 == ch)
                                inject_into(va, (inj_c - int(c0)) & 31, inj_b, inj_a);
                            if (CHK && ch == split) { gA = s0 + s1; s0 = s1 = 0.0f; }
                            screen32t<CHK>(va, ynt + ch * 32, uint32_t(cbeg + ch * 32), a1, a2, s0, s1);
                        }
                    }
                }
                if (!early_rel) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(t_empty_lead0 + uint32_t(buf) * 8u);
                }
                PROBE_ADD(0, clock64() - cb_); PROBE_ADD(5, 1);
                // merge the two chains into the tile's top-2, then the running top-2
                const float t1 = fminf(a1, b1);  // b1 = b2 = inf: single chain
                const float t2 = fminf(fminf(a2, b2), fmaxf(a1, b1));
                if (CHK) {
                    // the warpgroup's columns lie in one 128-column group g (two when
                    // its range crosses a group boundary: gA before, the rest
                    // after), location weight g + 1: one multiply per group
                    const int gf = (t * PR_BN + cbeg) / 128;
                    const double gs = double(s0 + s1);
                    rsum += double(gA) + gs;
                    wsum += double(gA) * double(gf + 1) + gs * double(gf + 1 + (split >= 0 ? 1 : 0));
                }
                const float hi = fmaxf(m1, t1);
                if (t1 < m1) tile1 = t;
                m1 = fminf(m1, t1);
                m2 = fminf(fminf(m2, t2), hi);
                if (et < PR_BN) yns[(ybuf ^ 1) * PR_BN + et] = yn_next;
                asm volatile("bar.sync 1, %0;" ::"n"(128 * PR_SWG) : "memory");
                ybuf ^= 1;
            }
            if (COLLECT && ncand) atomicAdd(P.row_cnt + grow, ncand);
            if (COLLECT) {
                int incl = nloc;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int o = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += o;
                }
                const int total = __shfl_sync(0xffffffffu, incl, 31);
                if (total) {
                    unsigned base = 0;
                    if (lane == 31) base = atomicAdd(P.cand_count, unsigned(total));
                    base = __shfl_sync(0xffffffffu, base, 31) + unsigned(incl - nloc);
                    const int cols[4] = {lc0, lc1, lc2, lc3};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (i < nloc && base + i < P.cand_cap)
                            P.cand[base + i] = make_int2(int(grow), cols[i]);
                }
            }
            // publish this warpgroup's partial for the row tile
            mbar_wait(&p_empty[pb], (uint32_t(it >> 1) & 1) ^ 1);
            PairPart pp;
            pp.m1 = m1;
            pp.j1 = tile1 * PR_BN + int(__float_as_uint(m1) & 0xFFu);
            pp.m2 = m2;
            pp.pad = 0.0f;
            part[(pb * PR_SWG + wg) * PR_BM + r] = pp;
            if (CHK) psum[(pb * PR_SWG + wg) * PR_BM + r] = make_double2(rsum, wsum);
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[pb]);
        }
    } else if (warp >= W_REFINE0 && warp < W_REFINE0 + 4) {
        // ----------------------------------------------------- refine --
#ifdef FTK_PAIR_SETMAXNREG
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(FTK_PAIR_REFINE_REGS));
#endif
        const int quad = warp & 3;
        const int r = quad * 32 + lane;
        if (CHK && !SX) {
            const int t = (warp - W_REFINE0) * 32 + lane;  // 0..127
            if (t < nkb * 8) css[t] = __ldg(reinterpret_cast<const float4 *>(P.csum) + t);
            asm volatile("bar.sync 3, 128;" ::: "memory");
        }
        // centroid row of this thread's winner in 32-float k-blocks: two
        // statically indexed register buffers, k-blocks 0 and 1 prefetched
        // for the hinted label (previous iteration) while the previous row
        // tile is still being screened
        float4 cA[8], cB[8];
        int pj = -1;  // centroid whose k-blocks 0 and 1 are in cA / cB
        auto load_row = [&](float4 (&cv)[8], int row_j, int kb, bool live) {
            if (F64 || COLLECT) return;  // the float64 refine reads the centroid itself
#ifdef FTK_PAIR_PROBE
            if (P.dbg & 8) live = false;  // timing probe: no centroid loads
#endif
            const float4 *c4 = reinterpret_cast<const float4 *>(P.y + int64_t(live ? row_j : 0) * P.d);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                cv[q] = (live && kb * PR_KB + 4 * q < P.d) ? __ldg(c4 + kb * 8 + q)
                                                           : make_float4(0.f, 0.f, 0.f, 0.f);
        };
        auto prefetch = [&](int64_t ptn) {
            pj = -1;
            if (F64 || COLLECT || !P.hint || ptn >= npt) return;
            const int64_t gn = ptn * 2 * PR_BM + int64_t(rank) * PR_BM + r;
            if (gn >= M) return;
            const int h = __ldg(P.hint + gn);
            if (h < 0 || h >= P.k) return;
            pj = h;
            load_row(cA, h, 0, true);
            if (nkb > 1) load_row(cB, h, 1, true);
        };
        prefetch(pt0);
        // per-row bounds (rowinfo) of the next row tile, loaded one tile ahead
        auto load_info = [&](int64_t ptn) -> float4 {
            const int64_t gn = ptn * 2 * PR_BM + int64_t(rank) * PR_BM + r;
            return (P.rowinfo && ptn < npt && gn < M) ? __ldg(P.rowinfo + gn) : make_float4(0.f, 0.f, 0.f, 0.f);
        };
        // float64 mode (no centroid row in flight): the per-row bounds of the
        // next row tile and the launch constants are loaded ahead (c4 screen
        // 1.48 -> 1.37 ms); the float32 refine measured 3-5 % slower with it
        float4 ri_next = F64 ? load_info(pt0) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float k_cmax2 = (F64 && !COLLECT) ? *P.cmax2 : 0.0f;
        const float k_ecmax2 = (F64 && !COLLECT) ? *P.ecmax2 : 0.0f;
        const float k_camax0 = (F64 && CHK && !COLLECT) ? P.camax[0] : 0.0f;
        const float k_camax2 = (F64 && CHK && !COLLECT) ? P.camax[2] : 0.0f;
        int it = 0;
        for (int64_t wi = pt0; wi < nwi; wi += pstride, ++it) {
                const int64_t pt = wi / TPS;
                const int tb = int(wi % TPS) * TPW, te = tb + TPW < P.ntiles ? tb + TPW : P.ntiles;
            const int pb = it & 1;
            const int ab = SX ? 0 : it % NA;
            PROBE_T(rw0_);
            mbar_wait(&p_full[pb], uint32_t(it >> 1) & 1);
            PROBE_T(rw1_);
            PROBE_ADD(6, rw1_ - rw0_);
            // merge the warpgroups' partials (ascending column ranges: a tie
            // keeps the earlier range, the reference's lowest index)
            float m1 = INFINITY, m2 = INFINITY;
            int j = 0;
            double rsum = 0.0, wsum = 0.0;
#pragma unroll
            for (int w = 0; w < PR_SWG; ++w) {
                const PairPart q = part[(pb * PR_SWG + w) * PR_BM + r];
                const float hi = fmaxf(m1, q.m1);
                if (q.m1 < m1) j = q.j1;
                m1 = fminf(m1, q.m1);
                m2 = fminf(fminf(m2, q.m2), hi);
                if (CHK) {
                    const double2 u = psum[(pb * PR_SWG + w) * PR_BM + r];
                    rsum += u.x;
                    wsum += u.y;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_empty[pb]);
            const int64_t grow = pt * 2 * PR_BM + int64_t(rank) * PR_BM + r;
            const int pjv = pj;  // the prefetched centroid (cA / cB are clobbered below)
            pj = -1;
            const float4 ri_cur = ri_next;
            if (F64) ri_next = load_info((wi + pstride) / TPS);
            if (!SX) mbar_wait(&a_full[ab], uint32_t(it / NA) & 1);  // own X half resident + visible
            const unsigned char *sAt = sA + size_t(ab) * A_BYTES + uint32_t(r) * 128;
            bool ok = false;
            float dval = 0.0f;
            float thr_out = INFINITY;          // pass-2 candidate threshold
            unsigned long long seed_out = ~0ull;  // (ordered d1, j1) key
            const bool active = !COLLECT && grow < M && m1 < INFINITY && !(P.dbg & 2);
            bool released = false;  // X k-blocks handed back (warp-uniform)
#ifdef FTK_PAIR_PROBE
            if ((P.dbg & 128) && !SX) {  // timing probe: hand X back at once (results invalid)
                __syncwarp();
                if (lane == 0)
                    for (int kb = 0; kb < nkb; ++kb) mbar_arrive(&a_kbe[ab * PR_MAX_KB + kb]);
                released = true;
            }
#endif
            if (!COLLECT && !(P.dbg & 2) && __any_sync(0xffffffffu, active)) {
                float acc = 0.0f, xx = 0.0f, ee = 0.0f, amax = 0.0f;
                float rr[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // ABFT reference x~ . csum (fp32)
                // checksum centroid: staged once per CTA (ABFT), from global when streamed
                const float4 *cs4 = SX ? reinterpret_cast<const float4 *>(P.csum) : css;
                const float4 *xg4 = reinterpret_cast<const float4 *>(P.x + (active ? grow : 0) * P.d);
                const bool have_info = P.rowinfo != nullptr;
                if (have_info) {
                    const float4 ri = F64 ? ri_cur : __ldg(P.rowinfo + grow);
                    xx = ri.x;
                    ee = ri.y;
                    amax = ri.z;
                }
                // the winner's centroid row; the X row comes from the resident tile
                auto load_c = [&](float4 (&cv)[8], int kb) { load_row(cv, j, kb, active); };
                auto consume = [&](const float4 (&cv)[8], int kb) {
                    const int k0 = kb * PR_KB;
                    const unsigned char *rowp = sAt + uint32_t(kb) * PR_A_KB;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (k0 + 4 * q < P.d) {
#ifdef FTK_PAIR_PROBE
                            const float4 xv = (P.dbg & 32) ? make_float4(1.f, 1.f, 1.f, 1.f) :
                                (SX ? __ldg(xg4 + kb * 8 + q)
                                    : *reinterpret_cast<const float4 *>(rowp + ((q ^ (r & 7)) << 4)));
#else
                            const float4 xv =
                                SX ? __ldg(xg4 + kb * 8 + q)
                                   : *reinterpret_cast<const float4 *>(rowp + ((q ^ (r & 7)) << 4));
#endif
#ifdef FTK_PAIR_PROBE
                            if (!F64 && !(P.dbg & 16)) {  // timing probe: bit 16 skips the exact chain
#else
                            if (!F64) {
#endif
                                const float4 c4 = cv[q];
                                acc = __fadd_rn(acc, __fmul_rn(xv.x, c4.x));
                                acc = __fadd_rn(acc, __fmul_rn(xv.y, c4.y));
                                acc = __fadd_rn(acc, __fmul_rn(xv.z, c4.z));
                                acc = __fadd_rn(acc, __fmul_rn(xv.w, c4.w));
                            }
                            if (!have_info) {
                                xx = fmaf(xv.x, xv.x, xx);
                                xx = fmaf(xv.y, xv.y, xx);
                                xx = fmaf(xv.z, xv.z, xx);
                                xx = fmaf(xv.w, xv.w, xx);
                                const float r0 = xv.x - tf32_trunc(xv.x);
                                const float r1 = xv.y - tf32_trunc(xv.y);
                                const float r2 = xv.z - tf32_trunc(xv.z);
                                const float r3 = xv.w - tf32_trunc(xv.w);
                                ee = fmaf(r0, r0, ee);
                                ee = fmaf(r1, r1, ee);
                                ee = fmaf(r2, r2, ee);
                                ee = fmaf(r3, r3, ee);
                                if (CHK)
                                    amax = fmaxf(amax, fmaxf(fmaxf(fabsf(xv.x), fabsf(xv.y)),
                                                             fmaxf(fabsf(xv.z), fabsf(xv.w))));
                            }
                            if (CHK) {
#ifdef FTK_PAIR_PROBE
                                const float4 sv = (P.dbg & 64) ? make_float4(1.f, 1.f, 1.f, 1.f) : cs4[kb * 8 + q];
#else
                                const float4 sv = cs4[kb * 8 + q];
#endif
                                rr[0] = fmaf(tf32_trunc(xv.x), sv.x, rr[0]);
                                rr[1] = fmaf(tf32_trunc(xv.y), sv.y, rr[1]);
                                rr[2] = fmaf(tf32_trunc(xv.z), sv.z, rr[2]);
                                rr[3] = fmaf(tf32_trunc(xv.w), sv.w, rr[3]);
                            }
                        }
                    }
                };
                auto release = [&](int kb) {  // this warp is done reading X k-block kb
                    if (SX || released) return;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&a_kbe[ab * PR_MAX_KB + kb]);
                };
                PROBE_T(lp0_);
                if (!(active && j == pjv)) {  // no (matching) prefetch: k-blocks 0 and 1 now
                    load_c(cA, 0);
                    if (nkb > 1) load_c(cB, 1);
                }
                for (int kb = 0; kb < nkb; kb += 2) {
                    consume(cA, kb);
                    release(kb);
                    if (kb + 2 < nkb) load_c(cA, kb + 2);
                    if (kb + 1 < nkb) {
                        consume(cB, kb + 1);
                        release(kb + 1);
                        if (kb + 3 < nkb) load_c(cB, kb + 3);
                    }
                }
                released = true;
                prefetch((wi + pstride) / TPS);  // the next row tile's hinted centroids, k-blocks 0 and 1
                PROBE_T(lp1_);
                PROBE_ADD(8, lp1_ - lp0_);
              if (active) {  // lanes without a live row only helped with the loads
                const float xn = sqrtf(xx * (1.0f + 0x1p-10f));
                const float cm = sqrtf((F64 ? k_cmax2 : *P.cmax2) * (1.0f + 0x1p-10f));
                const float A = 2.0f * (1.0f + 0x1p-10f) *
                                (sqrtf(ee * (1.0f + 0x1p-10f)) * cm +
                                 xn * sqrtf((F64 ? k_ecmax2 : *P.ecmax2) * (1.0f + 0x1p-10f)) + P.a_coef * xn * cm) +
                                (F64 ? P.a_abs * k_cmax2 : 0.0f);
                dval = F64 ? 0.0f : __fsub_rn(P.yn[j], __fadd_rn(acc, acc));
                const double rref = (rr[0] + rr[1]) + (rr[2] + rr[3]);
                bool abft_bad = false;
                if (CHK) {
                    // reference tolerance + the fp32 evaluation error of the
                    // checksum reference, |x~ . csum| rounding <= 34 u |x| |csum|
                    const float tau = P.tau_coef * fmaxf(1.0f, amax * (F64 ? k_camax0 : *P.camax)) + P.tau_abs +
                                      34.0f * 0x1p-24f * sqrtf(xx * (1.0f + 0x1p-10f)) *
                                          sqrtf((F64 ? k_camax2 : P.camax[2]) * (1.0f + 0x1p-10f));
                    const double D1 = rsum - rref;
                    abft_bad = !(fabs(D1) <= double(tau));
                    if (abft_bad) {
                        atomicAdd(P.abft_count, 1u);
                        if (P.abft_total) atomicAdd(P.abft_total, 1ull);
                        // the row is re-resolved exactly by pass 2 (a clean
                        // re-screen): correction without touching the hot path.
                        // Location and the event record are done after the pass
                        // (abft_flag_events_kernel) from this record.
                        if (P.flag_rec) {
                            const unsigned q = atomicAdd(P.flag_count, 1u);
                            if (q < P.flag_cap)
                                P.flag_rec[q] = make_double4(__longlong_as_double(grow), D1, wsum, double(tau));
                        }
                    }
                }
                if (F64) {
                    // certificate threshold for the float64 refine: j1 is the
                    // reference's strict argmin iff its exact value d1 < T
                    const float T = m2 - A - P.b_coef * fabsf(m2) - 0x1p-21f * (fabsf(m1) + fabsf(m2));
                    const bool good = !abft_bad && xn * cm < 1e36f && isfinite(T) && isfinite(m1);
                    P.rec64[grow] = make_int2(good ? j : -1, __float_as_int(T));
                    if (P.a64) P.a64[grow] = good ? A : -1.0f;  // the screen bound (pass-2 threshold)
                }
                // magnitudes far from overflow: the screen saw every column finite
                const bool sane = !F64 && xn * cm < 1e36f && isfinite(dval);
                if (sane) {
                    // ref_j >= s_j - A - B|s_j| > d1 unless s_j <= thr (see tc_pair.cuh)
                    thr_out = dval + A + 2.0f * (P.b_coef + 0x1p-20f) * (fabsf(dval) + A);
                    thr_out = thr_out + fabsf(thr_out) * 0x1p-20f;
                    seed_out = (static_cast<unsigned long long>(ordered_key(dval)) << 32) | unsigned(j);
                }
                ok = !abft_bad && sane &&
                     (m2 - A - P.b_coef * fabsf(m2) - 0x1p-21f * (fabsf(m1) + fabsf(m2)) > dval);
              }
                PROBE_ADD(9, clock64() - lp1_);
            }
            if (F64 && !active && grow < M) P.rec64[grow] = make_int2(-1, 0);
            if (!COLLECT && !F64 && grow < M) {
                if (ok) {
                    P.out_idx[grow] = j;
                    P.out_val[grow] = dval;
                }
            }
            // warp-aggregated append of the uncertified rows, with what pass 2
            // needs: the candidate threshold and the seed (exact d1, j1)
            const bool need = !COLLECT && !F64 && grow < M && !ok;
            const unsigned bal = __ballot_sync(0xffffffffu, need);
            if (bal) {
                unsigned base = 0;
                if (lane == 0) base = atomicAdd(P.fb_count, unsigned(__popc(bal)));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (need) {
                    const unsigned q = base + __popc(bal & ((1u << lane) - 1u));
                    P.fb_rows[q] = int32_t(grow);
                    if (P.fb_thr) {
                        P.fb_thr[q] = thr_out;
                        P.fb_seed[q] = seed_out;
                    }
                }
            }
            __syncwarp();
            if (!SX && !released && lane == 0)
                for (int kb = 0; kb < nkb; ++kb) mbar_arrive(&a_kbe[ab * PR_MAX_KB + kb]);
            PROBE_ADD(7, clock64() - rw1_);
        }
    }

#ifdef FTK_PAIR_PROBE
    if (P.clk && lane == 0 && (warp == W_SCREEN0 || warp == W_MMA || warp == W_REFINE0 || warp == W_XPROD))
        for (int q = 0; q < 10; ++q) atomicAdd(reinterpret_cast<unsigned long long *>(P.clk) + q,
                                              (unsigned long long)clk[q]);
#endif
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == W_MMA) {
        tc_fence_after();
        tmem_dealloc_pair(tmem, 512);
    }
}

// ------------------------------------------------------------- host ------
size_t pair_smem_bytes(int nkb, int abufs, int stages, bool sx) {
    return 1024 + size_t(abufs) * PR_A_KB * nkb + size_t(stages) * (sx ? PR_B_HALF + PR_A_KB : PR_B_HALF) +
           2 * PR_SWG * PR_BM * (sizeof(PairPart) + sizeof(double2)) + 8 * PR_BN * sizeof(float) +
           8 * 8 * sizeof(float4) +
           (2 * size_t(stages) + 2 * PR_MAX_NA + 4 + 2 * PR_NBUF + PR_MAX_NA * PR_MAX_KB) * 8 + 64;
}

int pair_plan(int64_t d, int64_t k, int *abufs, int *stages) {
    const int nkb = int((d + PR_KB - 1) / PR_KB);
    const bool sx = nkb > PR_MAX_KB;  // X streamed through the stages
    const size_t cap = 227 * 1024;
    int na = sx ? 0 : 2;
    if (!sx && pair_smem_bytes(nkb, 2, 3, false) > cap) na = 1;
    // few centroid k-blocks per row tile (small k and d): a row tile's MMAs are
    // short, so the X half-tiles are the stream to keep in flight -- up to four
    // X buffers, as long as four centroid stages remain
    const int64_t kblocks = int64_t(nkb) * ((k + PR_BN - 1) / PR_BN);
    if (!sx && kblocks <= 4 && !getenv("FTK_PAIR_NA2"))
        for (int cand = PR_MAX_NA; cand > na; --cand)
            if (pair_smem_bytes(nkb, cand, 4, false) <= cap) {
                na = cand;
                break;
            }
    int s = 12;
    while (s >= 2 && pair_smem_bytes(nkb, na, s, sx) > cap) --s;
    if (s < 2) return -1;
    *abufs = na;
    *stages = s;
    return 0;
}

int pair_screen_launch(const CUtensorMap &mx, const CUtensorMap &mc, PairParams P, bool chk,
                       cudaStream_t st) {
    if (pair_plan(P.d, P.k, &P.abufs, &P.stages)) {
        set_error("tc pair: tile exceeds shared memory");
        return FTK_ERR_UNSUPPORTED;
    }
    if (const char *e = getenv("FTK_PAIR_STAGES")) {  // tuning knob
        const int s = atoi(e);
        if (s >= 2 && s < P.stages) P.stages = s;
    }
    P.nkb = int((P.d + PR_KB - 1) / PR_KB);
    P.ntiles = int((P.k + PR_BN - 1) / PR_BN);
    const bool sx = P.nkb > PR_MAX_KB;  // streamed X: re-read per column tile (from L2)
    const size_t smem = pair_smem_bytes(P.nkb, P.abufs, P.stages, sx);
    const int64_t npt = (P.m + 2 * PR_BM - 1) / (2 * PR_BM);
    if (npt == 0) return FTK_OK;
    int nsm = 148;
    nsm = current_sm_count();
    const int64_t nwork = (P.thr && FTK_PAIR_COLLECT_SPLIT) ? npt * P.ntiles : npt;  // COLLECT: one item per (row tile, column tile)
    const int64_t ncl = nwork < nsm / 2 ? nwork : nsm / 2;
    if (P.rec64) {  // float64 data, fp32 copy resident (d <= 256)
        if (sx) {
            set_error("tc pair f64: d > 256");
            return FTK_ERR_UNSUPPORTED;
        }
        auto k64 = chk ? pair_screen_kernel<true, false, false, false, true>
                       : pair_screen_kernel<false, false, false, false, true>;
        FTK_CUDA(cudaFuncSetAttribute(k64, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k64<<<dim3(unsigned(2 * ncl)), dim3(PR_THREADS), smem, st>>>(mx, mc, P);
        FTK_LAUNCHED("pair_screen_kernel");
        return FTK_OK;
    }
    auto kern = sx ? (chk ? (P.thr ? pair_screen_kernel<true, true, false, true>
                                   : (P.inj_col ? pair_screen_kernel<true, false, true, true>
                                                : pair_screen_kernel<true, false, false, true>))
                          : (P.thr ? pair_screen_kernel<false, true, false, true>
                                   : pair_screen_kernel<false, false, false, true>))
                   : (chk ? (P.thr ? pair_screen_kernel<true, true, false, false>
                                   : (P.inj_col ? pair_screen_kernel<true, false, true, false>
                                                : pair_screen_kernel<true, false, false, false>))
                          : (P.thr ? pair_screen_kernel<false, true, false, false>
                                   : pair_screen_kernel<false, false, false, false>));
    FTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<dim3(unsigned(2 * ncl)), dim3(PR_THREADS), smem, st>>>(mx, mc, P);
    FTK_LAUNCHED("pair_screen_kernel");
    return FTK_OK;
}

}  // namespace ftk

namespace ftk {
// ------------------------------------------------ pass 2: exact candidates --
// One thread per (row, centroid) candidate: the reference's exact value
// (sequential fp32 products and sums, k ascending, then yn - (acc + acc)),
// folded into the row's (value, index) key with an atomic minimum -- the
// reference's "first strict minimum" rule is "smallest value, then smallest
// index".  Non-finite values never win (the reference starts from +inf).
__global__ void cand_exact_kernel(const float *g, const float *y, const float *yn, int64_t d,
                                  const int2 *cand, const unsigned *count, unsigned cap,
                                  const unsigned *row_cnt, unsigned row_cap,
                                  unsigned long long *key) {
    const unsigned n = min(*count, cap);
    for (unsigned c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        const int2 e = cand[c];
        if (row_cnt[e.x] > row_cap) continue;  // row goes to the exact kernel
        const float *xr = g + int64_t(e.x) * d;
        const float *cr = y + int64_t(e.y) * d;
        float acc = 0.0f;
        int64_t f = 0;
        if ((d & 31) == 0 && ((reinterpret_cast<uintptr_t>(xr) | reinterpret_cast<uintptr_t>(cr)) & 15) == 0) {
            // the chain is sequential (the reference's order); the loads are
            // not: 8-vector batches, the next batch in flight while the
            // current one is chained (one L2 round trip per 32 features
            // instead of one per 4)
            const float4 *x4 = reinterpret_cast<const float4 *>(xr);
            const float4 *c4 = reinterpret_cast<const float4 *>(cr);
            const int64_t nb = d / 32;
            float4 xa[8], ca[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) { xa[u] = __ldg(x4 + u); ca[u] = __ldg(c4 + u); }
            for (int64_t b = 0; b < nb; ++b) {
                float4 xn[8], cn[8];
                const int64_t o = (b + 1 < nb ? b + 1 : b) * 8;
#pragma unroll
                for (int u = 0; u < 8; ++u) { xn[u] = __ldg(x4 + o + u); cn[u] = __ldg(c4 + o + u); }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    acc = __fadd_rn(acc, __fmul_rn(xa[u].x, ca[u].x));
                    acc = __fadd_rn(acc, __fmul_rn(xa[u].y, ca[u].y));
                    acc = __fadd_rn(acc, __fmul_rn(xa[u].z, ca[u].z));
                    acc = __fadd_rn(acc, __fmul_rn(xa[u].w, ca[u].w));
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) { xa[u] = xn[u]; ca[u] = cn[u]; }
            }
        } else if ((d & 3) == 0) {
            const float4 *x4 = reinterpret_cast<const float4 *>(xr);
            const float4 *c4 = reinterpret_cast<const float4 *>(cr);
            for (; f < d / 4; ++f) {
                const float4 a = __ldg(x4 + f), b = __ldg(c4 + f);
                acc = __fadd_rn(acc, __fmul_rn(a.x, b.x));
                acc = __fadd_rn(acc, __fmul_rn(a.y, b.y));
                acc = __fadd_rn(acc, __fmul_rn(a.z, b.z));
                acc = __fadd_rn(acc, __fmul_rn(a.w, b.w));
            }
        } else {
            for (; f < d; ++f) acc = __fadd_rn(acc, __fmul_rn(__ldg(xr + f), __ldg(cr + f)));
        }
        const float v = __fsub_rn(__ldg(yn + e.y), __fadd_rn(acc, acc));
        if (v < INFINITY)
            atomicMin(key + e.x,
                      (static_cast<unsigned long long>(ordered_key(v)) << 32) | unsigned(e.y));
    }
}

// Resolved rows write their outputs; rows whose candidate set overflowed,
// rows beyond the pass-2 capacity (or the whole pass when the global list
// did) go to the exact kernel.
__global__ void cand_finalize_kernel(const int32_t *rows, const unsigned *n_rows, unsigned row_cap_n,
                                     const unsigned long long *key, const unsigned *row_cnt,
                                     unsigned row_cap, const unsigned *count, unsigned cap,
                                     int32_t *out_idx, float *out_val, int32_t *rows2,
                                     unsigned *n2) {
    const unsigned n = *n_rows;
    const bool global_over = *count > cap;
    for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int32_t row = rows[q];
        if (q >= row_cap_n || global_over || row_cnt[q] > row_cap) {
            rows2[atomicAdd(n2, 1u)] = row;
            continue;
        }
        const unsigned long long k = key[q];
        if (k == ~0ull) {  // nothing finite: the reference keeps (+inf, 0)
            out_idx[row] = 0;
            out_val[row] = INFINITY;
        } else {
            const uint32_t u = uint32_t(k >> 32);
            out_idx[row] = int32_t(k & 0xFFFFFFFFu);
            out_val[row] = __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
        }
    }
}

// Gather the pass-1 uncertified rows (device count, clamped to the pass-2
// capacity) and initialise their candidate keys (the pass-1 seed) and counts.
__global__ void pass2_gather_kernel(const float *x, int64_t d, const int32_t *rows,
                                    const unsigned *count, unsigned cap_rows,
                                    const unsigned long long *seed, float *g,
                                    unsigned long long *key, unsigned *row_cnt) {
    const unsigned n = min(*count, cap_rows);
    // one warp per row (16-byte copies when the rows are aligned): no
    // per-element 64-bit division
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const bool v4 = (d & 3) == 0 && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(g)) & 15) == 0;
    for (int64_t q = w0; q < n; q += nw) {
        const float *src = x + int64_t(rows[q]) * d;
        float *dst = g + q * d;
        if (v4) {
            const float4 *s4 = reinterpret_cast<const float4 *>(src);
            float4 *d4 = reinterpret_cast<float4 *>(dst);
            for (int64_t f = lane; f < d / 4; f += 32) d4[f] = __ldg(s4 + f);
        } else {
            for (int64_t f = lane; f < d; f += 32) dst[f] = __ldg(src + f);
        }
        if (lane == 0) {
            key[q] = seed[q];
            row_cnt[q] = 0u;
        }
    }
}

// Exact resolution of the (rare) rows no screen resolved: one warp per row,
// lanes take centroids j = lane, lane + 32, ...; each distance is the
// reference's sequential chain, the winner the first strict minimum.
__global__ void exact_rows_kernel(const float *x, const float *y, const float *yn, int64_t k,
                                  int64_t d, const int32_t *rows, const unsigned *count,
                                  int32_t *out_idx, float *out_val) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const unsigned n = *count;
    for (int64_t q = w0; q < n; q += nw) {
        const int32_t row = rows[q];
        const float *xr = x + int64_t(row) * d;
        float bv = INFINITY;
        int32_t bj = 0;
        for (int64_t j = lane; j < k; j += 32) {
            const float *cr = y + j * d;
            float acc = 0.0f;
            for (int64_t f = 0; f < d; ++f) acc = __fadd_rn(acc, __fmul_rn(__ldg(xr + f), __ldg(cr + f)));
            const float v = __fsub_rn(__ldg(yn + j), __fadd_rn(acc, acc));
            if (v < bv) {
                bv = v;
                bj = int32_t(j);
            }
        }
        for (int off = 16; off; off >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
            const int32_t oj = __shfl_xor_sync(0xffffffffu, bj, off);
            if (ov < bv || (ov == bv && oj < bj)) {
                bv = ov;
                bj = oj;
            }
        }
        if (lane == 0) {
            out_idx[row] = bj;
            out_val[row] = bv;
        }
    }
}

// One warp per flagged row: the reference of the group-weighted checksum
// x~ . csumw (lane partials, fixed shuffle tree), the error's 128-column group
// g = rint(D2 / D1) - 1 when consistent, and a DetectionEvent unless the row
// carries a scheduled flip (those get the reference's own record from the
// exact replay).  The row itself is re-resolved exactly by pass 2 -- the
// correction -- so every record is detected-corrected; loc_j = -1 (the
// column within the group is not resolved), tile_j = the group's tile.
__global__ void abft_flag_events_kernel(FlagEvents F) {
    const int lane = threadIdx.x & 31;
    const unsigned n = min(*F.count, F.cap);
    const unsigned w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned nw = (gridDim.x * blockDim.x) >> 5;
    for (unsigned q = w0; q < n; q += nw) {
        const double4 r = F.rec[q];
        const int64_t row = __double_as_longlong(r.x);
        const double D1 = r.y, wsum = r.z, tau = r.w;
        const float4 *x4 = reinterpret_cast<const float4 *>(F.x + row * F.d);
        const float4 *w4 = reinterpret_cast<const float4 *>(F.csumw);
        float wr = 0.0f, xx = 0.0f;
        for (int64_t f = lane; f < F.d / 4; f += 32) {
            const float4 xv = __ldg(x4 + f), wv = __ldg(w4 + f);
            wr = fmaf(tf32_trunc(xv.x), wv.x, wr);
            wr = fmaf(tf32_trunc(xv.y), wv.y, wr);
            wr = fmaf(tf32_trunc(xv.z), wv.z, wr);
            wr = fmaf(tf32_trunc(xv.w), wv.w, wr);
            xx = fmaf(xv.x, xv.x, fmaf(xv.y, xv.y, fmaf(xv.z, xv.z, fmaf(xv.w, xv.w, xx))));
        }
        for (int off = 16; off; off >>= 1) {
            wr += __shfl_xor_sync(0xffffffffu, wr, off);
            xx += __shfl_xor_sync(0xffffffffu, xx, off);
        }
        if (lane != 0) continue;
        const double D2 = wsum - double(wr);
        const int ng = int((F.k + 127) / 128);
        const double gf = rint(D2 / D1) - 1.0;
        int64_t col = 0;
        bool located = false;
        if (gf >= 0.0 && gf < double(ng)) {
            const double tw = double(ng + 1) * tau + fabs(D1) * double(ng) * 0x1p-18 +
                              64.0 * 0x1p-24 * sqrt(double(xx) * (1.0 + 0x1p-10)) *
                                  sqrt(double(F.camax[3]) * (1.0 + 0x1p-10));
            located = fabs(D2 - (gf + 1.0) * D1) <= tw;
            col = located ? int64_t(gf) * 128 : 0;
        }
        atomicAdd(F.corrected, 1u);
        if (F.ev.rec && (!F.inj_col || F.inj_col[row] < 0 || F.events_for_scheduled)) {
            const unsigned long long c = atomicAdd(reinterpret_cast<unsigned long long *>(F.ev.count), 1ull);
            if (c < (unsigned long long)F.ev.cap) {
                int64_t *rec = F.ev.rec + c * 7;
                rec[0] = F.iteration;
                rec[1] = row / F.bm;
                rec[2] = col / F.bn;
                rec[3] = 0;  // EV_CORRECTED: the row is re-resolved exactly
                rec[4] = row % F.bm;
                rec[5] = -1;
                rec[6] = F.interval;
                F.ev.delta[c] = D1;
            }
        }
        (void)located;
    }
}

int abft_flag_events_run(const FlagEvents &F, cudaStream_t st) {
    abft_flag_events_kernel<<<32, 256, 0, st>>>(F);
    FTK_LAUNCHED("abft_flag_events_kernel");
    return FTK_OK;
}

int pass2_gather_run(const float *x, int64_t d, const int32_t *rows, const unsigned *count,
                     unsigned cap_rows, const unsigned long long *seed, float *g,
                     unsigned long long *key, unsigned *row_cnt, cudaStream_t st) {
    pass2_gather_kernel<<<148 * 8, 256, 0, st>>>(x, d, rows, count, cap_rows, seed, g, key, row_cnt);
    FTK_LAUNCHED("pass2_gather_kernel");
    return FTK_OK;
}

int exact_rows_run(const float *x, const float *y, const float *yn, int64_t k, int64_t d,
                   const int32_t *rows, const unsigned *count, int32_t *out_idx, float *out_val,
                   cudaStream_t st) {
    exact_rows_kernel<<<148 * 2, 256, 0, st>>>(x, y, yn, k, d, rows, count, out_idx, out_val);
    FTK_LAUNCHED("exact_rows_kernel");
    return FTK_OK;
}

int pair_candidates_run(const float *g, const float *y, const float *yn, int64_t d,
                        const int2 *cand, const unsigned *count, unsigned cap,
                        const unsigned *row_cnt, unsigned row_cap, unsigned long long *key,
                        const int32_t *rows, const unsigned *n_rows, unsigned row_cap_n,
                        int32_t *out_idx, float *out_val, int32_t *rows2, unsigned *n2,
                        cudaStream_t st) {
    cand_exact_kernel<<<148 * 8, 256, 0, st>>>(g, y, yn, d, cand, count, cap, row_cnt, row_cap, key);
    FTK_LAUNCHED("cand_exact_kernel");
    cand_finalize_kernel<<<148, 256, 0, st>>>(rows, n_rows, row_cap_n, key, row_cnt, row_cap,
                                              count, cap, out_idx, out_val, rows2, n2);
    FTK_LAUNCHED("cand_finalize_kernel");
    return FTK_OK;
}
}  // namespace ftk
