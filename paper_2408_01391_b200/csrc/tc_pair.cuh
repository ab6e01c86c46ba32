// tc_pair.cuh -- parameters and launcher of the CTA-pair screen (tc_pair.cu)
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ftk_b200.h"

namespace ftk {

// centroids per accumulator tile (the TMEM holds 512 / PAIR_BN buffers);
// each CTA of the pair loads PAIR_BN / 2 centroid rows per k-block
#ifndef FTK_PAIR_BN  // A/B knob: 128 (four TMEM buffers) measured 40% slower at c2
#define FTK_PAIR_BN 256
#endif
constexpr int PAIR_BN = FTK_PAIR_BN;

struct PairParams {
    const float *x;  // rows (global, read by the refine warps)
    const float *y, *yn;
    int64_t m, k, d;
    int nkb, ntiles, stages, abufs;
    float a_coef, b_coef;
    const float *cmax2, *ecmax2;
    int32_t *out_idx;
    float *out_val;
    int32_t *fb_rows;
    unsigned *fb_count;
    // ABFT
    const float *csum, *camax;
    float tau_coef, tau_abs;
    const int32_t *inj_col;
    const float *inj_before, *inj_after;
    unsigned *abft_count;
    unsigned long long *abft_total;  // cumulative over launches (ftk_abft_flags_total)
    // ABFT: every row whose checksum fails is recorded as (row, D1 = row sum
    // - reference, the 128-column-group-weighted row sum, tau) for
    // abft_flag_events_run (location + event record after the pass)
    double4 *flag_rec;
    unsigned *flag_count;
    unsigned flag_cap;
    // pass 1: per uncertified row, the pass-2 threshold and the (d1, j1) seed key
    float *fb_thr;
    unsigned long long *fb_seed;
    // pass 2 (COLLECT mode, thr != null): rows are the gathered uncertified
    // rows; every column with s_j <= thr[row] is appended to cand
    const float *thr;
    int2 *cand;
    unsigned *cand_count;
    unsigned cand_cap;
    unsigned *row_cnt;
    const unsigned *m_dev;  // device-side row count (<= m) or null
    const float4 *rowinfo;  // per-fit row bounds (|x|^2, |x - tf32 x|^2, max|x|) or null
    // previous iteration's labels (m entries) or null: the refine prefetches
    // the hinted centroid's first two k-blocks during the previous row tile
    // (a speed hint only: a row whose winner differs reloads)
    const int32_t *hint;
    // float64 data screened in tf32 (tc64 path): per row (j1, T) -- T the
    // certificate threshold (j1 is the reference's argmin if its exact float64
    // value d1 < T); j1 = -1 when the row is not screenable (checksum flag,
    // non-finite).  The refine then skips the fp32 exact chain.
    int2 *rec64;
    float *a64;   // optional: per-row screen bound A (the float64 pass-2 candidate threshold)
    float a_abs;  // extra absolute screen error (the fp32 rounding of float64 norms)
    long long *clk;  // debug: per-role clock64 sums (screen busy/wait, MMA waits), or null
    int dbg;  // bit 0: skip the screen math, bit 1: skip the refine (pipeline timing only)
};

int pair_screen_launch(const CUtensorMap &mx, const CUtensorMap &mc, PairParams P, bool chk,
                       cudaStream_t st);

}  // namespace ftk

namespace ftk {
int pair_candidates_run(const float *g, const float *y, const float *yn, int64_t d,
                        const int2 *cand, const unsigned *count, unsigned cap,
                        const unsigned *row_cnt, unsigned row_cap, unsigned long long *key,
                        const int32_t *rows, const unsigned *n_rows, unsigned row_cap_n,
                        int32_t *out_idx, float *out_val, int32_t *rows2, unsigned *n2,
                        cudaStream_t st);
int pass2_gather_run(const float *x, int64_t d, const int32_t *rows, const unsigned *count,
                     unsigned cap_rows, const unsigned long long *seed, float *g,
                     unsigned long long *key, unsigned *row_cnt, cudaStream_t st);
int exact_rows_run(const float *x, const float *y, const float *yn, int64_t k, int64_t d,
                   const int32_t *rows, const unsigned *count, int32_t *out_idx, float *out_val,
                   cudaStream_t st);
// Location (128-column group, weighted checksum) and event records of the
// rows the CTA-pair screen flagged (see abft_flag_events_kernel).
struct FlagEvents {
    const float *x;
    int64_t d, k;
    const float *csumw, *camax;
    const double4 *rec;
    const unsigned *count;
    unsigned cap;
    const int32_t *inj_col;  // rows carrying a scheduled flip (replayed exactly), or null
    int events_for_scheduled;
    ftk_events ev;
    int64_t iteration, bm, bn, interval;
    unsigned *corrected;
};
int abft_flag_events_run(const FlagEvents &F, cudaStream_t st);
}  // namespace ftk

namespace ftk {
struct TcFt {  // checksum-protected (abft) mode of a screened assignment
    double delta_rel, abs_tol;
    int64_t bm, bn, bk, iteration;
    const ftk_injection *inj;
    ftk_events *ev;
};

// streamed-X narrow screen (tc_narrow.cu): K + 4 <= 256, any D % 4 == 0
struct NarrowIn {
    const float *x, *y, *yn;
    int64_t m, k, d;
    int32_t *out_idx;
    float *out_val;
    const float *cmax2, *ecmax2;  // device scalars (tc_prep_kernel)
    int32_t *fb_rows;             // m + 1 entries
    unsigned *cnt;                // [0] exact rows, [2] abft flags, [3] winner rows, [4] corrected
    const TcFt *ft;               // null: FT off
    const int32_t *inj_col;
    const float *inj_before, *inj_after;
};
bool narrow_supported(int64_t k, int64_t d, bool chk);
int narrow_assign_run(ftk_ctx *ctx, const NarrowIn &in, cudaStream_t st);

// The logical row blocks that carry scheduled flips are recomputed by the
// exact checked kernel (the reference's detection, location, correction and
// event record, bit for bit) and overwrite the screened results of those rows.
template <typename T>
int emulate_injected_blocks(ftk_ctx *ctx, const T *xf, const T *yf, const T *ynf, int64_t m,
                            int64_t k, int64_t d, const TcFt &ft, int32_t *out_idx, T *outv,
                            cudaStream_t st);
}  // namespace ftk
