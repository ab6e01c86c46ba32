// common.cuh -- shared helpers for the B200 FT K-means kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <string>

#include "../../include/ftk_b200.h"

namespace ftk {

// ---------------------------------------------------------------- errors --
void set_error(const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);
void count_launch(int n = 1);

#define FTK_CUDA(call)                                        \
    do {                                                      \
        cudaError_t e_ = (call);                              \
        if (e_ != cudaSuccess) return ::ftk::cuda_fail(e_, #call); \
    } while (0)

#define FTK_LAUNCHED(what)                                           \
    do {                                                             \
        ::ftk::count_launch();                                       \
        cudaError_t e_ = cudaGetLastError();                         \
        if (e_ != cudaSuccess) return ::ftk::cuda_fail(e_, what);    \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------------- scratch --
// Per-context cached device scratch (grown on demand, never shrunk).
struct Scratch {
    void *ptr = nullptr;
    size_t bytes = 0;
};

}  // namespace ftk

struct ftk_ctx {
    int device = 0;
    ftk::Scratch slots[32];
    // per-fit row bounds registered by ftk_ctx_set_rows (X constant for the fit)
    const void *rows_x = nullptr;
    int64_t rows_m = 0, rows_d = 0;
    const float *rows_info = nullptr;  // m x 4: |x|^2, |x - tf32(x)|^2, max|x|, 0
    const float *rows_x32 = nullptr;   // float64 data: the fp32 copy the tensor cores screen
    // diagnostics of the last screened assignment on this context
    unsigned last_fb[3] = {0, 0, 0};              // pass-1 uncertified, exact rows, ABFT flags
    int last_path = 0;                            // pass-1 kernel: 0 single-CTA, 1 CTA pair
    cudaEvent_t time_ev[2] = {nullptr, nullptr};  // around the last pass-1 launch
    const unsigned *stat_dev[3] = {nullptr, nullptr, nullptr};  // counters still on the device
    int64_t generation = 0;  // scratch (re)allocations: captured graphs go stale
    unsigned long long *abft_total = nullptr;  // cumulative TC/DMMA row-checksum flags (device)
    void *h2d = nullptr;  // staged pageable upload: pinned buffers, streams (h2d.cu)
    // label hint of the next assignment (ftk_ctx_set_label_hint): the previous
    // iteration's labels, used by the narrow screen to pick the exact chain
    const int32_t *hint = nullptr;
    int64_t hint_m = 0;
    int inj_replay = 1;  // FTK_OPT_INJ_REPLAY: replay blocks with scheduled flips exactly
    int family = 0;      // forced kernel family of the current call (0 auto, 1 pair, 2 narrow, 3 dmma, 4 dfma,
                         // 5 float64 through the tf32 CTA-pair screen)
};

namespace ftk {
// SM count of the CURRENT device (each rank of a multi-GPU run drives its own)
inline int current_sm_count() {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return nsm;
}
// Returns a device buffer of at least `bytes` for `slot` of this context.
void *scratch(ftk_ctx *ctx, int slot, size_t bytes, cudaStream_t st);
// The context's cumulative row-checksum flag counter (allocated and zeroed
// on first use, outside any capture; ftk_abft_flags_total reads it).
unsigned long long *abft_total_ptr(ftk_ctx *ctx, cudaStream_t st);

enum ScratchSlot {
    SLOT_BMAX = 0,
    SLOT_SORT_KEYS = 1,
    SLOT_SORT_VALS = 2,
    SLOT_SORT_TMP = 3,
    SLOT_OFFSETS = 4,
    SLOT_PAIRWISE = 5,
    SLOT_MISC = 6,
    SLOT_TC_A = 7,
    SLOT_TC_B = 8,
    SLOT_TC_ROWS = 9,
    SLOT_TC_MISC = 10,
    SLOT_INJ = 11,
    SLOT_SEG_BASE = 12,
    SLOT_SEG_PART = 13,
    SLOT_SEG_FB = 14,
    SLOT_TC_CSUM1 = 15,
    SLOT_TC_CSUM2 = 16,
    SLOT_TC_INJROWS = 17,
    SLOT_PAIR_FB = 18,    // pass-1 thresholds + seeds
    SLOT_PAIR_CAND = 19,  // pass-2 candidate list, keys, counters
    SLOT_DS = 20,         // float64 screen: bounds, counters, fallback rows
    SLOT_DS_G = 21,       // float64 screen: gathered fallback rows
    SLOT_EXACT_SPLIT = 22,  // per-(row, column split) argmin partials of the exact kernel
    SLOT_KPP = 23,          // k-means++: prefix scan of d2, counters, CUB temp
    SLOT_NARROW = 24,       // narrow screen: augmented centroids, tolerances, winner-pass rows
    SLOT_PAIR_FLAG = 25,    // CTA-pair screen: records of checksum-flagged rows
    SLOT_TC64_X = 26,       // float64 via tf32: per-call fp32 copy of X + row bounds
    SLOT_TC64_C = 27,       // float64 via tf32: fp32 centroids, norms, bounds, counters
    SLOT_TC64_REC = 28,     // float64 via tf32: per-row (j1, T) records, fallback rows
    SLOT_TC64_G = 29,       // float64 via tf32: gathered uncertified rows (DMMA pass 2)
    SLOT_TC64_P2 = 30,      // float64 via tf32: pass-2 thresholds, fp32 rows, candidates, keys
};

// ------------------------------------------------------- float helpers --
template <typename T> struct Bits;
template <> struct Bits<float> { using U = uint32_t; static constexpr int W = 32; };
template <> struct Bits<double> { using U = unsigned long long; static constexpr int W = 64; };

// Correctly rounded single operations that nvcc may not contract into FMA.
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

template <typename T>
__device__ __forceinline__ T flip_bit(T v, int64_t bit) {
    using U = typename Bits<T>::U;
    U u;
    memcpy(&u, &v, sizeof(T));
    u ^= (U(1) << U(bit));
    T r;
    memcpy(&r, &u, sizeof(T));
    return r;
}

// Lexicographic (value, index) minimum with the reference's candidate rule:
// a value only wins if it compares below the running best, so NaN and +inf
// never win and the default is (+inf, 0) (_kernels.py:88-102, 450-452).
template <typename T>
__device__ __forceinline__ void argmin_merge(T &bv, int32_t &bj, T v, int32_t j) {
    if (v < bv || (v == bv && j < bj)) {
        bv = v;
        bj = j;
    }
}

}  // namespace ftk
