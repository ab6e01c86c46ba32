// abi.cu -- extern "C" entry points (include/ftk_b200.h), context, errors.
#include <mutex>
#include <string>

#include "common.cuh"
#include "tc_pair.cuh"

namespace ftk {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string &msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return FTK_ERR_CUDA;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void *scratch(ftk_ctx *ctx, int slot, size_t bytes, cudaStream_t st) {
    Scratch &s = ctx->slots[slot];
    if (bytes == 0) bytes = 16;
    if (s.bytes >= bytes) return s.ptr;
    if (s.ptr) {
        cudaStreamSynchronize(st);
        cudaFree(s.ptr);
        s.ptr = nullptr;
        s.bytes = 0;
    }
    size_t want = bytes + bytes / 4;
    cudaError_t e = cudaMalloc(&s.ptr, want);
    if (e != cudaSuccess) {
        cuda_fail(e, "scratch cudaMalloc");
        s.ptr = nullptr;
        return nullptr;
    }
    s.bytes = want;
    ++ctx->generation;
    return s.ptr;
}

unsigned long long *abft_total_ptr(ftk_ctx *ctx, cudaStream_t st) {
    if (!ctx->abft_total) {
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(st, &cap);
        if (cap != cudaStreamCaptureStatusNone) return nullptr;  // counted from the next eager call
        if (cudaMalloc(&ctx->abft_total, sizeof(unsigned long long)) != cudaSuccess) {
            ctx->abft_total = nullptr;
            return nullptr;
        }
        cudaMemset(ctx->abft_total, 0, sizeof(unsigned long long));
    }
    return ctx->abft_total;
}

// implemented in exact.cu / update.cu / tc.cu / h2d.cu
void h2d_stage_free(void *);
int h2d_pageable_run(ftk_ctx *, void *, const void *, size_t, cudaStream_t);
int exact_run(ftk_ctx *, int, const void *, const void *, const void *, int64_t, int64_t, int64_t,
              int64_t, int64_t, int64_t, int32_t *, void *, void *, bool, double, double, int64_t,
              const ftk_injection *, ftk_events *, cudaStream_t);
int row_sq_norms_run(int, const void *, int64_t, int64_t, void *, cudaStream_t);
int row_info_run(const float *, int64_t, int64_t, float *, cudaStream_t);
int kpp_update_run(int, const void *, int64_t, int64_t, int64_t, const int64_t *, int, double *,
                   int64_t *, int64_t, cudaStream_t);
int kpp_search_run(ftk_ctx *, const double *, int64_t, double, int64_t *, unsigned long long *,
                   cudaStream_t);
int update_sums_run(ftk_ctx *, int, const void *, const int32_t *, int64_t, int64_t, int64_t,
                    double *, int64_t *, double *, int64_t *, cudaStream_t);
int dmr_compare_run(const double *, const int64_t *, const double *, const int64_t *, int64_t,
                    int64_t, int32_t *, cudaStream_t);
int finalize_run(int, const double *, const int64_t *, int64_t, int64_t, void *, int32_t *,
                 cudaStream_t);
int reseed_run(ftk_ctx *, int, const void *, int64_t, int64_t, const int64_t *, int64_t, double *,
               void *, cudaStream_t);
int sq_dists_run(int, const void *, const double *, int64_t, double *, cudaStream_t);
int pairwise_sum_run(ftk_ctx *, const double *, int64_t, double *, cudaStream_t);
int movement_run(ftk_ctx *, int, const void *, const void *, int64_t, int64_t, double, double *,
                 cudaStream_t);
int labels_equal_run(const int32_t *, const int32_t *, int64_t, int32_t *, cudaStream_t);
int own_sq_dists_run(ftk_ctx *, int, const void *, const int32_t *, const double *, int64_t,
                     int64_t, double *, cudaStream_t);
int flip_f64_run(double *, int64_t, int64_t, int64_t, int64_t, double *, cudaStream_t);
struct TcFt;
int tc_assign_run(ftk_ctx *, int, const void *, const void *, const void *, int64_t, int64_t,
                  int64_t, int32_t *, void *, cudaStream_t, float *raw, int split_only,
                  const TcFt *ft);
int tc_checked_run(ftk_ctx *, int, const void *, const void *, const void *, int64_t, int64_t,
                   int64_t, int64_t, int64_t, int64_t, double, double, int64_t, int32_t *, void *,
                   const ftk_injection *, ftk_events *, cudaStream_t);
int tc_supported(int dtype, int64_t m, int64_t k, int64_t d);
bool tc64_supported(int64_t m, int64_t k, int64_t d);
int tc64_assign_run(ftk_ctx *ctx, const double *x, const double *y, const double *yn, int64_t m,
                    int64_t k, int64_t d, int32_t *out_idx, double *out_val, const TcFt *ft,
                    cudaStream_t st);
int row_info64_run(const double *x, int64_t m, int64_t d, float *x32, float *info, cudaStream_t st);
int dscreen_run(ftk_ctx *, const double *, const double *, const double *, int64_t, int64_t,
                int64_t, int32_t *, double *, const TcFt *, cudaStream_t);
int tc_last_fallback(ftk_ctx *, unsigned *, cudaStream_t);
float tc_last_pass1_ms(ftk_ctx *);

static bool dtype_ok(int dt) { return dt == FTK_F32 || dt == FTK_F64; }

// Variant code -> forced kernel family for the duration of one call.
struct FamilyScope {
    ftk_ctx *ctx;
    bool ok = true;
    FamilyScope(ftk_ctx *c, int dtype, int variant) : ctx(c) {
        int fam = 0;
        switch (variant) {
            case FTK_VARIANT_TC_PAIR: fam = dtype == FTK_F64 ? 5 : 1; break;
            case FTK_VARIANT_TC_NARROW: fam = 2; break;
            case FTK_VARIANT_F64_DMMA: fam = 3; break;
            case FTK_VARIANT_F64_DFMA: fam = 4; break;
            case FTK_VARIANT_AUTO: case FTK_VARIANT_EXACT: case FTK_VARIANT_TC: break;
            default: ok = false;
        }
        if ((fam == 1 || fam == 2) && dtype != FTK_F32) ok = false;
        if ((fam == 3 || fam == 4) && dtype != FTK_F64) ok = false;
        if (!ok) set_error("variant does not apply to this dtype");
        ctx->family = ok ? fam : 0;
    }
    ~FamilyScope() { ctx->family = 0; }
};
// float64 through the tf32 CTA-pair screen: forced, or by default on shapes
// large enough to amortise the per-call fp32 copy of the centroids
static bool use_tc64(ftk_ctx *ctx, int64_t m, int64_t k, int64_t d) {
    if (ctx->family == 5) return true;
    if (ctx->family != 0) return false;
    if (const char *e = getenv("FTK_F64_TC")) return atoi(e) != 0 && tc64_supported(m, k, d);
    return m >= 65536 && tc64_supported(m, k, d);
}
static bool forced_tc(int v) { return v == FTK_VARIANT_TC || v == FTK_VARIANT_TC_PAIR || v == FTK_VARIANT_TC_NARROW; }
static bool forced_any(int v) { return v != FTK_VARIANT_AUTO && v != FTK_VARIANT_EXACT; }

}  // namespace ftk

using namespace ftk;

extern "C" {

const char *ftk_last_error(void) { return g_err.c_str(); }
int ftk_version(void) { return 1; }
int64_t ftk_launch_count(void) { return g_launches.load(); }

ftk_ctx *ftk_ctx_create(int device) {
    if (cudaSetDevice(device) != cudaSuccess) {
        set_error("cudaSetDevice failed");
        return nullptr;
    }
    ftk_ctx *c = new ftk_ctx();
    c->device = device;
    return c;
}

void ftk_ctx_destroy(ftk_ctx *ctx) {
    if (!ctx) return;
    cudaDeviceSynchronize();
    for (auto &s : ctx->slots)
        if (s.ptr) cudaFree(s.ptr);
    for (auto &e : ctx->time_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->abft_total) cudaFree(ctx->abft_total);
    h2d_stage_free(ctx->h2d);
    delete ctx;
}

int ftk_row_info(ftk_ctx *ctx, const float *x, int64_t m, int64_t d, float *info, void *stream) {
    if (!ctx || d < 1 || m < 0) { set_error("bad ctx/shape"); return FTK_ERR_ARG; }
    return row_info_run(x, m, d, info, as_stream(stream));
}

int ftk_kpp_d2(ftk_ctx *ctx, int dtype, const void *x, int64_t m, int64_t d, int64_t pick,
               int first, double *d2, void *stream) {
    if (!ctx || !dtype_ok(dtype) || d < 1 || m < 1 || pick < 0 || pick >= m) { set_error("bad ctx/dtype/pick"); return FTK_ERR_ARG; }
    return kpp_update_run(dtype, x, m, d, pick, nullptr, first, d2, nullptr, 0, as_stream(stream));
}

int ftk_kpp_update(ftk_ctx *ctx, int dtype, const void *x, int64_t m, int64_t d, int64_t host_pick,
                   const int64_t *pick_dev, int first, double *d2, int64_t *picks, int64_t c,
                   void *stream) {
    if (!ctx || !dtype_ok(dtype) || d < 1 || m < 1 || host_pick >= m || (host_pick < 0 && !pick_dev)) {
        set_error("bad ctx/shape/pick");
        return FTK_ERR_ARG;
    }
    return kpp_update_run(dtype, x, m, d, host_pick, pick_dev, first, d2, picks, c, as_stream(stream));
}

int ftk_kpp_search(ftk_ctx *ctx, const double *d2, int64_t m, double r, int64_t *pick_dev,
                   uint64_t *n_replays, void *stream) {
    if (!ctx || m < 1 || !pick_dev || !n_replays) { set_error("bad ctx/args"); return FTK_ERR_ARG; }
    return kpp_search_run(ctx, d2, m, r, pick_dev, reinterpret_cast<unsigned long long *>(n_replays),
                          as_stream(stream));
}

int64_t ftk_ctx_generation(ftk_ctx *ctx) { return ctx ? ctx->generation : -1; }

int ftk_ctx_set_rows(ftk_ctx *ctx, const void *x, int64_t m, int64_t d, const float *info) {
    if (!ctx) { set_error("bad ctx"); return FTK_ERR_ARG; }
    ctx->rows_x = x;
    ctx->rows_m = x ? m : 0;
    ctx->rows_d = x ? d : 0;
    ctx->rows_info = x ? info : nullptr;
    ctx->rows_x32 = nullptr;
    return FTK_OK;
}

int ftk_row_info64(ftk_ctx *ctx, const double *x, int64_t m, int64_t d, float *x32, float *info,
                   void *stream) {
    if (!ctx || d < 1 || m < 0 || (m > 0 && (!x || !x32 || !info))) { set_error("bad ctx/shape"); return FTK_ERR_ARG; }
    return row_info64_run(x, m, d, x32, info, as_stream(stream));
}

int ftk_ctx_set_rows64(ftk_ctx *ctx, const double *x, int64_t m, int64_t d, const float *x32,
                       const float *info) {
    if (!ctx) { set_error("bad ctx"); return FTK_ERR_ARG; }
    ctx->rows_x = x;
    ctx->rows_m = x ? m : 0;
    ctx->rows_d = x ? d : 0;
    ctx->rows_info = x ? info : nullptr;
    ctx->rows_x32 = x ? x32 : nullptr;
    return FTK_OK;
}

int ftk_ctx_set_label_hint(ftk_ctx *ctx, const int32_t *labels, int64_t m) {
    if (!ctx || m < 0) { set_error("bad ctx/m"); return FTK_ERR_ARG; }
    ctx->hint = labels;
    ctx->hint_m = labels ? m : 0;
    return FTK_OK;
}

int ftk_ctx_set_option(ftk_ctx *ctx, int option, int64_t value) {
    if (!ctx) { set_error("bad ctx"); return FTK_ERR_ARG; }
    switch (option) {
        case FTK_OPT_INJ_REPLAY: ctx->inj_replay = value != 0; return FTK_OK;
        default: set_error("unknown option"); return FTK_ERR_ARG;
    }
}

int ftk_row_sq_norms(ftk_ctx *ctx, int dtype, const void *x, int64_t m, int64_t n, void *out,
                     void *stream) {
    (void)ctx;
    if (!dtype_ok(dtype) || n < 1) { set_error("bad dtype/shape"); return FTK_ERR_ARG; }
    return row_sq_norms_run(dtype, x, m, n, out, as_stream(stream));
}

int ftk_assign(ftk_ctx *ctx, int dtype, int variant, const void *x, const void *y,
               const void *ynorms, int64_t m, int64_t k, int64_t d, int64_t bm, int64_t bn,
               int64_t bk, int32_t *out_idx, void *out_val, const ftk_injection *inj,
               void *stream) {
    if (!ctx || !dtype_ok(dtype)) { set_error("bad ctx/dtype"); return FTK_ERR_ARG; }
    FamilyScope fs(ctx, dtype, variant);
    if (!fs.ok) return FTK_ERR_ARG;
    cudaStream_t st = as_stream(stream);
    bool has_inj = inj && inj->n > 0;
    if (dtype == FTK_F64 && variant != FTK_VARIANT_EXACT && !has_inj && use_tc64(ctx, m, k, d)) {
        // float64 screened on the tf32 tensor cores, certified in float64 (tc64.cu)
        int rc = tc64_assign_run(ctx, static_cast<const double *>(x), static_cast<const double *>(y),
                                 static_cast<const double *>(ynorms), m, k, d, out_idx,
                                 static_cast<double *>(out_val), nullptr, st);
        if (rc != FTK_ERR_UNSUPPORTED || ctx->family == 5) return rc;
    }
    if (dtype == FTK_F64 && variant != FTK_VARIANT_EXACT && !has_inj) {
        // float64: DMMA / DFMA screen + certified exact refine (dscreen.cu)
        int rc = dscreen_run(ctx, static_cast<const double *>(x), static_cast<const double *>(y),
                             static_cast<const double *>(ynorms), m, k, d, out_idx,
                             static_cast<double *>(out_val), nullptr, st);
        if (rc != FTK_ERR_UNSUPPORTED || forced_any(variant)) return rc;
    }
    // scheduled flips in an unprotected pass: the reference's corrupted
    // result is the exact kernel's (the screens apply flips only when checked)
    if (!has_inj && (forced_tc(variant) || variant == FTK_VARIANT_AUTO)) {
        int rc = tc_assign_run(ctx, dtype, x, y, ynorms, m, k, d, out_idx, out_val, st, nullptr, 0,
                               nullptr);
        if (rc != FTK_ERR_UNSUPPORTED || forced_tc(variant)) return rc;
    }
    return exact_run(ctx, dtype, x, y, ynorms, m, k, d, bm, bn, bk, out_idx, out_val, nullptr,
                     false, 0.0, 0.0, 0, inj, nullptr, st);
}

int ftk_checked_assign(ftk_ctx *ctx, int dtype, int variant, const void *x, const void *y,
                       const void *ynorms, int64_t m, int64_t k, int64_t d, int64_t bm,
                       int64_t bn, int64_t bk, double delta_rel, double abs_tol,
                       int64_t iteration, int32_t *out_idx, void *out_val,
                       const ftk_injection *inj, ftk_events *ev, void *stream) {
    if (!ctx || !dtype_ok(dtype)) { set_error("bad ctx/dtype"); return FTK_ERR_ARG; }
    FamilyScope fs(ctx, dtype, variant);
    if (!fs.ok) return FTK_ERR_ARG;
    cudaStream_t st = as_stream(stream);
    if (dtype == FTK_F64 && variant != FTK_VARIANT_EXACT && bn >= 1 && bm >= 1 &&
        use_tc64(ctx, m, k, d)) {
        TcFt ft{delta_rel, abs_tol, bm, bn, bk, iteration, inj, ev};
        int rc = tc64_assign_run(ctx, static_cast<const double *>(x), static_cast<const double *>(y),
                                 static_cast<const double *>(ynorms), m, k, d, out_idx,
                                 static_cast<double *>(out_val), &ft, st);
        if (rc != FTK_ERR_UNSUPPORTED || ctx->family == 5) return rc;
    }
    if (dtype == FTK_F64 && variant != FTK_VARIANT_EXACT && bn >= 1 && bm >= 1) {
        TcFt ft{delta_rel, abs_tol, bm, bn, bk, iteration, inj, ev};
        int rc = dscreen_run(ctx, static_cast<const double *>(x), static_cast<const double *>(y),
                             static_cast<const double *>(ynorms), m, k, d, out_idx,
                             static_cast<double *>(out_val), &ft, st);
        if (rc != FTK_ERR_UNSUPPORTED || forced_any(variant)) return rc;
    }
    // TC path: screened assignment with per-tile row checksums; flagged rows
    // and the logical blocks carrying scheduled flips are resolved exactly
    if ((forced_tc(variant) || variant == FTK_VARIANT_AUTO) && bn >= 1 && bm >= 1) {
        if (tc_supported(dtype, m, k, d))
            return tc_checked_run(ctx, dtype, x, y, ynorms, m, k, d, bm, bn, bk, delta_rel, abs_tol,
                                  iteration, out_idx, out_val, inj, ev, st);
        if (forced_tc(variant)) {
            set_error("tensor-core variant: unsupported shape");
            return FTK_ERR_UNSUPPORTED;
        }
    }
    return exact_run(ctx, dtype, x, y, ynorms, m, k, d, bm, bn, bk, out_idx, out_val, nullptr,
                     true, delta_rel, abs_tol, iteration, inj, ev, st);
}

int ftk_gemm(ftk_ctx *ctx, int dtype, const void *x, const void *y, int64_t m, int64_t k,
             int64_t d, int64_t bm, int64_t bn, int64_t bk, double delta_rel, double abs_tol,
             int64_t iteration, void *out, const ftk_injection *inj, ftk_events *ev,
             void *stream) {
    if (!ctx || !dtype_ok(dtype)) { set_error("bad ctx/dtype"); return FTK_ERR_ARG; }
    return exact_run(ctx, dtype, x, y, nullptr, m, k, d, bm, bn, bk, nullptr, nullptr, out,
                     ev != nullptr, delta_rel, abs_tol, iteration, inj, ev, as_stream(stream));
}

int ftk_update_sums(ftk_ctx *ctx, int dtype, const void *x, const int32_t *labels, int64_t m,
                    int64_t d, int64_t k, double *sums_a, int64_t *counts_a, double *sums_b,
                    int64_t *counts_b, void *stream) {
    if (!ctx || !dtype_ok(dtype)) { set_error("bad ctx/dtype"); return FTK_ERR_ARG; }
    return update_sums_run(ctx, dtype, x, labels, m, d, k, sums_a, counts_a, sums_b, counts_b,
                           as_stream(stream));
}

int ftk_dmr_compare(ftk_ctx *ctx, const double *sums_a, const int64_t *counts_a,
                    const double *sums_b, const int64_t *counts_b, int64_t k, int64_t d,
                    int32_t *out_mismatch, void *stream) {
    (void)ctx;
    return dmr_compare_run(sums_a, counts_a, sums_b, counts_b, k, d, out_mismatch,
                           as_stream(stream));
}

int ftk_update_finalize(ftk_ctx *ctx, int dtype, const double *sums, const int64_t *counts,
                        int64_t k, int64_t d, void *centroids, int32_t *n_empty, void *stream) {
    (void)ctx;
    if (!dtype_ok(dtype)) { set_error("bad dtype"); return FTK_ERR_ARG; }
    return finalize_run(dtype, sums, counts, k, d, centroids, n_empty, as_stream(stream));
}

int ftk_reseed_empty(ftk_ctx *ctx, int dtype, const void *x, int64_t m, int64_t d,
                     const int64_t *counts, int64_t k, double *sq_dists, void *centroids,
                     void *stream) {
    if (!ctx || !dtype_ok(dtype)) { set_error("bad ctx/dtype"); return FTK_ERR_ARG; }
    return reseed_run(ctx, dtype, x, m, d, counts, k, sq_dists, centroids, as_stream(stream));
}

int ftk_sq_dists(ftk_ctx *ctx, int dtype, const void *min_dists, const double *x_sq, int64_t m,
                 double *sq, void *stream) {
    (void)ctx;
    return sq_dists_run(dtype, min_dists, x_sq, m, sq, as_stream(stream));
}

int ftk_pairwise_sum(ftk_ctx *ctx, const double *a, int64_t n, double *out, void *stream) {
    if (!ctx) { set_error("bad ctx"); return FTK_ERR_ARG; }
    return pairwise_sum_run(ctx, a, n, out, as_stream(stream));
}

int ftk_movement(ftk_ctx *ctx, int dtype, const void *new_c, const void *old_c, int64_t k,
                 int64_t d, double eps, double *moved, void *stream) {
    if (!ctx || !dtype_ok(dtype)) { set_error("bad ctx/dtype"); return FTK_ERR_ARG; }
    return movement_run(ctx, dtype, new_c, old_c, k, d, eps, moved, as_stream(stream));
}

int ftk_labels_equal(ftk_ctx *ctx, const int32_t *a, const int32_t *b, int64_t m, int32_t *out,
                     void *stream) {
    (void)ctx;
    return labels_equal_run(a, b, m, out, as_stream(stream));
}

int ftk_own_sq_dists(ftk_ctx *ctx, int dtype, const void *x, const int32_t *labels,
                     const double *cent64, int64_t m, int64_t d, double *out, void *stream) {
    if (!ctx || !dtype_ok(dtype)) { set_error("bad ctx/dtype"); return FTK_ERR_ARG; }
    return own_sq_dists_run(ctx, dtype, x, labels, cent64, m, d, out, as_stream(stream));
}

int ftk_flip_f64(ftk_ctx *ctx, double *a, int64_t d, int64_t i, int64_t j, int64_t bit,
                 double *before_after, void *stream) {
    (void)ctx;
    return flip_f64_run(a, d, i, j, bit, before_after, as_stream(stream));
}

int ftk_tc_fallback_rows(ftk_ctx *ctx, int64_t *out, void *stream) {
    if (!ctx) { set_error("bad ctx"); return FTK_ERR_ARG; }
    unsigned v[3] = {0, 0, 0};
    int rc = tc_last_fallback(ctx, v, as_stream(stream));
    out[0] = int64_t(v[0]);
    out[1] = int64_t(v[1]);
    out[2] = int64_t(v[2]);
    return rc;
}

void ftk_add_launches(int64_t n) { count_launch(int(n)); }

int ftk_h2d(ftk_ctx *ctx, void *dst, const void *src, int64_t nbytes, void *stream) {
    if (!ctx || nbytes < 0 || (nbytes && (!dst || !src))) { set_error("bad ctx/args"); return FTK_ERR_ARG; }
    return h2d_pageable_run(ctx, dst, src, size_t(nbytes), as_stream(stream));
}

int ftk_abft_flags_total(ftk_ctx *ctx, int64_t *out, int reset, void *stream) {
    if (!ctx || !out) { set_error("bad ctx"); return FTK_ERR_ARG; }
    *out = 0;
    if (!ctx->abft_total) return FTK_OK;
    cudaStream_t st = as_stream(stream);
    unsigned long long v = 0;
    FTK_CUDA(cudaMemcpyAsync(&v, ctx->abft_total, sizeof(v), cudaMemcpyDeviceToHost, st));
    FTK_CUDA(cudaStreamSynchronize(st));
    *out = int64_t(v);
    if (reset) FTK_CUDA(cudaMemsetAsync(ctx->abft_total, 0, sizeof(v), st));
    return FTK_OK;
}

int ftk_tc_last_kernel_ms(ftk_ctx *ctx, float *ms) {
    if (!ctx || !ms) { set_error("bad ctx"); return FTK_ERR_ARG; }
    *ms = tc_last_pass1_ms(ctx);
    return FTK_OK;
}

int ftk_tc_raw_dots(ftk_ctx *ctx, int split, const float *x, const float *y, const float *ynorms,
                    int64_t m, int64_t k, int64_t d, float *raw, int32_t *out_idx,
                    float *out_val, void *stream) {
    if (!ctx || !raw) { set_error("bad ctx/raw"); return FTK_ERR_ARG; }
    return tc_assign_run(ctx, FTK_F32, x, y, ynorms, m, k, d, out_idx, out_val,
                         as_stream(stream), raw, split, nullptr);
}

}  // extern "C"
