// h2d.cu -- host -> device upload of a PAGEABLE buffer (the reference's
// numpy input) at pinned-copy speed.
//
// A plain cudaMemcpy from pageable memory is staged by the driver through a
// small bounce buffer, one chunk at a time, with the host copy and the DMA
// serialised (~10-20 GB/s).  Here T host threads each own two page-locked
// staging buffers and a stream: thread t copies chunks t, t+T, ... of the
// source into its staging buffer (memcpy, parallel across threads) and
// queues the DMA; the next chunk's memcpy overlaps that DMA.  The caller's
// stream then waits on every thread's last DMA, so work queued after the
// upload is ordered behind it without a host synchronisation.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"

namespace ftk {

struct H2DStage {
    static constexpr int T = 16;                   // max copy threads (FTK_H2D_THREADS, default 6)
    static constexpr size_t CH = size_t(8) << 20;  // bytes per chunk
    void *buf[T][2] = {};
    cudaEvent_t ev[T][2] = {};
    cudaStream_t st[T] = {};
    int ready = 0;  // threads whose buffers, events and stream exist
};

static int stage_init(H2DStage &S, int nt) {
    for (int t = S.ready; t < nt; ++t) {
        FTK_CUDA(cudaStreamCreateWithFlags(&S.st[t], cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            FTK_CUDA(cudaHostAlloc(&S.buf[t][b], H2DStage::CH, cudaHostAllocDefault));
            FTK_CUDA(cudaEventCreateWithFlags(&S.ev[t][b], cudaEventDisableTiming));
        }
        S.ready = t + 1;
    }
    return FTK_OK;
}

void h2d_stage_free(void *p) {
    auto *S = static_cast<H2DStage *>(p);
    if (!S) return;
    for (int t = 0; t < H2DStage::T; ++t) {
        for (int b = 0; b < 2; ++b) {
            if (S->buf[t][b]) cudaFreeHost(S->buf[t][b]);
            if (S->ev[t][b]) cudaEventDestroy(S->ev[t][b]);
        }
        if (S->st[t]) cudaStreamDestroy(S->st[t]);
    }
    delete S;
}

int h2d_pageable_run(ftk_ctx *ctx, void *dst, const void *src, size_t n, cudaStream_t st) {
    if (n == 0) return FTK_OK;
    if (!ctx->h2d) ctx->h2d = new H2DStage();
    H2DStage &S = *static_cast<H2DStage *>(ctx->h2d);
    // copy threads: the host cores but two, up to 14 (a 10-iteration c2 fit from
    // numpy: 4 threads 255, 6 332, 10 371, 14 385 iter/s, profiles/r3z)
    const int hw = int(std::thread::hardware_concurrency());
    int want = std::max(2, std::min(14, hw > 2 ? hw - 2 : 2));
    if (const char *e = getenv("FTK_H2D_THREADS")) want = std::max(1, std::min(H2DStage::T, atoi(e)));
    // the upload may overwrite memory the caller's stream still reads
    cudaEvent_t start;
    FTK_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    FTK_CUDA(cudaEventRecord(start, st));
    const size_t nch = (n + H2DStage::CH - 1) / H2DStage::CH;
    const int nt = int(std::min<size_t>(size_t(want), nch));
    if (int rc = stage_init(S, nt)) return rc;
    std::vector<int> rc(nt, FTK_OK);
    std::vector<std::string> err(nt);
    auto work = [&](int t) {
        cudaSetDevice(ctx->device);
        if (cudaStreamWaitEvent(S.st[t], start, 0) != cudaSuccess) { rc[t] = FTK_ERR_CUDA; return; }
        int b = 0;
        for (size_t c = size_t(t); c < nch; c += size_t(nt), b ^= 1) {
            const size_t off = c * H2DStage::CH;
            const size_t len = std::min(H2DStage::CH, n - off);
            // the DMA that last read this staging buffer must be done
            if (cudaEventSynchronize(S.ev[t][b]) != cudaSuccess) { rc[t] = FTK_ERR_CUDA; return; }
            std::memcpy(S.buf[t][b], static_cast<const char *>(src) + off, len);
            if (cudaMemcpyAsync(static_cast<char *>(dst) + off, S.buf[t][b], len, cudaMemcpyHostToDevice,
                                S.st[t]) != cudaSuccess ||
                cudaEventRecord(S.ev[t][b], S.st[t]) != cudaSuccess) {
                rc[t] = FTK_ERR_CUDA;
                return;
            }
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto &h : th) h.join();
    cudaEventDestroy(start);
    for (int t = 0; t < nt; ++t)
        if (rc[t]) {
            set_error("h2d staged upload: CUDA call failed");
            return rc[t];
        }
    // the caller's stream is ordered behind every thread's last DMA
    for (int t = 0; t < nt; ++t) {
        const int last_b = int(((nch - 1 - size_t(t)) / size_t(nt)) & 1);
        FTK_CUDA(cudaStreamWaitEvent(st, S.ev[t][last_b], 0));
    }
    return FTK_OK;
}

}  // namespace ftk
