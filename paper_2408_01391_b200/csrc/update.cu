// update.cu -- centroid update, inertia and convergence kernels (sm_100a).
//
// The reference accumulates per-cluster sums with numpy.bincount: float64,
// ascending sample order, one pass per feature (kmeans.py:167-171).  Floating
// point addition is not associative, so to reproduce those bits the update
// walks each cluster's members in ascending sample index: a stable radix sort
// of the labels gives every cluster its member list, then one warp per
// (cluster, 32-feature group) runs the float64 chains with coalesced row
// loads.  The chain for DMR mode carries two independent accumulators over
// the same loaded values (the reference's duplicated accumulation,
// kmeans.py:176-189); the compare is bitwise.
//
// Inertia uses numpy's pairwise summation tree (kmeans.py:275, 307) and the
// movement test np.linalg.norm's per-row pairwise reduce (kmeans.py:289-293),
// both evaluated on the device with the same association.
//
// Compiled with --fmad=false.

#include <cub/cub.cuh>

#include <algorithm>
#include <functional>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace ftk {

// --------------------------------------------------------------- counts --
__global__ void histogram_kernel(const int32_t *labels, int64_t m, int64_t k,
                                 unsigned long long *counts) {
    extern __shared__ unsigned int hist[];
    for (int64_t c = threadIdx.x; c < k; c += blockDim.x) hist[c] = 0;
    __syncthreads();
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x)
        atomicAdd(&hist[labels[i]], 1u);
    __syncthreads();
    for (int64_t c = threadIdx.x; c < k; c += blockDim.x)
        if (hist[c]) atomicAdd(&counts[c], (unsigned long long)hist[c]);
}

__global__ void histogram_global_kernel(const int32_t *labels, int64_t m,
                                        unsigned long long *counts) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x)
        atomicAdd(&counts[labels[i]], 1ull);
}

// Independent second count (DMR): segment boundaries of the sorted labels.
__global__ void boundary_count_kernel(const int32_t *sorted, int64_t m, int64_t k,
                                      unsigned long long *counts) {
    // counts must be zeroed; segment end adds end, segment start subtracts
    // start (two's complement wrap makes the unsigned atomics exact).
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x) {
        int32_t c = sorted[i];
        if (i == m - 1 || sorted[i + 1] != c) atomicAdd(&counts[c], (unsigned long long)(i + 1));
        if (i == 0 || sorted[i - 1] != c) atomicAdd(&counts[c], (unsigned long long)(-i));
    }
}

__global__ void exclusive_scan_small_kernel(const int64_t *counts, int64_t k, int64_t *offsets) {
    // single block; k up to a few hundred thousand is fine
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < k; base += blockDim.x) {
        int64_t i = base + threadIdx.x;
        int64_t v = i < k ? counts[i] : 0;
        // block inclusive scan via warp shuffles + smem
        __shared__ int64_t warp_tot[32];
        int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        int64_t s = v;
        for (int off = 1; off < 32; off <<= 1) {
            int64_t o = __shfl_up_sync(0xffffffffu, s, off);
            if (lane >= off) s += o;
        }
        if (lane == 31) warp_tot[w] = s;
        __syncthreads();
        if (w == 0) {
            int64_t t = lane < int(blockDim.x / 32) ? warp_tot[lane] : 0;
            for (int off = 1; off < 32; off <<= 1) {
                int64_t o = __shfl_up_sync(0xffffffffu, t, off);
                if (lane >= off) t += o;
            }
            warp_tot[lane] = t;
        }
        __syncthreads();
        int64_t incl = s + (w ? warp_tot[w - 1] : 0);
        if (i < k) offsets[i] = carry + incl - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) offsets[k] = carry;
}

// ------------------------------------------------- stable counting sort --
// Member lists (rows of each cluster in ascending sample order) for K up to
// CS_MAX_K: per-block label histograms, a per-label scan over blocks, and a
// stable scatter -- four small kernels in place of iota + a two-pass radix
// sort + boundary counting + the count scan.  Block b owns rows
// [b*chunk, (b+1)*chunk); within it, warp w owns a contiguous sub-chunk, so
// (block, warp, lane) order is sample order.
constexpr int CS_MAX_K = 8192;
constexpr int CS_WARPS_MAX = 8;

__host__ __device__ inline int cs_warps(int64_t k) {
    // per-warp label counters in shared memory: <= 64 KB
    int w = CS_WARPS_MAX;
    while (w > 1 && int64_t(w) * k * 4 > 64 * 1024) w /= 2;
    return w;
}

__global__ void cs_hist_kernel(const int32_t *labels, int64_t m, int64_t k, int64_t chunk,
                               int32_t *hist, int64_t nb) {
    extern __shared__ int32_t cnt[];
    for (int64_t b = threadIdx.x; b < k; b += blockDim.x) cnt[b] = 0;
    __syncthreads();
    const int64_t r0 = int64_t(blockIdx.x) * chunk;
    const int64_t r1 = r0 + chunk < m ? r0 + chunk : m;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const int32_t lab = labels[i];
        if (uint32_t(lab) < uint32_t(k)) atomicAdd(&cnt[lab], 1);  // out-of-range rows: no member
    }
    __syncthreads();
    for (int64_t b = threadIdx.x; b < k; b += blockDim.x) hist[b * nb + blockIdx.x] = cnt[b];
}

// one warp per label: exclusive prefix over blocks (in place), label total
__global__ void cs_binscan_kernel(int32_t *hist, int64_t nb, int64_t k, int64_t *counts) {
    const int64_t bin = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (bin >= k) return;
    int32_t *h = hist + bin * nb;
    int64_t run = 0;
    for (int64_t j0 = 0; j0 < nb; j0 += 32) {
        const int32_t v = j0 + lane < nb ? h[j0 + lane] : 0;
        int32_t s = v;
        for (int off = 1; off < 32; off <<= 1) {
            const int32_t o = __shfl_up_sync(0xffffffffu, s, off);
            if (lane >= off) s += o;
        }
        if (j0 + lane < nb) h[j0 + lane] = int32_t(run) + s - v;
        run += __shfl_sync(0xffffffffu, s, 31);
    }
    if (lane == 0) counts[bin] = run;
}

// Stable scatter: the block's per-label bases come from the scans; each warp
// first counts its sub-chunk per label, the block turns those into per-warp
// bases, then every warp walks its rows in order, 32 at a time, ranking equal
// labels with __match_any_sync.
__global__ void cs_scatter_kernel(const int32_t *labels, int64_t m, int64_t k, int64_t chunk,
                                  const int32_t *hist, int64_t nb, const int64_t *offsets,
                                  int32_t *perm) {
    extern __shared__ int32_t wcnt[];  // [warps][k]
    const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t e = threadIdx.x; e < int64_t(nw) * k; e += blockDim.x) wcnt[e] = 0;
    __syncthreads();
    const int64_t r0 = int64_t(blockIdx.x) * chunk;
    const int64_t r1 = r0 + chunk < m ? r0 + chunk : m;
    const int64_t sub = (chunk + nw - 1) / nw;
    const int64_t w0 = r0 + int64_t(w) * sub < r1 ? r0 + int64_t(w) * sub : r1;
    const int64_t w1 = w0 + sub < r1 ? w0 + sub : r1;
    int32_t *mine = wcnt + int64_t(w) * k;
    for (int64_t i = w0 + lane; i < w1; i += 32) {
        const int32_t lab = labels[i];
        if (uint32_t(lab) < uint32_t(k)) atomicAdd(&mine[lab], 1);
    }
    __syncthreads();
    // per-warp bases: global label start + this block's prefix + earlier warps
    for (int64_t b = threadIdx.x; b < k; b += blockDim.x) {
        int32_t run = int32_t(offsets[b]) + hist[b * nb + blockIdx.x];
        for (int q = 0; q < nw; ++q) {
            const int32_t c = wcnt[int64_t(q) * k + b];
            wcnt[int64_t(q) * k + b] = run;
            run += c;
        }
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t base = w0; base < w1; base += 128) {
        int32_t labs[4];  // four rounds of labels in flight
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = base + 32 * u + lane;
            labs[u] = i < w1 ? labels[i] : -1;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = base + 32 * u + lane;
            int32_t lab = labs[u];
            const bool live = uint32_t(lab) < uint32_t(k);
            if (!live) lab = -1 - lane;  // tail / out-of-range lanes: unique dummies
            const unsigned peers = __match_any_sync(0xffffffffu, lab);
            if (live) {
                const int32_t pos = mine[lab] + __popc(peers & lt);
                perm[pos] = int32_t(i);
            }
            __syncwarp();
            if (live && (peers & lt) == 0) mine[lab] += __popc(peers);
            __syncwarp();
        }
    }
}

// Single block: offsets = exclusive scan of the member counts and, for the
// segmented update, the segment table -- seg_base = exclusive scan of
// ceil(count / SEG), seg_cl[s] = cluster owning segment s.  Also zeroes the
// replay queue counter.
template <typename F>
__device__ void block_exclusive_scan(F val, int64_t k, int64_t *out) {
    __shared__ int64_t carry;
    __shared__ int64_t warp_tot[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t base = 0; base < k; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const int64_t v = i < k ? val(i) : 0;
        int64_t s = v;
        for (int off = 1; off < 32; off <<= 1) {
            const int64_t o = __shfl_up_sync(0xffffffffu, s, off);
            if (lane >= off) s += o;
        }
        if (lane == 31) warp_tot[w] = s;
        __syncthreads();
        if (w == 0) {
            int64_t t = lane < int(blockDim.x / 32) ? warp_tot[lane] : 0;
            for (int off = 1; off < 32; off <<= 1) {
                const int64_t o = __shfl_up_sync(0xffffffffu, t, off);
                if (lane >= off) t += o;
            }
            warp_tot[lane] = t;
        }
        __syncthreads();
        const int64_t incl = s + (w ? warp_tot[w - 1] : 0);
        if (i < k) out[i] = carry + incl - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[k] = carry;
    __syncthreads();
}

constexpr int SEG_MEMBERS = 256;  // == SEG (segment length of the certified update)

__global__ void offsets_segs_kernel(const int64_t *counts, int64_t k, int64_t *offsets,
                                    int64_t *seg_base, int32_t *seg_cl, unsigned *zero,
                                    unsigned *done = nullptr) {
    if (zero && threadIdx.x == 0) *zero = 0u;
    if (done)
        for (int64_t c = threadIdx.x; c < k; c += blockDim.x) done[c] = 0u;
    block_exclusive_scan([&](int64_t i) { return counts[i]; }, k, offsets);
    if (!seg_base) return;
    block_exclusive_scan([&](int64_t i) { return (counts[i] + SEG_MEMBERS - 1) / SEG_MEMBERS; }, k,
                         seg_base);
    for (int64_t c = threadIdx.x; c < k; c += blockDim.x)
        for (int64_t s = seg_base[c]; s < seg_base[c + 1]; ++s) seg_cl[s] = int32_t(c);
}

__global__ void iota_kernel(int32_t *v, int64_t m) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x)
        v[i] = int32_t(i);
}

// ----------------------------------------------------- ordered chains --
// One warp per (cluster, 32-feature group).  Lane f accumulates feature
// g*32+f over the cluster's members in ascending sample order.
template <typename T, bool DMR>
__global__ void __launch_bounds__(256) chain_sums_kernel(const T *x, int64_t d,
                                                         const int32_t *perm,
                                                         const int64_t *offsets, int64_t k,
                                                         double *sums_a, double *sums_b) {
    const int warps_per_block = blockDim.x / 32;
    const int64_t ngroups = (d + 31) / 32;
    const int64_t wid = int64_t(blockIdx.x) * warps_per_block + (threadIdx.x >> 5);
    if (wid >= k * ngroups) return;
    const int64_t c = wid / ngroups;
    const int64_t f = (wid % ngroups) * 32 + (threadIdx.x & 31);
    const int lane = threadIdx.x & 31;
    const bool live = f < d;
    const int64_t lo = offsets[c], hi = offsets[c + 1];
    double acc_a = 0.0, acc_b = 0.0;
    constexpr int U = 8;
    for (int64_t base = lo; base < hi; base += 32) {
        const int nb = int(hi - base < 32 ? hi - base : 32);
        const int32_t my_row = lane < nb ? perm[base + lane] : 0;
        int t = 0;
        for (; t + U <= nb; t += U) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int32_t row = __shfl_sync(0xffffffffu, my_row, t + u);
                v[u] = live ? double(x[int64_t(row) * d + f]) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc_a = __dadd_rn(acc_a, v[u]);
                if (DMR) acc_b = __dadd_rn(acc_b, v[u]);
            }
        }
        for (; t < nb; ++t) {
            int32_t row = __shfl_sync(0xffffffffu, my_row, t);
            double v = live ? double(x[int64_t(row) * d + f]) : 0.0;
            acc_a = __dadd_rn(acc_a, v);
            if (DMR) acc_b = __dadd_rn(acc_b, v);
        }
    }
    if (live) {
        sums_a[c * d + f] = acc_a;
        if (DMR) sums_b[c * d + f] = acc_b;
    }
}

// ------------------------------------------------ pipelined ordered chains --
// The reference's chain verbatim (one float64 accumulator per (cluster,
// feature), members in ascending sample order), latency-hidden: each warp
// owns (cluster, 32-feature group) and streams member rows through a shared
// memory ring with cp.async (CH_RING rows in flight, CH_GROUP rows per
// commit group), so the chain runs at DADD latency instead of load latency.
// Used when the chains are long and few (K * D/32 fits one wave): small K or
// float64 data, where certified segment folding rarely applies.
constexpr int CH_RING = 256, CH_GROUP = 32, CH_WARPS = 1;

__device__ __forceinline__ void cp_async_8(void *dst, const void *src, bool pred) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
                 "@p cp.async.ca.shared.global [%0], [%1], 8;\n\t}" ::"r"(s),
                 "l"(src), "r"(int(pred))
                 : "memory");
}
__device__ __forceinline__ void cp_async_4(void *dst, const void *src, bool pred) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
                 "@p cp.async.ca.shared.global [%0], [%1], 4;\n\t}" ::"r"(s),
                 "l"(src), "r"(int(pred))
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <typename T, bool DMR>
__global__ void __launch_bounds__(32 * CH_WARPS) chain_pipe_kernel(
    const T *x, int64_t d, const int32_t *perm, const int64_t *offsets, int64_t k,
    double *sums_a, double *sums_b) {
    extern __shared__ __align__(16) unsigned char ch_smem[];
    T(*ring)[CH_RING][32] = reinterpret_cast<T(*)[CH_RING][32]>(ch_smem);  // [CH_WARPS]
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ngroups = (d + 31) / 32;
    const int64_t wid = int64_t(blockIdx.x) * CH_WARPS + w;
    if (wid >= k * ngroups) return;
    const int64_t c = wid / ngroups;
    const int64_t f = (wid % ngroups) * 32 + lane;
    const bool live = f < d;
    const int64_t lo = offsets[c], hi = offsets[c + 1];
    const int64_t n = hi - lo;
    T(*rb)[32] = ring[w];
    // issue the copies of members [t, t + CH_GROUP) into their ring slots;
    // `rows` holds those members' sample indices (lanes 0..CH_GROUP-1),
    // loaded one group ahead so the shuffles never wait on global memory
    auto load_rows = [&](int64_t t) -> int32_t {
        const int64_t idx = t + lane;
        return (lane < CH_GROUP && idx < n) ? __ldg(perm + lo + idx) : 0;
    };
    const T *xf = x + f;
    auto issue = [&](int64_t t, int32_t rows) {
        // t is a multiple of CH_GROUP, which divides CH_RING: one slot base
        // per group, and no per-member bound test for full groups
        T(*slot)[32] = rb + int(t % CH_RING);
        const bool full = t + CH_GROUP <= n;
#pragma unroll
        for (int u = 0; u < CH_GROUP; ++u) {
            const int32_t row = __shfl_sync(0xffffffffu, rows, u);
            const bool p = full ? live : (live && (t + u < n));
            T *dst = &slot[u][lane];
            if (sizeof(T) == 8) cp_async_8(dst, xf + int64_t(row) * d, p);
            else cp_async_4(dst, xf + int64_t(row) * d, p);
        }
        cp_async_commit();
    };
    constexpr int NG = CH_RING / CH_GROUP;
    // sample indices run three groups ahead of the copies that need them
    int32_t r0 = load_rows(0), r1 = load_rows(CH_GROUP), r2 = load_rows(2 * CH_GROUP);
#pragma unroll
    for (int g = 0; g < NG - 1; ++g) {
        issue(int64_t(g) * CH_GROUP, r0);
        r0 = r1;
        r1 = r2;
        r2 = load_rows(int64_t(g + 3) * CH_GROUP);
    }
    double acc_a = 0.0, acc_b = 0.0;
    for (int64_t t = 0; t < n; t += CH_GROUP) {
        const int64_t ti = t + int64_t(NG - 1) * CH_GROUP;
        issue(ti, r0);  // may be empty: keeps the group count uniform
        r0 = r1;
        r1 = r2;
        r2 = load_rows(ti + 3 * CH_GROUP);
        cp_async_wait<NG - 1>();  // group of rows [t, t + CH_GROUP) landed
        __syncwarp();
        const int cnt = int(n - t < CH_GROUP ? n - t : CH_GROUP);
        const T(*slot)[32] = rb + int(t % CH_RING);
        if (cnt == CH_GROUP) {
            if (live) {  // full group: no per-member tests
                double v[CH_GROUP];
#pragma unroll
                for (int u = 0; u < CH_GROUP; ++u) v[u] = double(slot[u][lane]);
#pragma unroll
                for (int u = 0; u < CH_GROUP; ++u) {
                    acc_a = __dadd_rn(acc_a, v[u]);
                    if (DMR) acc_b = __dadd_rn(acc_b, v[u]);
                }
            }
        } else if (live) {
            for (int u = 0; u < cnt; ++u) {
                const double v = double(slot[u][lane]);
                acc_a = __dadd_rn(acc_a, v);
                if (DMR) acc_b = __dadd_rn(acc_b, v);
            }
        }
        __syncwarp();  // slots of this group are refilled next iteration
    }
    cp_async_wait<0>();
    if (live) {
        sums_a[c * d + f] = acc_a;
        if (DMR) sums_b[c * d + f] = acc_b;
    }
}

// ------------------------------------- warp-specialised ordered chains ----
// The same ordered chains, with the gathers decoupled from the chain.  One
// CTA per (cluster, slab of 32*VEC features = 512 bytes of a row): warp 0 is
// the CONSUMER (each lane folds VEC = 16/sizeof(T) independent float64
// chains, members in ascending sample order, from 16-byte shared reads);
// warps 1..CS_LOADERS are LOADERS that take 16-member groups round-robin and
// gather them into a ring of CS_NG slots with 16-byte cp.async (one
// instruction per member row), signalling each slot's mbarrier through
// cp.async.mbarrier.arrive.  A single warp's outstanding copies cap a
// gather at ~10 GB/s per SM (measured: the 1-warp kernels above, with 8- and
// 16-byte copies alike, run c4's update in 4.3 ms); seven loader warps keep
// ~56 KB per CTA in flight, so the longest cluster's chain -- the kernel's
// critical path -- is no longer fed by one warp.
#ifndef FTK_CS_LOADERS
#define FTK_CS_LOADERS 7
#define FTK_CS_NG 8
#endif
#ifndef FTK_CS_GS
#define FTK_CS_GS 16
#endif
constexpr int CS_GS = FTK_CS_GS, CS_NG = FTK_CS_NG, CS_LOADERS = FTK_CS_LOADERS;
// a loader's next group reuses a slot at most one phase ahead only if there
// are more slots than loaders (parity waits cannot tell phases two apart)
static_assert(CS_LOADERS < CS_NG, "chain ring needs more slots than loader warps");

__device__ __forceinline__ void cs_cp16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cs_bar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(bar))), "r"(count));
}
__device__ __forceinline__ void cs_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(bar)))
                 : "memory");
}
__device__ __forceinline__ void cs_cp_arrive(uint64_t *bar) {  // arrives when this thread's copies land
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(bar)))
                 : "memory");
}
__device__ __forceinline__ void cs_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "CSW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra CSW_%=;\n\t}" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
        "r"(parity)
        : "memory");
}

// SLAB: bytes of a member row per CTA (512, 256 or 128; FTK_CS_SLAB): narrower
// slabs split a cluster's features over more CTAs.
template <typename T, bool DMR, int SLAB>
__global__ void __launch_bounds__(32 * (1 + CS_LOADERS)) chain_spec_kernel(
    const T *x, int64_t d, int64_t nslab, const int32_t *perm, const int64_t *offsets, double *sums_a,
    double *sums_b) {
    constexpr int VEC = 16 / sizeof(T);
    constexpr int LPR = SLAB / 16;        // lanes per row (16 bytes each)
    constexpr int RPI = 32 / LPR;         // rows per copy instruction
    constexpr int W = SLAB / sizeof(T);   // features per slab
    extern __shared__ __align__(128) unsigned char cs_smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(cs_smem);
    uint64_t *empty = full + CS_NG;
    unsigned char *ring = cs_smem + 256;  // [CS_NG][CS_GS][SLAB bytes]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c = int64_t(blockIdx.x) / nslab, s = int64_t(blockIdx.x) % nslab;
    const int64_t f0 = s * W;
    const int fw = int(d - f0 < W ? d - f0 : W);  // a multiple of VEC
    const int64_t lo = offsets[c], n = offsets[c + 1] - lo;
    const int64_t ngrp = (n + CS_GS - 1) / CS_GS;
    if (threadIdx.x == 0) {
        for (int g = 0; g < CS_NG; ++g) {
            cs_bar_init(&full[g], 32);  // the 32 lanes of one loader warp
            cs_bar_init(&empty[g], 1);  // the consumer
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp > 0) {
        // ------------------------------------------------ loaders --
        const int ri = lane / LPR, ch = lane % LPR;  // row within the instruction, 16-byte chunk
        const bool live = ch * VEC < fw;
        const T *xs = x + f0 + ch * VEC;
        const uint32_t rbase = static_cast<uint32_t>(__cvta_generic_to_shared(ring)) + ri * SLAB + ch * 16;
        int64_t g = warp - 1;
        int32_t rows = (g < ngrp && lane < CS_GS && g * CS_GS + lane < n) ? __ldg(perm + lo + g * CS_GS + lane) : 0;
        for (; g < ngrp; g += CS_LOADERS) {
            const int slot = int(g % CS_NG);
            const int64_t gn = g + CS_LOADERS;  // this warp's next group: indices in flight early
            const int32_t next = (gn < ngrp && lane < CS_GS && gn * CS_GS + lane < n)
                                     ? __ldg(perm + lo + gn * CS_GS + lane) : 0;
            cs_wait(&empty[slot], (uint32_t(g / CS_NG) & 1u) ^ 1u);
            const int cnt = int(n - g * CS_GS < CS_GS ? n - g * CS_GS : CS_GS);
            const uint32_t dst = rbase + uint32_t(slot) * (CS_GS * SLAB);
            if (cnt == CS_GS) {
#pragma unroll
                for (int u = 0; u < CS_GS; u += RPI) {
                    const int32_t row = __shfl_sync(0xffffffffu, rows, u + ri);
                    if (live) cs_cp16(dst + u * SLAB, xs + int64_t(row) * d);
                }
            } else {
                for (int u = 0; u < cnt; u += RPI) {
                    const int32_t row = __shfl_sync(0xffffffffu, rows, (u + ri) & 31);
                    if (live && u + ri < cnt) cs_cp16(dst + u * SLAB, xs + int64_t(row) * d);
                }
            }
            cs_cp_arrive(&full[slot]);
            rows = next;
        }
    } else {
        // ----------------------------------------------- consumer --
        double acc_a[VEC], acc_b[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc_a[v] = acc_b[v] = 0.0;
        const bool live = lane < LPR && lane * VEC < fw;
        const T *base = reinterpret_cast<const T *>(ring) + lane * VEC;
        for (int64_t g = 0; g < ngrp; ++g) {
            const int slot = int(g % CS_NG);
            cs_wait(&full[slot], uint32_t(g / CS_NG) & 1u);
            const int cnt = int(n - g * CS_GS < CS_GS ? n - g * CS_GS : CS_GS);
            const T *sl = base + size_t(slot) * CS_GS * W;
            if (live) {
                auto fold = [&](int u) {
                    T v[VEC];
                    *reinterpret_cast<uint4 *>(v) = *reinterpret_cast<const uint4 *>(sl + u * W);
#pragma unroll
                    for (int e = 0; e < VEC; ++e) {
                        acc_a[e] = __dadd_rn(acc_a[e], double(v[e]));
                        if (DMR) acc_b[e] = __dadd_rn(acc_b[e], double(v[e]));
                    }
                };
                if (cnt == CS_GS) {
#pragma unroll
                    for (int u = 0; u < CS_GS; ++u) fold(u);
                } else {
                    for (int u = 0; u < cnt; ++u) fold(u);
                }
            }
            __syncwarp();
            if (lane == 0) cs_arrive(&empty[slot]);
        }
        if (live) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                sums_a[c * d + f0 + lane * VEC + e] = acc_a[e];
                if (DMR) sums_b[c * d + f0 + lane * VEC + e] = acc_b[e];
            }
        }
    }
}

template <typename T, bool DMR>
static int chain_spec_launch(const T *x, int64_t d, int64_t k, const int32_t *perm, const int64_t *offsets,
                             double *sums_a, double *sums_b, cudaStream_t st) {
    // 512-byte slabs: narrower ones (more CTAs per cluster) measured no faster
    // at c4 (2.2 / 2.2 / 2.4 ms for 512 / 256 / 128): the chains are bound by
    // the random-row gather rate (~2.4 TB/s), not by one SM's share
    int slab = 512;
    const int64_t row_bytes = d * int64_t(sizeof(T));
    if (const char *e = getenv("FTK_CS_SLAB")) {
        const int v = atoi(e);
        if (v == 128 || v == 256 || v == 512) slab = v;
    }
    const int64_t nslab = (row_bytes + slab - 1) / slab;
    const size_t smem = 256 + size_t(CS_NG) * CS_GS * slab;
    auto kern = slab == 512 ? chain_spec_kernel<T, DMR, 512>
                            : (slab == 256 ? chain_spec_kernel<T, DMR, 256> : chain_spec_kernel<T, DMR, 128>);
    FTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<unsigned(k * nslab), 32 * (1 + CS_LOADERS), smem, st>>>(x, d, nslab, perm, offsets, sums_a, sums_b);
    FTK_LAUNCHED("chain_spec_kernel");
    return FTK_OK;
}

// ------------------------------------------------ certified segmented sums --
// The reference's float64 chain is order-dependent only if some partial sum
// rounds.  For a (cluster, feature) chain whose values are all multiples of
// 2^q (q = smallest ulp exponent among them), every partial sum of ANY subset
// is a multiple of 2^q bounded by S = sum |v|; if S < 2^(53+q) all of them
// are exact float64 numbers, so any association yields the reference's bits.
// Segments of SEG members are summed in parallel; the combine step checks
// the certificate and queues uncertified chains for the ordered kernel.
constexpr int SEG = 256;
static_assert(SEG == SEG_MEMBERS, "segment length");

template <typename T> __device__ __forceinline__ int ulp_exp(T v);
template <> __device__ __forceinline__ int ulp_exp<float>(float v) {
    const uint32_t e = (__float_as_uint(v) >> 23) & 0xFFu;
    return int(e == 0 ? 1 : e) - 150;
}
template <> __device__ __forceinline__ int ulp_exp<double>(double v) {
    const uint64_t e = (uint64_t(__double_as_longlong(v)) >> 52) & 0x7FFu;
    return int(e == 0 ? 1 : e) - 1075;
}


// Per segment and feature: the float64 partial sum of the segment's members
// (in member order), max |v| and min (|v| bits - 1) -- the smallest nonzero
// magnitude, whose exponent bounds the ulp exponent of every value.  V
// consecutive features per thread (16-byte loads for V = 4); the segment's
// owner comes from the segment table (seg_cl), not a search.
template <int V> struct FVec;
template <> struct FVec<4> { using T = float4; };
template <> struct FVec<2> { using T = float2; };
template <> struct FVec<1> { using T = float; };

template <int V>
__device__ __forceinline__ void fvec_load(const float *p, float (&v)[V]) {
    if constexpr (V == 4) {
        const float4 t = *reinterpret_cast<const float4 *>(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else if constexpr (V == 2) {
        const float2 t = *reinterpret_cast<const float2 *>(p);
        v[0] = t.x; v[1] = t.y;
    } else {
        v[0] = *p;
    }
}

// The certificate of one (cluster, feature) chain from its segment summaries
// (seg_fold_kernel and the fused fold below): values multiples of 2^q and
// sum |v| < 2^(53+q); the bound's own rounding stays far below the margin.
__device__ __forceinline__ bool chain_exact(double bnd, int q) {
    return q == INT_MAX || (q > -1000 && bnd * (1.0 + 0x1p-20) < ldexp(1.0, 53 + q));
}

// FOLD: the block that completes a cluster's last segment (per-cluster
// arrival counter) folds that cluster's chains -- the separate fold pass and
// its launch disappear.  Threads split into nsub = 256/d sub-lanes per feature
// (adjacent lanes, combined by shuffles); any association is exact when the
// certificate holds, failing chains are queued for seg_replay_kernel.
// Surplus blocks (the grid is sized for the largest segment count) write the
// zero sums of empty clusters.
template <bool DMR>
struct SegFold {
    double *sums_a, *sums_b;
    int64_t *fail_list;
    unsigned *fail_count;
    unsigned *done;  // per-cluster arrivals, zeroed by offsets_segs_kernel
};

template <bool DMR, int V, bool FOLD = false>
__global__ void __launch_bounds__(256) seg_partials_kernel(
    const float *x, int64_t d, const int32_t *perm, const int64_t *offsets, const int64_t *seg_base,
    const int32_t *seg_cl, int64_t k, double *ps_a, double *ps_b, double *ps_abs, int32_t *ps_q,
    SegFold<DMR> fo = SegFold<DMR>{}) {
    // The segment partial is only used when the whole chain is certified
    // exact (then any association gives the reference's bits), so the
    // members of a segment are split across `nph` thread phases and the
    // phase partials are combined through shared memory.
    __shared__ int64_t rowoff[SEG];
    __shared__ double red_a[256 * V], red_b[DMR ? 256 * V : 1];
    __shared__ uint32_t red_mx[256 * V], red_mn[256 * V];
    const int64_t s = blockIdx.x;
    if (s >= seg_base[k]) {  // launched for the largest possible segment count
        if (FOLD) {
            const int64_t extra = int64_t(gridDim.x) - seg_base[k];
            for (int64_t c = s - seg_base[k]; c < k; c += extra)
                if (offsets[c + 1] == offsets[c])
                    for (int64_t f = threadIdx.x; f < d; f += blockDim.x) {
                        fo.sums_a[c * d + f] = 0.0;
                        if (DMR) fo.sums_b[c * d + f] = 0.0;
                    }
        }
        return;
    }
    const int64_t c = seg_cl[s];
    const int64_t beg = offsets[c] + (s - seg_base[c]) * SEG;
    const int64_t end = offsets[c + 1];
    const int n = int(end - beg < SEG ? end - beg : SEG);
    for (int t = threadIdx.x; t < n; t += blockDim.x) rowoff[t] = int64_t(perm[beg + t]) * d;
    __syncthreads();
    const int64_t nf = d / V;
    const int nph = nf >= int64_t(blockDim.x) ? 1 : int(blockDim.x / nf);
    const int ph = nph > 1 ? int(threadIdx.x / nf) : 0;
    constexpr int U = V == 4 ? 4 : 8;  // vector loads in flight per thread
    for (int64_t f = nph > 1 ? int64_t(threadIdx.x % nf) : int64_t(threadIdx.x); f < nf;
         f += (nph > 1 ? nf : int64_t(blockDim.x))) {
        double a[V], b[V];
        uint32_t mx[V], mn[V];
#pragma unroll
        for (int h = 0; h < V; ++h) {
            a[h] = 0.0;
            b[h] = 0.0;
            mx[h] = 0;
            mn[h] = 0xFFFFFFFFu;
        }
        if (ph < nph) {
            const float *xb = x + V * f;
            for (int t = ph; t < n; t += U * nph) {
                float v[U][V];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int tt = t + u * nph;
                    if (tt < n) {
                        fvec_load<V>(xb + rowoff[tt], v[u]);
                    } else {
#pragma unroll
                        for (int h = 0; h < V; ++h) v[u][h] = 0.0f;
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
#pragma unroll
                    for (int h = 0; h < V; ++h) {
                        a[h] = __dadd_rn(a[h], double(v[u][h]));
                        if (DMR) b[h] = __dadd_rn(b[h], double(v[u][h]));
                        const uint32_t w = __float_as_uint(v[u][h]) & 0x7FFFFFFFu;
                        mx[h] = max(mx[h], w);
                        mn[h] = min(mn[h], w - 1u);  // zeros wrap to 0xFFFFFFFF: ignored
                    }
                }
            }
        }
        if (nph > 1) {
            // combine the phases of feature group f
            const int slot = ph * int(nf) + int(f);
#pragma unroll
            for (int h = 0; h < V; ++h) {
                red_a[V * slot + h] = a[h];
                if (DMR) red_b[V * slot + h] = b[h];
                red_mx[V * slot + h] = mx[h];
                red_mn[V * slot + h] = mn[h];
            }
            __syncthreads();  // nph > 1: every thread runs exactly one f iteration
            if (ph != 0) continue;
            for (int q = 1; q < nph; ++q) {
                const int sl = q * int(nf) + int(f);
#pragma unroll
                for (int h = 0; h < V; ++h) {
                    a[h] = __dadd_rn(a[h], red_a[V * sl + h]);
                    if (DMR) b[h] = __dadd_rn(b[h], red_b[V * sl + h]);
                    mx[h] = max(mx[h], red_mx[V * sl + h]);
                    mn[h] = min(mn[h], red_mn[V * sl + h]);
                }
            }
        }
        // q = exponent of the ulp of the smallest nonzero magnitude (a lower
        // bound of every value's ulp exponent); bound = n * max|v|
#pragma unroll
        for (int h = 0; h < V; ++h) {
            const int64_t ff = V * f + h;
            int q = INT_MAX;
            if (mn[h] != 0xFFFFFFFFu) {
                const int e = int((mn[h] + 1u) >> 23);
                q = (e == 0 ? 1 : e) - 150;
            }
            ps_a[s * d + ff] = a[h];
            if (DMR) ps_b[s * d + ff] = b[h];
            ps_abs[s * d + ff] = double(n) * double(__uint_as_float(mx[h]));
            ps_q[s * d + ff] = q;
        }
    }
    if (!FOLD) return;
    __shared__ int is_last;
    __threadfence();  // this block's partials are visible before its arrival
    __syncthreads();
    if (threadIdx.x == 0)
        is_last = atomicAdd(fo.done + c, 1u) == unsigned(seg_base[c + 1] - seg_base[c] - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    const int64_t s0 = seg_base[c], s1 = seg_base[c + 1];
    int nsub = 1;
    while (nsub < 32 && int64_t(nsub) * 2 * d <= int64_t(blockDim.x)) nsub *= 2;
    const int sub = int(threadIdx.x) & (nsub - 1);
    const int64_t fstride = int64_t(blockDim.x) / nsub;
    // whole warps iterate together (the shuffles): the trip count follows the
    // warp's first feature
    const int64_t fw = int64_t(threadIdx.x & ~31u) / nsub;
    for (int64_t r = 0; fw + r * fstride < d; ++r) {
        const int64_t f0 = int64_t(threadIdx.x) / nsub + r * fstride;
        const bool live = f0 < d;
        const int64_t f = live ? f0 : 0;
        double a = 0.0, b = 0.0, bnd = 0.0;
        int q = INT_MAX;
        if (live)
            for (int64_t t = s0 + sub; t < s1; t += nsub) {
                a = __dadd_rn(a, __ldcg(ps_a + t * d + f));
                if (DMR) b = __dadd_rn(b, __ldcg(ps_b + t * d + f));
                bnd = __dadd_rn(bnd, __ldcg(ps_abs + t * d + f));
                q = min(q, __ldcg(ps_q + t * d + f));
            }
        for (int off = nsub / 2; off; off >>= 1) {
            a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, off, nsub));
            if (DMR) b = __dadd_rn(b, __shfl_xor_sync(0xffffffffu, b, off, nsub));
            bnd = __dadd_rn(bnd, __shfl_xor_sync(0xffffffffu, bnd, off, nsub));
            q = min(q, __shfl_xor_sync(0xffffffffu, q, off, nsub));
        }
        if (!live || sub != 0) continue;
        const int64_t e = c * d + f;
        if (chain_exact(bnd, q)) {
            fo.sums_a[e] = a;
            if (DMR) fo.sums_b[e] = b;
        } else {
            fo.fail_list[atomicAdd(fo.fail_count, 1u)] = e;
        }
    }
}

// Fold one (cluster, feature) chain.  If every value of the chain is a
// multiple of 2^q and sum |v| < 2^(53+q), every partial sum of the
// reference's sequential chain is an exact float64 number, so the segment
// partials combined in any order give the reference's bits.  Chains that
// fail (values of tiny magnitude next to large sums) are queued for
// seg_replay_kernel, which recomputes them in member order.
template <bool DMR>
__global__ void seg_fold_kernel(const int64_t *seg_base, int64_t k, int64_t d,
                                const double *ps_a, const double *ps_b, const double *ps_abs,
                                const int32_t *ps_q, double *sums_a, double *sums_b,
                                int64_t *fail_list, unsigned *fail_count, int lanes) {
    // `lanes` (a power of two <= 32) threads per chain stride over its
    // segments and combine by shuffles: any association is exact when the
    // certificate holds, and the bound's rounding stays far below its margin
    const int sub = int(threadIdx.x) & (lanes - 1);
    const int64_t groups = (int64_t(gridDim.x) * blockDim.x) / lanes;
    const int64_t mine = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / lanes;
    const int64_t first = (int64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u)) / lanes;
    // the trip count follows the warp's first group, so whole warps shuffle
    for (int64_t r = 0; first + r * groups < k * d; ++r) {
        const int64_t e0 = mine + r * groups;
        const bool live = e0 < k * d;
        const int64_t e = live ? e0 : 0;
        const int64_t c = e / d, f = e % d;
        const int64_t s0 = live ? seg_base[c] : 0, s1 = live ? seg_base[c + 1] : 0;
        double a = 0.0, b = 0.0, bnd = 0.0;
        int q = INT_MAX;
        for (int64_t s = s0 + sub; s < s1; s += lanes) {
            a = __dadd_rn(a, ps_a[s * d + f]);
            if (DMR) b = __dadd_rn(b, ps_b[s * d + f]);
            bnd = __dadd_rn(bnd, ps_abs[s * d + f]);
            q = min(q, ps_q[s * d + f]);
        }
        for (int off = lanes / 2; off; off >>= 1) {
            a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, off, lanes));
            if (DMR) b = __dadd_rn(b, __shfl_xor_sync(0xffffffffu, b, off, lanes));
            bnd = __dadd_rn(bnd, __shfl_xor_sync(0xffffffffu, bnd, off, lanes));
            q = min(q, __shfl_xor_sync(0xffffffffu, q, off, lanes));
        }
        if (!live || sub != 0) continue;
        if (chain_exact(bnd, q)) {
            sums_a[e] = a;
            if (DMR) sums_b[e] = b;
        } else {
            fail_list[atomicAdd(fail_count, 1u)] = e;
        }
    }
}

// Exponent of the lowest set bit of a float64 (s = odd * 2^e), INT_MAX for 0.
__device__ __forceinline__ int lowbit_exp(double s) {
    const uint64_t u = uint64_t(__double_as_longlong(s));
    const uint64_t ef = (u >> 52) & 0x7FFu;
    uint64_t mant = u & 0xFFFFFFFFFFFFFull;
    if (ef == 0 && mant == 0) return INT_MAX;
    if (ef != 0) mant |= (1ull << 52);
    return int(ef == 0 ? 1 : ef) - 1075 + __ffsll((long long)mant) - 1;
}

// One block per failing chain.  The leading segments whose partial sums
// provably join the running sum exactly (per-segment certificate against the
// running sum's lowest set bit) are folded directly.  At the first segment
// that fails, the block gathers a WINDOW of up to RW segments' member values
// into shared memory in one parallel pass (one gather latency instead of one
// per segment) and summarises them in 32-member sub-segments; one thread then
// walks the window: a segment that certifies against the running sum is
// added whole, else each of its sub-segments that certifies, else its members
// one by one -- the reference's sequential float64 chain wherever a partial
// sum can round.
constexpr int RW = 8;  // segments per staged window (8 KB of member values)

__device__ __forceinline__ bool joins_exactly(double a, double part_abs, int qpart) {
    const int qa = lowbit_exp(a);
    const int q = qa < qpart ? qa : qpart;
    return q > -1000 && fabs(a) + part_abs * (1.0 + 0x1p-20) < ldexp(1.0, 53 + q);
}

template <bool DMR>
__global__ void __launch_bounds__(256) seg_replay_kernel(
    const float *x, int64_t d, const int32_t *perm, const int64_t *offsets,
    const int64_t *seg_base, const double *ps_a, const double *ps_b, const double *ps_abs,
    const int32_t *ps_q, const int64_t *fail_list, const unsigned *fail_count, double *sums_a,
    double *sums_b) {
    constexpr int SB = 256;  // summaries staged per round (== blockDim.x)
    constexpr int NSUB = RW * SEG / 32;
    __shared__ __align__(16) float vals[RW * SEG];
    __shared__ double sub_a[NSUB], sub_abs[NSUB];
    __shared__ int sub_q[NSUB];
    __shared__ double sp_a[SB], sp_b[DMR ? SB : 1], sp_abs[SB];
    __shared__ int32_t sp_q[SB];
    __shared__ double run[2];
    __shared__ int next;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned nfail = *fail_count;
    for (unsigned w = blockIdx.x; w < nfail; w += gridDim.x) {
        const int64_t e = fail_list[w];
        const int64_t c = e / d, f = e % d;
        const int64_t s0 = seg_base[c], s1 = seg_base[c + 1];
        const int64_t m0 = offsets[c], m1 = offsets[c + 1];
        if (threadIdx.x == 0) run[0] = run[1] = 0.0;
        for (int64_t sb = s0; sb < s1; sb += SB) {
            const int cnt = int(s1 - sb < SB ? s1 - sb : SB);
            __syncthreads();
            if (int(threadIdx.x) < cnt) {
                const int64_t q = (sb + threadIdx.x) * d + f;
                sp_a[threadIdx.x] = ps_a[q];
                if (DMR) sp_b[threadIdx.x] = ps_b[q];
                sp_abs[threadIdx.x] = ps_abs[q];
                sp_q[threadIdx.x] = ps_q[q];
            }
            __syncthreads();
            int j = 0;
            while (true) {
                if (threadIdx.x == 0) {
                    double a = run[0], b = run[1];
                    for (; j < cnt; ++j) {
                        if (sp_q[j] == INT_MAX) continue;  // all-zero segment
                        if (!joins_exactly(a, sp_abs[j], sp_q[j]) || (DMR && a != b)) break;
                        a = __dadd_rn(a, sp_a[j]);
                        if (DMR) b = __dadd_rn(b, sp_b[j]);
                    }
                    run[0] = a;
                    run[1] = b;
                    next = j;
                }
                __syncthreads();
                j = next;
                if (j >= cnt) break;
                // stage the window's member values (segments j .. j+nw-1)
                const int nw = cnt - j < RW ? cnt - j : RW;
                const int64_t t0 = m0 + (sb + j - s0) * SEG;
                const int64_t tend = m1 - t0 < int64_t(nw) * SEG ? m1 : t0 + int64_t(nw) * SEG;
                const int n = int(tend - t0);
#pragma unroll 4
                for (int t = threadIdx.x; t < n; t += 256) vals[t] = x[int64_t(perm[t0 + t]) * d + f];
                __syncthreads();
                // 32-member sub-segment summaries (warp w: sub-segments w, w+8, ...)
                for (int sj = wid; sj * 32 < n; sj += 8) {
                    const float v = sj * 32 + lane < n ? vals[sj * 32 + lane] : 0.0f;
                    double ps = double(v);
                    uint32_t mx = __float_as_uint(v) & 0x7FFFFFFFu, mn = mx - 1u;
                    for (int off = 16; off; off >>= 1) {
                        ps = __dadd_rn(ps, __shfl_xor_sync(0xffffffffu, ps, off));
                        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
                        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
                    }
                    if (lane == 0) {
                        sub_a[sj] = ps;
                        sub_abs[sj] = 32.0 * double(__uint_as_float(mx));
                        int q = INT_MAX;
                        if (mn != 0xFFFFFFFFu) {
                            const int ex = int((mn + 1u) >> 23);
                            q = (ex == 0 ? 1 : ex) - 150;
                        }
                        sub_q[sj] = q;
                    }
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    double a = run[0], b = run[1];
                    for (int g = 0; g < nw; ++g) {
                        const int jj = j + g;
                        if (sp_q[jj] == INT_MAX) continue;
                        if (joins_exactly(a, sp_abs[jj], sp_q[jj]) && (!DMR || a == b)) {
                            a = __dadd_rn(a, sp_a[jj]);
                            if (DMR) b = __dadd_rn(b, sp_b[jj]);
                            continue;
                        }
                        const int te = min(n, (g + 1) * SEG);
                        for (int sj = g * (SEG / 32); sj * 32 < te; ++sj) {
                            if (sub_q[sj] == INT_MAX) continue;  // all-zero sub-segment
                            if (joins_exactly(a, sub_abs[sj], sub_q[sj]) && (!DMR || a == b)) {
                                a = __dadd_rn(a, sub_a[sj]);
                                if (DMR) b = __dadd_rn(b, sub_a[sj]);
                                continue;
                            }
                            const int ue = min(te, sj * 32 + 32);
                            if (ue == sj * 32 + 32) {
                                // a whole sub-segment: its 32 values loaded up
                                // front (8 x LDS.128), then the dependent chain
                                const float4 *v4 = reinterpret_cast<const float4 *>(vals + sj * 32);
                                float4 r[8];
#pragma unroll
                                for (int u = 0; u < 8; ++u) r[u] = v4[u];
#pragma unroll
                                for (int u = 0; u < 8; ++u) {
                                    const float vv[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
                                    for (int h = 0; h < 4; ++h) {
                                        a = __dadd_rn(a, double(vv[h]));
                                        if (DMR) b = __dadd_rn(b, double(vv[h]));
                                    }
                                }
                                continue;
                            }
                            for (int t = sj * 32; t < ue; ++t) {
                                a = __dadd_rn(a, double(vals[t]));
                                if (DMR) b = __dadd_rn(b, double(vals[t]));
                            }
                        }
                    }
                    run[0] = a;
                    run[1] = b;
                    next = j + nw;
                }
                __syncthreads();
                j = next;
            }
        }
        if (threadIdx.x == 0) {
            sums_a[e] = run[0];
            if (DMR) sums_b[e] = run[1];
        }
        __syncthreads();
    }
}

__global__ void u64_to_i64_kernel(const unsigned long long *a, int64_t *b, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        b[i] = int64_t(a[i]);
}

// ----------------------------------------------------------- finalize --
template <typename T>
__global__ void finalize_kernel(const double *sums, const int64_t *counts, int64_t k, int64_t d,
                                T *cent, int32_t *n_empty) {
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < k * d;
         e += int64_t(gridDim.x) * blockDim.x) {
        int64_t c = e / d;
        int64_t n = counts[c];
        double v = n > 0 ? __ddiv_rn(sums[e], double(n)) : 0.0;
        cent[e] = T(v);
        if (n <= 0 && e % d == 0 && n_empty) atomicAdd(n_empty, 1);
    }
}

__global__ void dmr_compare_kernel(const unsigned long long *a, const unsigned long long *b,
                                   int64_t n, int32_t *flag) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        if (a[i] != b[i]) atomicExch(flag, 1);
}

// ------------------------------------------------------ reseed empties --
// argmax with numpy semantics (first maximum; NaN counts as the maximum).
struct ArgMax {
    double v;
    int64_t i;
};
__device__ __forceinline__ bool am_better(double v, int64_t i, double bv, int64_t bi) {
    bool vn = isnan(v), bn = isnan(bv);
    if (vn != bn) return vn;  // NaN wins over non-NaN
    if (vn && bn) return i < bi;
    return v > bv || (v == bv && i < bi);
}

__global__ void argmax_partial_kernel(const double *a, int64_t n, ArgMax *part) {
    double bv = -INFINITY;
    int64_t bi = INT64_MAX;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        if (am_better(a[i], i, bv, bi)) { bv = a[i]; bi = i; }
    }
    for (int off = 16; off; off >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, bv, off);
        int64_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (am_better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
    }
    __shared__ ArgMax sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = {bv, bi};
    __syncthreads();
    if (threadIdx.x == 0) {
        ArgMax r = sh[0];
        for (int w = 1; w < int(blockDim.x / 32); ++w)
            if (am_better(sh[w].v, sh[w].i, r.v, r.i)) r = sh[w];
        part[blockIdx.x] = r;
    }
}

template <typename T>
__global__ void reseed_apply_kernel(const ArgMax *part, int nparts, const T *x, int64_t d,
                                    int64_t j, double *sq, T *cent) {
    __shared__ int64_t far;
    if (threadIdx.x == 0) {
        ArgMax r = part[0];
        for (int p = 1; p < nparts; ++p)
            if (am_better(part[p].v, part[p].i, r.v, r.i)) r = part[p];
        far = r.i == INT64_MAX ? 0 : r.i;
    }
    __syncthreads();
    for (int64_t f = threadIdx.x; f < d; f += blockDim.x) cent[j * d + f] = x[far * d + f];
    __syncthreads();
    if (threadIdx.x == 0) sq[far] = -INFINITY;
}

// ------------------------------------------------------------ inertia --
template <typename T>
__global__ void sq_dists_kernel(const T *md, const double *xsq, int64_t m, double *sq) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x)
        sq[i] = __dadd_rn(double(md[i]), xsq[i]);
}

// numpy pairwise_sum leaf (n <= 128): 8 strided accumulators.
__device__ double pairwise_leaf(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

// Full recursion with an explicit stack (per-thread; used for rows of <= a
// few thousand elements).  Post-order evaluation keeps numpy's association.
__device__ double pairwise_sum_dev(const double *a, int64_t n) {
    if (n <= 128) return pairwise_leaf(a, n);
    struct Fr { int64_t off, n; int state; double left; };
    Fr st[48];
    int sp = 0;
    st[0] = {0, n, 0, 0.0};
    double ret = 0.0;
    while (sp >= 0) {
        Fr &f = st[sp];
        if (f.n <= 128) {
            ret = pairwise_leaf(a + f.off, f.n);
            --sp;
            continue;
        }
        int64_t n2 = f.n / 2;
        n2 -= n2 % 8;
        if (f.state == 0) {
            f.state = 1;
            st[sp + 1] = {f.off, n2, 0, 0.0};
            ++sp;
        } else if (f.state == 1) {
            f.left = ret;
            f.state = 2;
            st[sp + 1] = {f.off + n2, f.n - n2, 0, 0.0};
            ++sp;
        } else {
            ret = __dadd_rn(f.left, ret);
            --sp;
        }
    }
    return ret;
}

// Leaf sums: 8 lanes per leaf (one per accumulator), 4 leaves per warp.
__global__ void pairwise_leaves_kernel(const double *a, const int64_t *leaf_start, int64_t nleaves,
                                       double *vals) {
    const int64_t gl = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 8;
    const int j = threadIdx.x & 7;
    const bool live = gl < nleaves;
    int64_t off = 0, n = 0;
    if (live) {
        off = leaf_start[gl];
        n = leaf_start[gl + 1] - off;
    }
    const double *p = a + off;
    double r = 0.0;
    const bool small = n < 8;
    int64_t lim = n - (n % 8);
    if (live && !small) {
        r = p[j];
        for (int64_t i = 8; i < lim; i += 8) r = __dadd_rn(r, p[i + j]);
    }
    // ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)) within the 8-lane group
    const unsigned mask = 0xffffffffu;
    double o1 = __shfl_xor_sync(mask, r, 1);
    double s1 = (j & 1) ? __dadd_rn(o1, r) : __dadd_rn(r, o1);  // pair sums (even lane has r_even+r_odd)
    double o2 = __shfl_xor_sync(mask, s1, 2);
    double s2 = (j & 2) ? __dadd_rn(o2, s1) : __dadd_rn(s1, o2);
    double o4 = __shfl_xor_sync(mask, s2, 4);
    double s4 = (j & 4) ? __dadd_rn(o4, s2) : __dadd_rn(s2, o4);
    if (live && j == 0) {
        double res;
        if (small) {
            res = 0.0;
            for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, p[i]);
        } else {
            res = s4;
            for (int64_t i = lim; i < n; ++i) res = __dadd_rn(res, p[i]);
        }
        vals[gl] = res;
    }
}

// Internal nodes, level by level (height order), single block.
// SM: the whole tree (leaf values, node values, child lists) is staged in
// shared memory, so each of the ~log2(n/128) levels costs a shared-memory
// round trip instead of an L2 one (c2: 15 -> ~3 us).
template <bool SM>
__global__ void pairwise_tree_kernel(double *vals, const int2 *nodes, const int64_t *level_start,
                                     int nlevels, int64_t nleaves, double *out) {
    extern __shared__ __align__(16) unsigned char pt_smem[];
    const int64_t nnodes = level_start[nlevels];
    double *v = vals;
    const int2 *nd = nodes;
    if (SM) {
        double *sv = reinterpret_cast<double *>(pt_smem);
        int2 *sn = reinterpret_cast<int2 *>(sv + nleaves + nnodes);
        for (int64_t i = threadIdx.x; i < nleaves; i += blockDim.x) sv[i] = vals[i];
        for (int64_t i = threadIdx.x; i < nnodes; i += blockDim.x) sn[i] = nodes[i];
        __syncthreads();
        v = sv;
        nd = sn;
    }
    for (int L = 0; L < nlevels; ++L) {
        for (int64_t q = level_start[L] + threadIdx.x; q < level_start[L + 1]; q += blockDim.x) {
            int2 ch = nd[q];
            v[nleaves + q] = __dadd_rn(v[ch.x], v[ch.y]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = nnodes > 0 ? v[nleaves + nnodes - 1] : v[0];
}

// ---------------------------------------------------------- movement --
template <typename T>
__global__ void movement_kernel(const T *nc, const T *oc, int64_t k, int64_t d, double eps,
                                double *tmp, unsigned long long *moved_bits) {
    int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= k) return;
    double *a = tmp + j * 2 * d;
    double *b = a + d;
    for (int64_t f = 0; f < d; ++f) {
        double o = double(oc[j * d + f]);
        double diff = __dsub_rn(double(nc[j * d + f]), o);
        a[f] = __dmul_rn(diff, diff);
        b[f] = __dmul_rn(o, o);
    }
    double num = sqrt(pairwise_sum_dev(a, d));
    double den = __dadd_rn(sqrt(pairwise_sum_dev(b, d)), eps);
    double r = __ddiv_rn(num, den);
    unsigned long long bits = isnan(r) ? 0x7ff8000000000000ull : __double_as_longlong(r);
    atomicMax(moved_bits, bits);  // non-negative doubles order like their bits
}

// Warp per centroid (d <= 128: numpy's pairwise reduce is a single leaf):
// lanes 0-7 hold the 8 strided accumulators of ||new - old||^2, lanes 8-15
// those of ||old||^2; the leaf's fixed combine tree and tail follow.
template <typename T>
__global__ void movement_warp_kernel(const T *nc, const T *oc, int64_t k, int64_t d, double eps,
                                     unsigned long long *moved_bits) {
    const int lane = threadIdx.x & 31;
    const int64_t j = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (j >= k) return;
    const T *nr = nc + j * d, *orow = oc + j * d;
    const int which = lane >> 3, jj = lane & 7;  // which: 0 num, 1 den
    double r = 0.0;
    const int64_t lim = d - (d % 8);
    if (which < 2 && d >= 8) {
        for (int64_t i = jj; i < lim; i += 8) {
            const double o = double(orow[i]);
            const double v = which == 0 ? __dsub_rn(double(nr[i]), o) : o;
            const double sq = __dmul_rn(v, v);
            r = i == jj ? sq : __dadd_rn(r, sq);
        }
    }
    // ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)) within each 8-lane group
    const double s1 = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    const double s2 = __dadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, 2));
    const double s4 = __dadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, 4));
    double tot[2];
    tot[0] = __shfl_sync(0xffffffffu, s4, 0);
    tot[1] = __shfl_sync(0xffffffffu, s4, 8);
    if (lane == 0) {
        for (int w = 0; w < 2; ++w) {
            double res = d >= 8 ? tot[w] : 0.0;
            for (int64_t i = d >= 8 ? lim : 0; i < d; ++i) {
                const double o = double(orow[i]);
                const double v = w == 0 ? __dsub_rn(double(nr[i]), o) : o;
                res = __dadd_rn(res, __dmul_rn(v, v));
            }
            tot[w] = res;
        }
        const double num = sqrt(tot[0]);
        const double den = __dadd_rn(sqrt(tot[1]), eps);
        const double q = __ddiv_rn(num, den);
        const unsigned long long bits = isnan(q) ? 0x7ff8000000000000ull : __double_as_longlong(q);
        atomicMax(moved_bits, bits);  // non-negative doubles order like their bits
    }
}

// sq[i] = pairwise_sum_f((x[i,f] - cent64[label[i], f])^2)  (kmeans.py:199-201)
template <typename T>
__global__ void own_sq_dists_kernel(const T *x, const int32_t *lab, const double *c64, int64_t m,
                                    int64_t d, double *tmp, double *out) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    double *a = tmp + tid * d;
    for (int64_t i = tid; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        const double *c = c64 + int64_t(lab[i]) * d;
        for (int64_t f = 0; f < d; ++f) {
            double diff = __dsub_rn(double(x[i * d + f]), c[f]);
            a[f] = __dmul_rn(diff, diff);
        }
        out[i] = pairwise_sum_dev(a, d);
    }
}

__global__ void labels_equal_kernel(const int32_t *a, const int32_t *b, int64_t m, int32_t *flag) {
    // vectorised compare, one warp vote per 4 x 32 labels, one store per
    // differing warp (no contended atomics)
    bool diff = false;
    const int64_t m4 = m / 4;
    const int4 *a4 = reinterpret_cast<const int4 *>(a), *b4 = reinterpret_cast<const int4 *>(b);
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m4;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int4 u = a4[i], v = b4[i];
        diff |= (u.x != v.x) | (u.y != v.y) | (u.z != v.z) | (u.w != v.w);
    }
    for (int64_t i = m4 * 4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x)
        diff |= a[i] != b[i];
    if (__any_sync(0xffffffffu, diff) && (threadIdx.x & 31) == 0) *flag = 0;
}

__global__ void flip_f64_kernel(double *a, int64_t idx, int64_t bit, double *ba) {
    double before = a[idx];
    double after = flip_bit(before, bit);
    a[idx] = after;
    if (ba) { ba[0] = before; ba[1] = after; }
}

__global__ void set_i32_kernel(int32_t *p, int32_t v) { *p = v; }

// =================================================================== host ==
static unsigned grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    return unsigned(g);
}

int update_sums_run(ftk_ctx *ctx, int dtype, const void *x, const int32_t *labels, int64_t m,
                    int64_t d, int64_t k, double *sums_a, int64_t *counts_a, double *sums_b,
                    int64_t *counts_b, cudaStream_t st) {
    if (k <= 0) return FTK_OK;
    // counts: from the segment boundaries of the sorted labels (below); the
    // DMR duplicate (counts_b) comes from an independent histogram
    FTK_CUDA(cudaMemsetAsync(counts_a, 0, sizeof(int64_t) * k, st));
    if (m > 0 && counts_b) {
        FTK_CUDA(cudaMemsetAsync(counts_b, 0, sizeof(int64_t) * k, st));
        if (k <= 12 * 1024) {
            histogram_kernel<<<grid_for(m, 512), 512, sizeof(unsigned) * k, st>>>(
                labels, m, k, reinterpret_cast<unsigned long long *>(counts_b));
        } else {
            histogram_global_kernel<<<grid_for(m, 512), 512, 0, st>>>(
                labels, m, reinterpret_cast<unsigned long long *>(counts_b));
        }
        FTK_LAUNCHED("histogram_kernel");
    }
    // update path (decided up front: the member-offset scan also builds the
    // segment table of the certified segmented sums)
    const bool dmr = sums_b != nullptr;
    const int64_t nwarps = k * ((d + 31) / 32);
    // float64 data: every partial sum rounds (full 53-bit values), so the
    // reference's ordered chain runs as is; float32: certified segments,
    // whatever the chain count (measured faster at c1, c3 and c2)
    bool pipe_chains = m > 0 && dtype == FTK_F64;
    if (const char *e = getenv("FTK_UPD_PATH"))  // A/B knob: "seg" or "pipe" (float32 data)
        if (dtype == FTK_F32 && m > 0) pipe_chains = e[0] == 'p';
    const bool use_seg = dtype == FTK_F32 && m > 0 && !pipe_chains;
    const int64_t max_seg = (m + SEG - 1) / SEG + k;
    int64_t *seg_base = nullptr;
    int32_t *seg_cl = nullptr;
    int64_t *fail_list = nullptr;
    unsigned *fail_count = nullptr;
    if (use_seg) {
        seg_base = static_cast<int64_t *>(scratch(ctx, SLOT_SEG_BASE, sizeof(int64_t) * (k + 2) +
                                                                          sizeof(int32_t) * max_seg, st));
        fail_list = static_cast<int64_t *>(scratch(ctx, SLOT_SEG_FB, sizeof(int64_t) * (k * d + 2) +
                                                                        sizeof(unsigned) * (k + 2), st));
        if (!seg_base || !fail_list) return FTK_ERR_CUDA;
        seg_cl = reinterpret_cast<int32_t *>(seg_base + (k + 2));
        fail_count = reinterpret_cast<unsigned *>(fail_list + k * d);
    }
    // fused fold (seg_partials_kernel<FOLD>: the last segment block of a
    // cluster folds its chains, no separate fold pass) -- an A/B knob, off by default: measured slower at c2 (partials 93 -> 124 us
    // against the 15 us fold pass it removes, profiles/r6_ab_experiments.txt)
    bool fused_fold = false;
    if (const char *e = getenv("FTK_UPD_FUSED_FOLD")) fused_fold = use_seg && atoi(e) != 0;
    unsigned *done = fused_fold ? reinterpret_cast<unsigned *>(fail_list + k * d + 2) : nullptr;
    // stable sort of (label, index) -> member lists in ascending sample order
    int bits = 1;
    while ((int64_t(1) << bits) < k) ++bits;
    int32_t *keys_out = static_cast<int32_t *>(scratch(ctx, SLOT_SORT_KEYS, sizeof(int32_t) * (m + 1) * 2, st));
    int32_t *vals = static_cast<int32_t *>(scratch(ctx, SLOT_SORT_VALS, sizeof(int32_t) * (m + 1) * 2, st));
    int64_t *offsets = static_cast<int64_t *>(scratch(ctx, SLOT_OFFSETS, sizeof(int64_t) * (k + 1), st));
    if (!keys_out || !vals || !offsets) return FTK_ERR_CUDA;
    int32_t *vals_in = vals, *vals_out = vals + (m + 1);
    if (m > 0 && k <= CS_MAX_K && m < (int64_t(1) << 31)) {
        const int64_t chunk = std::max<int64_t>(2048, (m + 2047) / 2048);
        const int64_t nb = (m + chunk - 1) / chunk;
        int32_t *hist = keys_out;  // k x nb counters (<= 4 * 2048 * CS_MAX_K bytes)
        if (k * nb > 2 * (m + 1)) {
            hist = static_cast<int32_t *>(scratch(ctx, SLOT_SORT_TMP, sizeof(int32_t) * k * nb, st));
            if (!hist) return FTK_ERR_CUDA;
        }
        const int nw = cs_warps(k);
        cs_hist_kernel<<<unsigned(nb), 256, sizeof(int32_t) * k, st>>>(labels, m, k, chunk, hist, nb);
        FTK_LAUNCHED("cs_hist_kernel");
        cs_binscan_kernel<<<unsigned((k * 32 + 255) / 256), 256, 0, st>>>(hist, nb, k, counts_a);
        FTK_LAUNCHED("cs_binscan_kernel");
        offsets_segs_kernel<<<1, 1024, 0, st>>>(counts_a, k, offsets, seg_base, seg_cl, fail_count, done);
        FTK_LAUNCHED("offsets_segs_kernel");
        const size_t smw = sizeof(int32_t) * size_t(nw) * k;
        if (smw > 48 * 1024)
            FTK_CUDA(cudaFuncSetAttribute(cs_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(smw)));
        cs_scatter_kernel<<<unsigned(nb), 32 * nw, smw, st>>>(labels, m, k, chunk, hist, nb, offsets,
                                                            vals_out);
        FTK_LAUNCHED("cs_scatter_kernel");
    } else if (m > 0) {
        iota_kernel<<<grid_for(m, 256), 256, 0, st>>>(vals_in, m);
        FTK_LAUNCHED("iota_kernel");
        size_t tmp_bytes = 0;
        FTK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, labels, keys_out, vals_in,
                                                 vals_out, int(m), 0, bits, st));
        void *tmp = scratch(ctx, SLOT_SORT_TMP, tmp_bytes, st);
        if (!tmp) return FTK_ERR_CUDA;
        FTK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, labels, keys_out, vals_in,
                                                 vals_out, int(m), 0, bits, st));
        count_launch((bits + 7) / 8 * 3);
        boundary_count_kernel<<<grid_for(m, 256), 256, 0, st>>>(
            keys_out, m, k, reinterpret_cast<unsigned long long *>(counts_a));
        FTK_LAUNCHED("boundary_count_kernel");
        offsets_segs_kernel<<<1, 1024, 0, st>>>(counts_a, k, offsets, seg_base, seg_cl, fail_count, done);
        FTK_LAUNCHED("offsets_segs_kernel");
    } else {
        offsets_segs_kernel<<<1, 1024, 0, st>>>(counts_a, k, offsets, seg_base, seg_cl, fail_count, done);
        FTK_LAUNCHED("offsets_segs_kernel");
    }
    const int64_t warps = k * ((d + 31) / 32);
    const int block = 256;
    const unsigned grid = unsigned((warps * 32 + block - 1) / block);
    const int vec = dtype == FTK_F32 ? 4 : 2;
    if (pipe_chains && d % vec == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
        !(getenv("FTK_UPD_CHAIN") && atoi(getenv("FTK_UPD_CHAIN")) == 0)) {
        // ordered chains: warp-specialised gathers of row slabs
        if (dtype == FTK_F32)
            return dmr ? chain_spec_launch<float, true>(static_cast<const float *>(x), d, k, vals_out, offsets,
                                                        sums_a, sums_b, st)
                       : chain_spec_launch<float, false>(static_cast<const float *>(x), d, k, vals_out, offsets,
                                                         sums_a, nullptr, st);
        return dmr ? chain_spec_launch<double, true>(static_cast<const double *>(x), d, k, vals_out, offsets,
                                                     sums_a, sums_b, st)
                   : chain_spec_launch<double, false>(static_cast<const double *>(x), d, k, vals_out, offsets,
                                                      sums_a, nullptr, st);
    }
    if (pipe_chains) {
        // few long chains: the reference's ordered chain, latency-hidden
        const unsigned g = unsigned((nwarps + CH_WARPS - 1) / CH_WARPS);
        const size_t sm = size_t(CH_WARPS) * CH_RING * 32 * (dtype == FTK_F32 ? 4 : 8);
        if (dtype == FTK_F32) {
            auto xx = static_cast<const float *>(x);
            auto kern = dmr ? chain_pipe_kernel<float, true> : chain_pipe_kernel<float, false>;
            FTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
            kern<<<g, 32 * CH_WARPS, sm, st>>>(xx, d, vals_out, offsets, k, sums_a, dmr ? sums_b : nullptr);
        } else {
            auto xx = static_cast<const double *>(x);
            auto kern = dmr ? chain_pipe_kernel<double, true> : chain_pipe_kernel<double, false>;
            FTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
            kern<<<g, 32 * CH_WARPS, sm, st>>>(xx, d, vals_out, offsets, k, sums_a, dmr ? sums_b : nullptr);
        }
        FTK_LAUNCHED("chain_pipe_kernel");
        return FTK_OK;
    }
    if (use_seg) {
        // certified segmented sums (float32 data): segments fold exactly
        // unless their certificate fails, in which case only that segment is
        // re-walked in member order
        size_t pbytes = size_t(max_seg) * d * (3 * sizeof(double) + sizeof(int32_t)) + 64;
        char *pbuf = static_cast<char *>(scratch(ctx, SLOT_SEG_PART, pbytes, st));
        if (!pbuf) return FTK_ERR_CUDA;
        double *ps_a = reinterpret_cast<double *>(pbuf);
        double *ps_b = ps_a + max_seg * d;
        double *ps_abs = ps_b + max_seg * d;
        int32_t *ps_q = reinterpret_cast<int32_t *>(ps_abs + max_seg * d);
        auto xx = static_cast<const float *>(x);
        // replay: one block per failing chain (the count is on the device, so
        // size for many); fold: enough lanes per chain to cover its segments
        const unsigned rgrid = unsigned(std::min<int64_t>(k * d, 148 * 32));
        int lanes = 1;
        while (lanes < 32 && int64_t(lanes) * k < max_seg) lanes *= 2;
        const unsigned fgrid = grid_for(k * d * lanes, 128);
        if (dmr) {
            const SegFold<true> fo{sums_a, sums_b, fail_list, fail_count, done};
            if (fused_fold) {
                auto kp = d % 4 == 0 ? seg_partials_kernel<true, 4, true>
                          : (d % 2 == 0 ? seg_partials_kernel<true, 2, true> : seg_partials_kernel<true, 1, true>);
                kp<<<unsigned(max_seg), 256, 0, st>>>(xx, d, vals_out, offsets, seg_base, seg_cl, k, ps_a,
                                                      ps_b, ps_abs, ps_q, fo);
                FTK_LAUNCHED("seg_partials_kernel");
            } else {
                auto kp = d % 4 == 0 ? seg_partials_kernel<true, 4>
                          : (d % 2 == 0 ? seg_partials_kernel<true, 2> : seg_partials_kernel<true, 1>);
                kp<<<unsigned(max_seg), 256, 0, st>>>(xx, d, vals_out, offsets, seg_base, seg_cl, k, ps_a,
                                                      ps_b, ps_abs, ps_q, fo);
                FTK_LAUNCHED("seg_partials_kernel");
                seg_fold_kernel<true><<<fgrid, 128, 0, st>>>(
                    seg_base, k, d, ps_a, ps_b, ps_abs, ps_q, sums_a, sums_b, fail_list, fail_count, lanes);
                FTK_LAUNCHED("seg_fold_kernel");
            }
            seg_replay_kernel<true><<<rgrid, 256, 0, st>>>(xx, d, vals_out, offsets, seg_base, ps_a,
                                                          ps_b, ps_abs, ps_q, fail_list, fail_count,
                                                          sums_a, sums_b);
        } else {
            const SegFold<false> fo{sums_a, nullptr, fail_list, fail_count, done};
            if (fused_fold) {
                auto kp = d % 4 == 0 ? seg_partials_kernel<false, 4, true>
                          : (d % 2 == 0 ? seg_partials_kernel<false, 2, true> : seg_partials_kernel<false, 1, true>);
                kp<<<unsigned(max_seg), 256, 0, st>>>(xx, d, vals_out, offsets, seg_base, seg_cl, k, ps_a,
                                                      nullptr, ps_abs, ps_q, fo);
                FTK_LAUNCHED("seg_partials_kernel");
            } else {
                auto kp = d % 4 == 0 ? seg_partials_kernel<false, 4>
                          : (d % 2 == 0 ? seg_partials_kernel<false, 2> : seg_partials_kernel<false, 1>);
                kp<<<unsigned(max_seg), 256, 0, st>>>(xx, d, vals_out, offsets, seg_base, seg_cl, k, ps_a,
                                                      nullptr, ps_abs, ps_q, fo);
                FTK_LAUNCHED("seg_partials_kernel");
                seg_fold_kernel<false><<<fgrid, 128, 0, st>>>(
                    seg_base, k, d, ps_a, nullptr, ps_abs, ps_q, sums_a, nullptr, fail_list, fail_count, lanes);
                FTK_LAUNCHED("seg_fold_kernel");
            }
            seg_replay_kernel<false><<<rgrid, 256, 0, st>>>(xx, d, vals_out, offsets, seg_base, ps_a,
                                                           nullptr, ps_abs, ps_q, fail_list,
                                                           fail_count, sums_a, nullptr);
        }
        FTK_LAUNCHED("seg_replay_kernel");
        if (getenv("FTK_UPD_DEBUG")) {  // diagnostics: chains the certificate sent to the replay
            unsigned nf = 0;
            cudaMemcpyAsync(&nf, fail_count, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            fprintf(stderr, "update: %u of %lld chains replayed in order\n", nf, (long long)(k * d));
        }
        return FTK_OK;
    }
    if (dtype == FTK_F32) {
        auto xx = static_cast<const float *>(x);
        if (dmr) chain_sums_kernel<float, true><<<grid, block, 0, st>>>(xx, d, vals_out, offsets, k, sums_a, sums_b);
        else chain_sums_kernel<float, false><<<grid, block, 0, st>>>(xx, d, vals_out, offsets, k, sums_a, nullptr);
    } else {
        auto xx = static_cast<const double *>(x);
        if (dmr) chain_sums_kernel<double, true><<<grid, block, 0, st>>>(xx, d, vals_out, offsets, k, sums_a, sums_b);
        else chain_sums_kernel<double, false><<<grid, block, 0, st>>>(xx, d, vals_out, offsets, k, sums_a, nullptr);
    }
    FTK_LAUNCHED("chain_sums_kernel");
    return FTK_OK;
}

int dmr_compare_run(const double *sa, const int64_t *ca, const double *sb, const int64_t *cb,
                    int64_t k, int64_t d, int32_t *flag, cudaStream_t st) {
    set_i32_kernel<<<1, 1, 0, st>>>(flag, 0);
    FTK_LAUNCHED("set_i32_kernel");
    dmr_compare_kernel<<<grid_for(k * d, 256), 256, 0, st>>>(
        reinterpret_cast<const unsigned long long *>(sa),
        reinterpret_cast<const unsigned long long *>(sb), k * d, flag);
    FTK_LAUNCHED("dmr_compare_kernel");
    dmr_compare_kernel<<<grid_for(k, 256), 256, 0, st>>>(
        reinterpret_cast<const unsigned long long *>(ca),
        reinterpret_cast<const unsigned long long *>(cb), k, flag);
    FTK_LAUNCHED("dmr_compare_kernel");
    return FTK_OK;
}

int finalize_run(int dtype, const double *sums, const int64_t *counts, int64_t k, int64_t d,
                 void *cent, int32_t *n_empty, cudaStream_t st) {
    if (n_empty) {
        set_i32_kernel<<<1, 1, 0, st>>>(n_empty, 0);
        FTK_LAUNCHED("set_i32_kernel");
    }
    if (dtype == FTK_F32)
        finalize_kernel<float><<<grid_for(k * d, 256), 256, 0, st>>>(sums, counts, k, d, static_cast<float *>(cent), n_empty);
    else
        finalize_kernel<double><<<grid_for(k * d, 256), 256, 0, st>>>(sums, counts, k, d, static_cast<double *>(cent), n_empty);
    FTK_LAUNCHED("finalize_kernel");
    return FTK_OK;
}

int reseed_run(ftk_ctx *ctx, int dtype, const void *x, int64_t m, int64_t d,
               const int64_t *counts, int64_t k, double *sq, void *cent, cudaStream_t st) {
    std::vector<int64_t> hc(k);
    FTK_CUDA(cudaMemcpyAsync(hc.data(), counts, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, st));
    FTK_CUDA(cudaStreamSynchronize(st));
    const int nparts = 256;
    ArgMax *part = static_cast<ArgMax *>(scratch(ctx, SLOT_MISC, sizeof(ArgMax) * nparts, st));
    if (!part) return FTK_ERR_CUDA;
    for (int64_t j = 0; j < k; ++j) {
        if (hc[j] > 0) continue;
        argmax_partial_kernel<<<nparts, 256, 0, st>>>(sq, m, part);
        FTK_LAUNCHED("argmax_partial_kernel");
        if (dtype == FTK_F32)
            reseed_apply_kernel<float><<<1, 256, 0, st>>>(part, nparts, static_cast<const float *>(x), d, j, sq, static_cast<float *>(cent));
        else
            reseed_apply_kernel<double><<<1, 256, 0, st>>>(part, nparts, static_cast<const double *>(x), d, j, sq, static_cast<double *>(cent));
        FTK_LAUNCHED("reseed_apply_kernel");
    }
    return FTK_OK;
}

int sq_dists_run(int dtype, const void *md, const double *xsq, int64_t m, double *sq,
                 cudaStream_t st) {
    if (m <= 0) return FTK_OK;
    if (dtype == FTK_F32)
        sq_dists_kernel<float><<<grid_for(m, 256), 256, 0, st>>>(static_cast<const float *>(md), xsq, m, sq);
    else
        sq_dists_kernel<double><<<grid_for(m, 256), 256, 0, st>>>(static_cast<const double *>(md), xsq, m, sq);
    FTK_LAUNCHED("sq_dists_kernel");
    return FTK_OK;
}

// Host-built numpy pairwise tree for length n (cached per context+n).
struct PairwiseTree {
    int64_t n = -1, nleaves = 0, nnodes = 0;
    int nlevels = 0;
    int64_t *d_leaf_start = nullptr;
    int2 *d_nodes = nullptr;
    int64_t *d_level_start = nullptr;
};

static std::mutex g_tree_mu;
static std::map<std::pair<ftk_ctx *, int64_t>, PairwiseTree> g_trees;

static int build_tree(int64_t n, std::vector<int64_t> &leaf_start, std::vector<int2> &nodes,
                      std::vector<int64_t> &level_start) {
    // returns the number of levels; node ids: leaves 0..L-1, internal L+q
    struct Item { int64_t off, n; };
    std::vector<int64_t> starts;
    std::vector<std::pair<int, int>> height_node;  // (height, q) for sorting
    std::vector<int2> raw;
    std::vector<int> heights;
    // recursive lambda returning (id, height)
    std::function<std::pair<int, int>(int64_t, int64_t)> rec = [&](int64_t off, int64_t len) -> std::pair<int, int> {
        if (len <= 128) {
            starts.push_back(off);
            return {int(starts.size() - 1), 0};
        }
        int64_t n2 = len / 2;
        n2 -= n2 % 8;
        auto L = rec(off, n2);
        auto R = rec(off + n2, len - n2);
        raw.push_back(int2{L.first, R.first});  // ids fixed up below (leaf vs internal)
        int h = 1 + (L.second > R.second ? L.second : R.second);
        heights.push_back(h);
        return {-int(raw.size()), h};  // negative: internal node index (1-based)
    };
    auto root = rec(0, n);
    (void)root;
    int64_t L = int64_t(starts.size());
    leaf_start = starts;
    leaf_start.push_back(n);
    // convert ids: leaf id stays; internal -q -> L + (q-1)
    for (auto &c : raw) {
        if (c.x < 0) c.x = int(L + (-c.x - 1));
        if (c.y < 0) c.y = int(L + (-c.y - 1));
    }
    // order internal nodes by height, keeping creation order within a height
    int maxh = 0;
    for (int h : heights) maxh = h > maxh ? h : maxh;
    std::vector<int> new_index(raw.size());
    level_start.assign(maxh + 1, 0);
    std::vector<int> order;
    for (int h = 1; h <= maxh; ++h) {
        level_start[h - 1] = int64_t(order.size());
        for (size_t q = 0; q < raw.size(); ++q)
            if (heights[q] == h) order.push_back(int(q));
    }
    level_start[maxh] = int64_t(order.size());
    for (size_t p = 0; p < order.size(); ++p) new_index[order[p]] = int(p);
    nodes.resize(raw.size());
    for (size_t p = 0; p < order.size(); ++p) {
        int2 c = raw[order[p]];
        if (c.x >= L) c.x = int(L + new_index[c.x - L]);
        if (c.y >= L) c.y = int(L + new_index[c.y - L]);
        nodes[p] = c;
    }
    return maxh;
}

int pairwise_sum_run(ftk_ctx *ctx, const double *a, int64_t n, double *out, cudaStream_t st) {
    if (n <= 0) {
        FTK_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
        return FTK_OK;
    }
    PairwiseTree *T;
    {
        std::lock_guard<std::mutex> lk(g_tree_mu);
        T = &g_trees[{ctx, n}];
        if (T->n != n) {
            std::vector<int64_t> ls, lev;
            std::vector<int2> nodes;
            int nl = build_tree(n, ls, nodes, lev);
            T->n = n;
            T->nleaves = int64_t(ls.size()) - 1;
            T->nnodes = int64_t(nodes.size());
            T->nlevels = nl;
            FTK_CUDA(cudaMalloc(&T->d_leaf_start, sizeof(int64_t) * ls.size()));
            FTK_CUDA(cudaMalloc(&T->d_nodes, sizeof(int2) * (nodes.size() + 1)));
            FTK_CUDA(cudaMalloc(&T->d_level_start, sizeof(int64_t) * (lev.size() + 1)));
            FTK_CUDA(cudaMemcpy(T->d_leaf_start, ls.data(), sizeof(int64_t) * ls.size(), cudaMemcpyHostToDevice));
            if (!nodes.empty())
                FTK_CUDA(cudaMemcpy(T->d_nodes, nodes.data(), sizeof(int2) * nodes.size(), cudaMemcpyHostToDevice));
            FTK_CUDA(cudaMemcpy(T->d_level_start, lev.data(), sizeof(int64_t) * lev.size(), cudaMemcpyHostToDevice));
        }
    }
    double *vals = static_cast<double *>(scratch(ctx, SLOT_PAIRWISE, sizeof(double) * (T->nleaves + T->nnodes + 1), st));
    if (!vals) return FTK_ERR_CUDA;
    int64_t threads = T->nleaves * 8;
    pairwise_leaves_kernel<<<unsigned((threads + 255) / 256), 256, 0, st>>>(a, T->d_leaf_start, T->nleaves, vals);
    FTK_LAUNCHED("pairwise_leaves_kernel");
    const size_t tree_smem = sizeof(double) * size_t(T->nleaves + T->nnodes) + sizeof(int2) * size_t(T->nnodes) + 16;
    if (tree_smem <= 200 * 1024) {
        // opt in to > 48 KB (per call: cheap, and right for every device)
        FTK_CUDA(cudaFuncSetAttribute(pairwise_tree_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        pairwise_tree_kernel<true><<<1, 1024, tree_smem, st>>>(vals, T->d_nodes, T->d_level_start,
                                                               T->nlevels, T->nleaves, out);
    } else {
        pairwise_tree_kernel<false><<<1, 1024, 0, st>>>(vals, T->d_nodes, T->d_level_start, T->nlevels,
                                                        T->nleaves, out);
    }
    FTK_LAUNCHED("pairwise_tree_kernel");
    return FTK_OK;
}

int movement_run(ftk_ctx *ctx, int dtype, const void *nc, const void *oc, int64_t k, int64_t d,
                 double eps, double *moved, cudaStream_t st) {
    double *tmp = static_cast<double *>(scratch(ctx, SLOT_MISC, sizeof(double) * 2 * k * d + 64, st));
    if (!tmp) return FTK_ERR_CUDA;
    FTK_CUDA(cudaMemsetAsync(moved, 0, sizeof(double), st));
    auto mb = reinterpret_cast<unsigned long long *>(moved);
    if (d <= 128) {
        const unsigned g = unsigned((k * 32 + 255) / 256);
        if (dtype == FTK_F32)
            movement_warp_kernel<float><<<g, 256, 0, st>>>(static_cast<const float *>(nc), static_cast<const float *>(oc), k, d, eps, mb);
        else
            movement_warp_kernel<double><<<g, 256, 0, st>>>(static_cast<const double *>(nc), static_cast<const double *>(oc), k, d, eps, mb);
        FTK_LAUNCHED("movement_warp_kernel");
        return FTK_OK;
    }
    unsigned grid = unsigned((k + 127) / 128);
    if (dtype == FTK_F32)
        movement_kernel<float><<<grid, 128, 0, st>>>(static_cast<const float *>(nc), static_cast<const float *>(oc), k, d, eps, tmp, mb);
    else
        movement_kernel<double><<<grid, 128, 0, st>>>(static_cast<const double *>(nc), static_cast<const double *>(oc), k, d, eps, tmp, mb);
    FTK_LAUNCHED("movement_kernel");
    return FTK_OK;
}

int own_sq_dists_run(ftk_ctx *ctx, int dtype, const void *x, const int32_t *lab,
                     const double *c64, int64_t m, int64_t d, double *out, cudaStream_t st) {
    if (m <= 0) return FTK_OK;
    const int block = 128, grid = 148 * 2;
    double *tmp = static_cast<double *>(scratch(ctx, SLOT_MISC, sizeof(double) * block * grid * d, st));
    if (!tmp) return FTK_ERR_CUDA;
    if (dtype == FTK_F32)
        own_sq_dists_kernel<float><<<grid, block, 0, st>>>(static_cast<const float *>(x), lab, c64, m, d, tmp, out);
    else
        own_sq_dists_kernel<double><<<grid, block, 0, st>>>(static_cast<const double *>(x), lab, c64, m, d, tmp, out);
    FTK_LAUNCHED("own_sq_dists_kernel");
    return FTK_OK;
}

int labels_equal_run(const int32_t *a, const int32_t *b, int64_t m, int32_t *out, cudaStream_t st) {
    set_i32_kernel<<<1, 1, 0, st>>>(out, 1);
    FTK_LAUNCHED("set_i32_kernel");
    if (m > 0) {
        labels_equal_kernel<<<grid_for(m, 256), 256, 0, st>>>(a, b, m, out);
        FTK_LAUNCHED("labels_equal_kernel");
    }
    return FTK_OK;
}

int flip_f64_run(double *a, int64_t d, int64_t i, int64_t j, int64_t bit, double *ba,
                 cudaStream_t st) {
    flip_f64_kernel<<<1, 1, 0, st>>>(a, i * d + j, bit, ba);
    FTK_LAUNCHED("flip_f64_kernel");
    return FTK_OK;
}

}  // namespace ftk
