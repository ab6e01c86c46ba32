// tc_ptx.cuh -- inline-PTX wrappers for sm_100a: mbarrier, TMA, tcgen05
// (alloc / mma kind::tf32 / commit / ld), UMMA descriptors, and the screening
// epilogue primitive shared by the tensor-core kernels.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace ftk {

// ----------------------------------------------------------- PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifndef FTK_WAIT_TICKS
#define FTK_WAIT_TICKS 0x989680u
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#if FTK_WAIT_TICKS
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(FTK_WAIT_TICKS)  // suspend hint: sleep in the barrier, not in an issue-slot spin
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
}
// 64 consecutive TMEM columns in one load: columns 0-31 to a, 32-63 to b
__device__ __forceinline__ void tmem_ld64_issue(uint32_t taddr, uint32_t (&a)[32], uint32_t (&b)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
        "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]),
          "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15]),
          "=r"(a[16]), "=r"(a[17]), "=r"(a[18]), "=r"(a[19]), "=r"(a[20]), "=r"(a[21]), "=r"(a[22]), "=r"(a[23]),
          "=r"(a[24]), "=r"(a[25]), "=r"(a[26]), "=r"(a[27]), "=r"(a[28]), "=r"(a[29]), "=r"(a[30]), "=r"(a[31]),
          "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]),
          "=r"(b[8]), "=r"(b[9]), "=r"(b[10]), "=r"(b[11]), "=r"(b[12]), "=r"(b[13]), "=r"(b[14]), "=r"(b[15]),
          "=r"(b[16]), "=r"(b[17]), "=r"(b[18]), "=r"(b[19]), "=r"(b[20]), "=r"(b[21]), "=r"(b[22]), "=r"(b[23]),
          "=r"(b[24]), "=r"(b[25]), "=r"(b[26]), "=r"(b[27]), "=r"(b[28]), "=r"(b[29]), "=r"(b[30]), "=r"(b[31])
        : "r"(taddr));
}
// no instruction: orders every later use of `v` after the preceding wait::ld
__device__ __forceinline__ void tmem_pin(uint32_t (&v)[32]) {
    asm volatile(""
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                   "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                   "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]),
                   "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                   "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]),
                   "+r"(v[30]), "+r"(v[31])
                 :
                 : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// wait::ld that also pins the destination registers, so no use of `v` can be
// scheduled before the load has completed
__device__ __forceinline__ void tmem_ld_wait(uint32_t (&v)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                   "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                   "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]),
                   "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]),
                   "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]),
                   "+r"(v[30]), "+r"(v[31])
                 :
                 : "memory");
}

__device__ __forceinline__ float tf32_trunc(float v) {
    return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
}

// Scheduled flip on the TMEM-loaded accumulator of column e (0..31): the
// screened value moves by the reference's delta (after - before of the exact
// accumulator) or becomes the non-finite flipped value.  Static indexing only.
__device__ __forceinline__ void inject_into(uint32_t (&v)[32], int e, float before, float after) {
#pragma unroll
    for (int u = 0; u < 32; ++u)
        if (u == e) {
            const float cur = __uint_as_float(v[u]);
            v[u] = __float_as_uint(isfinite(after) ? cur + (after - before) : after);
        }
}

// Running top-2 (t1 <= t2) update with two new values: 5 min/max ops per
// pair (the compiler emits FMNMX3 for the 3-input minimum).
__device__ __forceinline__ void top2_pair(float a, float b, float &t1, float &t2) {
    const float u = fminf(t1, a), v = fmaxf(t1, a);
    const float w = fmaxf(u, b);
    t2 = fminf(fminf(t2, v), w);
    t1 = fminf(u, b);
}

__device__ __forceinline__ float pack_col(float dd, uint32_t col, uint32_t mask) {
    return __uint_as_float((__float_as_uint(dd) & ~mask) | col);
}

// Screen 32 accumulator columns: s = yn - 2 acc with the index packed into
// the low 7 mantissa bits (column within the <=128-wide tile), folded into
// the running top-2.  yn_s points at this chunk's 32 norms in SHARED memory
// (broadcast reads); `live` = valid columns in the chunk (<= 0: none).
template <bool CHK = false>
__device__ __forceinline__ void screen_chunk(const uint32_t (&v)[32], const float *yn_s,
                                             int cbase, int live, uint32_t mask, float &t1,
                                             float &t2, float &tsum) {
    if (live >= 32) {
        const float4 *yn4 = reinterpret_cast<const float4 *>(yn_s);
        float part[2] = {0.0f, 0.0f};
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 yv = yn4[q];
            const int e = q * 4;
            if (CHK) {  // ABFT row checksum over the raw accumulators (shallow tree)
                const float s01 = __uint_as_float(v[e + 0]) + __uint_as_float(v[e + 1]);
                const float s23 = __uint_as_float(v[e + 2]) + __uint_as_float(v[e + 3]);
                part[q & 1] += s01 + s23;
            }
            const float p0 = pack_col(fmaf(-2.0f, __uint_as_float(v[e + 0]), yv.x), cbase + e + 0, mask);
            const float p1 = pack_col(fmaf(-2.0f, __uint_as_float(v[e + 1]), yv.y), cbase + e + 1, mask);
            const float p2 = pack_col(fmaf(-2.0f, __uint_as_float(v[e + 2]), yv.z), cbase + e + 2, mask);
            const float p3 = pack_col(fmaf(-2.0f, __uint_as_float(v[e + 3]), yv.w), cbase + e + 3, mask);
            top2_pair(p0, p1, t1, t2);
            top2_pair(p2, p3, t1, t2);
        }
        if (CHK) tsum += part[0] + part[1];
    } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            if (e < live) {
                if (CHK) tsum += __uint_as_float(v[e]);
                const float p =
                    pack_col(fmaf(-2.0f, __uint_as_float(v[e]), yn_s[e]), cbase + e, mask);
                const float hi = fmaxf(t1, p);
                t1 = fminf(t1, p);
                t2 = fminf(t2, hi);
            }
        }
    }
}

// K-major, 128-byte swizzled operand tile (rows of 128 B, 8-row atoms of
// 1024 B): start address >> 4, SBO = 1024 B, version 1, layout SWIZZLE_128B.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t(1) << 16;                 // LBO (unused for swizzled K-major)
    d |= uint64_t(1024 >> 4) << 32;         // SBO
    d |= uint64_t(1) << 46;                 // descriptor version (sm100)
    d |= uint64_t(2) << 61;                 // SWIZZLE_128B
    return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) |
           (uint32_t(M >> 4) << 24);
}


}  // namespace ftk

// ------------------------------------------------ CTA-pair (cluster) PTX --
namespace ftk {
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t ncluster_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
// shared::cta address -> shared::cluster address of the same offset in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
// wait with cluster-scope acquire (barriers that receive arrivals from the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA 2-D load into this CTA's shared memory, completion counted on an
// mbarrier that may live in either CTA of the pair (cluster address)
__device__ __forceinline__ void tma_load_2d_pair(void *dst, const CUtensorMap *map,
                                                 uint32_t bar_cluster, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
// D[tmem] (+)= A[smem, both CTAs: 128 rows each] . B[smem, both CTAs: N/2 rows each]^T
__device__ __forceinline__ void mma_tf32_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// completion of all prior pair MMAs -> one arrive on `bar` in every CTA of `mask`
__device__ __forceinline__ void mma_commit_pair(uint64_t *bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"(mask)
        : "memory");
}
}  // namespace ftk

namespace ftk {
// screen_chunk with the 32 centroid norms read from GLOBAL memory (uniform
// addresses across the warp: one broadcast transaction per float4)
template <bool CHK = false>
__device__ __forceinline__ void screen_chunk_g(const uint32_t (&v)[32], const float *yn_g,
                                               int cbase, int live, uint32_t mask, float &t1,
                                               float &t2, float &tsum) {
    if (live >= 32) {
        const float4 *yn4 = reinterpret_cast<const float4 *>(yn_g);
        float part[2] = {0.0f, 0.0f};
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 yv = __ldg(yn4 + q);
            const int e = q * 4;
            if (CHK) {
                const float s01 = __uint_as_float(v[e + 0]) + __uint_as_float(v[e + 1]);
                const float s23 = __uint_as_float(v[e + 2]) + __uint_as_float(v[e + 3]);
                part[q & 1] += s01 + s23;
            }
            const float p0 = pack_col(fmaf(-2.0f, __uint_as_float(v[e + 0]), yv.x), cbase + e + 0, mask);
            const float p1 = pack_col(fmaf(-2.0f, __uint_as_float(v[e + 1]), yv.y), cbase + e + 1, mask);
            const float p2 = pack_col(fmaf(-2.0f, __uint_as_float(v[e + 2]), yv.z), cbase + e + 2, mask);
            const float p3 = pack_col(fmaf(-2.0f, __uint_as_float(v[e + 3]), yv.w), cbase + e + 3, mask);
            top2_pair(p0, p1, t1, t2);
            top2_pair(p2, p3, t1, t2);
        }
        if (CHK) tsum += part[0] + part[1];
    } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            if (e < live) {
                if (CHK) tsum += __uint_as_float(v[e]);
                const float p =
                    pack_col(fmaf(-2.0f, __uint_as_float(v[e]), __ldg(yn_g + e)), cbase + e, mask);
                const float hi = fmaxf(t1, p);
                t1 = fminf(t1, p);
                t2 = fminf(t2, hi);
            }
        }
    }
}
}  // namespace ftk

namespace ftk {
// arrive on a (possibly remote) cluster barrier with default (CTA-scope
// release) semantics -- no GPU-scope fence; ordering of tensor-memory reads
// is carried by tcgen05.fence::before_thread_sync on the arriving side
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
}  // namespace ftk

namespace ftk {
// d = a * (-2, -2) + c on the paired FP32 pipe (FFMA2); a, c adjacent registers
__device__ __forceinline__ void ffma2_m2(float a0, float a1, float c0, float c1, float &d0,
                                         float &d1) {
    asm("{.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\tmov.b64 rc, {%5, %6};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(-2.0f), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void fadd2(float &s0, float &s1, float a0, float a1) {
    asm("{.reg .b64 ra, rs;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rs, {%0, %1};\n\t"
        "add.rn.f32x2 rs, rs, ra;\n\tmov.b64 {%0, %1}, rs;}"
        : "+f"(s0), "+f"(s1)
        : "f"(a0), "f"(a1));
}

// Screen 32 accumulator columns (no partial chunks: padded columns carry
// yn = +inf, so their packed value is a NaN that fminf never selects; their
// accumulators are exactly 0 from the zero-filled TMA tile, so the ABFT sum
// is unaffected).  Two independent running top-2 states (a: even pairs,
// b: odd pairs) halve the dependency chain; merged by the caller.
template <bool CHK>
__device__ __forceinline__ void screen32(const uint32_t (&v)[32], const float *yn_s, uint32_t cbase,
                                         float &a1, float &a2, float &b1, float &b2, float &s0,
                                         float &s1) {
    const float4 *yn4 = reinterpret_cast<const float4 *>(yn_s);
    // the four packed column indices of quad q live in the bytes of one
    // register: idx4 = (cbase + 4q) * 0x01010101 + 0x03020100; PRMT moves
    // byte i into the low byte of element i (1.25 instructions per element
    // instead of an add and a mask-or)
    const uint32_t base4 = cbase * 0x01010101u + 0x03020100u;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const float4 yv = yn4[q];
        const int e = q * 4;
        if (CHK) {
            fadd2(s0, s1, __uint_as_float(v[e + 0]), __uint_as_float(v[e + 1]));
            fadd2(s0, s1, __uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
        }
        float d0, d1, d2, d3;
        ffma2_m2(__uint_as_float(v[e + 0]), __uint_as_float(v[e + 1]), yv.x, yv.y, d0, d1);
        ffma2_m2(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]), yv.z, yv.w, d2, d3);
        const uint32_t idx4 = base4 + uint32_t(e) * 0x01010101u;
        const float p0 = __uint_as_float(__byte_perm(__float_as_uint(d0), idx4, 0x3214));
        const float p1 = __uint_as_float(__byte_perm(__float_as_uint(d1), idx4, 0x3215));
        const float p2 = __uint_as_float(__byte_perm(__float_as_uint(d2), idx4, 0x3216));
        const float p3 = __uint_as_float(__byte_perm(__float_as_uint(d3), idx4, 0x3217));
        top2_pair(p0, p1, a1, a2);
        top2_pair(p2, p3, b1, b2);
    }
}
}  // namespace ftk

namespace ftk {
// (a0, a1) + (b0, b1) and (a0, a1) - (b0, b1) on the paired FP32 pipe
__device__ __forceinline__ void fadd2v(float a0, float a1, float b0, float b1, float &d0, float &d1) {
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void fsub2v(float a0, float a1, float b0, float b1, float &d0, float &d1) {
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// Tournament screen of 32 accumulator columns.
//
// Packed values p (index in the low byte, see screen32) play a knockout
// tournament: each match keeps lo = min(a, b) on the ALU pipe and the loser
// hi = (a + b) - lo on the paired FP32 pipe (FADD2).  The chunk minimum is the
// champion (exact, index included) and the second smallest value is the
// smallest loser, min over all hi (every non-champion is >= the runner-up,
// who only loses to the champion).  The FP32 reconstruction of hi is within
// 2^-23 (|a| + |b| + |hi|) of the true loser; the caller's certificate
// subtracts that margin, so the runner-up bound stays a lower bound.  This
// needs ~1.5 ALU + 1 PRMT per column instead of 2.5 + 1 for a running top-2.
// Padded columns (yn = +inf) pack to NaN: fminf drops them and their sums
// are NaN, which every later minimum ignores.
template <bool CHK>
__device__ __forceinline__ void screen32t(const uint32_t (&v)[32], const float *yn_s,
                                          uint32_t cbase, float &L1, float &M2, float &s0,
                                          float &s1) {
    const float4 *yn4 = reinterpret_cast<const float4 *>(yn_s);
    const uint32_t base4 = cbase * 0x01010101u + 0x03020100u;
    float p[32];
    if (CHK) {
        // row-sum of the raw accumulators: a pairwise tree (FADD2), not a chain
        float t[16];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            fadd2v(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                   __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]), t[2 * i], t[2 * i + 1]);
#pragma unroll
        for (int i = 0; i < 4; ++i) fadd2v(t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3], t[2 * i], t[2 * i + 1]);
#pragma unroll
        for (int i = 0; i < 2; ++i) fadd2v(t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3], t[2 * i], t[2 * i + 1]);
        fadd2v(t[0], t[1], t[2], t[3], t[0], t[1]);
        fadd2(s0, s1, t[0], t[1]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const float4 yv = yn4[q];
        const int e = q * 4;
        float d0, d1, d2, d3;
        ffma2_m2(__uint_as_float(v[e + 0]), __uint_as_float(v[e + 1]), yv.x, yv.y, d0, d1);
        ffma2_m2(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]), yv.z, yv.w, d2, d3);
        const uint32_t idx4 = base4 + uint32_t(e) * 0x01010101u;
        p[e + 0] = __uint_as_float(__byte_perm(__float_as_uint(d0), idx4, 0x3214));
        p[e + 1] = __uint_as_float(__byte_perm(__float_as_uint(d1), idx4, 0x3215));
        p[e + 2] = __uint_as_float(__byte_perm(__float_as_uint(d2), idx4, 0x3216));
        p[e + 3] = __uint_as_float(__byte_perm(__float_as_uint(d3), idx4, 0x3217));
    }
    // rounds: matches (x[4j], x[4j+2]) and (x[4j+1], x[4j+3]) so both sums are
    // one FADD2 of adjacent register pairs
    float h[32];
    int nh = 0;
#pragma unroll
    for (int n = 32; n >= 4; n >>= 1) {
#pragma unroll
        for (int j = 0; j < n / 4; ++j) {
            float sa, sb, la, lb, ha, hb;
            fadd2v(p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3], sa, sb);
            la = fminf(p[4 * j], p[4 * j + 2]);
            lb = fminf(p[4 * j + 1], p[4 * j + 3]);
            fsub2v(sa, sb, la, lb, ha, hb);
            h[nh++] = ha;
            h[nh++] = hb;
            p[2 * j] = la;
            p[2 * j + 1] = lb;
        }
    }
    // final match of the two remaining finalists
    const float c1 = fminf(p[0], p[1]);
    h[nh++] = (p[0] + p[1]) - c1;
    // smallest loser: 31 values in 15 three-input minima
    float r[11];
#pragma unroll
    for (int i = 0; i < 10; ++i) r[i] = fminf(fminf(h[3 * i], h[3 * i + 1]), h[3 * i + 2]);
    r[10] = h[30];
    const float u0 = fminf(fminf(r[0], r[1]), r[2]);
    const float u1 = fminf(fminf(r[3], r[4]), r[5]);
    const float u2 = fminf(fminf(r[6], r[7]), r[8]);
    const float w0 = fminf(fminf(u0, u1), u2);
    const float hmin = fminf(fminf(w0, r[9]), r[10]);
    // a chunk with no live column has c1 = NaN: it must not demote the
    // running champion to runner-up (fmaxf would return L1)
    M2 = fminf(fminf(M2, hmin), c1 == c1 ? fmaxf(L1, c1) : INFINITY);
    L1 = fminf(L1, c1);
}
}  // namespace ftk

namespace ftk {
// 16 consecutive TMEM columns of this warp's 32 lanes (one row per thread)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                   "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                   "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
                 :
                 : "memory");
}
}  // namespace ftk
