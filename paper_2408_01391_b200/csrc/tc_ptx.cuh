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
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
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
