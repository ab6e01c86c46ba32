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

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace ftk {

constexpr int TC_BM = 128;       // rows per CTA (UMMA M)
constexpr int TC_KB = 32;        // fp32 elements per 128-byte swizzle row
constexpr int TC_THREADS = 192;  // 6 warps
constexpr int TC_MAX_D = 256;    // resident-A limit

struct TcParams {
    const float *x;      // rows x d  (exact values; pass 2: the gathered rows)
    const float *y;      // k x d
    const float *yn;     // k         (exact fp32 squared norms, reference order)
    int64_t m, k, d;
    int nkb;             // ceil(d / 32)
    int ntiles;          // ceil(k / BN)
    int stages;
    float a_coef;        // see header
    float b_coef;
    const float *cmax2;  // device scalar: upper bound of max_j ||c_j||^2
    const int32_t *rows; // pass 2: row r of the tile is global row rows[r]
    int32_t *out_idx;
    float *out_val;
    int32_t *fb_rows;    // uncertified rows (global indices)
    unsigned *fb_count;
    float *raw;          // debug: materialise the raw screened dot products
};

// ------------------------------------------------------------- kernel ----
template <int BN, bool SPLIT>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_screen_kernel(const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ CUtensorMap tmXl,
                     const __grid_constant__ CUtensorMap tmC,
                     const __grid_constant__ CUtensorMap tmCl, TcParams P) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int NOP = SPLIT ? 2 : 1;             // hi (+ lo) operand copies
    const int nkb = P.nkb, S = P.stages;
    const uint32_t A_KB_BYTES = TC_BM * 128;       // one k-block of X
    const uint32_t B_BYTES = BN * 128;             // one k-block of C
    unsigned char *sA = smem;                      // NOP x nkb x 16 KB (hi first)
    unsigned char *sB = sA + size_t(NOP) * nkb * A_KB_BYTES;  // S x NOP x B_BYTES
    uint64_t *bars = reinterpret_cast<uint64_t *>(sB + size_t(S) * NOP * B_BYTES);
    uint64_t *full = bars, *empty = bars + S;
    uint64_t *a_full = bars + 2 * S;
    uint64_t *t_full = a_full + 1, *t_empty = a_full + 3;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(a_full + 5);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = int64_t(blockIdx.x) * TC_BM;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmX);
        prefetch_tmap(&tmC);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(a_full, 1);
        mbar_init(&t_full[0], 1);
        mbar_init(&t_full[1], 1);
        mbar_init(&t_empty[0], 4);
        mbar_init(&t_empty[1], 4);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 2 * BN);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(a_full, A_KB_BYTES * nkb * NOP);
            for (int kb = 0; kb < nkb; ++kb) {
                tma_load_2d(sA + size_t(kb) * A_KB_BYTES, &tmX, a_full, kb * TC_KB, int(row0));
                if (SPLIT)
                    tma_load_2d(sA + size_t(nkb + kb) * A_KB_BYTES, &tmXl, a_full, kb * TC_KB,
                                int(row0));
            }
            int stage = 0;
            uint32_t phase = 0;
            for (int t = 0; t < P.ntiles; ++t) {
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], B_BYTES * NOP);
                    unsigned char *dst = sB + size_t(stage) * NOP * B_BYTES;
                    tma_load_2d(dst, &tmC, &full[stage], kb * TC_KB, t * BN);
                    if (SPLIT) tma_load_2d(dst + B_BYTES, &tmCl, &full[stage], kb * TC_KB, t * BN);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_tf32(TC_BM, BN);
            const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
            const uint32_t a_lo = a_base + uint32_t(nkb) * A_KB_BYTES;
            mbar_wait(a_full, 0);
            int stage = 0;
            uint32_t phase = 0;
            for (int t = 0; t < P.ntiles; ++t) {
                const int buf = t & 1;
                const uint32_t use = uint32_t(t >> 1) & 1;
                mbar_wait(&t_empty[buf], use ^ 1);
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
    } else {
        // ---------------------------------------------------- epilogue --
        const int quad = warp & 3;              // TMEM lane group this warp may access
        const int r = quad * 32 + lane;         // accumulator row
        const int64_t grow = row0 + r;          // row within this pass
        const uint32_t lane_base = uint32_t(quad * 32) << 16;
        float m1 = INFINITY, m2 = INFINITY;
        int tile1 = 0;
        for (int t = 0; t < P.ntiles; ++t) {
            const int buf = t & 1;
            const uint32_t use = uint32_t(t >> 1) & 1;
            mbar_wait(&t_full[buf], use);
            tc_fence_after();
            float t1 = INFINITY, t2 = INFINITY;
            const int64_t c0 = int64_t(t) * BN;
            const int live = int(P.k - c0 < BN ? P.k - c0 : BN);
            const uint32_t tbase = tmem + lane_base + uint32_t(buf * BN);
            // software-pipelined TMEM drain: chunk ch+1 in flight while ch is screened
            uint32_t va[32], vb[32];
            tmem_ld32_issue(tbase, va);
            tmem_ld_wait(va);
#pragma unroll
            for (int ch = 0; ch < BN / 32; ch += 2) {
                if (ch + 1 < BN / 32) tmem_ld32_issue(tbase + uint32_t((ch + 1) * 32), vb);
                if (P.raw && grow < P.m)
                    for (int e = 0; e < 32 && ch * 32 + e < live; ++e)
                        P.raw[grow * P.k + c0 + ch * 32 + e] = __uint_as_float(va[e]);
                screen_chunk(va, P.yn + c0 + ch * 32, ch * 32, live - ch * 32, t1, t2);
                if (ch + 1 < BN / 32) {
                    tmem_ld_wait(vb);
                    if (ch + 2 < BN / 32) tmem_ld32_issue(tbase + uint32_t((ch + 2) * 32), va);
                    if (P.raw && grow < P.m)
                        for (int e = 0; e < 32 && (ch + 1) * 32 + e < live; ++e)
                            P.raw[grow * P.k + c0 + (ch + 1) * 32 + e] = __uint_as_float(vb[e]);
                    screen_chunk(vb, P.yn + c0 + (ch + 1) * 32, (ch + 1) * 32,
                                 live - (ch + 1) * 32, t1, t2);
                    if (ch + 2 < BN / 32) tmem_ld_wait(va);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&t_empty[buf]);
            // merge the tile's top-2 into the running top-2
            const float hi = fmaxf(m1, t1);
            if (t1 < m1) tile1 = t;
            m1 = fminf(m1, t1);
            m2 = fminf(fminf(m2, t2), hi);
        }

        if (grow < P.m) {
            const int j = tile1 * BN + int(__float_as_uint(m1) & 0x7Fu);
            const int64_t orow = P.rows ? int64_t(P.rows[grow]) : grow;
            // one pass over the resident X row: ||x||^2 (bound) and the exact
            // sequential dot product with the screened winner.  The winner row
            // is fetched 32 floats (8 x 16 B) at a time so the L2 round trips
            // overlap; x comes from the swizzled tile (chunk q of row r sits at
            // chunk position q ^ (r & 7)); in split mode x = x_hi + x_lo exactly.
            const float4 *cj4 = reinterpret_cast<const float4 *>(P.y + int64_t(j) * P.d);
            float acc = 0.0f, xx = 0.0f;
            for (int kb = 0; kb < nkb; ++kb) {
                const int k0 = kb * TC_KB;
                float4 cv[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    cv[q] = (k0 + 4 * q < P.d) ? __ldg(cj4 + (k0 >> 2) + q)
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
                const unsigned char *rowp = sA + uint32_t(kb) * A_KB_BYTES + uint32_t(r) * 128;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (k0 + 4 * q < P.d) {
                        const uint32_t off = (q ^ (r & 7)) << 4;
                        // the hi tile holds the full fp32 x (the MMA truncates it)
                        const float4 xv = *reinterpret_cast<const float4 *>(rowp + off);
                        acc = __fadd_rn(acc, __fmul_rn(xv.x, cv[q].x));
                        acc = __fadd_rn(acc, __fmul_rn(xv.y, cv[q].y));
                        acc = __fadd_rn(acc, __fmul_rn(xv.z, cv[q].z));
                        acc = __fadd_rn(acc, __fmul_rn(xv.w, cv[q].w));
                        xx = fmaf(xv.x, xv.x, xx);
                        xx = fmaf(xv.y, xv.y, xx);
                        xx = fmaf(xv.z, xv.z, xx);
                        xx = fmaf(xv.w, xv.w, xx);
                    }
                }
            }
            const float A = P.a_coef * sqrtf(xx * (1.0f + 0x1p-10f)) * sqrtf(*P.cmax2);
            const float gap_need = 2.0f * A + P.b_coef * (fabsf(m1) + fabsf(m2));
            if (m2 - m1 > gap_need && m1 < INFINITY) {
                P.out_idx[orow] = j;
                P.out_val[orow] = __fsub_rn(P.yn[j], __fadd_rn(acc, acc));
            } else {
                const unsigned slot = atomicAdd(P.fb_count, 1u);
                P.fb_rows[slot] = int32_t(orow);
            }
        }
    }

    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 2 * BN);
    }
}

// --------------------------------------------------------- small kernels --
// Upper bound of max_j ||c_j||^2 from the exact fp32 norms; resets counters.
__global__ void tc_prep_kernel(const float *yn, int64_t k, float *cmax2, unsigned *counters) {
    float m = 0.0f;
    for (int64_t j = threadIdx.x; j < k; j += blockDim.x) m = fmaxf(m, yn[j]);
    for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    __shared__ float sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        float mm = 0.0f;
        for (int w = 0; w < int(blockDim.x / 32); ++w) mm = fmaxf(mm, sh[w]);
        *cmax2 = mm * (1.0f + 0x1p-10f);  // yn is a rounded sum
        counters[0] = counters[1] = 0u;
    }
}

__device__ __forceinline__ float tf32_trunc(float v) {
    return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
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

template <int BN, bool SPLIT>
static int launch_screen(TcParams P, const CUtensorMap &mx, const CUtensorMap &mxl,
                         const CUtensorMap &mc, const CUtensorMap &mcl, cudaStream_t st) {
    constexpr int NOP = SPLIT ? 2 : 1;
    const size_t a_bytes = size_t(P.nkb) * TC_BM * 128 * NOP;
    const size_t b_bytes = size_t(BN) * 128 * NOP;
    // Two CTAs per SM (one's refine/prologue overlaps the other's MMAs) when
    // the resident X tile leaves room for >= 2 centroid stages in ~113 KB.
    const size_t fixed = 1024 + a_bytes + 256;
    const size_t two_cta = 113 * 1024;
    int stages = fixed + 2 * b_bytes <= two_cta ? int((two_cta - fixed) / b_bytes)
                                                : int((227 * 1024 - fixed) / b_bytes);
    if (stages > 6) stages = 6;
    if (stages < 2) {
        set_error("tc: tile exceeds shared memory");
        return FTK_ERR_UNSUPPORTED;
    }
    P.stages = stages;
    const size_t smem = fixed + size_t(stages) * b_bytes;
    const int64_t grid = (P.m + TC_BM - 1) / TC_BM;
    if (grid == 0) return FTK_OK;
    auto kern = tc_screen_kernel<BN, SPLIT>;
    FTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<dim3(unsigned(grid)), dim3(TC_THREADS), smem, st>>>(mx, mxl, mc, mcl, P);
    FTK_LAUNCHED("tc_screen_kernel");
    return FTK_OK;
}

template <bool SPLIT>
static int screen(int bn, const TcParams &P, const CUtensorMap &mx, const CUtensorMap &mxl,
                  const CUtensorMap &mc, const CUtensorMap &mcl, cudaStream_t st) {
    switch (bn) {
        case 32: return launch_screen<32, SPLIT>(P, mx, mxl, mc, mcl, st);
        case 64: return launch_screen<64, SPLIT>(P, mx, mxl, mc, mcl, st);
        default: return launch_screen<128, SPLIT>(P, mx, mxl, mc, mcl, st);
    }
}

int tc_supported(int dtype, int64_t m, int64_t k, int64_t d) {
    return dtype == FTK_F32 && d >= 8 && d % 4 == 0 && d <= TC_MAX_D && k >= 1 && m >= 1 &&
           m < (int64_t(1) << 31) && k < (int64_t(1) << 24);
}

// exact.cu: the tiled exact kernel (used on gathered tie rows)
int exact_run(ftk_ctx *, int, const void *, const void *, const void *, int64_t, int64_t, int64_t,
              int64_t, int64_t, int64_t, int32_t *, void *, void *, bool, double, double, int64_t,
              const ftk_injection *, ftk_events *, cudaStream_t);

static unsigned g_last_fb[3] = {0, 0, 0};  // pass-1 flagged, pass-2 flagged (diagnostics)

int tc_assign_run(ftk_ctx *ctx, int dtype, const void *x, const void *y, const void *yn,
                  int64_t m, int64_t k, int64_t d, int32_t *out_idx, void *out_val,
                  cudaStream_t st, float *raw, int split_only) {
    if (!tc_supported(dtype, m, k, d)) {
        set_error("tc variant: unsupported shape/dtype");
        return FTK_ERR_UNSUPPORTED;
    }
    const float *xf = static_cast<const float *>(x), *yf = static_cast<const float *>(y);
    const float *ynf = static_cast<const float *>(yn);
    float *outv = static_cast<float *>(out_val);
    const int bn = k >= 128 ? 128 : (k > 32 ? 64 : 32);
    const int bn2 = k >= 64 ? 64 : 32;  // pass 2 carries hi+lo operands: narrower tiles
    float *misc = static_cast<float *>(scratch(ctx, SLOT_TC_MISC, 256, st));
    int32_t *rows1 = static_cast<int32_t *>(scratch(ctx, SLOT_TC_ROWS, sizeof(int32_t) * 2 * (m + 1), st));
    float *c_lo = static_cast<float *>(scratch(ctx, SLOT_TC_B, sizeof(float) * k * d, st));
    if (!misc || !rows1 || !c_lo) return FTK_ERR_CUDA;
    int32_t *rows2 = rows1 + (m + 1);
    unsigned *cnt = reinterpret_cast<unsigned *>(misc + 8);  // [0] pass-1 flagged, [1] pass-2
    tc_prep_kernel<<<1, 256, 0, st>>>(ynf, k, misc, cnt);
    FTK_LAUNCHED("tc_prep_kernel");

    TcParams P{};
    P.x = xf; P.y = yf; P.yn = ynf;
    P.m = m; P.k = k; P.d = d;
    P.nkb = int((d + TC_KB - 1) / TC_KB);
    P.b_coef = float((0x1p-15 + 0x1p-22) * 1.01);
    P.cmax2 = misc;
    P.out_idx = out_idx;
    P.out_val = outv;
    P.raw = raw;
    CUtensorMap mx, mc, mcl;
    int rc = make_map(&mc, yf, k, d, uint32_t(bn));
    if (rc) return rc;
    unsigned n1 = unsigned(m);
    const int32_t *pass2_rows = nullptr;
    if (!split_only) {
        // ---------------- pass 1: 1xTF32 over every row
        rc = make_map(&mx, xf, m, d, TC_BM);
        if (rc) return rc;
        P.ntiles = int((k + bn - 1) / bn);
        P.a_coef = float(2.0 * (0x1p-9 + 0x1p-20 + 3.0 * double(d) * 0x1p-24) * (1.0 + 0x1p-10));
        P.fb_rows = rows1;
        P.fb_count = cnt;
        rc = screen<false>(bn, P, mx, mx, mc, mc, st);
        if (rc) return rc;
        FTK_CUDA(cudaMemcpyAsync(&n1, cnt, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        FTK_CUDA(cudaStreamSynchronize(st));
        pass2_rows = rows1;
    }
    g_last_fb[0] = n1;
    g_last_fb[1] = 0;
    if (n1 == 0) return FTK_OK;
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
    rc = screen<true>(bn2, Q, mg, mgl, mc2, mcl2, st);
    unsigned n2 = 0;
    if (rc == FTK_ERR_UNSUPPORTED) {
        // hi+lo X tile does not fit (large D): every pass-1 tie goes exact
        rows2 = const_cast<int32_t *>(pass2_rows);
        n2 = n1;
        rc = FTK_OK;
    } else {
        if (rc) return rc;
        FTK_CUDA(cudaMemcpyAsync(&n2, cnt + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        FTK_CUDA(cudaStreamSynchronize(st));
        cnt += 1;
    }
    g_last_fb[1] = n2;
    if (n2 == 0) return FTK_OK;
    // ---------------- exact resolution of the remaining ties (tiled SIMT kernel)
    float *g2 = g;  // reuse: n2 <= n1 rows
    gather_rows_kernel<<<148 * 4, 256, 0, st>>>(xf, d, rows2, cnt, g2, nullptr);
    FTK_LAUNCHED("gather_rows_kernel");
    int32_t *idx2 = reinterpret_cast<int32_t *>(g_lo);
    float *val2 = g_lo + n2;
    rc = exact_run(ctx, FTK_F32, g2, yf, ynf, n2, k, d, 32, 256, 16, idx2, val2, nullptr, false,
                   0.0, 0.0, 0, nullptr, nullptr, st);
    if (rc) return rc;
    scatter_rows_kernel<float><<<148, 256, 0, st>>>(rows2, cnt, idx2, val2, out_idx, outv);
    FTK_LAUNCHED("scatter_rows_kernel");
    return FTK_OK;
}

int tc_last_fallback(ftk_ctx *, unsigned *out, cudaStream_t) {
    out[0] = g_last_fb[0];
    out[1] = g_last_fb[1];
    return FTK_OK;
}

}  // namespace ftk
