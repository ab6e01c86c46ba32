// kpp.cu -- k-means++ D^2 seeding on the device (reference kmeans.py:86-103).
//
// The reference, per pick c = 1..k-1 (numpy, float64):
//     total = d2.sum()                                   (pairwise sum)
//     r     = rng.random() * total                       (host Generator draw)
//     pick  = min(searchsorted(cumsum(d2), r, "right"), m - 1)
//     d2    = minimum(d2, ((x64 - x64[pick])**2).sum(axis=1))
// Everything except the Generator draw runs here, with no host round trip
// beyond the one scalar `total` the draw needs:
//
//   kpp_update_kernel   the D^2 row update; numpy's pairwise reduce over the
//                       feature axis (8 strided accumulators per <=128 leaf,
//                       recursive halving above 128) evaluated on the fly,
//                       any D.  The pick index comes from device memory.
//   search              cumsum(d2) is a SEQUENTIAL float64 running sum.  A
//                       parallel inclusive scan P~ (CUB) differs from it by at
//                       most E_i = 2 gamma_i P~_i (both are sums of the same
//                       non-negative terms, each within gamma_i = i u/(1-i u)
//                       of the exact prefix).  searchsorted(.., "right") of a
//                       non-decreasing array is the count of entries <= r:
//                       entries with P~_i + E_i <= r are certainly counted,
//                       entries with P~_i - E_i > r certainly not.  With no
//                       entry in between the count IS the reference's pick.
//   resolve             otherwise (rare: r within ~1e-10 relative of a
//                       boundary) one thread replays the reference's exact
//                       sequential cumsum up to the ambiguous window.
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"

namespace ftk {

// numpy pairwise_sum leaf over f(off..off+n-1), n <= 128 (loops_utils.h.src).
// f.group(i) is called before each run of up to 8 consecutive elements
// starting at a multiple of 8 (leaf offsets are multiples of 8), so a staged
// source can fetch once per group; f(i) returns element i.
template <class F>
__device__ __forceinline__ double pw_leaf(F &f, int64_t off, int64_t n) {
    if (n < 8) {
        f.group(off);
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s = __dadd_rn(s, f(off + i));
        return s;
    }
    double r[8];
    f.group(off);
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = f(off + j);
    int64_t i = 8;
#pragma unroll 1
    for (; i < n - (n % 8); i += 8) {
        f.group(off + i);
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(off + i + j));
    }
    double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    if (i < n) f.group(off + i);
    for (; i < n; ++i) s = __dadd_rn(s, f(off + i));
    return s;
}

// recursive halving (n2 = n/2 rounded down to a multiple of 8), post-order
template <class F>
__device__ double pw_sum(F &f, int64_t n) {
    if (n <= 128) return pw_leaf(f, 0, n);
    struct Fr { int64_t off, n; int state; double left; };
    Fr st[40];
    int sp = 0;
    st[0] = {0, n, 0, 0.0};
    double ret = 0.0;
    while (sp >= 0) {
        Fr &fr = st[sp];
        if (fr.n <= 128) {
            ret = pw_leaf(f, fr.off, fr.n);
            --sp;
            continue;
        }
        int64_t n2 = fr.n / 2;
        n2 -= n2 % 8;
        if (fr.state == 0) {
            fr.state = 1;
            st[sp + 1] = {fr.off, n2, 0, 0.0};
            ++sp;
        } else if (fr.state == 1) {
            fr.left = ret;
            fr.state = 2;
            st[sp + 1] = {fr.off + n2, fr.n - n2, 0, 0.0};
            ++sp;
        } else {
            ret = __dadd_rn(fr.left, ret);
            --sp;
        }
    }
    return ret;
}

// d2[i] = pairwise_sum_f((x64[i,f] - x64[pick,f])^2), then np.minimum with the
// previous d2 unless `first`.  pick: `host_pick` if >= 0, else *pick_dev.
// Block 0 records the pick in picks[c].
//
// One warp per 32 rows, lane = row.  Every lane walks the same feature
// sequence (the pairwise schedule depends only on d), so the warp stages its
// 32 rows 32 features at a time in shared memory with coalesced 128-byte row
// loads, and each lane reads its own row back from the staged tile.
template <typename T>
struct StagedSq {
    const T *x, *cr;
    int64_t d, r0;
    int rows, lane;
    T (*tile)[33];
    int64_t loaded;
    __device__ void group(int64_t f) {
        const int64_t ch = f >> 5;
        if (ch == loaded) return;  // warp-uniform
        __syncwarp();
        const int64_t col = ch * 32 + lane;
#pragma unroll 4
        for (int rr = 0; rr < 32; ++rr)
            tile[rr][lane] = (rr < rows && col < d) ? x[(r0 + rr) * d + col] : T(0);
        __syncwarp();
        loaded = ch;
    }
    __device__ double operator()(int64_t f) const {
        const double df = __dsub_rn(double(tile[lane][f & 31]), double(cr[f]));
        return __dmul_rn(df, df);
    }
};

template <typename T, int W>
__global__ void __launch_bounds__(W * 32) kpp_update_kernel(const T *x, int64_t m, int64_t d,
                                                            int64_t host_pick, const int64_t *pick_dev,
                                                            int first, double *d2, int64_t *picks,
                                                            int64_t c) {
    __shared__ T tile_all[W][32][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t pick = host_pick >= 0 ? host_pick : *pick_dev;
    if (picks && blockIdx.x == 0 && threadIdx.x == 0) picks[c] = pick;
    StagedSq<T> f{x, x + pick * d, d, 0, 0, lane, tile_all[w], -1};
    const int64_t ngroups = (m + 31) / 32;
    for (int64_t g = int64_t(blockIdx.x) * W + w; g < ngroups; g += int64_t(gridDim.x) * W) {
        f.r0 = g * 32;
        f.rows = m - f.r0 < 32 ? int(m - f.r0) : 32;
        f.loaded = -1;
        const double s = pw_sum(f, d);
        if (lane < f.rows) {
            const int64_t i = f.r0 + lane;
            if (first) {
                d2[i] = s;
            } else {
                const double o = d2[i];
                d2[i] = (s != s || o != o) ? s + o : (s < o ? s : o);  // np.minimum (NaN propagates)
            }
        }
    }
}

// Classify every prefix against r: cnt[0] += certainly <= r, cnt[1] +=
// ambiguous, cnt[2] = min ambiguous index, cnt[3] = max ambiguous index,
// cnt[4] = max certainly-<= index + 1.
__global__ void kpp_classify_kernel(const double *P, int64_t m, double r,
                                    unsigned long long *cnt) {
    unsigned long long le = 0, amb = 0, amin = ~0ull, amax = 0, lmax = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x) {
        const double p = P[i];
        // E_i = 2 gamma_{i+1} p (1 + slack): |cumsum_i - P~_i| <= E_i
        const double g = double(i + 1) * 0x1p-53;
        const double e = 2.0 * g / (1.0 - g) * p * (1.0 + 0x1p-20) + 0x1p-1074;
        if (p + e <= r) {
            ++le;
            lmax = max(lmax, (unsigned long long)(i + 1));
        } else if (!(p - e > r)) {
            ++amb;
            amin = min(amin, (unsigned long long)i);
            amax = max(amax, (unsigned long long)i);
        }
    }
    typedef cub::BlockReduce<unsigned long long, 256> BR;
    __shared__ typename BR::TempStorage tmp;
    le = BR(tmp).Sum(le);
    __syncthreads();
    amb = BR(tmp).Sum(amb);
    __syncthreads();
    amin = BR(tmp).Reduce(amin, cub::Min());
    __syncthreads();
    amax = BR(tmp).Reduce(amax, cub::Max());
    __syncthreads();
    lmax = BR(tmp).Reduce(lmax, cub::Max());
    if (threadIdx.x == 0) {
        if (le) {
            atomicAdd(cnt + 0, le);
            atomicMax(cnt + 4, lmax);
        }
        if (amb) {
            atomicAdd(cnt + 1, amb);
            atomicMin(cnt + 2, amin);
            atomicMax(cnt + 3, amax);
        }
    }
}

// pick = min(count(cumsum <= r), m - 1); ambiguous: the reference's exact
// sequential cumsum, walked to the end of the ambiguous window
__global__ void kpp_resolve_kernel(const double *d2, int64_t m, double r,
                                   const unsigned long long *cnt, int64_t *pick,
                                   unsigned long long *n_replays) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t count = int64_t(cnt[0]);
    if (cnt[1]) {
        // every entry past both the ambiguous window and the last certain
        // "<= r" entry is certainly > r: the walk's count is the exact count
        const int64_t hi = max(int64_t(cnt[3]) + 1, int64_t(cnt[4]));
        double cs = 0.0;
        int64_t le = 0;
        for (int64_t i = 0; i < hi; ++i) {
            cs = __dadd_rn(cs, d2[i]);
            le += cs <= r ? 1 : 0;
        }
        count = le;
        atomicAdd(n_replays, 1ull);
    }
    *pick = count < m - 1 ? count : m - 1;
}

template <typename T>
static int update_launch(const void *x, int64_t m, int64_t d, int64_t host_pick,
                         const int64_t *pick_dev, int first, double *d2, int64_t *picks, int64_t c,
                         cudaStream_t st) {
    constexpr int W = sizeof(T) == 8 ? 4 : 8;  // warps per block (staging tile <= 34 KB)
    const int64_t groups = (m + 31) / 32;
    const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>((groups + W - 1) / W, 148 * 16)));
    kpp_update_kernel<T, W><<<grid, W * 32, 0, st>>>(static_cast<const T *>(x), m, d, host_pick, pick_dev,
                                                     first, d2, picks, c);
    FTK_LAUNCHED("kpp_update_kernel");
    return FTK_OK;
}

int kpp_update_run(int dtype, const void *x, int64_t m, int64_t d, int64_t host_pick,
                   const int64_t *pick_dev, int first, double *d2, int64_t *picks, int64_t c,
                   cudaStream_t st) {
    if (m < 1 || d < 1) return FTK_OK;
    return dtype == FTK_F32 ? update_launch<float>(x, m, d, host_pick, pick_dev, first, d2, picks, c, st)
                            : update_launch<double>(x, m, d, host_pick, pick_dev, first, d2, picks, c, st);
}

int kpp_search_run(ftk_ctx *ctx, const double *d2, int64_t m, double r, int64_t *pick,
                   unsigned long long *n_replays, cudaStream_t st) {
    if (m < 1) return FTK_OK;
    size_t tmp_bytes = 0;
    FTK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, d2, static_cast<double *>(nullptr),
                                           m, st));
    const size_t pbytes = (sizeof(double) * size_t(m) + 255) & ~size_t(255);
    char *buf = static_cast<char *>(scratch(ctx, SLOT_KPP, pbytes + 256 + tmp_bytes, st));
    if (!buf) return FTK_ERR_CUDA;
    double *P = reinterpret_cast<double *>(buf);
    unsigned long long *cnt = reinterpret_cast<unsigned long long *>(buf + pbytes);
    void *tmp = buf + pbytes + 256;
    FTK_CUDA(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, d2, P, m, st));
    FTK_CUDA(cudaMemsetAsync(cnt, 0, 5 * sizeof(unsigned long long), st));
    FTK_CUDA(cudaMemsetAsync(cnt + 2, 0xFF, sizeof(unsigned long long), st));  // min index
    const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 148 * 4)));
    kpp_classify_kernel<<<grid, 256, 0, st>>>(P, m, r, cnt);
    FTK_LAUNCHED("kpp_classify_kernel");
    kpp_resolve_kernel<<<1, 32, 0, st>>>(d2, m, r, cnt, pick, n_replays);
    FTK_LAUNCHED("kpp_resolve_kernel");
    return FTK_OK;
}

}  // namespace ftk
