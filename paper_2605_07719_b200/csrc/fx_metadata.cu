// fx_metadata.cu -- K1: Quest block metadata (element-wise min / max keys per
// logical block), block_index.cpp:10-39.
//
// Batched builder: one streaming pass over every (b, g) cpu segment produces
// all four candidate granularities {16, 32, 64, 128} (selector.hpp:12).  A
// CTA owns a 128-row slab: each warp reduces 16 rows with 128-bit loads
// (level 16), then the CTA folds pairs in shared memory (32, 64, 128).
// Folding is bit-identical to a direct build because min/max are exact and
// every fold keeps the EARLIER operand on ties, like the reference's
// sequential `mn = (row < mn) ? row : mn` (std::min keeps its first argument).
//
// HBM layout of a level: [B][Hkv][nblk][2][D] in the KV dtype -- the min row
// and the max row of a block are adjacent, so scoring reads 2*D*s contiguous
// bytes per block.
#include "fx_common.cuh"

namespace fx {
namespace {

template <int DT>
__device__ __forceinline__ void unpack16(const uint4& w, float* out);
template <>
__device__ __forceinline__ void unpack16<FX_BF16>(const uint4& w, float* out) {
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        out[2 * i] = bf16lo_to_f(u[i]);
        out[2 * i + 1] = bf16hi_to_f(u[i]);
    }
}
template <>
__device__ __forceinline__ void unpack16<FX_F32>(const uint4& w, float* out) {
    out[0] = __uint_as_float(w.x);
    out[1] = __uint_as_float(w.y);
    out[2] = __uint_as_float(w.z);
    out[3] = __uint_as_float(w.w);
}
template <int DT>
__device__ __forceinline__ uint4 pack16(const float* v);
template <>
__device__ __forceinline__ uint4 pack16<FX_BF16>(const float* v) {
    // values are exact bf16 (they came from bf16 storage): truncation is exact
    uint4 w;
    w.x = (__float_as_uint(v[0]) >> 16) | (__float_as_uint(v[1]) & 0xffff0000u);
    w.y = (__float_as_uint(v[2]) >> 16) | (__float_as_uint(v[3]) & 0xffff0000u);
    w.z = (__float_as_uint(v[4]) >> 16) | (__float_as_uint(v[5]) & 0xffff0000u);
    w.w = (__float_as_uint(v[6]) >> 16) | (__float_as_uint(v[7]) & 0xffff0000u);
    return w;
}
template <>
__device__ __forceinline__ uint4 pack16<FX_F32>(const float* v) {
    return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]),
                      __float_as_uint(v[3]));
}

// keep-first folds (L holds earlier rows than R)
__device__ __forceinline__ float fold_min(float L, float R) { return (R < L) ? R : L; }
__device__ __forceinline__ float fold_max(float L, float R) { return (L < R) ? R : L; }

constexpr int kSlab = 128;  // rows per CTA
constexpr int kWarps = 8;   // 16 rows per warp

template <int DT, int D>
__global__ void __launch_bounds__(256) k_meta_levels(const typename Elem<DT>::T* __restrict__ k,
                                                     int64_t l_cap, int64_t l_sink, int64_t l_cpu,
                                                     typename Elem<DT>::T* __restrict__ m16,
                                                     typename Elem<DT>::T* __restrict__ m32,
                                                     typename Elem<DT>::T* __restrict__ m64,
                                                     typename Elem<DT>::T* __restrict__ m128,
                                                     float* __restrict__ absmax) {
    using T = typename Elem<DT>::T;
    constexpr int V = 16 / Elem<DT>::kBytes;  // elements per 128-bit vector
    constexpr int LPR = D / V;                // lanes per row
    static_assert(LPR >= 1 && LPR <= 32 && (32 % LPR) == 0, "row must fit one warp");
    constexpr int RPW = 32 / LPR;             // rows per warp load
    constexpr int RPS = kBoxRows / RPW;       // rows per lane slot (contiguous)

    __shared__ float s16[kWarps][2][D];
    __shared__ float s32[4][2][D];
    __shared__ float s64[2][2][D];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t bg = blockIdx.y;
    const int64_t slab = blockIdx.x;
    const int slot = lane / LPR, col = (lane % LPR) * V;
    const T* kb = k + (bg * l_cap + l_sink) * D;

    float mn[V], mx[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
        mn[i] = __int_as_float(0x7f800000);
        mx[i] = -__int_as_float(0x7f800000);
    }
    const int64_t r0 = slab * kSlab + warp * kBoxRows + slot * RPS;
    uint4 raw[RPS];
#pragma unroll
    for (int i = 0; i < RPS; ++i) {
        const int64_t r = r0 + i;
        raw[i] = r < l_cpu ? __ldg(reinterpret_cast<const uint4*>(kb + r * D + col))
                           : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < RPS; ++i) {
        if (r0 + i < l_cpu) {
            float x[V];
            unpack16<DT>(raw[i], x);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                mn[j] = fold_min(mn[j], x[j]);
                mx[j] = fold_max(mx[j], x[j]);
            }
        }
    }
    // fold the RPW row slots of the warp in row order
#pragma unroll
    for (int step = LPR; step < 32; step <<= 1) {
        const bool lower = ((lane / step) & 1) == 0;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const float pmn = __shfl_xor_sync(0xffffffffu, mn[j], step);
            const float pmx = __shfl_xor_sync(0xffffffffu, mx[j], step);
            mn[j] = lower ? fold_min(mn[j], pmn) : fold_min(pmn, mn[j]);
            mx[j] = lower ? fold_max(mx[j], pmx) : fold_max(pmx, mx[j]);
        }
    }
    const int64_t j16 = slab * kWarps + warp;
    const int64_t n16 = cdiv_dev(l_cpu, 16);
    if (slot == 0) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
            s16[warp][0][col + j] = mn[j];
            s16[warp][1][col + j] = mx[j];
        }
        if (j16 < n16) {
            T* dst = m16 + (bg * n16 + j16) * 2 * D;
            *reinterpret_cast<uint4*>(dst + col) = pack16<DT>(mn);
            *reinterpret_cast<uint4*>(dst + D + col) = pack16<DT>(mx);
        }
    }
    __syncthreads();
    // level 32
    {
        const int64_t n32 = cdiv_dev(l_cpu, 32);
        for (int e = threadIdx.x; e < 4 * 2 * D; e += blockDim.x) {
            const int i = e / (2 * D), which = (e / D) & 1, d = e % D;
            const float L = s16[2 * i][which][d], R = s16[2 * i + 1][which][d];
            const float val = which ? fold_max(L, R) : fold_min(L, R);
            s32[i][which][d] = val;
            const int64_t j = slab * 4 + i;
            if (j < n32) m32[((bg * n32 + j) * 2 + which) * D + d] = Elem<DT>::from_f(val);
        }
    }
    __syncthreads();
    {
        const int64_t n64 = cdiv_dev(l_cpu, 64);
        for (int e = threadIdx.x; e < 2 * 2 * D; e += blockDim.x) {
            const int i = e / (2 * D), which = (e / D) & 1, d = e % D;
            const float L = s32[2 * i][which][d], R = s32[2 * i + 1][which][d];
            const float val = which ? fold_max(L, R) : fold_min(L, R);
            s64[i][which][d] = val;
            const int64_t j = slab * 2 + i;
            if (j < n64) m64[((bg * n64 + j) * 2 + which) * D + d] = Elem<DT>::from_f(val);
        }
    }
    __syncthreads();
    {
        const int64_t n128 = cdiv_dev(l_cpu, 128);
        for (int e = threadIdx.x; e < D; e += blockDim.x) {
            const float lo = fold_min(s64[0][0][e], s64[1][0][e]);
            const float hi = fold_max(s64[0][1][e], s64[1][1][e]);
            if (slab < n128) {
                T* dst = m128 + (bg * n128 + slab) * 2 * D;
                dst[e] = Elem<DT>::from_f(lo);
                dst[D + e] = Elem<DT>::from_f(hi);
            }
            if (absmax) {
                const float a = fmaxf(fabsf(lo), fabsf(hi));
                atomicMax(reinterpret_cast<int*>(absmax + bg * D + e), __float_as_int(a));
            }
        }
    }
}

// Any granularity >= 1: one CTA per block, threads over dims, rows in order.
template <int DT>
__global__ void k_meta_generic(const typename Elem<DT>::T* __restrict__ k, int64_t rows, int dim,
                               int blk, typename Elem<DT>::T* __restrict__ meta) {
    const int64_t b = blockIdx.x;
    const int64_t r0 = b * blk;
    const int64_t r1 = min(rows, r0 + blk);
    for (int d = threadIdx.x; d < dim; d += blockDim.x) {
        float mn = Elem<DT>::to_f(k[r0 * dim + d]), mx = mn;
        for (int64_t r = r0 + 1; r < r1; ++r) {
            const float x = Elem<DT>::to_f(k[r * dim + d]);
            mn = fold_min(mn, x);
            mx = fold_max(mx, x);
        }
        meta[(b * 2) * dim + d] = Elem<DT>::from_f(mn);
        meta[(b * 2 + 1) * dim + d] = Elem<DT>::from_f(mx);
    }
}

template <int DT, int D>
void meta_levels_t(const fx_layout& L, const void* k, void* m16, void* m32, void* m64, void* m128,
                   float* absmax, cudaStream_t s) {
    using T = typename Elem<DT>::T;
    const dim3 grid((unsigned)cdiv(L.l_cpu, kSlab), (unsigned)(L.batch * L.kv_heads));
    k_meta_levels<DT, D><<<grid, 256, 0, s>>>(
        static_cast<const T*>(k), L.l_cap, L.l_sink, L.l_cpu, static_cast<T*>(m16),
        static_cast<T*>(m32), static_cast<T*>(m64), static_cast<T*>(m128), absmax);
}

}  // namespace

void launch_meta_levels(const fx_layout& L, const void* k, void* m16, void* m32, void* m64,
                        void* m128, float* absmax, cudaStream_t s) {
    FX_REQUIRE(L.l_cpu > 0, FX_ERR_INVALID, "empty-context: cpu segment is empty");
    if (absmax)
        FX_CUDA(cudaMemsetAsync(absmax, 0, sizeof(float) * L.batch * L.kv_heads * L.head_dim, s));
    const int D = L.head_dim;
    if (L.dtype == FX_BF16 && D == 128) meta_levels_t<FX_BF16, 128>(L, k, m16, m32, m64, m128, absmax, s);
    else if (L.dtype == FX_BF16 && D == 64) meta_levels_t<FX_BF16, 64>(L, k, m16, m32, m64, m128, absmax, s);
    else if (L.dtype == FX_F32 && D == 128) meta_levels_t<FX_F32, 128>(L, k, m16, m32, m64, m128, absmax, s);
    else if (L.dtype == FX_F32 && D == 64) meta_levels_t<FX_F32, 64>(L, k, m16, m32, m64, m128, absmax, s);
    else fail(FX_ERR_INVALID, "bad-shape: batched metadata supports head_dim 64 or 128");
    FX_CUDA(cudaGetLastError());
}

void launch_meta_generic(const void* k, int dtype, int64_t rows, int dim, int blk, void* meta,
                         cudaStream_t s) {
    FX_REQUIRE(blk > 0, FX_ERR_INVALID, "invalid-granularity: block size must be >= 1");
    const int64_t nblk = cdiv(rows, blk);
    if (nblk == 0) return;
    const int threads = dim >= 256 ? 256 : ((dim + 31) / 32) * 32;
    if (dtype == FX_BF16)
        k_meta_generic<FX_BF16><<<(unsigned)nblk, threads, 0, s>>>(
            static_cast<const __nv_bfloat16*>(k), rows, dim, blk, static_cast<__nv_bfloat16*>(meta));
    else
        k_meta_generic<FX_F32><<<(unsigned)nblk, threads, 0, s>>>(
            static_cast<const float*>(k), rows, dim, blk, static_cast<float*>(meta));
    FX_CUDA(cudaGetLastError());
}

}  // namespace fx
