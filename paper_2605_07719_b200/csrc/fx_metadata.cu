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

// Streaming builder: every warp owns whole level-128 blocks (128 rows) and
// walks them in 16-row sub-blocks -- with 16 lanes per row, slot 0 folds rows
// 0..7, slot 1 rows 8..15 (contiguous, so the slot combine keeps the earlier
// rows first) -- keeping the running level-32 / -64 / -128 folds and the
// absmax in registers.  Each warp streams its rows through a private ring of
// 1-D bulk copies (TMA engine, one mbarrier per stage, ~16 KB in flight per
// warp, 128 KB per SM) -- no CTA barrier between loads -- and each level's
// rows leave as one 16-byte store per lane (min from slot 0, max from slot 1).  A CTA covers a
// contiguous range of one (b, g)'s blocks and reduces absmax once per
// dimension (one atomic per dim per CTA).  Optional per-block mean keys
// (f32, sum / rows; north-star item 1, not used by the reference's Quest
// score) come from the same pass.
constexpr int kMW = 8;    // warps per CTA
constexpr int kMB = 16;   // level-128 blocks per warp (the ring's ramp is paid once per warp)
constexpr int kSub = 16;  // rows per sub-block (= level 16)

template <int DT, int D>
struct MetaOut {
    typename Elem<DT>::T* lv[4];  // levels 16 / 32 / 64 / 128: [B*Hkv][nblk][2][D]
    float* mean[4];               // optional per-block means [B*Hkv][nblk][D] (f32)
};

template <int DT, int D, bool MEAN>
__global__ void __launch_bounds__(kMW * 32, 2) k_meta_stream(const typename Elem<DT>::T* __restrict__ k,
                                                          int64_t l_cap, int64_t l_sink, int64_t l_cpu,
                                                          MetaOut<DT, D> out, float* __restrict__ absmax) {
    using T = typename Elem<DT>::T;
    constexpr int V = 16 / Elem<DT>::kBytes;  // elements per 128-bit vector
    constexpr int LPR = D / V;                // lanes per row
    static_assert(LPR >= 1 && LPR <= 32 && (32 % LPR) == 0, "row must fit one warp");
    constexpr int NSLOT = 32 / LPR;           // row slots of the warp
    constexpr int RPS = kSub / NSLOT;         // contiguous rows per slot
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int slot = lane / LPR, col = (lane % LPR) * V;
    const int64_t bg = blockIdx.y;
    const T* kb = k + (bg * l_cap + l_sink) * D;
    const int64_t n16 = cdiv_dev(l_cpu, 16), n32 = cdiv_dev(l_cpu, 32), n64 = cdiv_dev(l_cpu, 64),
                  n128 = cdiv_dev(l_cpu, 128);
    const int64_t nlev[4] = {n16, n32, n64, n128};
    constexpr bool want_mean = MEAN;
    float amax[V];
#pragma unroll
    for (int j = 0; j < V; ++j) amax[j] = 0.f;
    // this warp's level-128 blocks: kMB consecutive ones of the CTA's range
    const int64_t jb0 = ((int64_t)blockIdx.x * kMW + warp) * kMB;
    const int nsub = (int)max((int64_t)0, min((int64_t)kMB * 8, cdiv_dev(l_cpu - jb0 * 128, kSub)));
    // this warp's bulk-copy ring: NST sub-blocks of kSub rows in flight
    constexpr int SB = kSub * D * (int)sizeof(T);
    constexpr int NST = SB >= 4096 ? 2 : 8192 / SB;
    extern __shared__ __align__(128) unsigned char msm[];
    T* ring = reinterpret_cast<T*>(msm) + (size_t)warp * NST * kSub * D;
    __shared__ __align__(8) uint64_t s_full[kMW][16];
    uint64_t* full = s_full[warp];
    auto issue = [&](int sidx) {  // lane 0: rows of sub-block sidx -> stage sidx % NST
        const int64_t r0 = jb0 * 128 + (int64_t)sidx * kSub;
        const int rows = (int)min((int64_t)kSub, l_cpu - r0);
        const int st = sidx % NST;
        fence_proxy_async();  // the stage's previous rows were read through the generic proxy
        mbar_arrive_expect_tx(&full[st], (uint32_t)(rows * D * sizeof(T)));
        bulk_g2s(ring + (size_t)st * kSub * D, kb + r0 * D, (uint32_t)(rows * D * sizeof(T)), &full[st]);
    };
    if (lane == 0) {
        for (int i = 0; i < NST; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
        for (int i = 0; i < NST && i < nsub; ++i) issue(i);
    }
    __syncwarp();
    float m32[2][V], m64[2][V], m128[2][V];  // running folds (min, max)
    float s32[V], s64[V], s128[V];           // running sums (means)
    auto emit = [&](int lvl, int64_t jl, const float* lo, const float* hi, const float* sum, int rows_per) {
        if (jl >= nlev[lvl]) return;
        T* dst = out.lv[lvl] + (bg * nlev[lvl] + jl) * 2 * D + col;
        if (NSLOT == 1) {  // one lane per vector: both rows
            *reinterpret_cast<uint4*>(dst) = pack16<DT>(lo);
            *reinterpret_cast<uint4*>(dst + D) = pack16<DT>(hi);
        } else if (slot < 2) {  // slot 0 the min row, slot 1 the max row
            *reinterpret_cast<uint4*>(dst + slot * D) = pack16<DT>(slot == 0 ? lo : hi);
        }
        if (MEAN && slot == 0) {
            const float n = (float)min((int64_t)rows_per, l_cpu - jl * rows_per);
            float4* md = reinterpret_cast<float4*>(out.mean[lvl] + (bg * nlev[lvl] + jl) * D + col);
#pragma unroll
            for (int j = 0; j < V; j += 4) md[j / 4] = make_float4(sum[j] / n, sum[j + 1] / n, sum[j + 2] / n, sum[j + 3] / n);
        }
    };
    // one sub-block: fold this slot's RPS rows in order, combine the slots in
    // row order, emit level 16 and carry the level 32 / 64 / 128 folds
    auto process = [&](int si) {
        const int st = si % NST;
        mbar_wait(&full[st], (uint32_t)((si / NST) & 1));
        const T* rw = ring + (size_t)st * kSub * D + (size_t)(slot * RPS) * D + col;
        float mn[V], mx[V], sm[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            mn[j] = __int_as_float(0x7f800000);
            mx[j] = -__int_as_float(0x7f800000);
            sm[j] = 0.f;
        }
        const int64_t rbase = jb0 * 128 + (int64_t)si * kSub + slot * RPS;
#pragma unroll
        for (int i = 0; i < RPS; ++i) {
            if (rbase + i < l_cpu) {
                float x[V];
                unpack16<DT>(*reinterpret_cast<const uint4*>(rw + (size_t)i * D), x);
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    mn[j] = fold_min(mn[j], x[j]);
                    mx[j] = fold_max(mx[j], x[j]);
                    if (MEAN) sm[j] += x[j];
                }
            }
        }
#pragma unroll
        for (int step = LPR; step < 32; step <<= 1) {  // slots in row order: the lower slot is earlier
            const bool lower = ((lane / step) & 1) == 0;
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const float pmn = __shfl_xor_sync(0xffffffffu, mn[j], step);
                const float pmx = __shfl_xor_sync(0xffffffffu, mx[j], step);
                mn[j] = lower ? fold_min(mn[j], pmn) : fold_min(pmn, mn[j]);
                mx[j] = lower ? fold_max(mx[j], pmx) : fold_max(pmx, mx[j]);
                if (MEAN) {
                    const float psm = __shfl_xor_sync(0xffffffffu, sm[j], step);
                    sm[j] = lower ? sm[j] + psm : psm + sm[j];
                }
            }
        }
        const int64_t j16 = jb0 * 8 + si;
        emit(0, j16, mn, mx, sm, 16);
        const int q32 = si & 1, q64 = si & 3, q128 = si & 7;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            m32[0][j] = q32 ? fold_min(m32[0][j], mn[j]) : mn[j];
            m32[1][j] = q32 ? fold_max(m32[1][j], mx[j]) : mx[j];
            if (MEAN) s32[j] = q32 ? s32[j] + sm[j] : sm[j];
        }
        if (q32 == 1 || si + 1 == nsub) {
            emit(1, j16 >> 1, m32[0], m32[1], s32, 32);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                m64[0][j] = (q64 >> 1) ? fold_min(m64[0][j], m32[0][j]) : m32[0][j];
                m64[1][j] = (q64 >> 1) ? fold_max(m64[1][j], m32[1][j]) : m32[1][j];
                if (MEAN) s64[j] = (q64 >> 1) ? s64[j] + s32[j] : s32[j];
            }
            if (q64 == 3 || si + 1 == nsub) {
                emit(2, j16 >> 2, m64[0], m64[1], s64, 64);
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    m128[0][j] = (q128 >> 2) ? fold_min(m128[0][j], m64[0][j]) : m64[0][j];
                    m128[1][j] = (q128 >> 2) ? fold_max(m128[1][j], m64[1][j]) : m64[1][j];
                    if (MEAN) s128[j] = (q128 >> 2) ? s128[j] + s64[j] : s64[j];
                }
                if (q128 == 7 || si + 1 == nsub) {
                    emit(3, j16 >> 3, m128[0], m128[1], s128, 128);
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        amax[j] = fmaxf(amax[j], fmaxf(fabsf(m128[0][j]), fabsf(m128[1][j])));
                }
            }
        }
    };
    for (int si = 0; si < nsub; ++si) {
        process(si);
        __syncwarp();  // every lane has read the stage
        if (lane == 0 && si + NST < nsub) issue(si + NST);
    }
    // absmax: fold the two slots, then the CTA's warps, one atomic per dim
    __shared__ float s_amax[kMW][D];
#pragma unroll
    for (int step = LPR; step < 32; step <<= 1)
#pragma unroll
        for (int j = 0; j < V; ++j) amax[j] = fmaxf(amax[j], __shfl_xor_sync(0xffffffffu, amax[j], step));
    if (slot == 0)
#pragma unroll
        for (int j = 0; j < V; ++j) s_amax[warp][col + j] = amax[j];
    __syncthreads();
    if (absmax)
        for (int d = threadIdx.x; d < D; d += blockDim.x) {
            float a = 0.f;
#pragma unroll
            for (int w = 0; w < kMW; ++w) a = fmaxf(a, s_amax[w][d]);
            if (a > 0.f) atomicMax(reinterpret_cast<int*>(absmax + bg * D + d), __float_as_int(a));
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
void meta_levels_t(const fx_layout& L, const void* k, void* const lv[4], float* const mean[4], float* absmax,
                   cudaStream_t s) {
    using T = typename Elem<DT>::T;
    MetaOut<DT, D> out;
    for (int i = 0; i < 4; ++i) {
        out.lv[i] = static_cast<T*>(lv[i]);
        out.mean[i] = mean ? mean[i] : nullptr;
    }
    const int64_t n128 = cdiv(L.l_cpu, 128);
    const dim3 grid((unsigned)cdiv(n128, kMW * kMB), (unsigned)(L.batch * L.kv_heads));
    constexpr int SB = kSub * D * (int)sizeof(T);
    constexpr int NST = SB >= 4096 ? 2 : 8192 / SB;
    const size_t smem = (size_t)kMW * NST * SB;
    auto kern = mean ? k_meta_stream<DT, D, true> : k_meta_stream<DT, D, false>;
    FX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, kMW * 32, smem, s>>>(static_cast<const T*>(k), L.l_cap, L.l_sink, L.l_cpu, out, absmax);
}

}  // namespace

void launch_meta_levels(const fx_layout& L, const void* k, void* m16, void* m32, void* m64,
                        void* m128, float* absmax, cudaStream_t s, float* const mean[4]) {
    FX_REQUIRE(L.l_cpu > 0, FX_ERR_INVALID, "empty-context: cpu segment is empty");
    if (mean) {
        bool all = true, none = true;
        for (int i = 0; i < 4; ++i) {
            all = all && mean[i] != nullptr;
            none = none && mean[i] == nullptr;
        }
        FX_REQUIRE(all || none, FX_ERR_INVALID, "bad-shape: per-block means need all four levels or none");
        if (none) mean = nullptr;
    }
    if (absmax)
        FX_CUDA(cudaMemsetAsync(absmax, 0, sizeof(float) * L.batch * L.kv_heads * L.head_dim, s));
    void* const lv[4] = {m16, m32, m64, m128};
    const int D = L.head_dim;
    if (L.dtype == FX_BF16 && D == 128) meta_levels_t<FX_BF16, 128>(L, k, lv, mean, absmax, s);
    else if (L.dtype == FX_BF16 && D == 64) meta_levels_t<FX_BF16, 64>(L, k, lv, mean, absmax, s);
    else if (L.dtype == FX_F32 && D == 128) meta_levels_t<FX_F32, 128>(L, k, lv, mean, absmax, s);
    else if (L.dtype == FX_F32 && D == 64) meta_levels_t<FX_F32, 64>(L, k, lv, mean, absmax, s);
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
