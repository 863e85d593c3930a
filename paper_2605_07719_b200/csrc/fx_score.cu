// fx_score.cu -- K2a: approximate Quest scores of every block of every head,
// the prefilter of the bit-exact selection (fx_topk.cu).
//
// The reference score (block_index.cpp:41-53) is
//     s = sum_d max(q_d * min_d, q_d * max_d) = sum_d q-_d min_d + q+_d max_d
// (q+ = max(q, 0), q- = min(q, 0); exactly one term of each pair is non-zero)
// -- a contraction of the block's [min row | max row] (2*D contiguous values in
// the metadata layout) with [q- ; q+].  For bf16 metadata it runs on the tensor
// cores: S^T[16 blocks x 8 heads] += Meta[16 x 16] . Q[16 x 8] (mma.sync
// m16n8k16, f32 accumulate), all G <= 8 heads of the group in one MMA column
// block, q split into bf16 hi + lo.  The contraction index is permuted so that
// every lane's A fragment for two consecutive k-steps is ONE 16-byte vector load
// straight from global memory (4 lanes cover 64 contiguous bytes of a row):
//     k-step 2p   : a0,a2 <- row[32p + 8t + {0,1}], row[32p + 8t + {2,3}]
//     k-step 2p+1 : a0,a2 <- row[32p + 8t + {4,5}], row[32p + 8t + {6,7}]
// (t = lane % 4), and the B fragment (q) uses the same permutation.
//
// Error bound handed to the selection: |s_approx - s| <= c * sum_d |q_d| absmax_d
// with c = 16 * 2^-24 for the f32 CUDA-core path (at most 13 roundings on any
// path of the summation tree) and c = 2^-14 for the MMA path (bf16 split of q
// leaves <= 2^-16 relative; tensor-core f32 accumulation adds a few ulp per
// MMA over 32 MMAs -- tests/test_gpu_parity.py::test_approx_score_error_bound
// measures the realized ratio, ~1e-6, against this 6e-5 budget).
#include "fx_common.cuh"

namespace fx {
namespace {

constexpr int kTileBlocks = 512;  // blocks per CTA (8 MMA m-tiles per warp)

struct MetaPtrs {
    const void* p[4];
};

__device__ __forceinline__ const void* level_ptr(const void* const* meta, int blk) {
    return meta[blk == 16 ? 0 : blk == 32 ? 1 : blk == 64 ? 2 : 3];
}

// Shared prologue: which (b, g, tile) this CTA scores, or false to exit.
struct TileCtx {
    int bg, b, g, blk;
    int64_t nblk, t0, head0;
};
__device__ __forceinline__ bool tile_ctx(const int32_t* blk_arr, const int32_t* kblocks, int Hkv,
                                         int G, int64_t l_cpu, TileCtx& c) {
    c.bg = blockIdx.y;
    c.b = c.bg / Hkv;
    c.g = c.bg % Hkv;
    c.blk = blk_arr[c.bg];
    if (c.blk <= 0) return false;
    c.nblk = cdiv_dev(l_cpu, c.blk);
    c.t0 = (int64_t)blockIdx.x * kTileBlocks;
    if (c.t0 >= c.nblk) return false;
    c.head0 = (int64_t)c.b * Hkv * G + (int64_t)c.g * G;
    bool any = false;
    for (int h = 0; h < G; ++h) {
        const int32_t kk = kblocks[c.head0 + h];
        any |= (kk > 0 && kk < c.nblk);  // k = 0 or k >= nblk needs no ranking
    }
    return any;
}

// ---------------------------------------------------------------------------
// tensor-core path (bf16 metadata)
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(128) k_approx_scores_mma(MetaPtrs meta,
                                                           const float* __restrict__ q,
                                                           const int32_t* __restrict__ blk_arr,
                                                           const int32_t* __restrict__ kblocks,
                                                           int Hkv, int G, int64_t l_cpu,
                                                           float* __restrict__ approx,
                                                           int64_t stride) {
    pdl_wait();
    pdl_trigger();
    constexpr int KW = 2 * D;   // min row | max row
    constexpr int NP = KW / 32;  // k-step pairs
    TileCtx c;
    if (!tile_ctx(blk_arr, kblocks, Hkv, G, l_cpu, c)) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hq = lane >> 2, t = lane & 3;
    const __nv_bfloat16* base =
        static_cast<const __nv_bfloat16*>(level_ptr(meta.p, c.blk)) + (int64_t)c.bg * c.nblk * KW;

    // B fragments of [q- ; q+] for head hq, permuted like the A loads
    uint32_t bh[NP][4], bl[NP][4];
    {
        const float* qh = q + (c.head0 + (hq < G ? hq : 0)) * D;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            float hi[8], lo[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int col = 32 * p + 8 * t + e;
                const int d = col % D;
                float x = hq < G ? __ldg(qh + d) : 0.f;
                x = col < D ? fminf(x, 0.f) : fmaxf(x, 0.f);
                hi[e] = __bfloat162float(__float2bfloat16_rn(x));
                lo[e] = x - hi[e];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                bh[p][i] = pack_bf16(hi[2 * i], hi[2 * i + 1]);
                bl[p][i] = pack_bf16(lo[2 * i], lo[2 * i + 1]);
            }
        }
    }
    for (int mt = warp; mt < kTileBlocks / 16; mt += 4) {
        const int64_t j0 = c.t0 + mt * 16;
        if (j0 >= c.nblk) break;
        const int64_t r0 = min(j0 + hq, c.nblk - 1), r1 = min(j0 + hq + 8, c.nblk - 1);
        uint4 va[NP], vb[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            va[p] = __ldg(reinterpret_cast<const uint4*>(base + r0 * KW + 32 * p + 8 * t));
            vb[p] = __ldg(reinterpret_cast<const uint4*>(base + r1 * KW + 32 * p + 8 * t));
        }
        float ch[4] = {0.f, 0.f, 0.f, 0.f}, cl[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            mma_bf16_16816(ch, va[p].x, vb[p].x, va[p].y, vb[p].y, bh[p][0], bh[p][1]);
            mma_bf16_16816(cl, va[p].x, vb[p].x, va[p].y, vb[p].y, bl[p][0], bl[p][1]);
            mma_bf16_16816(ch, va[p].z, vb[p].z, va[p].w, vb[p].w, bh[p][2], bh[p][3]);
            mma_bf16_16816(cl, va[p].z, vb[p].z, va[p].w, vb[p].w, bl[p][2], bl[p][3]);
        }
        const int h0 = 2 * t;
        const int64_t ja = j0 + hq, jb = j0 + hq + 8;
        if (h0 < G) {
            if (ja < c.nblk) approx[(c.head0 + h0) * stride + ja] = ch[0] + cl[0];
            if (jb < c.nblk) approx[(c.head0 + h0) * stride + jb] = ch[2] + cl[2];
        }
        if (h0 + 1 < G) {
            if (ja < c.nblk) approx[(c.head0 + h0 + 1) * stride + ja] = ch[1] + cl[1];
            if (jb < c.nblk) approx[(c.head0 + h0 + 1) * stride + jb] = ch[3] + cl[3];
        }
    }
}

// ---------------------------------------------------------------------------
// CUDA-core path (f32 metadata): lanes split the head dimension
// ---------------------------------------------------------------------------
template <int D, int G>
__global__ void __launch_bounds__(256) k_approx_scores_f32(MetaPtrs meta, const float* __restrict__ q,
                                                           const int32_t* __restrict__ blk_arr,
                                                           const int32_t* __restrict__ kblocks,
                                                           int Hkv, int64_t l_cpu,
                                                           float* __restrict__ approx,
                                                           int64_t stride) {
    pdl_wait();
    pdl_trigger();
    constexpr int LPR = D / 4;  // lanes per block row pair (4 dims per lane)
    static_assert(LPR <= 32 && 32 % LPR == 0, "head_dim");
    constexpr int RPW = 32 / LPR;
    constexpr int GP = G <= 1 ? 1 : G <= 2 ? 2 : G <= 4 ? 4 : 8;
    static_assert(GP <= LPR, "group too wide for the lane split");
    TileCtx c;
    if (!tile_ctx(blk_arr, kblocks, Hkv, G, l_cpu, c)) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int col = (lane % LPR) * 4;
    const float* base = static_cast<const float*>(level_ptr(meta.p, c.blk)) + (int64_t)c.bg * c.nblk * 2 * D;
    float qp[G][4], qn[G][4];
#pragma unroll
    for (int h = 0; h < G; ++h) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(q + (c.head0 + h) * D + col));
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            qp[h][i] = fmaxf(vv[i], 0.0f);
            qn[h][i] = fminf(vv[i], 0.0f);
        }
    }
    int my_h = 0;  // head this lane owns after the halving reduction
    {
        int cc = GP;
#pragma unroll
        for (int s = LPR / 2; s >= 1; s >>= 1)
            if (cc > 1) {
                if (lane & s) my_h += cc / 2;
                cc >>= 1;
            }
    }
    const bool writer = (lane % (LPR / GP)) == 0 && my_h < G;
    const int64_t t1 = min(c.nblk, c.t0 + kTileBlocks);
    constexpr int U = 4;
    for (int64_t j0 = c.t0 + warp * RPW * U; j0 < t1; j0 += 8 * RPW * U) {
        float4 mn[U], mx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = j0 + u * RPW + lane / LPR;
            if (j < t1) {
                mn[u] = __ldg(reinterpret_cast<const float4*>(base + j * 2 * D + col));
                mx[u] = __ldg(reinterpret_cast<const float4*>(base + j * 2 * D + D + col));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = j0 + u * RPW + lane / LPR;
            const float a[4] = {mn[u].x, mn[u].y, mn[u].z, mn[u].w};
            const float z[4] = {mx[u].x, mx[u].y, mx[u].z, mx[u].w};
            float v[GP];
#pragma unroll
            for (int h = 0; h < GP; ++h) v[h] = 0.0f;
            if (j < t1) {
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    float s = 0.0f;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        s = fmaf(qp[h][i], z[i], s);
                        s = fmaf(qn[h][i], a[i], s);
                    }
                    v[h] = s;
                }
            }
            int cc = GP;  // halving butterfly: each step hands half the values over
#pragma unroll
            for (int s = LPR / 2; s >= 1; s >>= 1) {
                if (cc > 1) {
                    const bool up = (lane & s) != 0;
#pragma unroll
                    for (int i = 0; i < GP / 2; ++i) {
                        if (i < cc / 2) {
                            const float send = up ? v[i] : v[i + cc / 2];
                            const float keep = up ? v[i + cc / 2] : v[i];
                            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
                        }
                    }
                    cc >>= 1;
                } else {
                    v[0] += __shfl_xor_sync(0xffffffffu, v[0], s);
                }
            }
            if (writer && j < t1) approx[(c.head0 + my_h) * stride + j] = v[0];
        }
    }
}

template <int D>
void launch_f32(const fx_layout& L, MetaPtrs mp, const float* q, const int32_t* blk,
                const int32_t* kblocks, float* approx, int64_t stride, dim3 grid,
                cudaStream_t s) {
#define FX_G(GG)                                                                                \
    case GG:                                                                                    \
        launch_pdl(k_approx_scores_f32<D, GG>, grid, 256, 0, s, mp, q, blk, kblocks, L.kv_heads,       \
                                                        L.l_cpu, approx, stride);               \
        break;
    switch (L.group_size) {
        FX_G(1) FX_G(2) FX_G(3) FX_G(4) FX_G(5) FX_G(6) FX_G(7) FX_G(8)
        default: fail(FX_ERR_INVALID, "bad-shape: group_size must be <= 8");
    }
#undef FX_G
}

}  // namespace

double approx_eps_scale(const fx_layout& L) {
    return L.dtype == FX_BF16 ? 1.0 / 16384.0 : 16.0 / 16777216.0;
}

void launch_approx_scores(const fx_layout& L, const void* const meta[4], const float* q,
                          const int32_t* blk, const int32_t* kblocks, float* approx,
                          int64_t approx_stride, cudaStream_t s) {
    MetaPtrs mp{{meta[0], meta[1], meta[2], meta[3]}};
    const int D = L.head_dim;
    FX_REQUIRE(L.group_size <= 8, FX_ERR_INVALID, "bad-shape: group_size must be <= 8");
    const dim3 grid((unsigned)cdiv(level_blocks(L.l_cpu, 16), kTileBlocks),
                    (unsigned)(L.batch * L.kv_heads));
    if (L.dtype == FX_BF16 && D == 128)
        launch_pdl(k_approx_scores_mma<128>, grid, 128, 0, s, mp, q, blk, kblocks, L.kv_heads, L.group_size,
                                                      L.l_cpu, approx, approx_stride);
    else if (L.dtype == FX_BF16 && D == 64)
        launch_pdl(k_approx_scores_mma<64>, grid, 128, 0, s, mp, q, blk, kblocks, L.kv_heads, L.group_size,
                                                     L.l_cpu, approx, approx_stride);
    else if (L.dtype == FX_F32 && D == 128) launch_f32<128>(L, mp, q, blk, kblocks, approx, approx_stride, grid, s);
    else if (L.dtype == FX_F32 && D == 64) launch_f32<64>(L, mp, q, blk, kblocks, approx, approx_stride, grid, s);
    else fail(FX_ERR_INVALID, "bad-shape: batched scoring supports head_dim 64 or 128");
    FX_CUDA(cudaGetLastError());
}

}  // namespace fx
