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
#include <algorithm>

#include "fx_common.cuh"

namespace fx {
namespace {


#ifdef FX_TRACE  // profiling build only: per-CTA phase times of the TMA scorer
__device__ long long g_score_trace[8 * 512];
__device__ __forceinline__ long long stimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SC_MARK(i) g_score_trace[blockIdx.x * 8 + (i)] = stimer();
#else
#define SC_MARK(i)
#endif

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
                                         int G, int64_t l_cpu, TileCtx& c, int rank_all, int tile) {
    c.bg = blockIdx.y;
    c.b = c.bg / Hkv;
    c.g = c.bg % Hkv;
    c.blk = blk_arr[c.bg];
    if (c.blk <= 0) return false;
    c.nblk = cdiv_dev(l_cpu, c.blk);
    c.t0 = (int64_t)blockIdx.x * tile;
    if (c.t0 >= c.nblk) return false;
    c.head0 = (int64_t)c.b * Hkv * G + (int64_t)c.g * G;
    bool any = false;
    for (int h = 0; h < G; ++h) {
        const int32_t kk = kblocks[c.head0 + h];
        any |= (kk > 0 && (rank_all || kk < c.nblk));  // k = 0 or k >= nblk needs no ranking
    }
    return any;
}

// ---------------------------------------------------------------------------
// tensor-core path (bf16 metadata): TMA-fed, warp-specialized, persistent
// ---------------------------------------------------------------------------
// Work item: 64 consecutive blocks (metadata rows) of one (b, g) = one 3-D
// TMA box {64 columns, 64 rows, 2D/64 chunks} with 128-byte swizzle (32 KB
// at D = 128), the same row-box layout the attention kernel streams K with.
// One CTA per SM: a producer warp walks the CTA's contiguous range of the
// flattened item sequence (only groups that need ranking) issuing one TMA per
// item into a kSStages ring; 4 consumer warps take 16 rows each:
// S^T[16 blocks x 8 heads] = Meta[16 x 2D] . [q- ; q+] (ldmatrix + mma.sync
// m16n8k16, f32 accumulate, q split into bf16 hi + lo).
constexpr int kSRows = 64;
constexpr int kSStages = 5;
constexpr int kSCWarps = 4;
constexpr int kSThreads = (kSCWarps + 1) * 32;
constexpr int kMaxScoreGroups = 4096;

struct MetaMaps {
    CUtensorMap lvl[4];  // blk 16 / 32 / 64 / 128
};

struct ItemHdr {
    int32_t bg, j0, n, end;
};

template <int D>
struct ScoreCfg {
    static constexpr int RB = 2 * D * 2;       // bytes of one [min | max] row
    static constexpr int NCH = RB / 128;       // 128-byte chunks per row
    static constexpr int STAGE = kSRows * RB;  // one box
    static constexpr int NT = 2 * D / 16;      // k-steps
    static constexpr size_t HDR = (size_t)kSStages * STAGE;
    static constexpr size_t BAR = HDR + kSStages * sizeof(ItemHdr);
    static constexpr size_t PREF = BAR + 2 * kSStages * sizeof(uint64_t);
    static constexpr size_t BLK = PREF + (kMaxScoreGroups + 1) * sizeof(int);
    static constexpr size_t TOTAL = BLK + kMaxScoreGroups * sizeof(int) + 1024;
};

__device__ __forceinline__ int level_of(int blk) { return blk == 16 ? 0 : blk == 32 ? 1 : blk == 64 ? 2 : 3; }

// items of group bg (0: streaming, or no head needs ranking); blk and the
// G per-head k load together (one round trip)
__device__ __forceinline__ int group_items(const int32_t* blk_arr, const int32_t* kblocks, int bg,
                                           int G, int64_t l_cpu, int* blk_out, int rank_all) {
    int32_t kk[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) kk[h] = h < G ? __ldg(kblocks + (int64_t)bg * G + h) : 0;
    const int blk = __ldg(blk_arr + bg);
    *blk_out = blk;
    if (blk <= 0) return 0;
    const int64_t nblk = cdiv_dev(l_cpu, blk);
    bool any = false;
#pragma unroll
    for (int h = 0; h < 8; ++h) any |= (kk[h] > 0 && (rank_all || kk[h] < nblk));  // k = 0 or >= nblk: no ranking
    return any ? (int)cdiv_dev(nblk, kSRows) : 0;
}

template <int D>
__global__ void __launch_bounds__(kSThreads, 1) k_score_tma(
    const __grid_constant__ MetaMaps maps, const float* __restrict__ q,
    const int32_t* __restrict__ blk_arr, const int32_t* __restrict__ kblocks, int n_bg, int G,
    int64_t l_cpu, float* __restrict__ approx, int64_t stride, int rank_all) {
    if (threadIdx.x == kSCWarps * 32)  // descriptors: independent of the preceding kernels
        for (int l = 0; l < 4; ++l) tma_prefetch_desc(&maps.lvl[l]);
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) { SC_MARK(0) }
    using C = ScoreCfg<D>;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    ItemHdr* hdr = reinterpret_cast<ItemHdr*>(smem + C::HDR);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR);
    uint64_t* empty = full + kSStages;
    int* s_pref = reinterpret_cast<int*>(smem + C::PREF);
    int* s_blk = reinterpret_cast<int*>(smem + C::BLK);
    __shared__ int s_wsum[kSThreads / 32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int NW = kSThreads / 32;
    // exclusive prefix of items over the groups
    int carry = 0;
    for (int c0 = 0; c0 < n_bg; c0 += kSThreads) {
        const int i = c0 + tid;
        int bv = 0;
        const int v = i < n_bg ? group_items(blk_arr, kblocks, i, G, l_cpu, &bv, rank_all) : 0;
        if (i < n_bg) s_blk[i] = bv;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_wsum[warp] = x;
        __syncthreads();
        int off = carry, tot = 0;
        for (int w = 0; w < NW; ++w) {
            if (w < warp) off += s_wsum[w];
            tot += s_wsum[w];
        }
        if (i < n_bg) s_pref[i] = off + x - v;
        __syncthreads();
        carry += tot;
    }
    if (tid == 0) {
        s_pref[n_bg] = carry;
        for (int i = 0; i < kSStages; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, kSCWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t total = carry;
    const int64_t i0 = total * blockIdx.x / gridDim.x, i1 = total * (blockIdx.x + 1) / gridDim.x;

    if (warp == kSCWarps) {
        // ------------------------------ producer ------------------------------
        if (lane == 0) {
            SC_MARK(1)
            int st = 0;
            uint32_t ph = 0;
            int bg = 0, cur = -1, lvl = 0;
            int64_t nblk = 0;
            if (i0 < i1) {
                int lo = 0, hi = n_bg - 1;  // last group with s_pref[bg] <= i0
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_pref[mid] <= i0) lo = mid;
                    else hi = mid - 1;
                }
                bg = lo;
            }
            for (int64_t it = i0; it < i1; ++it) {
                while (s_pref[bg + 1] <= it) ++bg;
                if (bg != cur) {
                    cur = bg;
                    const int blk = s_blk[bg];
                    lvl = level_of(blk);
                    nblk = cdiv_dev(l_cpu, blk);
                }
                const int64_t j0 = (it - s_pref[bg]) * kSRows;
                mbar_wait(empty + st, ph ^ 1u);
                ItemHdr& H = hdr[st];
                H.bg = bg;
                H.j0 = (int32_t)j0;
                H.n = (int32_t)(nblk - j0 < kSRows ? nblk - j0 : kSRows);
                H.end = 0;
                mbar_arrive_expect_tx(full + st, (uint32_t)C::STAGE);
                tma_load_3d(smem + (size_t)st * C::STAGE, &maps.lvl[lvl], full + st, 0,
                            (int)((int64_t)bg * nblk + j0), 0);
                if (++st == kSStages) {
                    st = 0;
                    ph ^= 1u;
                }
            }
            SC_MARK(4)
#ifdef FX_TRACE
            g_score_trace[blockIdx.x * 8 + 5] = i1 - i0;
#endif
            mbar_wait(empty + st, ph ^ 1u);
            hdr[st].end = 1;
            mbar_arrive(full + st);
        }
        return;
    }

    // ------------------------------- consumers -------------------------------
    constexpr int NT = C::NT;
    const int hq = lane >> 2, tq = lane & 3;
    uint32_t bh[NT][2], bl[NT][2];
    int cur = -1;
    int64_t head0 = 0;
    int st = 0;
    uint32_t ph = 0;
    const int r = (lane & 7) + ((lane >> 3) & 1) * 8;
    int first_bg = -1;  // the CTA's first group: its q fragments load while the first box is in flight
    if (i0 < i1) {
        int lo = 0, hi = n_bg - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_pref[mid] <= i0) lo = mid;
            else hi = mid - 1;
        }
        while (s_pref[lo + 1] <= i0) ++lo;
        first_bg = lo;
    }
    while (true) {
        int want = first_bg;
        ItemHdr H;
        if (want < 0) {
            mbar_wait(full + st, ph);
            H = hdr[st];
            if (H.end) break;
            want = H.bg;
        }
        if (want != cur) {  // B fragments of [q- ; q+] for head hq of the group
            cur = want;
            head0 = (int64_t)cur * G;
            const float* qh = q + (head0 + (hq < G ? hq : 0)) * D;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                float x[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int col = 16 * j + 2 * tq + (e & 1) + (e >> 1) * 8;
                    float v = hq < G ? __ldg(qh + (col % D)) : 0.f;
                    x[e] = col < D ? fminf(v, 0.f) : fmaxf(v, 0.f);
                }
                const float h0 = __bfloat162float(__float2bfloat16_rn(x[0]));
                const float h1 = __bfloat162float(__float2bfloat16_rn(x[1]));
                const float h2 = __bfloat162float(__float2bfloat16_rn(x[2]));
                const float h3 = __bfloat162float(__float2bfloat16_rn(x[3]));
                bh[j][0] = pack_bf16(h0, h1);
                bh[j][1] = pack_bf16(h2, h3);
                bl[j][0] = pack_bf16(x[0] - h0, x[1] - h1);
                bl[j][1] = pack_bf16(x[2] - h2, x[3] - h3);
            }
        }
        if (first_bg >= 0) {  // prefetched; now wait for the first box
            first_bg = -1;
            mbar_wait(full + st, ph);
            if (tid == 0) { SC_MARK(2) }
            H = hdr[st];
            if (H.end) break;
            if (H.bg != cur) continue;  // (cannot happen: same range arithmetic)
        }
        if (warp * 16 < H.n) {
            const uint32_t ka = smem_u32(smem + (size_t)st * C::STAGE) + warp * 16 * 128;
            float ch[4] = {0.f, 0.f, 0.f, 0.f}, cl[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int u = ((j & 3) << 1) + (lane >> 4);
                const uint32_t off = r * 128 + ((u ^ (r & 7)) << 4);
                uint32_t a0, a1, a2, a3;
                ldsm_x4(ka + (j >> 2) * (kSRows * 128) + off, a0, a1, a2, a3);
                mma_bf16_16816(ch, a0, a1, a2, a3, bh[j][0], bh[j][1]);
                mma_bf16_16816(cl, a0, a1, a2, a3, bl[j][0], bl[j][1]);
            }
            const int h0 = 2 * tq;
            const int ra = warp * 16 + hq, rb = ra + 8;
            const int64_t ja = H.j0 + ra, jb = H.j0 + rb;
            if (h0 < G) {
                if (ra < H.n) approx[(head0 + h0) * stride + ja] = ch[0] + cl[0];
                if (rb < H.n) approx[(head0 + h0) * stride + jb] = ch[2] + cl[2];
            }
            if (h0 + 1 < G) {
                if (ra < H.n) approx[(head0 + h0 + 1) * stride + ja] = ch[1] + cl[1];
                if (rb < H.n) approx[(head0 + h0 + 1) * stride + jb] = ch[3] + cl[3];
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
        if (++st == kSStages) {
            st = 0;
            ph ^= 1u;
        }
    }
    if (tid == 0) { SC_MARK(3) }
}

// ---------------------------------------------------------------------------
// CUDA-core path (f32 metadata): lanes split the head dimension
// ---------------------------------------------------------------------------
// f32 scorer tile: one pass of the CTA's 8 warps (U = 4 rows per lane group),
// so a batch-1 layer's few groups still spread over many SMs
template <int D>
constexpr int kTileF32 = 8 * (32 / (D / 4)) * 4;

template <int D, int G>
__global__ void __launch_bounds__(256) k_approx_scores_f32(MetaPtrs meta, const float* __restrict__ q,
                                                           const int32_t* __restrict__ blk_arr,
                                                           const int32_t* __restrict__ kblocks,
                                                           int Hkv, int64_t l_cpu,
                                                           float* __restrict__ approx,
                                                           int64_t stride, int rank_all) {
    pdl_wait();
    pdl_trigger();
    constexpr int LPR = D / 4;  // lanes per block row pair (4 dims per lane)
    static_assert(LPR <= 32 && 32 % LPR == 0, "head_dim");
    constexpr int RPW = 32 / LPR;
    constexpr int GP = G <= 1 ? 1 : G <= 2 ? 2 : G <= 4 ? 4 : 8;
    static_assert(GP <= LPR, "group too wide for the lane split");
    TileCtx c;
    if (!tile_ctx(blk_arr, kblocks, Hkv, G, l_cpu, c, rank_all, kTileF32<D>)) return;
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
    const int64_t t1 = min(c.nblk, c.t0 + kTileF32<D>);
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
                cudaStream_t s, int rank_all) {
#define FX_G(GG)                                                                                \
    case GG:                                                                                    \
        launch_pdl(k_approx_scores_f32<D, GG>, grid, 256, 0, s, mp, q, blk, kblocks, L.kv_heads,       \
                                                        L.l_cpu, approx, stride, rank_all);     \
        break;
    switch (L.group_size) {
        FX_G(1) FX_G(2) FX_G(3) FX_G(4) FX_G(5) FX_G(6) FX_G(7) FX_G(8)
        default: fail(FX_ERR_INVALID, "bad-shape: group_size must be <= 8");
    }
#undef FX_G
}

template <int D>
void launch_score_tma(const fx_layout& L, const void* const meta[4], const float* q,
                      const int32_t* blk, const int32_t* kblocks, float* approx, int64_t stride,
                      int num_sms, cudaStream_t s, int rank_all) {
    const int n_bg = L.batch * L.kv_heads;
    FX_REQUIRE(n_bg <= kMaxScoreGroups, FX_ERR_INVALID, "bad-shape: more than 4096 (b, g) groups");
    MetaMaps maps;
    for (int l = 0; l < 4; ++l) {
        const int64_t rows = (int64_t)n_bg * level_blocks(L.l_cpu, kLevels[l]);
        maps.lvl[l] = make_row_map(meta[l], 2 * D, std::max<int64_t>(rows, kSRows), kSRows);
    }
    const size_t smem = ScoreCfg<D>::TOTAL;
    FX_CUDA(cudaFuncSetAttribute(k_score_tma<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch_pdl(k_score_tma<D>, (unsigned)std::max(1, num_sms), kSThreads, smem, s, maps, q, blk,
               kblocks, n_bg, L.group_size, L.l_cpu, approx, stride, rank_all);
}

}  // namespace

double approx_eps_scale(const fx_layout& L) {
    return L.dtype == FX_BF16 ? 1.0 / 16384.0 : 16.0 / 16777216.0;
}

void launch_approx_scores(const fx_layout& L, const void* const meta[4], const float* q,
                          const int32_t* blk, const int32_t* kblocks, float* approx,
                          int64_t approx_stride, int num_sms, cudaStream_t s, bool rank_all) {
    MetaPtrs mp{{meta[0], meta[1], meta[2], meta[3]}};
    const int D = L.head_dim;
    FX_REQUIRE(L.group_size <= 8, FX_ERR_INVALID, "bad-shape: group_size must be <= 8");
    const int n_bg = L.batch * L.kv_heads;
    if (L.dtype == FX_BF16 && D == 128)
        launch_score_tma<128>(L, meta, q, blk, kblocks, approx, approx_stride, num_sms, s, rank_all);
    else if (L.dtype == FX_BF16 && D == 64)
        launch_score_tma<64>(L, meta, q, blk, kblocks, approx, approx_stride, num_sms, s, rank_all);
    else if (L.dtype == FX_F32 && D == 128)
        launch_f32<128>(L, mp, q, blk, kblocks, approx, approx_stride,
                        dim3((unsigned)cdiv(level_blocks(L.l_cpu, 16), kTileF32<128>), (unsigned)n_bg), s, rank_all);
    else if (L.dtype == FX_F32 && D == 64)
        launch_f32<64>(L, mp, q, blk, kblocks, approx, approx_stride,
                       dim3((unsigned)cdiv(level_blocks(L.l_cpu, 16), kTileF32<64>), (unsigned)n_bg), s, rank_all);
    else fail(FX_ERR_INVALID, "bad-shape: batched scoring supports head_dim 64 or 128");
    FX_CUDA(cudaGetLastError());
}

#ifdef FX_TRACE
extern "C" FX_API int fx_debug_score_trace(long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_score_trace, sizeof(long long) * n) == cudaSuccess ? 0 : -2;
}
#endif

}  // namespace fx
