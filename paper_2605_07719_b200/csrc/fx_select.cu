// fx_select.cu -- K2: Quest block scoring and budgeted top-k selection,
// block_index.cpp:41-83, bit-exact against the reference.
//
// The reference ranks blocks by an f64 score summed in dimension order over
// exact f32 x f32 products (block_score) with ties to the lower block id.
// Doing that f64 work for every block would make the scan FP64-bound, so the
// selection is two-phase:
//
//  1. k_approx_scores: a streaming, 128-bit-coalesced pass over the group's
//     metadata at its planned granularity computes f32 scores for all G heads
//     (warp lanes split the head dimension; the reduction order is free
//     because only a bound is needed).  |s32 - s64| <= eps with
//         eps = 16 * 2^-24 * sum_d |q_d| * absmax_d     (+ tiny)
//     (at most 13 roundings on any path of the summation tree, each of
//     relative size <= 2^-24 of the partial sums, which are bounded by
//     sum_d |q_d * sel_d| <= sum_d |q_d| absmax_d).
//  2. k_select (one CTA per head): radix-select the k-th largest f32 score
//     A_k.  Blocks with s32 > A_k + 2 eps are in the reference top-k for
//     sure, blocks with s32 < A_k - 2 eps are out for sure; the few blocks
//     in between are re-scored with the reference's exact f64 recipe
//     (sequential d, unfused) and ranked by (score desc, id asc).
//
// Output is a per-head bitmask over blocks; k_worklist turns the union of a
// group's masks into 16-row boxes with per-box head masks for K3.
#include <algorithm>

#include "fx_common.cuh"

namespace fx {
namespace {

constexpr int kSelThreads = 512;
constexpr int kMaxWords = 4096;      // nblk <= 131072 per (b, g) at the chosen blk
constexpr int kSmemKeys = 24576;     // approx scores staged in smem up to this many blocks
constexpr int kSmallCand = 1024;     // candidates ranked in smem by counting

template <int DT>
__device__ __forceinline__ void load4(const typename Elem<DT>::T* p, float* out);
template <>
__device__ __forceinline__ void load4<FX_BF16>(const __nv_bfloat16* p, float* out) {
    const uint2 w = __ldg(reinterpret_cast<const uint2*>(p));
    out[0] = bf16lo_to_f(w.x);
    out[1] = bf16hi_to_f(w.x);
    out[2] = bf16lo_to_f(w.y);
    out[3] = bf16hi_to_f(w.y);
}
template <>
__device__ __forceinline__ void load4<FX_F32>(const float* p, float* out) {
    const float4 w = __ldg(reinterpret_cast<const float4*>(p));
    out[0] = w.x;
    out[1] = w.y;
    out[2] = w.z;
    out[3] = w.w;
}

__device__ __forceinline__ const void* level_ptr(const void* const* meta, int blk) {
    return meta[blk == 16 ? 0 : blk == 32 ? 1 : blk == 64 ? 2 : 3];
}

struct MetaPtrs {
    const void* p[4];
};

// ---------------------------------------------------------------------------
// phase 1: approximate f32 scores
// ---------------------------------------------------------------------------
constexpr int kTileBlocks = 128;

template <int DT, int D, int G>
__global__ void __launch_bounds__(256) k_approx_scores(MetaPtrs meta, const float* __restrict__ q,
                                                       const int32_t* __restrict__ blk_arr,
                                                       const int32_t* __restrict__ kblocks,
                                                       int Hkv, int64_t l_cpu,
                                                       float* __restrict__ approx,
                                                       int64_t stride) {
    using T = typename Elem<DT>::T;
    constexpr int LPR = D / 4;  // lanes per metadata row pair (4 dims per lane)
    static_assert(LPR <= 32 && 32 % LPR == 0, "head_dim");
    constexpr int RPW = 32 / LPR;
    constexpr int GP = G <= 1 ? 1 : G <= 2 ? 2 : G <= 4 ? 4 : 8;
    static_assert(GP <= LPR, "group too wide for the lane split");
    const int bg = blockIdx.y;
    const int b = bg / Hkv, g = bg % Hkv;
    const int blk = blk_arr[bg];
    if (blk <= 0) return;
    const int64_t nblk = cdiv_dev(l_cpu, blk);
    const int64_t t0 = (int64_t)blockIdx.x * kTileBlocks;
    if (t0 >= nblk) return;
    const int64_t H = (int64_t)Hkv * G;
    const int64_t head0 = (int64_t)b * H + (int64_t)g * G;
    bool any = false;
#pragma unroll
    for (int h = 0; h < G; ++h) {
        const int32_t kk = kblocks[head0 + h];
        any |= (kk > 0 && kk < nblk);
    }
    if (!any) return;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int col = (lane % LPR) * 4;
    const T* base = static_cast<const T*>(level_ptr(meta.p, blk)) + (int64_t)bg * nblk * 2 * D;
    float qp[G][4], qn[G][4];
#pragma unroll
    for (int h = 0; h < G; ++h) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(q + (head0 + h) * D + col));
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            qp[h][i] = fmaxf(vv[i], 0.0f);
            qn[h][i] = fminf(vv[i], 0.0f);
        }
    }
    // head owned by this lane after the halving reduction
    int my_h = 0;
    {
        int c = GP;
#pragma unroll
        for (int s = LPR / 2; s >= 1; s >>= 1)
            if (c > 1) {
                if (lane & s) my_h += c / 2;
                c >>= 1;
            }
    }
    const bool writer = (lane % (LPR / GP)) == 0 && my_h < G;
    const int64_t t1 = min(nblk, t0 + kTileBlocks);
    constexpr int U = 4;
    for (int64_t j0 = t0 + warp * RPW * U; j0 < t1; j0 += 8 * RPW * U) {
        float mn[U][4], mx[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = j0 + u * RPW + lane / LPR;
            if (j < t1) {
                load4<DT>(base + j * 2 * D + col, mn[u]);
                load4<DT>(base + j * 2 * D + D + col, mx[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = j0 + u * RPW + lane / LPR;
            float v[GP];
#pragma unroll
            for (int h = 0; h < GP; ++h) v[h] = 0.0f;
            if (j < t1) {
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    float s = 0.0f;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        s = fmaf(qp[h][i], mx[u][i], s);
                        s = fmaf(qn[h][i], mn[u][i], s);
                    }
                    v[h] = s;
                }
            }
            // halving butterfly: each step hands half of the values to the partner
            int c = GP;
#pragma unroll
            for (int s = LPR / 2; s >= 1; s >>= 1) {
                if (c > 1) {
                    const bool up = (lane & s) != 0;
#pragma unroll
                    for (int i = 0; i < GP / 2; ++i) {
                        if (i < c / 2) {
                            const float send = up ? v[i] : v[i + c / 2];
                            const float keep = up ? v[i + c / 2] : v[i];
                            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
                        }
                    }
                    c >>= 1;
                } else {
                    v[0] += __shfl_xor_sync(0xffffffffu, v[0], s);
                }
            }
            if (writer && j < t1) approx[(head0 + my_h) * stride + j] = v[0];
        }
    }
}

// ---------------------------------------------------------------------------
// phase 2: selection
// ---------------------------------------------------------------------------

// Exact reference score (block_index.cpp:41-53): f64, dimension order, unfused.
template <typename T>
__device__ double exact_score(const float* __restrict__ q, const T* __restrict__ mn,
                              const T* __restrict__ mx, int D) {
    double s = 0.0;
    for (int d = 0; d < D; ++d) {
        const double qd = (double)q[d];
        const double lo = __dmul_rn(qd, (double)tofl(mn[d]));
        const double hi = __dmul_rn(qd, (double)tofl(mx[d]));
        s = __dadd_rn(s, (lo < hi) ? hi : lo);
    }
    return s;
}

// Find digit `d` such that (#keys with larger digit) < rem <= (#keys with digit >= d).
__device__ __forceinline__ void find_digit(const uint32_t* hist, int64_t rem, int* out) {
    const int lane = threadIdx.x & 31;
    uint32_t loc[8];
    uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        loc[i] = hist[lane * 8 + i];
        t += loc[i];
    }
    uint32_t incl = t;  // sum over lanes >= lane (descending digit order)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_down_sync(0xffffffffu, incl, o);
        if (lane + o < 32) incl += v;
    }
    const uint32_t excl = incl - t;
    if ((int64_t)excl < rem && rem <= (int64_t)incl) {
        uint32_t above = excl;
#pragma unroll
        for (int i = 7; i >= 0; --i) {
            if ((int64_t)(above + loc[i]) >= rem) {
                out[0] = lane * 8 + i;
                out[1] = (int)above;
                break;
            }
            above += loc[i];
        }
    }
}

// Block-wide radix select: kth-largest (1-based) 32-bit key of `n` keys
// produced by key_of(i).  Returns the key; *gt = #keys strictly greater.
template <class KeyOf>
__device__ uint32_t radix_kth32(int64_t n, int64_t kth, KeyOf key_of, uint32_t* hist, int* sh,
                                int64_t* gt) {
    uint32_t prefix = 0, mask = 0;
    int64_t rem = kth, above_total = 0;
    const int lane = threadIdx.x & 31;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int64_t i0 = 0; i0 < n; i0 += blockDim.x) {
            const int64_t i = i0 + threadIdx.x;
            const bool act = i < n;
            const uint32_t key = act ? key_of(i) : 0u;
            const bool match = act && (key & mask) == prefix;
            const uint32_t dig = (key >> shift) & 255u;
            const uint32_t m = __match_any_sync(0xffffffffu, match ? dig : 0x100u);
            if (match && lane == __ffs(m) - 1) atomicAdd(&hist[dig], (uint32_t)__popc(m));
        }
        __syncthreads();
        if (threadIdx.x < 32) find_digit(hist, rem, sh);
        __syncthreads();
        const int d = sh[0];
        const int ab = sh[1];
        prefix |= (uint32_t)d << shift;
        mask |= 255u << shift;
        rem -= ab;
        above_total += ab;
        __syncthreads();
    }
    *gt = above_total;
    return prefix;
}

template <class KeyOf>
__device__ uint64_t radix_kth64(int64_t n, int64_t kth, KeyOf key_of, uint32_t* hist, int* sh,
                                int64_t* gt) {
    uint64_t prefix = 0, mask = 0;
    int64_t rem = kth, above_total = 0;
    const int lane = threadIdx.x & 31;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int64_t i0 = 0; i0 < n; i0 += blockDim.x) {
            const int64_t i = i0 + threadIdx.x;
            const bool act = i < n;
            const uint64_t key = act ? key_of(i) : 0ull;
            const bool match = act && (key & mask) == prefix;
            const uint32_t dig = (uint32_t)(key >> shift) & 255u;
            const uint32_t m = __match_any_sync(0xffffffffu, match ? dig : 0x100u);
            if (match && lane == __ffs(m) - 1) atomicAdd(&hist[dig], (uint32_t)__popc(m));
        }
        __syncthreads();
        if (threadIdx.x < 32) find_digit(hist, rem, sh);
        __syncthreads();
        prefix |= (uint64_t)sh[0] << shift;
        mask |= 255ull << shift;
        rem -= sh[1];
        above_total += sh[1];
        __syncthreads();
    }
    *gt = above_total;
    return prefix;
}

// Exclusive block scan of cnt[0..n) in place (n <= kMaxWords); returns total.
__device__ int64_t block_exclusive_scan(int32_t* cnt, int n, int64_t* wsum) {
    const int t = threadIdx.x, nt = blockDim.x;
    const int per = (n + nt - 1) / nt;
    const int a = min(n, t * per), e = min(n, a + per);
    int64_t s = 0;
    for (int i = a; i < e; ++i) s += cnt[i];
    wsum[t] = s;
    __syncthreads();
    if (t == 0) {
        int64_t run = 0;
        for (int i = 0; i < nt; ++i) {
            const int64_t v = wsum[i];
            wsum[i] = run;
            run += v;
        }
        wsum[nt] = run;
    }
    __syncthreads();
    int64_t run = wsum[t];
    for (int i = a; i < e; ++i) {
        const int32_t v = cnt[i];
        cnt[i] = (int32_t)run;
        run += v;
    }
    __syncthreads();
    return wsum[nt];
}

template <int DT>
__global__ void __launch_bounds__(kSelThreads) k_select(
    MetaPtrs meta, const float* __restrict__ absmax, const float* __restrict__ q,
    const int32_t* __restrict__ blk_arr, const int32_t* __restrict__ kblocks, int Hkv, int G,
    int D, int64_t l_cpu, const float* __restrict__ approx, int64_t astride,
    uint32_t* __restrict__ sel_bits, int sel_words, uint64_t* __restrict__ cand_keys,
    uint32_t* __restrict__ cand_ids, int64_t cand_stride) {
    using T = typename Elem<DT>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* s_keys = reinterpret_cast<float*>(smem_raw);  // [kSmemKeys] when staged
    __shared__ uint32_t hist[256];
    __shared__ int sh[4];
    __shared__ int32_t wcnt[kMaxWords];
    __shared__ int64_t wsum[kSelThreads + 1];
    __shared__ uint64_t ck[kSmallCand];
    __shared__ uint32_t ci[kSmallCand];
    __shared__ double s_eps;
    __shared__ unsigned long long s_ndef;

    const int64_t head = blockIdx.x;
    const int64_t H = (int64_t)Hkv * G;
    const int b = (int)(head / H), h = (int)(head % H), g = h / G;
    const int bg = b * Hkv + g;
    const int blk = blk_arr[bg];
    const int64_t k = kblocks[head];
    uint32_t* bits = sel_bits + head * sel_words;
    const int64_t nblk = blk > 0 ? cdiv_dev(l_cpu, blk) : 0;
    const int W = (int)cdiv_dev(nblk, 32);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = kSelThreads / 32;

    if (nblk == 0 || k <= 0) {
        for (int j = t; j < W; j += kSelThreads) bits[j] = 0u;
        return;
    }
    if (k >= nblk) {  // clamp: every block (block_index.cpp:61-64)
        for (int j = t; j < W; j += kSelThreads) {
            const int64_t rem = nblk - (int64_t)j * 32;
            bits[j] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
        }
        return;
    }
    const T* mbase = static_cast<const T*>(level_ptr(meta.p, blk)) + (int64_t)bg * nblk * 2 * D;
    const float* qh = q + head * D;
    const float* sc = approx + head * astride;
    const bool staged = nblk <= kSmemKeys;
    if (staged)
        for (int64_t i = t; i < nblk; i += kSelThreads) s_keys[i] = sc[i];
    if (warp == 0) {  // error bound of the f32 prefilter
        double a = 0.0;
        for (int d = lane; d < D; d += 32) a += fabs((double)qh[d]) * (double)absmax[(int64_t)bg * D + d];
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) {
            s_eps = a * (16.0 * 1.01 / 16777216.0) + 1e-30;
            s_ndef = 0;
        }
    }
    __syncthreads();
    const float* src = staged ? s_keys : sc;
    int64_t gt_unused;
    const uint32_t tkey =
        radix_kth32(nblk, k, [&](int64_t i) { return f32_key(src[i]); }, hist, sh, &gt_unused);
    const double ak = (double)key_f32(tkey);
    const double eps = s_eps;
    const bool sane = isfinite(ak) && isfinite(eps);
    const double hi = ak + 2.0 * eps, lo = ak - 2.0 * eps;

    // classify: definite-in bits now, candidate masks to smem
    for (int j = warp; j < W; j += nwarps) {
        const int64_t i = (int64_t)j * 32 + lane;
        const bool in = i < nblk;
        const double a = in ? (double)src[i] : 0.0;
        const bool fin = isfinite(a);
        const bool def = in && sane && fin && a > hi;
        const bool cand = in && !def && (!sane || !fin || a >= lo);
        const uint32_t bd = __ballot_sync(0xffffffffu, def);
        const uint32_t bc = __ballot_sync(0xffffffffu, cand);
        if (lane == 0) {
            bits[j] = bd;
            wcnt[j] = __popc(bc);
            if (bd) atomicAdd(&s_ndef, (unsigned long long)__popc(bd));
        }
        // stash candidate mask in the (unused) tail of hist-sized scratch: recompute later
    }
    __syncthreads();
    const int64_t n_def = (int64_t)s_ndef;
    const int64_t n_cand = block_exclusive_scan(wcnt, W, wsum);
    const int64_t need = k - n_def;
    // compact candidate ids in ascending id order
    uint32_t* cids = cand_ids + head * cand_stride;
    uint64_t* ckeys = cand_keys + head * cand_stride;
    for (int j = warp; j < W; j += nwarps) {
        const int64_t i = (int64_t)j * 32 + lane;
        const bool in = i < nblk;
        const double a = in ? (double)src[i] : 0.0;
        const bool fin = isfinite(a);
        const bool def = in && sane && fin && a > hi;
        const bool cand = in && !def && (!sane || !fin || a >= lo);
        const uint32_t bc = __ballot_sync(0xffffffffu, cand);
        if (cand) {
            const int64_t pos = wcnt[j] + __popc(bc & ((1u << lane) - 1u));
            if (n_cand <= kSmallCand) ci[pos] = (uint32_t)i;
            else cids[pos] = (uint32_t)i;
        }
    }
    __syncthreads();
    if (n_cand <= kSmallCand) {
        for (int64_t c = t; c < n_cand; c += kSelThreads) {
            const uint32_t id = ci[c];
            ck[c] = f64_key(exact_score<T>(qh, mbase + (int64_t)id * 2 * D, mbase + (int64_t)id * 2 * D + D, D));
        }
        __syncthreads();
        for (int64_t c = t; c < n_cand; c += kSelThreads) {
            const uint64_t kc = ck[c];
            const uint32_t idc = ci[c];
            int64_t rank = 0;
            for (int64_t j = 0; j < n_cand; ++j) {
                const uint64_t kj = ck[j];
                rank += (kj > kc) || (kj == kc && ci[j] < idc);
            }
            if (rank < need) atomicOr(&bits[idc >> 5], 1u << (idc & 31));
        }
    } else {
        for (int64_t c = t; c < n_cand; c += kSelThreads) {
            const uint32_t id = cids[c];
            ckeys[c] = f64_key(exact_score<T>(qh, mbase + (int64_t)id * 2 * D, mbase + (int64_t)id * 2 * D + D, D));
        }
        __syncthreads();
        int64_t gt = 0;
        const uint64_t t64 = radix_kth64(n_cand, need, [&](int64_t i) { return ckeys[i]; }, hist, sh, &gt);
        __syncthreads();
        for (int64_t c = t; c < n_cand; c += kSelThreads)
            if (ckeys[c] > t64) atomicOr(&bits[cids[c] >> 5], 1u << (cids[c] & 31));
        if (t == 0) {  // ties at the threshold: lowest ids first (block_index.cpp:71)
            int64_t take = need - gt;
            for (int64_t c = 0; c < n_cand && take > 0; ++c)
                if (ckeys[c] == t64) {
                    atomicOr(&bits[cids[c] >> 5], 1u << (cids[c] & 31));
                    --take;
                }
        }
    }
}

// ---------------------------------------------------------------------------
// worklist: union of the group's selections -> 16-row boxes with head masks
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_worklist(int Hkv, int G, int64_t l_sink, int64_t l_cpu,
                                                  int64_t l_tail, const int32_t* __restrict__ blk_arr,
                                                  const uint32_t* __restrict__ sel_bits,
                                                  int sel_words, Box* __restrict__ boxes,
                                                  int64_t box_stride,
                                                  int32_t* __restrict__ bg_count,
                                                  int32_t* __restrict__ bg_start,
                                                  int32_t* __restrict__ done) {
    __shared__ int32_t wcnt[kMaxWords];
    __shared__ int64_t wsum[257];
    __shared__ int s_last;
    __shared__ int wtot[8];
    const int bg = blockIdx.x, n_bg = gridDim.x;
    const int b = bg / Hkv, g = bg % Hkv;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int blk = blk_arr[bg];
    const uint16_t all = (uint16_t)((1u << G) - 1u);
    Box* out = boxes + (int64_t)bg * box_stride;
    // defaults: sink, then local + decoded rows (attention.cpp:143-151)
    const int nb_s = (int)cdiv_dev(l_sink, kBoxRows);
    const int nb_t = (int)cdiv_dev(l_tail, kBoxRows);
    for (int i = t; i < nb_s + nb_t; i += blockDim.x) {
        Box bx;
        if (i < nb_s) {
            bx.row = i * kBoxRows;
            bx.n = (uint16_t)min((int64_t)kBoxRows, l_sink - (int64_t)i * kBoxRows);
        } else {
            const int r = i - nb_s;
            bx.row = (int32_t)(l_sink + l_cpu + (int64_t)r * kBoxRows);
            bx.n = (uint16_t)min((int64_t)kBoxRows, l_tail - (int64_t)r * kBoxRows);
        }
        bx.mask = all;
        out[i] = bx;
    }
    const int nd = nb_s + nb_t;
    int64_t total = nd;
    if (blk > 0) {
        const int64_t nblk = cdiv_dev(l_cpu, blk);
        const int W = (int)cdiv_dev(nblk, 32);
        const int bpb = blk / kBoxRows;
        const int64_t last = nblk - 1;
        const int nb_last = (int)cdiv_dev(l_cpu - last * blk, kBoxRows);
        const uint32_t* hb = sel_bits + ((int64_t)b * Hkv * G + (int64_t)g * G) * sel_words;
        for (int j = t; j < W; j += blockDim.x) {
            uint32_t u = 0;
            for (int h = 0; h < G; ++h) u |= hb[(int64_t)h * sel_words + j];
            int c = __popc(u) * bpb;
            if ((last >> 5) == j && ((u >> (last & 31)) & 1u)) c -= bpb - nb_last;
            wcnt[j] = c;
        }
        __syncthreads();
        total += block_exclusive_scan(wcnt, W, wsum);
        for (int j = warp; j < W; j += blockDim.x / 32) {
            uint32_t u = 0;
            uint32_t hw[16];
            for (int h = 0; h < G; ++h) {
                hw[h] = hb[(int64_t)h * sel_words + j];
                u |= hw[h];
            }
            if ((u >> lane) & 1u) {
                const int64_t i = (int64_t)j * 32 + lane;
                uint16_t m = 0;
                for (int h = 0; h < G; ++h) m |= (uint16_t)(((hw[h] >> lane) & 1u) << h);
                const int64_t r0 = i * blk;
                const int64_t len = min((int64_t)blk, l_cpu - r0);
                const int nb = (int)cdiv_dev(len, kBoxRows);
                const int64_t o = nd + wcnt[j] + (int64_t)__popc(u & ((1u << lane) - 1u)) * bpb;
                for (int x = 0; x < nb; ++x) {
                    Box bx;
                    bx.row = (int32_t)(l_sink + r0 + x * kBoxRows);
                    bx.n = (uint16_t)min((int64_t)kBoxRows, len - (int64_t)x * kBoxRows);
                    bx.mask = m;
                    out[o + x] = bx;
                }
            }
        }
    }
    if (t == 0) bg_count[bg] = (int32_t)total;
    __threadfence();
    __syncthreads();
    if (t == 0) s_last = atomicAdd(&done[n_bg], 1) == n_bg - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // last CTA: exclusive prefix of box counts over (b, g)
    for (int i0 = 0, run = 0; i0 < n_bg; i0 += blockDim.x) {
        const int i = i0 + t;
        int v = i < n_bg ? __ldcg(bg_count + i) : 0;
        // block inclusive scan of v
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wtot[warp] = x;
        __syncthreads();
        int wo = 0;
        for (int w = 0; w < warp; ++w) wo += wtot[w];
        int ctot = 0;
        for (int w = 0; w < 8; ++w) ctot += wtot[w];
        if (i < n_bg) bg_start[i] = run + wo + x - v;
        run += ctot;
        __syncthreads();
        if (i0 + (int)blockDim.x >= n_bg && t == 0) bg_start[n_bg] = run;
    }
}

// ---------------------------------------------------------------------------
// per-query API helpers
// ---------------------------------------------------------------------------
template <int DT>
__global__ void k_exact_scores(const float* __restrict__ q, const typename Elem<DT>::T* __restrict__ meta,
                               int64_t nblk, int D, double* __restrict__ scores) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nblk) scores[i] = exact_score(q, meta + i * 2 * D, meta + i * 2 * D + D, D);
}

// keys (exact score) and ids of every block, padded to `cap` with sentinels
template <int DT>
__global__ void k_score_keys(const float* __restrict__ q, const typename Elem<DT>::T* __restrict__ meta,
                             int64_t nblk, int D, uint64_t* __restrict__ keys,
                             uint32_t* __restrict__ ids, int64_t cap) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cap) return;
    if (i < nblk) {
        keys[i] = f64_key(exact_score(q, meta + i * 2 * D, meta + i * 2 * D + D, D));
        ids[i] = (uint32_t)i;
    } else {
        keys[i] = 0;  // below every finite key
        ids[i] = 0xffffffffu;
    }
}

template <int DT>
__global__ void k_meta_absmax(const typename Elem<DT>::T* __restrict__ meta, int64_t nblk, int D,
                              float* __restrict__ absmax) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= D) return;
    float a = 0.f;
    for (int64_t b = 0; b < 2 * nblk; ++b) a = fmaxf(a, fabsf(tofl(meta[b * D + d])));
    absmax[d] = a;
}

// (key desc, id asc) "less" = comes first
__device__ __forceinline__ bool first_of(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return ka != kb ? ka > kb : ia < ib;
}
__global__ void k_bitonic(uint64_t* keys, uint32_t* ids, int64_t n, int64_t j, int64_t kk) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t p = i ^ j;
    if (i >= n || p <= i) return;
    const bool up = (i & kk) == 0;
    const uint64_t a = keys[i], c = keys[p];
    const uint32_t ia = ids[i], ic = ids[p];
    const bool swap = up ? first_of(c, ic, a, ia) : first_of(a, ia, c, ic);
    if (swap) {
        keys[i] = c;
        keys[p] = a;
        ids[i] = ic;
        ids[p] = ia;
    }
}

}  // namespace

template <int DT, int D>
static void approx_dispatch_g(const fx_layout& L, MetaPtrs mp, const float* q, const int32_t* blk,
                              const int32_t* kblocks, float* approx, int64_t stride,
                              cudaStream_t s) {
    const dim3 grid((unsigned)cdiv(level_blocks(L.l_cpu, 16), kTileBlocks),
                    (unsigned)(L.batch * L.kv_heads));
#define FX_G(GG)                                                                              \
    case GG:                                                                                  \
        k_approx_scores<DT, D, GG><<<grid, 256, 0, s>>>(mp, q, blk, kblocks, L.kv_heads,    \
                                                        L.l_cpu, approx, stride);             \
        break;
    switch (L.group_size) {
        FX_G(1) FX_G(2) FX_G(3) FX_G(4) FX_G(5) FX_G(6) FX_G(7) FX_G(8)
        default: fail(FX_ERR_INVALID, "bad-shape: group_size must be <= 8");
    }
#undef FX_G
}

void launch_approx_scores(const fx_layout& L, const void* const meta[4], const float* q,
                          const int32_t* blk, const int32_t* kblocks, float* approx,
                          int64_t approx_stride, cudaStream_t s) {
    MetaPtrs mp{{meta[0], meta[1], meta[2], meta[3]}};
    const int D = L.head_dim;
    if (L.dtype == FX_BF16 && D == 128) approx_dispatch_g<FX_BF16, 128>(L, mp, q, blk, kblocks, approx, approx_stride, s);
    else if (L.dtype == FX_BF16 && D == 64) approx_dispatch_g<FX_BF16, 64>(L, mp, q, blk, kblocks, approx, approx_stride, s);
    else if (L.dtype == FX_F32 && D == 128) approx_dispatch_g<FX_F32, 128>(L, mp, q, blk, kblocks, approx, approx_stride, s);
    else if (L.dtype == FX_F32 && D == 64) approx_dispatch_g<FX_F32, 64>(L, mp, q, blk, kblocks, approx, approx_stride, s);
    else fail(FX_ERR_INVALID, "bad-shape: batched scoring supports head_dim 64 or 128");
    FX_CUDA(cudaGetLastError());
}

void launch_select(const fx_layout& L, const void* const meta[4], const float* absmax,
                   const float* q, const int32_t* blk, const int32_t* kblocks,
                   const float* approx, int64_t approx_stride, uint32_t* sel_bits, int sel_words,
                   uint64_t* cand_keys, uint32_t* cand_ids, cudaStream_t s) {
    MetaPtrs mp{{meta[0], meta[1], meta[2], meta[3]}};
    FX_REQUIRE(level_blocks(L.l_cpu, 16) <= (int64_t)kMaxWords * 32, FX_ERR_INVALID,
               "bad-shape: cpu segment too long for one selection CTA");
    const int64_t heads = (int64_t)L.batch * L.kv_heads * L.group_size;
    const int64_t nmax = level_blocks(L.l_cpu, 16);
    const size_t smem = (size_t)std::min<int64_t>(nmax, kSmemKeys) * sizeof(float);
    if (L.dtype == FX_BF16) {
        FX_CUDA(cudaFuncSetAttribute(k_select<FX_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_select<FX_BF16><<<(unsigned)heads, kSelThreads, smem, s>>>(
            mp, absmax, q, blk, kblocks, L.kv_heads, L.group_size, L.head_dim, L.l_cpu, approx,
            approx_stride, sel_bits, sel_words, cand_keys, cand_ids, approx_stride);
    } else {
        FX_CUDA(cudaFuncSetAttribute(k_select<FX_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_select<FX_F32><<<(unsigned)heads, kSelThreads, smem, s>>>(
            mp, absmax, q, blk, kblocks, L.kv_heads, L.group_size, L.head_dim, L.l_cpu, approx,
            approx_stride, sel_bits, sel_words, cand_keys, cand_ids, approx_stride);
    }
    FX_CUDA(cudaGetLastError());
}

void launch_worklist(const fx_layout& L, int64_t l_new, const int32_t* blk,
                     const uint32_t* sel_bits, int sel_words, Box* boxes, int64_t box_stride,
                     int32_t* bg_count, int32_t* bg_start, int32_t* done, cudaStream_t s) {
    FX_REQUIRE(L.group_size <= 16, FX_ERR_INVALID, "bad-shape: group_size must be <= 16");
    const int n_bg = L.batch * L.kv_heads;
    k_worklist<<<n_bg, 256, 0, s>>>(L.kv_heads, L.group_size, L.l_sink, L.l_cpu,
                                    L.l_local + l_new, blk, sel_bits, sel_words, boxes, box_stride,
                                    bg_count, bg_start, done);
    FX_CUDA(cudaGetLastError());
}

void launch_exact_scores(const float* q, const void* meta, int dtype, int64_t nblk, int dim,
                         double* scores, cudaStream_t s) {
    if (nblk <= 0) return;
    const unsigned grid = (unsigned)cdiv(nblk, 128);
    if (dtype == FX_BF16)
        k_exact_scores<FX_BF16><<<grid, 128, 0, s>>>(q, static_cast<const __nv_bfloat16*>(meta), nblk, dim, scores);
    else
        k_exact_scores<FX_F32><<<grid, 128, 0, s>>>(q, static_cast<const float*>(meta), nblk, dim, scores);
    FX_CUDA(cudaGetLastError());
}

void launch_topk_exact(const float* q, const void* meta, int dtype, int64_t nblk, int dim,
                       int64_t k, uint32_t* blocks_out, uint64_t* tmp_keys, uint32_t* tmp_ids,
                       int64_t cap, cudaStream_t s) {
    if (k <= 0 || nblk <= 0) return;
    const unsigned grid = (unsigned)cdiv(cap, 256);
    if (dtype == FX_BF16)
        k_score_keys<FX_BF16><<<grid, 256, 0, s>>>(q, static_cast<const __nv_bfloat16*>(meta), nblk, dim, tmp_keys, tmp_ids, cap);
    else
        k_score_keys<FX_F32><<<grid, 256, 0, s>>>(q, static_cast<const float*>(meta), nblk, dim, tmp_keys, tmp_ids, cap);
    FX_CUDA(cudaGetLastError());
    for (int64_t kk = 2; kk <= cap; kk <<= 1)
        for (int64_t j = kk >> 1; j > 0; j >>= 1) k_bitonic<<<grid, 256, 0, s>>>(tmp_keys, tmp_ids, cap, j, kk);
    FX_CUDA(cudaGetLastError());
    FX_CUDA(cudaMemcpyAsync(blocks_out, tmp_ids, sizeof(uint32_t) * std::min(k, nblk), cudaMemcpyDeviceToDevice, s));
}

void launch_meta_absmax(const void* meta, int dtype, int64_t nblk, int dim, float* absmax,
                        cudaStream_t s) {
    const unsigned grid = (unsigned)cdiv(dim, 128);
    if (dtype == FX_BF16)
        k_meta_absmax<FX_BF16><<<grid, 128, 0, s>>>(static_cast<const __nv_bfloat16*>(meta), nblk, dim, absmax);
    else
        k_meta_absmax<FX_F32><<<grid, 128, 0, s>>>(static_cast<const float*>(meta), nblk, dim, absmax);
    FX_CUDA(cudaGetLastError());
}

}  // namespace fx
