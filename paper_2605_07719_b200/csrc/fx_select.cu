// fx_select.cu -- the worklist that turns a group's per-head selections into
// attention boxes, and the per-query reference-API helpers (exact scores,
// ordered top-k).  Scoring lives in fx_score.cu, selection in fx_topk.cu.
#include <algorithm>

#include "fx_common.cuh"

namespace fx {
namespace {

constexpr int kMaxWords = 4096;      // nblk <= 131072 per (b, g) at the chosen blk

// Exclusive block scan of cnt[0..n) in place; returns the total.
__device__ int64_t block_exclusive_scan(int32_t* cnt, int n, int64_t* wsum) {
    const int t = threadIdx.x, nt = blockDim.x;
    const int per = (n + nt - 1) / nt;
    const int a = min(n, t * per), e = min(n, a + per);
    int64_t s = 0;
    for (int i = a; i < e; ++i) s += cnt[i];
    wsum[t] = s;
    __syncthreads();
    if (t < 32) {  // warp scan of the nt partial sums
        int64_t run = 0;
        for (int base = 0; base < nt; base += 32) {
            const int i = base + t;
            const int64_t v = i < nt ? wsum[i] : 0;
            int64_t x = v;
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (t >= o) x += y;
            }
            if (i < nt) wsum[i] = run + x - v;
            run += __shfl_sync(0xffffffffu, x, 31);
        }
        if (t == 0) wsum[nt] = run;
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
                                                  int32_t* __restrict__ done, int stage_words) {
    pdl_wait();
    pdl_trigger();
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
        const uint32_t* hg = sel_bits + ((int64_t)b * Hkv * G + (int64_t)g * G) * sel_words;
        // stage the group's G selection masks in smem (all loads in flight at once)
        extern __shared__ uint32_t s_bits[];
        const bool staged = (int64_t)G * W <= stage_words;
        if (staged) {
#pragma unroll 4
            for (int i = t; i < G * W; i += blockDim.x) s_bits[i] = hg[(int64_t)(i / W) * sel_words + i % W];
            __syncthreads();
        }
        const uint32_t* hb = staged ? s_bits : hg;
        const int64_t hstride = staged ? W : sel_words;
        for (int j = t; j < W; j += blockDim.x) {
            uint32_t u = 0;
            for (int h = 0; h < G; ++h) u |= hb[(int64_t)h * hstride + j];
            int c = __popc(u) * bpb;
            if ((last >> 5) == j && ((u >> (last & 31)) & 1u)) c -= bpb - nb_last;
            wcnt[j] = c;
        }
        __syncthreads();
        total += block_exclusive_scan(wcnt, W, wsum);
        for (int j = warp; j < W; j += blockDim.x / 32) {
            uint32_t u = 0, m = 0;  // union word; head mask of this lane's block
            for (int h = 0; h < G; ++h) {
                const uint32_t w = hb[(int64_t)h * hstride + j];
                u |= w;
                m |= ((w >> lane) & 1u) << h;
            }
            if ((u >> lane) & 1u) {
                const int i = j * 32 + lane;
                const int r0 = i * blk;  // < 2^31 (checked by the launcher)
                const int len = min(blk, (int)(l_cpu - r0));
                const int nb = (len + kBoxRows - 1) >> 4;
                const int64_t o = nd + wcnt[j] + (int64_t)__popc(u & ((1u << lane) - 1u)) * bpb;
                const int row0 = (int)l_sink + r0;
                for (int x = 0; x < nb; ++x) {
                    Box bx;
                    bx.row = row0 + x * kBoxRows;
                    bx.n = (uint16_t)min(kBoxRows, len - x * kBoxRows);
                    bx.mask = (uint16_t)m;
                    out[o + x] = bx;
                }
            }
        }
    }
    if (t == 0) bg_count[bg] = (int32_t)total;
    if (n_bg <= kMaxRunPrefix) return;  // the attention kernels rebuild the run starts from the counts
    __threadfence();
    __syncthreads();
    if (t == 0) s_last = atomicAdd(&done[n_bg], 1) == n_bg - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // last CTA: exclusive prefix of box counts over (b, g)
    for (int i0 = 0, run = 0; i0 < n_bg; i0 += blockDim.x) {
        const int i = i0 + t;
        int v = i < n_bg ? __ldcg(bg_count + i) + kRunPad : 0;  // + virtual run cost
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

void launch_worklist(const fx_layout& L, int64_t l_new, const int32_t* blk,
                     const uint32_t* sel_bits, int sel_words, Box* boxes, int64_t box_stride,
                     int32_t* bg_count, int32_t* bg_start, int32_t* done, cudaStream_t s) {
    FX_REQUIRE(L.group_size <= 16, FX_ERR_INVALID, "bad-shape: group_size must be <= 16");
    const int n_bg = L.batch * L.kv_heads;
    // stage up to 96 KB of selection words per group in smem
    const int64_t want = (int64_t)L.group_size * cdiv(std::max<int64_t>(1, level_blocks(L.l_cpu, 16)), 32);
    const int stage_words = (int)std::min<int64_t>(want, 24576);
    const size_t smem = (size_t)stage_words * 4;
    FX_CUDA(cudaFuncSetAttribute(k_worklist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch_pdl(k_worklist, n_bg, 256, smem, s, L.kv_heads, L.group_size, L.l_sink, L.l_cpu,
                                       L.l_local + l_new, blk, sel_bits, sel_words, boxes, box_stride,
                                       bg_count, bg_start, done, stage_words);
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
