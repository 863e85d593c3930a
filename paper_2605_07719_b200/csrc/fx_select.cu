// fx_select.cu -- the worklist that turns a group's per-head selections into
// attention boxes, and the per-query reference-API helpers (exact scores,
// ordered top-k).  Scoring lives in fx_score.cu, selection in fx_topk.cu.
#include <algorithm>

#include "fx_worklist.cuh"

namespace fx {
namespace {

constexpr int kMaxWords = 4096;      // nblk <= 131072 per (b, g) at the chosen blk

// ---------------------------------------------------------------------------
// worklist: union of the group's selections -> 16-row boxes with head masks.
// Standalone only when no k_select ran this step (given selection / empty cpu
// segment); otherwise the selection kernel's fused tail builds the boxes.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_worklist(WorklistArgs w) {
    pdl_wait();
    pdl_trigger();
    __shared__ int32_t wcnt[kMaxWords];
    __shared__ int64_t wsum[257];
    worklist_group(w, blockIdx.x, wcnt, wsum);
    worklist_publish(w, gridDim.x);
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
                     int32_t* bg_count, int32_t* bg_start, int32_t* done, cudaStream_t s,
                     const UnitQueue& uq) {
    FX_REQUIRE(L.group_size <= 16, FX_ERR_INVALID, "bad-shape: group_size must be <= 16");
    const int n_bg = L.batch * L.kv_heads;
    const WorklistArgs w{L.kv_heads, L.group_size, L.l_sink, L.l_cpu, L.l_local + l_new, blk, sel_bits,
                         sel_words, boxes, box_stride, bg_count, bg_start, done + n_bg, uq};
    launch_pdl(k_worklist, n_bg, 256, 0, s, w);
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
