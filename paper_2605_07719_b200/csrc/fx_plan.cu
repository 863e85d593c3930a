// fx_plan.cu -- K5: the granularity-budget selector and the head-property
// predictor, on device.
//
//   budget_at / volume / plan_group   selector.cpp:9-46  (Eq. 1, Eq. 3)
//   blocks_for_budget                  block_index.cpp:96-103
//   forward / predict                  predictor.cpp:161-185
//
// All f64 arithmetic uses explicit round-to-nearest intrinsics (__dmul_rn,
// __dadd_rn, ...) in the reference's operation order: the reference host
// build has no FMA (no -march), and contraction would move results by an
// ulp, which can flip k = ceil(.) at a boundary.
#include "fx_common.cuh"
#include "fx_selector_math.h"

namespace fx {
namespace {

using sel::budget_at;
using sel::clamp01;
__device__ __forceinline__ double volume_of(int blk, int64_t l_cpu, double clamped_sum) {
    return sel::volume_from_sum(blk, l_cpu, clamped_sum);
}
__device__ __forceinline__ int32_t blocks_for_budget(double budget, int64_t l_cpu, int blk) {
    return (int32_t)sel::blocks_for_budget(budget, l_cpu, blk);
}

// Sequential (head-order) sum of clamped budgets across the warp's G lanes.
__device__ __forceinline__ double seq_sum(double v, int G) {
    double s = 0.0;
    for (int h = 0; h < G; ++h) s = __dadd_rn(s, clamp01(__shfl_sync(0xffffffffu, v, h)));
    return s;
}

// One warp per (b, g): plan the group, derive per-head k, reset the step's
// per-group completion counter.
__global__ void k_prepare(int n_bg, int G, int64_t l_cpu, int mode, int fixed_blk,
                          double fixed_budget, const double* __restrict__ bgt0,
                          const double* __restrict__ kslope, const int32_t* __restrict__ streaming,
                          int32_t* __restrict__ blk_out, double* __restrict__ budgets,
                          double* __restrict__ volume, double* __restrict__ cand,
                          int32_t* __restrict__ kblocks, int32_t* __restrict__ bg_done,
                          AppendArgs ap, int32_t* __restrict__ err) {
    pdl_wait();
    pdl_trigger();
    const int bg = blockIdx.x;
    const int h = threadIdx.x;
    // fused append_new of the previous step's token (row ap.row of (b, g)): its
    // loads are issued with the head-property loads, its stores go out last
    constexpr int kAppendPerLane = 8;  // D <= 256
    float ak[kAppendPerLane], av[kAppendPerLane];
    if (ap.kn) {
#pragma unroll
        for (int j = 0; j < kAppendPerLane; ++j) {
            const int d = h + 32 * j;
            ak[j] = d < ap.D ? ap.kn[(int64_t)bg * ap.D + d] : 0.f;
            av[j] = d < ap.D ? ap.vn[(int64_t)bg * ap.D + d] : 0.f;
        }
    }
    const bool act = h < G;
    const int64_t head = (int64_t)bg * G + h;
    if (h == 0 && bg_done) {
        bg_done[bg] = 0;                 // attention contributors of (b, g)
        bg_done[n_bg + 1 + bg] = 0;      // selected heads of (b, g) (fused worklist)
        if (bg == 0) bg_done[n_bg] = 0;  // worklist publish counter
    }
    int blk = 0;
    double bud = 0.0, vol = 0.0, cv[4] = {0, 0, 0, 0};
    if (mode == FX_PLAN_PROPS) {
        const double b0 = act ? bgt0[head] : 0.0;
        const double ks = act ? kslope[head] : 0.0;
        const int st = act ? (streaming[head] != 0) : 1;
        const bool all_streaming = __all_sync(0xffffffffu, st != 0);
        if (!all_streaming) {  // plan_group, selector.cpp:21-46
            double best = 0.0;
            for (int c = 0; c < 4; ++c) {
                const int cb = 16 << c;
                const double b = budget_at(b0, ks, st, cb);
                const double v = volume_of(cb, l_cpu, seq_sum(b, G));
                cv[c] = v;
                if (blk == 0 || v <= best) {  // ties go to the larger blk
                    best = v;
                    blk = cb;
                    bud = b;
                }
            }
            vol = best;
        }
    } else if (mode == FX_PLAN_FIXED || mode == FX_PLAN_FULL) {
        const bool full = mode == FX_PLAN_FULL;
        blk = full ? 128 : fixed_blk;
        bud = full ? 1.0 : fixed_budget;
        const double s = seq_sum(bud, G);
        if (full) {  // pipeline.cpp:298-303
            vol = __dmul_rn(2.0, (double)l_cpu);
            for (int c = 0; c < 4; ++c) cv[c] = vol;
        } else {  // pipeline.cpp:304-311
            vol = volume_of(blk, l_cpu, s);
            for (int c = 0; c < 4; ++c) cv[c] = volume_of(16 << c, l_cpu, s);
        }
    } else {  // FX_PLAN_GIVEN
        blk = blk_out[bg];
        // a caller's block size outside {0} u kCandidateBlocks (selector.hpp:12) has no
        // metadata level: the group falls back to its resident defaults (blk 0) and the
        // ctx error word reports invalid-granularity at the next fx_ctx_synchronize
        if (blk != 0 && blk != 16 && blk != 32 && blk != 64 && blk != 128) {
            if (h == 0 && err) atomicExch(err, 1);
            blk = 0;
        }
        bud = act ? budgets[head] : 0.0;
        if (blk > 0) vol = volume_of(blk, l_cpu, seq_sum(bud, G));
    }
    __syncwarp();  // every lane has read blk_out[bg] before lane 0 rewrites it
    if (h == 0) {
        if (mode != FX_PLAN_GIVEN || blk == 0) blk_out[bg] = blk;
        if (volume) volume[bg] = vol;
        if (cand)
            for (int c = 0; c < 4; ++c) cand[bg * 4 + c] = cv[c];
    }
    if (act) {
        if (mode != FX_PLAN_GIVEN) budgets[head] = bud;
        if (kblocks) kblocks[head] = blk > 0 ? blocks_for_budget(bud, l_cpu, blk) : 0;
    }
    if (ap.kn) {
        const int64_t o = ((int64_t)bg * ap.l_cap + ap.row) * ap.D;
#pragma unroll
        for (int j = 0; j < kAppendPerLane; ++j) {
            const int d = h + 32 * j;
            if (d >= ap.D) break;
            if (ap.bf16) {
                static_cast<__nv_bfloat16*>(ap.k)[o + d] = __float2bfloat16_rn(ak[j]);
                static_cast<__nv_bfloat16*>(ap.v)[o + d] = __float2bfloat16_rn(av[j]);
            } else {
                static_cast<float*>(ap.k)[o + d] = ak[j];
                static_cast<float*>(ap.v)[o + d] = av[j];
            }
        }
    }
}

__global__ void k_blocks_for_budget(int n, const double* __restrict__ budgets,
                                    const int32_t* __restrict__ blk, int64_t l_cpu,
                                    int32_t* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = blocks_for_budget(budgets[i], l_cpu, blk[i]);
}

// predictor.cpp:40-53 linear_forward (bias-first, sequential, unfused) with
// weights stored transposed [in][out] so that thread o reads coalesced.
__device__ __forceinline__ double linear_row(const double* __restrict__ wt, double bias,
                                             const double* a, int in, int out, int o) {
    double s = bias;
    for (int i = 0; i < in; ++i) s = __dadd_rn(s, __dmul_rn(a[i], wt[(int64_t)i * out + o]));
    return s;
}

constexpr int kF = 41, kH1 = 256, kH2 = 384;

// One CTA (384 threads) per feature row: normalize -> 41->256->384->3.
__global__ void __launch_bounds__(384) k_predict(const double* __restrict__ w1t,
                                                 const double* __restrict__ b1,
                                                 const double* __restrict__ w2t,
                                                 const double* __restrict__ b2,
                                                 const double* __restrict__ w3t,
                                                 const double* __restrict__ b3,
                                                 const double* __restrict__ mu,
                                                 const double* __restrict__ sigma,
                                                 const double* __restrict__ feats,
                                                 double* __restrict__ bgt0, double* __restrict__ kslope,
                                                 int32_t* __restrict__ streaming,
                                                 double* __restrict__ zout) {
    __shared__ double x[kF], a1[kH1], a2[kH2];
    const int r = blockIdx.x, t = threadIdx.x;
    if (t < kF) {  // features.cpp:226-233
        const double sg = sigma[t];
        x[t] = sg > 0.0 ? __ddiv_rn(__dsub_rn(feats[(int64_t)r * kF + t], mu[t]), sg) : 0.0;
    }
    __syncthreads();
    if (t < kH1) {
        const double s = linear_row(w1t, b1[t], x, kF, kH1, t);
        a1[t] = s > 0.0 ? s : 0.0;
    }
    __syncthreads();
    {
        const double s = linear_row(w2t, b2[t], a1, kH1, kH2, t);
        a2[t] = s > 0.0 ? s : 0.0;
    }
    __syncthreads();
    if (t < 3) {
        const double z = linear_row(w3t, b3[t], a2, kH2, 3, t);
        if (zout) zout[(int64_t)r * 3 + t] = z;
        if (t == 0) bgt0[r] = clamp01(z);
        if (t == 1) kslope[r] = z;
        if (t == 2) {
            const double sp = 1.0 / (1.0 + exp(-z));  // sigmoid, predictor.cpp:20
            streaming[r] = sp >= 0.5 ? 1 : 0;          // pipeline.cpp:288
        }
    }
}

}  // namespace

void launch_prepare(const fx_layout& L, int64_t l_plan, int plan_mode, int fixed_blk, double fixed_budget,
                    const double* bgt0, const double* kslope, const int32_t* streaming,
                    int32_t* blk, double* budgets, double* volume, double* cand, int32_t* kblocks,
                    int32_t* bg_done, cudaStream_t s, const AppendArgs& ap, int32_t* err) {
    const int n_bg = L.batch * L.kv_heads;
    FX_REQUIRE(L.group_size >= 1 && L.group_size <= 32, FX_ERR_INVALID,
               "bad-shape: group_size must be in [1, 32]");
    FX_REQUIRE(ap.kn == nullptr || ap.D <= 256, FX_ERR_INVALID, "bad-shape: fused append needs head_dim <= 256");
    if (plan_mode == FX_PLAN_FIXED) {
        bool ok = false;
        for (int c = 0; c < 4; ++c) ok |= kLevels[c] == fixed_blk;
        FX_REQUIRE(ok, FX_ERR_INVALID, "invalid-granularity: blk must be one of 16/32/64/128");
    }
    launch_pdl(k_prepare, n_bg, 32, 0, s, n_bg, L.group_size, l_plan, plan_mode, fixed_blk, fixed_budget,
                                  bgt0, kslope, streaming, blk, budgets, volume, cand, kblocks,
                                  bg_done, ap, err);
    FX_CUDA(cudaGetLastError());
}

void launch_blocks_for_budget(int n, const double* budgets, const int32_t* blk, int64_t l_cpu,
                              int32_t* kblocks, cudaStream_t s) {
    if (n <= 0) return;
    k_blocks_for_budget<<<(n + 255) / 256, 256, 0, s>>>(n, budgets, blk, l_cpu, kblocks);
    FX_CUDA(cudaGetLastError());
}

void launch_predict(int n, const double* w1t, const double* b1, const double* w2t,
                    const double* b2, const double* w3t, const double* b3, const double* mu,
                    const double* sigma, const double* feats, double* bgt0, double* kslope,
                    int32_t* streaming, double* z, cudaStream_t s) {
    if (n <= 0) return;
    k_predict<<<n, kH2, 0, s>>>(w1t, b1, w2t, b2, w3t, b3, mu, sigma, feats, bgt0, kslope,
                                streaming, z);
    FX_CUDA(cudaGetLastError());
}

}  // namespace fx
