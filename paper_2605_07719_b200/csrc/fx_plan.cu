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
#include <algorithm>

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
        if (bg == 0) {
            bg_done[n_bg] = 0;  // worklist publish counter
            for (int i = 0; i < 4; ++i) bg_done[2 * n_bg + 1 + i] = 0;  // attention unit queue
        }
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

// predictor.cpp:40-53 linear_forward (bias first, inputs in order, unfused)
// as tiled f64 layers over all rows of the batch.  A CTA owns kMR rows x kMN
// neurons: the rows' inputs sit in shared memory, the weights (transposed
// [in][out]) stream through a 2-stage cp.async ring of kKC-input tiles, and
// each thread carries kMC independent chains (rows) of one neuron, adding the
// inputs in order -- each weight is read once per kMR rows, and the inner
// loop touches only shared memory and the FP64 pipe.
constexpr int kF = 41, kH1 = 256, kH2 = 384;
constexpr int kMR = 16, kMN = 64, kMT = 256, kKC = 32;  // rows, neurons, threads, inputs per tile
constexpr int kMC = kMR / (kMT / kMN);                   // chains per thread

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int IN, int OUT, bool NORM>
__global__ void __launch_bounds__(kMT) k_mlp_layer(int n, const double* __restrict__ x,
                                                   const double* __restrict__ wt,
                                                   const double* __restrict__ bias,
                                                   const double* __restrict__ mu,
                                                   const double* __restrict__ sigma,
                                                   double* __restrict__ y) {
    constexpr int NCH = (IN + kKC - 1) / kKC;
    extern __shared__ __align__(16) double msm[];
    double (*ws)[kKC * kMN] = reinterpret_cast<double (*)[kKC * kMN]>(msm);  // [2][kKC * kMN]
    double* xs = msm + 2 * kKC * kMN;                                       // [kMR][IN]
    const int r0 = blockIdx.x * kMR, n0 = blockIdx.y * kMN;
    const int t = threadIdx.x, nl = t % kMN, rg = t / kMN;
    auto load_tile = [&](int c, int st) {  // inputs [c*kKC, +kKC) x neurons [n0, +kMN)
        for (int e = t; e < kKC * kMN / 2; e += kMT) {
            const int row = e / (kMN / 2), col = (e % (kMN / 2)) * 2;
            const int i = c * kKC + row;
            if (i < IN) cp_async16(&ws[st][row * kMN + col], wt + (int64_t)i * OUT + n0 + col);
        }
        cp_async_commit();
    };
    load_tile(0, 0);  // weights do not depend on the preceding kernel
    pdl_wait();
    pdl_trigger();
    if (NORM) {  // features.cpp:226-233; all of a thread's loads are issued before any use
        constexpr int PER = (kMR * IN + kMT - 1) / kMT;
        double v[PER], m[PER], sg[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int e = t + u * kMT, r = r0 + e / IN, c = e % IN;
            const bool ok = e < kMR * IN && r < n;
            v[u] = ok ? x[(int64_t)r * IN + c] : 0.0;
            m[u] = e < kMR * IN ? mu[c] : 0.0;
            sg[u] = e < kMR * IN ? sigma[c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int e = t + u * kMT;
            if (e < kMR * IN) xs[e] = sg[u] > 0.0 ? __ddiv_rn(__dsub_rn(v[u], m[u]), sg[u]) : 0.0;
        }
    } else {  // rows of IN doubles (16-byte multiples): asynchronous copies, zero rows past n
        for (int e = t; e < kMR * IN / 2; e += kMT) {
            const int r = r0 + (2 * e) / IN;
            if (r < n) cp_async16(xs + 2 * e, x + (int64_t)r0 * IN + 2 * e);
            else reinterpret_cast<double2*>(xs)[e] = make_double2(0.0, 0.0);
        }
        cp_async_commit();
    }
    double acc[kMC];
    const double b = bias[n0 + nl];
#pragma unroll
    for (int j = 0; j < kMC; ++j) acc[j] = b;
    const double* xr = xs + rg * kMC * IN;
    for (int c = 0; c < NCH; ++c) {
        if (c + 1 < NCH) {
            load_tile(c + 1, (c + 1) & 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* w = ws[c & 1];
        const int kn = IN - c * kKC < kKC ? IN - c * kKC : kKC;
        // the products of 8 inputs first (independent), then the in-order adds:
        // the add chains never wait on a load or a multiply.  Full rounds read
        // each chain's 8 inputs as four 16-byte vectors (IN even: 16-byte rows)
        constexpr int PB = 8;
        for (int k0 = 0; k0 < kn; k0 += PB) {
            const int i0 = c * kKC + k0;
            double p[kMC][PB];
            if (k0 + PB <= kn && (IN % 2) == 0) {
                double wv[PB];
#pragma unroll
                for (int kk = 0; kk < PB; ++kk) wv[kk] = w[(k0 + kk) * kMN + nl];
#pragma unroll
                for (int j = 0; j < kMC; ++j) {
                    const double2* xv = reinterpret_cast<const double2*>(xr + j * IN + i0);
#pragma unroll
                    for (int v = 0; v < PB / 2; ++v) {
                        const double2 x2 = xv[v];
                        p[j][2 * v] = __dmul_rn(x2.x, wv[2 * v]);
                        p[j][2 * v + 1] = __dmul_rn(x2.y, wv[2 * v + 1]);
                    }
                }
            } else {
#pragma unroll
                for (int kk = 0; kk < PB; ++kk) {
                    const double wv = k0 + kk < kn ? w[(k0 + kk) * kMN + nl] : 0.0;
#pragma unroll
                    for (int j = 0; j < kMC; ++j) p[j][kk] = __dmul_rn(k0 + kk < kn ? xr[j * IN + i0 + kk] : 0.0, wv);
                }
            }
#pragma unroll
            for (int kk = 0; kk < PB; ++kk)
                if (k0 + kk < kn)
#pragma unroll
                    for (int j = 0; j < kMC; ++j) acc[j] = __dadd_rn(acc[j], p[j][kk]);
        }
        __syncthreads();  // the stage is refilled next round
    }
#pragma unroll
    for (int j = 0; j < kMC; ++j) {
        const int r = r0 + rg * kMC + j;
        if (r < n) y[(int64_t)r * OUT + n0 + nl] = acc[j] > 0.0 ? acc[j] : 0.0;  // ReLU
    }
}

// Hidden layer 2 (256 -> 384, ReLU), the predictor's FP64-bound layer: the
// same in-order unfused chains, tiled so every SM sub-partition carries
// chains: a CTA owns 16 rows x 32 neurons (4 warps, 8 rows x 16 neurons
// each), a thread 2 rows x 2 neurons = 4 interleaved chains (one weight
// load serves two rows, one input load two neurons).  The rows' inputs sit
// in shared memory (row stride padded by 16 bytes: the four row pairs a warp
// reads are in different banks); the weights are read from L2 / L1 directly,
// a window of 8 inputs ahead in registers, so the warps never synchronize
// inside the 256-input loop.  384 CTAs of 128 threads.
constexpr int kH2R = 16, kH2N = 32, kH2T = 128, kH2XS = kH1 + 2, kH2W = 8;
struct OutLayer {  // the output layer, run by the last neuron-tile CTA of each row tile
    const double* w3t;  // [384][3]
    const double* b3;
    double* bgt0;
    double* kslope;
    int32_t* streaming;
    double* z;        // raw logits [n][3] (nullable)
    int32_t* tiles;   // [row tiles] monotonic counters: + gridDim.y per call
};
__global__ void __launch_bounds__(kH2T) k_mlp_h2(int n, const double* __restrict__ x,
                                                 const double* __restrict__ wt,
                                                 const double* __restrict__ bias, double* __restrict__ y,
                                                 OutLayer ol) {
    extern __shared__ __align__(16) double h2sm[];
    double* xs = h2sm;  // [kH2R][kH2XS]
    const int r0 = blockIdx.x * kH2R, n0 = blockIdx.y * kH2N;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int rl = (warp >> 1) * 8 + (lane >> 3) * 2;  // this thread's rows rl, rl + 1 (in the tile)
    const int nl = (warp & 1) * 16 + (lane & 7) * 2;   // and neurons nl, nl + 1
    const double* wp = wt + n0 + nl;                   // + i * kH2: input i's weights of the two neurons
    double2 wc[kH2W], wn[kH2W];
#pragma unroll
    for (int k = 0; k < kH2W; ++k) wc[k] = __ldg(reinterpret_cast<const double2*>(wp + (int64_t)k * kH2));
    const double2 b = __ldg(reinterpret_cast<const double2*>(bias + n0 + nl));
    pdl_wait();
    pdl_trigger();
    for (int e = t; e < kH2R * kH1 / 2; e += kH2T) {
        const int r = (2 * e) / kH1, c = (2 * e) % kH1;
        if (r0 + r < n) cp_async16(xs + r * kH2XS + c, x + (int64_t)(r0 + r) * kH1 + c);
        else *reinterpret_cast<double2*>(xs + r * kH2XS + c) = make_double2(0.0, 0.0);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    double a00 = b.x, a01 = b.y, a10 = b.x, a11 = b.y;  // [row][neuron]
    const double* x0 = xs + rl * kH2XS;
    const double* x1 = x0 + kH2XS;
#pragma unroll 1
    for (int i0 = 0; i0 < kH1; i0 += kH2W) {
        if (i0 + kH2W < kH1) {
#pragma unroll
            for (int k = 0; k < kH2W; ++k)
                wn[k] = __ldg(reinterpret_cast<const double2*>(wp + (int64_t)(i0 + kH2W + k) * kH2));
        }
#pragma unroll
        for (int k0 = 0; k0 < kH2W; k0 += 2) {
            // products of 2 inputs first (independent), then the in-order adds,
            // the four chains interleaved
            const double2 xa = *reinterpret_cast<const double2*>(x0 + i0 + k0);
            const double2 xb = *reinterpret_cast<const double2*>(x1 + i0 + k0);
            const double2 wa = wc[k0], wb = wc[k0 + 1];
            const double p00 = __dmul_rn(xa.x, wa.x), p01 = __dmul_rn(xa.x, wa.y);
            const double p02 = __dmul_rn(xb.x, wa.x), p03 = __dmul_rn(xb.x, wa.y);
            const double p10 = __dmul_rn(xa.y, wb.x), p11 = __dmul_rn(xa.y, wb.y);
            const double p12 = __dmul_rn(xb.y, wb.x), p13 = __dmul_rn(xb.y, wb.y);
            a00 = __dadd_rn(a00, p00);
            a01 = __dadd_rn(a01, p01);
            a10 = __dadd_rn(a10, p02);
            a11 = __dadd_rn(a11, p03);
            a00 = __dadd_rn(a00, p10);
            a01 = __dadd_rn(a01, p11);
            a10 = __dadd_rn(a10, p12);
            a11 = __dadd_rn(a11, p13);
        }
#pragma unroll
        for (int k = 0; k < kH2W; ++k) wc[k] = wn[k];
    }
    const int ra = r0 + rl;
    if (ra < n)
        *reinterpret_cast<double2*>(y + (int64_t)ra * kH2 + n0 + nl) =
            make_double2(a00 > 0.0 ? a00 : 0.0, a01 > 0.0 ? a01 : 0.0);  // ReLU
    if (ra + 1 < n)
        *reinterpret_cast<double2*>(y + (int64_t)(ra + 1) * kH2 + n0 + nl) =
            make_double2(a10 > 0.0 ? a10 : 0.0, a11 > 0.0 ? a11 : 0.0);
    // The output layer (384 -> 3, no activation) and the head properties
    // (predictor.cpp:161-185, pipeline.cpp:288) of this row tile, by the CTA
    // that writes its last neurons: the barrier orders every thread's stores
    // before thread 0's acq_rel count (the counters only grow: gridDim.y per
    // call, so the last arrival sees a multiple of it).  Its 48 chains are 384
    // dependent adds long, overlapping the other row tiles' layer-2 work.
    __shared__ int s_last;
    __syncthreads();
    if (t == 0) s_last = (atomic_add_acq_rel_gpu(ol.tiles + blockIdx.x, 1) + 1) % (int)gridDim.y == 0;
    __syncthreads();
    if (!s_last) return;
    fence_acq_rel_gpu();
    double* w3s = h2sm;               // [384][3]
    double* as = h2sm + kH2 * 3;      // [kH2R][384]
    for (int e = t; e < kH2 * 3 / 2; e += kH2T) cp_async16(w3s + 2 * e, ol.w3t + 2 * e);
    for (int e = t; e < kH2R * kH2 / 2; e += kH2T) {
        const int r = r0 + (2 * e) / kH2;
        if (r < n) cp_async16(as + 2 * e, y + (int64_t)r0 * kH2 + 2 * e);
        else reinterpret_cast<double2*>(as)[e] = make_double2(0.0, 0.0);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const int lr = t / 3, o = t % 3, r = r0 + lr;
    if (lr >= kH2R || r >= n) return;
    const double* a = as + lr * kH2;
    double z = ol.b3[o];
    for (int k0 = 0; k0 < kH2; k0 += 32) {  // 32 products first, then the in-order adds
        double p[32];
#pragma unroll
        for (int kk = 0; kk < 32; ++kk) p[kk] = __dmul_rn(a[k0 + kk], w3s[(k0 + kk) * 3 + o]);
#pragma unroll
        for (int kk = 0; kk < 32; ++kk) z = __dadd_rn(z, p[kk]);
    }
    if (ol.z) ol.z[(int64_t)r * 3 + o] = z;
    if (o == 0) ol.bgt0[r] = clamp01(z);
    if (o == 1) ol.kslope[r] = z;
    if (o == 2) {
        const double sp = 1.0 / (1.0 + exp(-z));  // sigmoid, predictor.cpp:20
        ol.streaming[r] = sp >= 0.5 ? 1 : 0;      // pipeline.cpp:288
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

size_t predict_scratch_bytes(int n) { return (size_t)std::max(n, 1) * (kH1 + kH2) * sizeof(double); }

void launch_predict_tail(int n, const double* a1, const double* w2t, const double* b2, const double* w3t,
                         const double* b3, double* bgt0, double* kslope, int32_t* streaming, double* z,
                         double* a2, int32_t* tiles, cudaStream_t s) {
    if (n <= 0) return;
    const size_t s2 = std::max((size_t)kH2R * kH2XS, (size_t)kH2 * 3 + (size_t)kH2R * kH2) * sizeof(double);
    FX_CUDA(cudaFuncSetAttribute(k_mlp_h2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2));
    const OutLayer ol{w3t, b3, bgt0, kslope, streaming, z, tiles};
    launch_pdl(k_mlp_h2, dim3((unsigned)((n + kH2R - 1) / kH2R), kH2 / kH2N), kH2T, s2, s, n, a1, w2t, b2, a2, ol);
    FX_CUDA(cudaGetLastError());
}

int predict_row_tiles(int n) { return (std::max(n, 1) + kH2R - 1) / kH2R; }

void launch_predict(int n, const double* w1t, const double* b1, const double* w2t,
                    const double* b2, const double* w3t, const double* b3, const double* mu,
                    const double* sigma, const double* feats, double* bgt0, double* kslope,
                    int32_t* streaming, double* z, void* scratch, int32_t* tiles, cudaStream_t s) {
    if (n <= 0) return;
    double* a1 = static_cast<double*>(scratch);
    double* a2 = a1 + (size_t)n * kH1;
    const unsigned rt = (unsigned)((n + kMR - 1) / kMR);
    const size_t s1 = (size_t)(2 * kKC * kMN + kMR * kF) * sizeof(double);
    FX_CUDA(cudaFuncSetAttribute(k_mlp_layer<kF, kH1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1));
    launch_pdl(k_mlp_layer<kF, kH1, true>, dim3(rt, kH1 / kMN), kMT, s1, s, n, feats, w1t, b1, mu, sigma, a1);
    launch_predict_tail(n, a1, w2t, b2, w3t, b3, bgt0, kslope, streaming, z, a2, tiles, s);
}

}  // namespace fx
