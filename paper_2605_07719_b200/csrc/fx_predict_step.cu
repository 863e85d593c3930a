// fx_predict_step.cu -- decode features of every head (features.cpp:162-224)
// as two short kernels; fx_predict_props then runs the predictor's remaining
// layers (fx_plan.cu): features -> normalize -> 41-256-384-3 -> head
// properties (pipeline.cpp:277-290), which the decode step plans from.
//
// The per-step work of decode_features is the f64 attention of every head
// over its group's default segments -- sink and local for features 21/23/27/28
// (segment_summary, features.cpp:26-80), sink + local + decoded for the
// cross-head maximum output norm of feature 39 (gpu_output_norm,
// features.cpp:80-83, pipeline.cpp:279-282).  It is FP64-bound (~2 G D f64
// multiply-adds per row and head group), so it is spread over the machine:
//   k_feat_part   a persistent grid (3 CTAs of 128 threads per SM) walking
//                 contiguous ranges of (b, g, 64-row chunk) items; per item
//                 the chunk's K and V arrive by two 1-D bulk copies (a
//                 2-stage ring: the next item streams in meanwhile); f64
//                 scores of the G heads (lanes split D, q slice in registers,
//                 a head-splitting butterfly), the chunk max m, weights
//                 e = exp(s - m), z = sum e and sum e v -> one partial per
//                 (item, head).  With an append, the CTA holding the appended
//                 row writes it to the cache and patches its staged copy (the
//                 previous token, append_new after a step, pipeline.cpp:406-412).
//   k_feat_final  one CTA per (b, g), the sequence's Hkv CTAs in a cluster:
//                 the chunk partials merged per segment over all threads
//                 (lse, output, norm), the segments merged in order
//                 (merge_into, attention.cpp:89-104), the 41 features (lane i
//                 forms feature i), the per-sequence maximum of the default
//                 output norms (feature 39) exchanged through distributed
//                 shared memory; with a model, the normalization and the
//                 predictor's first layer for the CTA's G rows.
// Results agree with the reference within 1e-9 relative (sums associate
// differently), like fx_decode_features.
#include <algorithm>

#include <cooperative_groups.h>

#include "fx_common.cuh"

namespace fx {
namespace {

namespace cg = cooperative_groups;

constexpr int kPT = 256;  // threads per CTA
constexpr int kPW = kPT / 32;
constexpr int kF = 41;
constexpr int kCR = 64;             // rows per chunk
constexpr double kEmptyLse = -1e6;  // kEmptyLse, features.hpp:16

#ifdef FX_TRACE  // profiling build only: per-CTA phase times (%globaltimer) of the two kernels
__device__ long long g_fp_trace[16 * 2048];
#define FP_MARK(slot, i)                                                                  \
    if (threadIdx.x == 0 && (slot) < 2048) {                                              \
        long long t_;                                                                     \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
        g_fp_trace[(slot) * 16 + (i)] = t_;                                               \
    }
#else
#define FP_MARK(slot, i)
#endif

// f32 bits -> the f64 value x * 2^-896, with two integer ops (three for f32
// sources): the f32 sign / exponent / mantissa fields are moved into the f64
// fields without rebiasing the exponent, which is exact for every finite f32
// -- zero and denormals included (a zero exponent field stays zero and the
// mantissa m lands as the f64 denormal m * 2^29 * 2^-1074 = (m * 2^-149) *
// 2^-896) -- and needs no F2F (a quarter-rate MIO instruction; every K / V
// element is widened once per chunk).  The 2^896 comes back exactly through
// the q slice (scores) and the softmax weights (outputs), so every product
// and sum is the one of the unscaled values.  Non-finite K / V map to large
// finite values (the reference's features are NaN / inf there anyway).
constexpr double kUp = 0x1p896;
__device__ __forceinline__ double bits_to_f64_scaled(uint32_t u, bool low_bits) {
    const uint32_t hi = (uint32_t)((int32_t)u >> 3) & 0x8fffffffu;
    return __hiloint2double((int)hi, low_bits ? (int)(u << 29) : 0);
}

// N contiguous elements of a row (16-byte aligned slice) as scaled f64
template <typename T, int N>
__device__ __forceinline__ void load_row_slice(const T* p, double* out) {
    constexpr bool BF = sizeof(T) == 2;
    if constexpr (BF && N % 8 == 0) {
#pragma unroll
        for (int v = 0; v < N / 8; ++v) {
            const uint4 w = reinterpret_cast<const uint4*>(p)[v];
            const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                out[v * 8 + 2 * i] = bits_to_f64_scaled(u[i] << 16, false);
                out[v * 8 + 2 * i + 1] = bits_to_f64_scaled(u[i] & 0xffff0000u, false);
            }
        }
    } else if constexpr (BF && N == 4) {  // 8 bytes
        const uint2 w = *reinterpret_cast<const uint2*>(p);
        out[0] = bits_to_f64_scaled(w.x << 16, false);
        out[1] = bits_to_f64_scaled(w.x & 0xffff0000u, false);
        out[2] = bits_to_f64_scaled(w.y << 16, false);
        out[3] = bits_to_f64_scaled(w.y & 0xffff0000u, false);
    } else if constexpr (!BF && N % 4 == 0) {
#pragma unroll
        for (int v = 0; v < N / 4; ++v) {
            const uint4 w = reinterpret_cast<const uint4*>(p)[v];
            out[v * 4 + 0] = bits_to_f64_scaled(w.x, true);
            out[v * 4 + 1] = bits_to_f64_scaled(w.y, true);
            out[v * 4 + 2] = bits_to_f64_scaled(w.z, true);
            out[v * 4 + 3] = bits_to_f64_scaled(w.w, true);
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            if constexpr (BF) out[i] = bits_to_f64_scaled((uint32_t)__bfloat16_as_ushort(p[i]) << 16, false);
            else out[i] = bits_to_f64_scaled(__float_as_uint(p[i]), true);
        }
    }
}
// two adjacent elements as scaled f64
__device__ __forceinline__ void load_pair(const __nv_bfloat16* p, double& a, double& b) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(p);
    a = bits_to_f64_scaled(w << 16, false);
    b = bits_to_f64_scaled(w & 0xffff0000u, false);
}
__device__ __forceinline__ void load_pair(const float* p, double& a, double& b) {
    const uint2 w = *reinterpret_cast<const uint2*>(p);
    a = bits_to_f64_scaled(w.x, true);
    b = bits_to_f64_scaled(w.y, true);
}

// Sum of G values over the LPR lanes of a row group: the first levels of the
// butterfly halve the value set per lane (lanes with the offset bit set keep
// the upper half and send the lower), so each level moves half of what a
// plain butterfly of every value would; afterwards lane sl holds head
// sl / (LPR / GP) (GP = G rounded up to a power of two).
template <int G, int LPR>
__device__ __forceinline__ double reduce_heads(double (&p)[G], int sl) {
    constexpr int GP = G <= 1 ? 1 : G <= 2 ? 2 : G <= 4 ? 4 : 8;
    static_assert(GP <= LPR, "one head per lane group");
    double v[GP];
#pragma unroll
    for (int h = 0; h < GP; ++h) v[h] = h < G ? p[h] : 0.0;
    int o = LPR / 2;
#pragma unroll
    for (int n = GP; n > 1; n >>= 1, o >>= 1) {
        const bool up = (sl & o) != 0;
#pragma unroll
        for (int k = 0; k < n / 2; ++k) {
            const double send = up ? v[k] : v[k + n / 2];
            const double keep = up ? v[k + n / 2] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    double x = v[0];
#pragma unroll
    for (; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// chunks of the three default segments (sink, local, decoded) of a group
struct FeatChunks {
    int n[3];
    __host__ __device__ int total() const { return n[0] + n[1] + n[2]; }
};
__host__ __device__ inline FeatChunks feat_chunks(const fx_layout& L, int64_t l_new) {
    FeatChunks c;
    c.n[0] = (int)cdiv_dev(L.l_sink, kCR);
    c.n[1] = (int)cdiv_dev(L.l_local, kCR);
    c.n[2] = (int)cdiv_dev(l_new, kCR);
    return c;
}
template <int D>
constexpr int part_stride() { return D + 2; }  // m, z, sum e v [D] (f64)

struct FeatAppend {
    const float* kn = nullptr;  // [B][Hkv][D] f32: the row appended at `row`
    const float* vn = nullptr;
    int64_t row = -1;
};

template <typename T, int D>
constexpr size_t part_stage_bytes() { return (size_t)2 * kCR * D * sizeof(T); }
constexpr int kPartStages = 2;
constexpr int kPartCtasPerSm = 3;
constexpr int kPT2 = 128, kPW2 = kPT2 / 32;  // threads / warps of k_feat_part

// Chunk partials: a persistent grid, each CTA walking a contiguous range of
// (b, g, chunk) items (mostly one group, so the q slice is reloaded only at a
// group change) with a 2-stage ring of bulk copies -- the next chunk's K and V
// stream in while this one is computed.  Per item: f64 scores of the G heads
// (lanes split D) with each warp's running maximum per head, one exp per
// (row, head) over all threads with per-warp sums z, then sum e v (thread =
// dim pair x row slab)
// -> one partial (m, z, sum e v) per (item, head).
template <typename T, int G, int D>
__global__ void __launch_bounds__(kPT2, kPartCtasPerSm) k_feat_part(fx_layout L, void* kp, void* vp, int64_t l_new,
                                                                   const float* __restrict__ q, FeatAppend ap,
                                                                   double* __restrict__ part, int items) {
    extern __shared__ __align__(128) unsigned char fsm[];
    constexpr size_t STG = part_stage_bytes<T, D>();
    constexpr int NP = D / 2, NS = kPT2 / NP;  // dim pairs, row slabs of the P.V pass
    __shared__ double sc[kCR][G];
    __shared__ double red[NS][G][D];
    __shared__ double s_wm[kPW2][G], s_wz[kPW2][G];  // per warp and head: score max, sum of weights
    __shared__ __align__(8) uint64_t full[kPartStages];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const FeatChunks fc = feat_chunks(L, l_new);
    const int nch = fc.total();
    const int per = (items + gridDim.x - 1) / gridDim.x;
    const int i0 = blockIdx.x * per, i1 = min(items, i0 + per);
    if (i0 >= i1) return;
    FP_MARK(blockIdx.x, 0);
    // item -> (bg, chunk) -> rows
    auto locate = [&](int item, int64_t& bg, int& sg, int64_t& r0, int& nr) {
        bg = item / nch;
        const int c = item - (int)bg * nch;
        sg = c < fc.n[0] ? 0 : c < fc.n[0] + fc.n[1] ? 1 : 2;
        const int ci = c - (sg == 0 ? 0 : sg == 1 ? fc.n[0] : fc.n[0] + fc.n[1]);
        const int64_t seg_row = sg == 0 ? 0 : sg == 1 ? L.l_sink + L.l_cpu : L.l_sink + L.l_cpu + L.l_local;
        const int64_t seg_n = sg == 0 ? L.l_sink : sg == 1 ? L.l_local : l_new;
        r0 = seg_row + (int64_t)ci * kCR;
        nr = (int)min((int64_t)kCR, seg_n - (int64_t)ci * kCR);
    };
    auto issue = [&](int item, int st) {
        int64_t bg, r0;
        int sg, nr;
        locate(item, bg, sg, r0, nr);
        T* Ks = reinterpret_cast<T*>(fsm + st * STG);
        T* Vs = Ks + kCR * D;
        const uint32_t bytes = (uint32_t)nr * D * sizeof(T);
        mbar_arrive_expect_tx(&full[st], 2 * bytes);
        bulk_g2s(Ks, static_cast<const T*>(kp) + (bg * L.l_cap + r0) * D, bytes, &full[st]);
        bulk_g2s(Vs, static_cast<const T*>(vp) + (bg * L.l_cap + r0) * D, bytes, &full[st]);
    };
    pdl_wait();  // the cache rows of earlier steps' appends
    pdl_trigger();
    if (tid == 0) {
        for (int i = 0; i < kPartStages; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
        for (int i = 0; i < kPartStages && i0 + i < i1; ++i) issue(i0 + i, i);
    }
    __syncthreads();  // barrier init visible
    constexpr int LPR = G <= 4 ? 16 : 32, DPL = D / LPR, RPI = 32 / LPR;
    constexpr int GP = G <= 1 ? 1 : G <= 2 ? 2 : G <= 4 ? 4 : 8, LPH = LPR / GP;
    const int sub = lane / LPR, sl = lane % LPR;
    const double isd = 1.0 / sqrt((double)D);
    double qreg[DPL][G];
    int64_t q_bg = -1;
    for (int item = i0, it = 0; item < i1; ++item, ++it) {
        const int st = it % kPartStages;
        int64_t bg, r0;
        int sg, nr;
        locate(item, bg, sg, r0, nr);
        if (bg != q_bg) {  // this lane's q slice of the group's heads, times 2^896 (CTA-uniform)
#pragma unroll
            for (int h = 0; h < G; ++h)
#pragma unroll
                for (int j = 0; j < DPL; ++j) qreg[j][h] = (double)q[(bg * G + h) * D + sl * DPL + j] * kUp;
            q_bg = bg;
        }
        T* Ks = reinterpret_cast<T*>(fsm + st * STG);
        T* Vs = Ks + kCR * D;
        if (it == 1) FP_MARK(blockIdx.x, 12);
        mbar_wait(&full[st], (uint32_t)((it / kPartStages) & 1));
        if (it == 1) FP_MARK(blockIdx.x, 13);
        if (ap.kn != nullptr && ap.row >= r0 && ap.row < r0 + nr) {
            // the appended row: into the cache and over the staged (stale) copy
            const int rr = (int)(ap.row - r0);
            T* K = static_cast<T*>(kp) + bg * L.l_cap * D;
            T* V = static_cast<T*>(vp) + bg * L.l_cap * D;
            for (int d = tid; d < D; d += kPT2) {
                const float a = ap.kn[bg * D + d], b = ap.vn[bg * D + d];
                T ka, va;
                if constexpr (sizeof(T) == 2) {
                    ka = __float2bfloat16_rn(a);
                    va = __float2bfloat16_rn(b);
                } else {
                    ka = a;
                    va = b;
                }
                K[ap.row * D + d] = ka;
                V[ap.row * D + d] = va;
                Ks[rr * D + d] = ka;
                Vs[rr * D + d] = va;
            }
            __syncthreads();
        }
        // scores: LPR lanes per row, RPI rows per warp at a time; the warp's
        // running maximum per head on the lanes that hold the sums
        const bool writer = sl % LPH == 0 && sl / LPH < G;
        double mloc = -INFINITY;
        for (int rb = warp * RPI; rb < nr; rb += kPW2 * RPI) {
            const int r = rb + sub;
            const bool live = r < nr;
            double kv[DPL];
            load_row_slice<T, DPL>(Ks + (live ? r : rb) * D + sl * DPL, kv);
            double p[G];
#pragma unroll
            for (int h = 0; h < G; ++h) p[h] = 0.0;
#pragma unroll
            for (int j = 0; j < DPL; ++j)
#pragma unroll
                for (int h = 0; h < G; ++h) p[h] += qreg[j][h] * kv[j];
            const double v = reduce_heads<G, LPR>(p, sl) * isd;
            if (live && writer) {
                sc[r][sl / LPH] = v;
                mloc = fmax(mloc, v);
            }
        }
#pragma unroll
        for (int o = LPR; o < 32; o <<= 1) mloc = fmax(mloc, __shfl_xor_sync(0xffffffffu, mloc, o));
        if (sub == 0 && writer) s_wm[warp][sl / LPH] = mloc;
        __syncthreads();
        if (it == 1) FP_MARK(blockIdx.x, 9);
        double* out = part + (int64_t)item * G * part_stride<D>();
        // weights: one exp per (row, head) over all threads, scaled by 2^896
        // (the V elements carry 2^-896); z per warp and head
        {
            double zh[G];
#pragma unroll
            for (int h = 0; h < G; ++h) zh[h] = 0.0;
            for (int i = tid; i < nr * G; i += kPT2) {
                const int r = i / G, h = i - r * G;
                double M = s_wm[0][h];
#pragma unroll
                for (int w = 1; w < kPW2; ++w) M = fmax(M, s_wm[w][h]);
                const double e = exp(sc[r][h] - M) * kUp;
                sc[r][h] = e;
#pragma unroll
                for (int hh = 0; hh < G; ++hh) zh[hh] += hh == h ? e : 0.0;
            }
#pragma unroll
            for (int h = 0; h < G; ++h) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) zh[h] += __shfl_xor_sync(0xffffffffu, zh[h], o);
                if (lane == 0) s_wz[warp][h] = zh[h];
            }
        }
        __syncthreads();
        if (it == 1) FP_MARK(blockIdx.x, 10);
        {
            const int pi = tid % NP, slab = tid / NP;
            double a[G][2];
#pragma unroll
            for (int h = 0; h < G; ++h) a[h][0] = a[h][1] = 0.0;
#pragma unroll 4
            for (int r = slab; r < nr; r += NS) {
                double v0, v1;
                load_pair(Vs + r * D + 2 * pi, v0, v1);
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    const double w = sc[r][h];
                    a[h][0] += w * v0;
                    a[h][1] += w * v1;
                }
            }
#pragma unroll
            for (int h = 0; h < G; ++h) {
                red[slab][h][2 * pi] = a[h][0];
                red[slab][h][2 * pi + 1] = a[h][1];
            }
        }
        __syncthreads();  // the stage is consumed: refill it with the item two ahead
        if (it == 1) FP_MARK(blockIdx.x, 11);
        if (tid == 0 && item + kPartStages < i1) issue(item + kPartStages, st);
        for (int i = tid; i < G * D; i += kPT2) {
            const int h = i / D, d = i % D;
            double s2 = 0.0;
#pragma unroll
            for (int k = 0; k < NS; ++k) s2 += red[k][h][d];
            out[h * part_stride<D>() + 2 + d] = s2;
        }
        if (tid < G) {  // the chunk max and sum of weights (the 2^896 taken back exactly)
            double M = s_wm[0][tid], z = 0.0;
#pragma unroll
            for (int w = 1; w < kPW2; ++w) M = fmax(M, s_wm[w][tid]);
#pragma unroll
            for (int w = 0; w < kPW2; ++w) z += s_wz[w][tid];
            out[tid * part_stride<D>()] = M;
            out[tid * part_stride<D>() + 1] = z * 0x1p-896;
        }
        __syncthreads();  // sc / red are rewritten by the next item
        if (it < 6) FP_MARK(blockIdx.x, 2 + it);
    }
    FP_MARK(blockIdx.x, 1);
}

// The predictor's first layer inside the feature merge (the CTA holds its G
// heads' features): normalize (features.cpp:226-233) and 41 -> 256 + ReLU
// with the in-order unfused chains of k_mlp_layer (bit-identical).
struct Layer1 {
    const double* w1t = nullptr;  // [41][256]
    const double* b1 = nullptr;
    const double* mu = nullptr;
    const double* sigma = nullptr;
    double* a1 = nullptr;  // [heads][256]
};

// feature i of a head (features.cpp:172-224) from its record r, the step's
// reductions and the segment summaries; 39 (cross-head max) is set later
__device__ __forceinline__ double feature_value(int i, const double* r, double l_new, double qn, double qk,
                                                double qa, double nmk, double nmv, const double* lse,
                                                const double* nrm, const int64_t* seg_n, int D) {
    const double sd = sqrt((double)D);
    switch (i) {
        case 0: case 1: case 2: return r[i];
        case 3: return r[3] + r[4] + l_new;
        case 4: return r[6];
        case 5: return r[7];
        case 6: return sqrt(nmk);
        case 7: return sqrt(nmv);
        case 8: case 9: case 10: case 11: case 12: case 13: case 14: case 15: return r[i];
        case 16: return (qn > 0.0 && r[5] == 0.0) ? qk / (qn * sd) : 0.0;
        case 17: case 18: case 19: case 20: return r[i - 1];
        case 21: return seg_n[0] > 0 ? lse[0] : kEmptyLse;
        case 22: {  // approx_lse_cpu (features.cpp:159-170)
            const double l_cpu = r[2];
            if (l_cpu == 0.0) return kEmptyLse;
            if (qn == 0.0) return log(l_cpu);
            return log(l_cpu) + qn * (qk / (qn * sd)) + 0.5 * qn * qn * r[17];
        }
        case 23: return seg_n[1] > 0 ? lse[1] : kEmptyLse;
        case 24: case 25: case 26: return r[i - 4];
        case 27: return seg_n[0] > 0 ? nrm[0] : 0.0;
        case 28: return seg_n[1] > 0 ? nrm[1] : 0.0;
        case 29: case 30: case 31: return r[i - 6];
        case 32: return qn;
        case 33: return r[31];
        case 34: return (qn > 0.0 && r[31] > 0.0) ? qa / (qn * r[31]) : 0.0;
        case 35: case 36: case 37: case 38: return r[i - 9];
        case 40: return r[30];
        default: return 0.0;
    }
}

// Merge of a head's chunk partials and the 41 features; one CTA per (b, g),
// the sequence's Hkv CTAs form a cluster (feature 39).  A warp per head: the
// chunk maxima / weights are formed lane-parallel (lane = chunk), the chunk
// outputs' loads are all independent; lane i forms feature i (and i + 32).
template <int G, int D>
__global__ void __launch_bounds__(kPT, 2) k_feat_final(fx_layout L, int64_t l_new, const float* __restrict__ q,
                                                    const double* __restrict__ rec,
                                                    const double* __restrict__ part,
                                                    double* __restrict__ feats, Layer1 l1) {
    cg::cluster_group cluster = cg::this_cluster();
    constexpr int DV = D / 32;  // dims per lane (contiguous)
    constexpr int PS = part_stride<D>();
    static_assert(kPT == 256, "layer 1: one thread per hidden neuron");
    __shared__ double s_gn[8], s_seq_max;
    __shared__ double s_feat[8][kF + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = blockIdx.x, b = blockIdx.y;
    const int64_t bg = (int64_t)b * L.kv_heads + g;
    const FeatChunks fc = feat_chunks(L, l_new);
    const int64_t seg_n[3] = {L.l_sink, L.l_local, l_new};
    const int tslot = 1024 + blockIdx.y * gridDim.x + blockIdx.x;
    FP_MARK(tslot, 0);
#ifdef FX_TRACE
    if (tid == 0) g_fp_trace[tslot * 16 + 14] = clock64();
#endif
    // layer-1 weights into shared memory (independent of the features)
    extern __shared__ __align__(16) double w1s[];  // [kF][256] when l1.w1t
    if (l1.w1t) {
        for (int e = tid; e < kF * 256 / 2; e += kPT)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(w1s + 2 * e)),
                         "l"(l1.w1t + 2 * e)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // before the wait (independent of the chunk partials): the step's
    // reductions of q against the prefill record and the record fields
    const int h = warp;  // a warp per head
    const bool head_warp = h < G;
    double qn = 0.0, qk = 0.0, qa = 0.0, nmk = 0.0, nmv = 0.0;
    const int64_t head = bg * G + h;
    const double* r = rec + head * (32 + 3 * D);
    if (head_warp) {
        const double* mk = r + 32;
        const double* mv = mk + D;
        const double* an = mv + D;
        const float* qh = q + head * D;
        double qn2 = 0.0;
#pragma unroll
        for (int d = lane; d < D; d += 32) {
            const double qd = (double)qh[d];
            qn2 += qd * qd;
            qk += qd * mk[d];
            qa += qd * an[d];
            nmk += mk[d] * mk[d];
            nmv += mv[d] * mv[d];
        }
#pragma unroll
        for (int s2 = 16; s2 > 0; s2 >>= 1) {
            qn2 += __shfl_xor_sync(0xffffffffu, qn2, s2);
            qk += __shfl_xor_sync(0xffffffffu, qk, s2);
            qa += __shfl_xor_sync(0xffffffffu, qa, s2);
            nmk += __shfl_xor_sync(0xffffffffu, nmk, s2);
            nmv += __shfl_xor_sync(0xffffffffu, nmv, s2);
        }
        qn = sqrt(qn2);
        if (lane < 2) prefetch_l1(r + lane * 16);  // the record fields the features copy
    }
    FP_MARK(tslot, 1);
    pdl_wait();
    pdl_trigger();
    FP_MARK(tslot, 2);
    // The merge of the chunk partials, spread over all threads: (head, chunk)
    // scalars first (max per segment, weights), then (head, dim) outputs with
    // every chunk's load in flight at once, block-level norm reductions.
    const int T = fc.total();
    constexpr int PPT = (G * D + kPT - 1) / kPT;  // (head, dim) pairs per thread
    double* s_m = w1s + (l1.w1t ? kF * 256 : 0);  // [G][T] chunk maxima, then weights
    double* s_wz = s_m + G * T;                   // [G][T] z, then w * z
    __shared__ double s_M[8][3], s_Z[8][3], s_lse[8][3], s_nrm[8][3], s_wsg[8][3];
    __shared__ double s_sq[8][D / 32][3];
    auto seg_of = [&](int c) { return c < fc.n[0] ? 0 : c < fc.n[0] + fc.n[1] ? 1 : 2; };
    const double* pb = part + bg * T * G * PS;  // chunk c, head hh at + (c * G + hh) * PS
    for (int i = tid; i < G * T; i += kPT) {
        const int hh = i / T, c = i - hh * T;
        const double2 mz = *reinterpret_cast<const double2*>(pb + (int64_t)(c * G + hh) * PS);
        s_m[i] = mz.x;
        s_wz[i] = mz.y;
    }
    // the (head, dim) outputs of every chunk, loaded now (one round trip, in
    // flight while the chunk weights are formed) when they fit in registers
    constexpr int kMaxT = 16;
    const bool vreg = PPT <= 2 && T <= kMaxT;
    double pv[PPT <= 2 ? PPT : 1][kMaxT];
    if (vreg) {
#pragma unroll
        for (int pp = 0; pp < (PPT <= 2 ? PPT : 1); ++pp) {
            const int i = tid + pp * kPT;
            const int hh = min(i / D, G - 1), d = i % D;
            const double* pa = pb + (int64_t)hh * PS + 2 + d;
#pragma unroll
            for (int c = 0; c < kMaxT; ++c) pv[pp][c] = (c < T && i < G * D) ? pa[(int64_t)c * G * PS] : 0.0;
        }
    }
    __syncthreads();
    FP_MARK(tslot, 6);
    if (tid < G * 3) {  // per (head, segment): the maximum of the chunk maxima
        const int hh = tid / 3, sg = tid % 3;
        const int c0 = sg == 0 ? 0 : sg == 1 ? fc.n[0] : fc.n[0] + fc.n[1];
        double M = -INFINITY;
        for (int c = c0; c < c0 + fc.n[sg]; ++c) M = fmax(M, s_m[hh * T + c]);
        s_M[hh][sg] = M;
    }
    __syncthreads();
    for (int i = tid; i < G * T; i += kPT) {  // chunk weights
        const int hh = i / T, c = i - hh * T;
        const double w = exp(s_m[i] - s_M[hh][seg_of(c)]);
        s_m[i] = w;
        s_wz[i] *= w;
    }
    __syncthreads();
    FP_MARK(tslot, 7);
    if (tid < G * 3) {  // per (head, segment): the denominator and the LSE
        const int hh = tid / 3, sg = tid % 3;
        const int c0 = sg == 0 ? 0 : sg == 1 ? fc.n[0] : fc.n[0] + fc.n[1];
        double Z = 0.0;
        for (int c = c0; c < c0 + fc.n[sg]; ++c) Z += s_wz[hh * T + c];
        s_Z[hh][sg] = Z;
        s_lse[hh][sg] = fc.n[sg] > 0 ? s_M[hh][sg] + log(Z) : kEmptyLse;
    }
    // per (head, dim): the segment outputs, every chunk's value loaded at once
    double o[PPT][3];
#pragma unroll
    for (int pp = 0; pp < PPT; ++pp) {
        o[pp][0] = o[pp][1] = o[pp][2] = 0.0;
        const int i = tid + pp * kPT;
        if (i < G * D) {
            const int hh = i / D, d = i - hh * D;
            if (vreg) {
#pragma unroll
                for (int c = 0; c < kMaxT; ++c) {
                    if (c >= T) break;
                    const double v = pv[PPT <= 2 ? pp : 0][c] * s_m[hh * T + c];
                    const int sg = seg_of(c);
                    o[pp][0] += sg == 0 ? v : 0.0;
                    o[pp][1] += sg == 1 ? v : 0.0;
                    o[pp][2] += sg == 2 ? v : 0.0;
                }
            } else {
                const double* pa = pb + (int64_t)hh * PS + 2 + d;
#pragma unroll 8
                for (int c = 0; c < T; ++c) {
                    const double v = pa[(int64_t)c * G * PS] * s_m[hh * T + c];
                    const int sg = seg_of(c);
                    o[pp][0] += sg == 0 ? v : 0.0;
                    o[pp][1] += sg == 1 ? v : 0.0;
                    o[pp][2] += sg == 2 ? v : 0.0;
                }
            }
        }
    }
    __syncthreads();  // s_Z, s_lse
    FP_MARK(tslot, 8);
#pragma unroll
    for (int pp = 0; pp < PPT; ++pp) {
        const int i = tid + pp * kPT;
        double x[3] = {0.0, 0.0, 0.0};
        const int hh = min(i / D, G - 1);
        if (i < G * D) {
#pragma unroll
            for (int sg = 0; sg < 3; ++sg) {
                if (fc.n[sg] == 0) continue;
                o[pp][sg] /= s_Z[hh][sg];
                x[sg] = o[pp][sg] * o[pp][sg];
            }
        }
#pragma unroll
        for (int sg = 0; sg < 3; ++sg)
#pragma unroll
            for (int s2 = 16; s2 > 0; s2 >>= 1) x[sg] += __shfl_xor_sync(0xffffffffu, x[sg], s2);
        if (lane == 0 && i < G * D)
#pragma unroll
            for (int sg = 0; sg < 3; ++sg) s_sq[hh][(i % D) / 32][sg] = x[sg];
    }
    __syncthreads();
    if (tid < G * 3) {  // segment output norms
        const int hh = tid / 3, sg = tid % 3;
        double x = 0.0;
#pragma unroll
        for (int k = 0; k < D / 32; ++k) x += s_sq[hh][k][sg];
        s_nrm[hh][sg] = fc.n[sg] > 0 ? sqrt(x) : 0.0;
    }
    if (tid < G) {  // merge weights of the default output (sink, local, decoded in order, merge_into)
        double lsum = 0.0, wsg[3] = {0.0, 0.0, 0.0};
        bool any = false;
        for (int sg = 0; sg < 3; ++sg) {
            if (seg_n[sg] == 0) continue;
            if (!any) {
                lsum = s_lse[tid][sg];
                wsg[sg] = 1.0;
                any = true;
                continue;
            }
            const double p = s_lse[tid][sg];
            const double tot = lsum > p ? lsum + log1p(exp(p - lsum)) : p + log1p(exp(lsum - p));
            const double wa = exp(lsum - tot), wb = exp(p - tot);
            for (int s2 = 0; s2 < sg; ++s2) wsg[s2] *= wa;
            wsg[sg] = wb;
            lsum = tot;
        }
        for (int sg = 0; sg < 3; ++sg) s_wsg[tid][sg] = wsg[sg];
    }
    __syncthreads();  // s_sq is reused below
    FP_MARK(tslot, 9);
#pragma unroll
    for (int pp = 0; pp < PPT; ++pp) {
        const int i = tid + pp * kPT;
        const int hh = min(i / D, G - 1);
        double x = 0.0;
        if (i < G * D) {
            double od = 0.0;
#pragma unroll
            for (int sg = 0; sg < 3; ++sg)
                if (seg_n[sg] > 0) od += s_wsg[hh][sg] * o[pp][sg];
            x = od * od;
        }
#pragma unroll
        for (int s2 = 16; s2 > 0; s2 >>= 1) x += __shfl_xor_sync(0xffffffffu, x, s2);
        if (lane == 0 && i < G * D) s_sq[hh][(i % D) / 32][0] = x;
    }
    __syncthreads();
    if (head_warp) {
        if (lane == 0) {
            bool any = false;
            for (int sg = 0; sg < 3; ++sg) any |= seg_n[sg] > 0;
            double x = 0.0;
#pragma unroll
            for (int k = 0; k < D / 32; ++k) x += s_sq[h][k][0];
            s_gn[h] = any ? sqrt(x) : 0.0;
        }
        const double lse[3] = {s_lse[h][0], s_lse[h][1], s_lse[h][2]};
        const double nrm[3] = {s_nrm[h][0], s_nrm[h][1], s_nrm[h][2]};
        // lane i forms feature i (and i + 32)
        for (int i = lane; i < kF; i += 32)
            s_feat[h][i] = feature_value(i, r, (double)l_new, qn, qk, qa, nmk, nmv, lse, nrm, seg_n, D);
    }
    __syncthreads();
    FP_MARK(tslot, 3);
    if (tid == 0) {
        double m = 0.0;
        for (int h = 0; h < G; ++h) m = fmax(m, s_gn[h]);
        s_seq_max = m;
    }
    cluster.sync();  // every CTA of the sequence has its heads' maximum
    if (tid == 0) {
        double m = 0.0;
        for (unsigned c = 0; c < cluster.num_blocks(); ++c) m = fmax(m, *cluster.map_shared_rank(&s_seq_max, c));
        for (int h = 0; h < G; ++h) s_feat[h][39] = m;
    }
    cluster.sync();  // the peers' reads are done before any CTA moves on; s_feat complete
    FP_MARK(tslot, 4);
    if (feats)
        for (int i = tid; i < G * kF; i += kPT) feats[(bg * G + i / kF) * kF + i % kF] = s_feat[i / kF][i % kF];
    if (l1.w1t) {
        __syncthreads();  // every thread has read s_feat (the features) before it is normalized in place
        for (int i = tid; i < G * kF; i += kPT) {
            const int h = i / kF, c = i % kF;
            const double sg = l1.sigma[c];
            s_feat[h][c] = sg > 0.0 ? __ddiv_rn(__dsub_rn(s_feat[h][c], l1.mu[c]), sg) : 0.0;
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        const double bias = l1.b1[tid];
        double acc[G];
#pragma unroll
        for (int h = 0; h < G; ++h) acc[h] = bias;
#pragma unroll
        for (int i = 0; i < kF; ++i)
#pragma unroll
            for (int h = 0; h < G; ++h) acc[h] = __dadd_rn(acc[h], __dmul_rn(s_feat[h][i], w1s[i * 256 + tid]));
#pragma unroll
        for (int h = 0; h < G; ++h) l1.a1[(bg * G + h) * 256 + tid] = acc[h] > 0.0 ? acc[h] : 0.0;  // ReLU
    }
    FP_MARK(tslot, 5);
#ifdef FX_TRACE
    if (tid == 0) g_fp_trace[tslot * 16 + 15] = clock64();
#endif
}

template <typename T, int G, int D>
void launch_ff(const fx_layout& L, void* k, void* v, int64_t l_new, const float* q, const double* rec,
               double* feats, double* part, const FeatAppend& ap, const Layer1& l1, int num_sms, cudaStream_t s) {
    const FeatChunks fc = feat_chunks(L, l_new);
    const int n_bg = L.batch * L.kv_heads;
    if (fc.total() > 0) {
        const size_t smem = kPartStages * part_stage_bytes<T, D>();
        FX_CUDA(cudaFuncSetAttribute(k_feat_part<T, G, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int items = fc.total() * n_bg;
        const int grid = std::min(items, num_sms * kPartCtasPerSm);
        launch_pdl(k_feat_part<T, G, D>, dim3((unsigned)grid), kPT2, smem, s, L, k, v, l_new, q, ap, part, items);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)L.kv_heads, (unsigned)L.batch);
    cfg.blockDim = dim3(kPT);
    cfg.dynamicSmemBytes = ((l1.w1t ? (size_t)kF * 256 : 0) + (size_t)2 * G * fc.total()) * sizeof(double);
    FX_REQUIRE(cfg.dynamicSmemBytes <= 200 * 1024, FX_ERR_INVALID,
               "bad-shape: too many default rows for the feature merge");
    FX_CUDA(cudaFuncSetAttribute(k_feat_final<G, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max<size_t>(cfg.dynamicSmemBytes, 1)));
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)L.kv_heads;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    FX_CUDA(cudaLaunchKernelEx(&cfg, k_feat_final<G, D>, L, l_new, q, rec, (const double*)part, feats, l1));
}

template <typename T, int D>
void launch_ff_g(const fx_layout& L, void* k, void* v, int64_t l_new, const float* q, const double* rec,
                 double* feats, double* part, const FeatAppend& ap, const Layer1& l1, int num_sms, cudaStream_t s) {
    switch (L.group_size) {
#define FX_FG(GG)                                                          \
    case GG:                                                               \
        launch_ff<T, GG, D>(L, k, v, l_new, q, rec, feats, part, ap, l1, num_sms, s);   \
        break;
        FX_FG(1) FX_FG(2) FX_FG(4) FX_FG(7) FX_FG(8)
#undef FX_FG
        default: fail(FX_ERR_INVALID, "bad-shape: fused features support group sizes 1, 2, 4, 7, 8");
    }
}

}  // namespace

bool feat_fused_supported(const fx_layout& L) {
    const int G = L.group_size;
    return (G == 1 || G == 2 || G == 4 || G == 7 || G == 8) && (L.head_dim == 64 || L.head_dim == 128) &&
           L.kv_heads >= 1 && L.kv_heads <= 8;
}

size_t feat_fused_scratch_bytes(const fx_layout& L, int64_t l_new) {
    const FeatChunks fc = feat_chunks(L, l_new);
    return (size_t)L.batch * L.kv_heads * fc.total() * L.group_size * (L.head_dim + 2) * sizeof(double);
}

void launch_feat_fused(const fx_layout& L, void* k, void* v, int64_t l_new, const float* q, const double* rec,
                       double* feats, void* scratch, cudaStream_t s, const float* append_k,
                       const float* append_v, const double* const layer1[4], double* a1, int num_sms) {
    FX_REQUIRE(feat_fused_supported(L), FX_ERR_INVALID,
               "bad-shape: fused features need G in {1,2,4,7,8}, head_dim 64/128 and kv_heads <= 8");
    FeatAppend ap;
    if (append_k) {  // the row lands at the end of the decoded segment, which then holds l_new rows
        FX_REQUIRE(l_new >= 1, FX_ERR_INVALID, "bad-shape: an appended row needs l_new >= 1");
        ap.kn = append_k;
        ap.vn = append_v;
        ap.row = L.l_sink + L.l_cpu + L.l_local + l_new - 1;
    }
    Layer1 l1;
    if (layer1) {
        l1.w1t = layer1[0];
        l1.b1 = layer1[1];
        l1.mu = layer1[2];
        l1.sigma = layer1[3];
        l1.a1 = a1;
    }
    double* part = static_cast<double*>(scratch);
    const bool bf = L.dtype == FX_BF16;
    if (L.head_dim == 128) {
        if (bf) launch_ff_g<__nv_bfloat16, 128>(L, k, v, l_new, q, rec, feats, part, ap, l1, num_sms, s);
        else launch_ff_g<float, 128>(L, k, v, l_new, q, rec, feats, part, ap, l1, num_sms, s);
    } else {
        if (bf) launch_ff_g<__nv_bfloat16, 64>(L, k, v, l_new, q, rec, feats, part, ap, l1, num_sms, s);
        else launch_ff_g<float, 64>(L, k, v, l_new, q, rec, feats, part, ap, l1, num_sms, s);
    }
    FX_CUDA(cudaGetLastError());
}

#ifdef FX_TRACE
extern "C" FX_API int fx_debug_fp_trace(long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_fp_trace, sizeof(long long) * n) == cudaSuccess ? 0 : -2;
}
#endif

}  // namespace fx
