// fx_predict_step.cu -- decode features of every head (features.cpp:162-224)
// in ONE clustered launch; fx_predict_props then runs the tiled predictor
// (fx_plan.cu) on them: features -> normalize -> 41-256-384-3 -> head
// properties (pipeline.cpp:277-290), which the decode step plans from.
//
// One CTA per (b, g); the Hkv CTAs of a sequence form a thread-block cluster
// so feature 39 -- the maximum default-KV output norm over ALL heads of the
// sequence (features.cpp:218) -- is exchanged through distributed shared
// memory instead of a second kernel.  The default segments (sink, local,
// decoded; attention.cpp:26-55, 143-151) stream through a 2-stage ring of
// 1-D bulk copies (a chunk of K rows and of V rows: contiguous in the
// [B][Hkv][l_cap][D] cache); per chunk: warp-per-row scores (lanes split D,
// butterfly sum), per-head chunk max / weights / denominator with the
// segment's running max (online softmax), and 4 warps accumulate
// sum_r w_r v_r in registers (lanes own D/32 dims), reduced in a fixed order
// at the segment end.  Results agree with the reference within 1e-9
// relative (sums associate differently), like fx_decode_features.
#include <algorithm>

#include <cooperative_groups.h>

#include "fx_common.cuh"

namespace fx {
namespace {

namespace cg = cooperative_groups;

constexpr int kPT = 256;  // threads per CTA
constexpr int kPW = kPT / 32;
constexpr int kF = 41;
constexpr int kOW = 4;              // warps accumulating sum_r w_r v_r
constexpr double kEmptyLse = -1e6;  // kEmptyLse, features.hpp:16

template <typename T>
constexpr int chunk_rows() { return sizeof(T) == 2 ? 64 : 32; }

// f32 bits -> f64 with integer ops (exact for normal numbers: rebias the
// exponent, shift the mantissa); zero / denormal / non-finite take the F2F
// path.  F2F.F64.F32 is a low-throughput MIO instruction, and every K / V
// element of the default segments is widened once per head group.
__device__ __forceinline__ double f32bits_to_f64(uint32_t u) {
    const uint32_t e = u & 0x7f800000u;
    if (e == 0u || e == 0x7f800000u) return (double)__uint_as_float(u);
    const uint32_t hi = (u & 0x80000000u) | (((u & 0x7fffffffu) >> 3) + 0x38000000u);
    return __hiloint2double((int)hi, (int)(u << 29));
}
__device__ __forceinline__ double elem_f64(__nv_bfloat16 x) {
    return f32bits_to_f64((uint32_t)__bfloat16_as_ushort(x) << 16);
}
__device__ __forceinline__ double elem_f64(float x) { return f32bits_to_f64(__float_as_uint(x)); }

// N contiguous elements of a row (16-byte aligned slice) as f64, vector loads
template <typename T, int N>
__device__ __forceinline__ void load_row_slice(const T* p, double* out) {
    constexpr int EPV = 16 / (int)sizeof(T);
    if constexpr (N % EPV == 0) {
#pragma unroll
        for (int v = 0; v < N / EPV; ++v) {
            const uint4 w = reinterpret_cast<const uint4*>(p)[v];
            const uint32_t u[4] = {w.x, w.y, w.z, w.w};
            if constexpr (sizeof(T) == 2) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    out[v * 8 + 2 * i] = f32bits_to_f64(u[i] << 16);
                    out[v * 8 + 2 * i + 1] = f32bits_to_f64(u[i] & 0xffff0000u);
                }
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) out[v * 4 + i] = f32bits_to_f64(u[i]);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) out[i] = elem_f64(p[i]);
    }
}

#ifdef FX_TRACE  // profiling build only: per-CTA phase times
__device__ long long g_fp_trace[16 * 1024];
#define FP_MARK(i)                                                                        \
    if (threadIdx.x == 0 && blockIdx.y * gridDim.x + blockIdx.x < 1024) {                \
        long long t_;                                                                     \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
        g_fp_trace[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + (i)] = t_;                \
    }
#else
#define FP_MARK(i)
#endif

// smem bytes: ring [2][2][CR][D] T | qs [D][G] | sc [CR][G] | red [kOW][G][D] | oseg [3][G][D]
template <typename T, int G, int D>
constexpr size_t feat_smem_bytes() {
    return (size_t)2 * 2 * chunk_rows<T>() * D * sizeof(T) +
           ((size_t)D * G + (size_t)chunk_rows<T>() * G + (size_t)kOW * G * D + (size_t)3 * G * D) * 8;
}

template <typename T, int G, int D>
__global__ void __launch_bounds__(kPT, G <= 4 ? 2 : 1) k_feat_fused(fx_layout L, const void* __restrict__ kp,
                                                       const void* __restrict__ vp, int64_t l_new,
                                                       const float* __restrict__ q,
                                                       const double* __restrict__ rec,
                                                       double* __restrict__ feats) {
    constexpr int CR = chunk_rows<T>();
    constexpr size_t CHUNK = (size_t)CR * D * sizeof(T);
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(128) unsigned char fsm[];
    T* ring = reinterpret_cast<T*>(fsm);  // stage s: K rows at [s][0], V rows at [s][1]
    double* qs = reinterpret_cast<double*>(fsm + 4 * CHUNK);  // [D][G]
    double* sc = qs + D * G;                                   // [CR][G]
    double* red = sc + CR * G;                                 // [kOW][G][D]
    double* oseg = red + (size_t)kOW * G * D;                  // [3][G][D]
    __shared__ __align__(8) uint64_t full[2];
    __shared__ double s_m[8], s_z[8], s_scale[8], s_lse[3][8], s_norm[3][8], s_gn[8], s_seq_max;
    __shared__ double s_feat[8][kF];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = blockIdx.x, b = blockIdx.y;
    const int64_t bg = (int64_t)b * L.kv_heads + g;
    const T* K = static_cast<const T*>(kp) + bg * L.l_cap * D;
    const T* V = static_cast<const T*>(vp) + bg * L.l_cap * D;
    const int64_t seg_row[3] = {0, L.l_sink + L.l_cpu, L.l_sink + L.l_cpu + L.l_local};
    const int64_t seg_n[3] = {L.l_sink, L.l_local, l_new};
    const int nch0 = (int)cdiv_dev(seg_n[0], CR), nch1 = (int)cdiv_dev(seg_n[1], CR);
    const int nch = nch0 + nch1 + (int)cdiv_dev(seg_n[2], CR);
    // chunk c -> (segment, first row, rows)
    auto chunk = [&](int c, int& sg, int64_t& r0, int& nr) {
        sg = c < nch0 ? 0 : c < nch0 + nch1 ? 1 : 2;
        const int k = c - (sg == 0 ? 0 : sg == 1 ? nch0 : nch0 + nch1);
        r0 = seg_row[sg] + (int64_t)k * CR;
        nr = (int)min((int64_t)CR, seg_n[sg] - (int64_t)k * CR);
    };
    auto issue = [&](int c) {
        int sg, nr;
        int64_t r0;
        chunk(c, sg, r0, nr);
        const int st = c & 1;
        const uint32_t bytes = (uint32_t)nr * D * sizeof(T);
        mbar_arrive_expect_tx(&full[st], 2 * bytes);
        bulk_g2s(ring + (size_t)(2 * st) * CR * D, K + r0 * D, bytes, &full[st]);
        bulk_g2s(ring + (size_t)(2 * st + 1) * CR * D, V + r0 * D, bytes, &full[st]);
    };
    FP_MARK(0);
#ifdef FX_TRACE
    if (tid == 0 && blockIdx.y * gridDim.x + blockIdx.x < 1024)
        g_fp_trace[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + 14] = clock64();
#endif
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_mbar_init();
        for (int c = 0; c < 2 && c < nch; ++c) issue(c);
    }
    for (int i = tid; i < G * D; i += kPT) {
        const int h = i / D, d = i % D;
        qs[d * G + h] = (double)q[bg * G * D + i];
    }
    if (tid < G) {
        s_m[tid] = -INFINITY;
        s_z[tid] = 0.0;
    }
    __syncthreads();
    FP_MARK(1);
    const double isd = 1.0 / sqrt((double)D);
    constexpr int DV = D / 32;
    constexpr int LPR = G <= 4 ? 16 : 32, DPL = D / LPR, RPI = 32 / LPR;  // score-loop lane mapping
    const int sub = lane / LPR, sl = lane % LPR;
    double qreg[DPL][G];
#pragma unroll
    for (int j = 0; j < DPL; ++j)
#pragma unroll
        for (int h = 0; h < G; ++h) qreg[j][h] = qs[(sl * DPL + j) * G + h];
    double acc[G][DV];  // sum_r w_r v_r, lanes own DV dims (warps < kOW)
#pragma unroll
    for (int h = 0; h < G; ++h)
#pragma unroll
        for (int j = 0; j < DV; ++j) acc[h][j] = 0.0;
    for (int c = 0; c < nch; ++c) {
        int sg, nr;
        int64_t r0;
        chunk(c, sg, r0, nr);
        const int st = c & 1;
        if (c == nch0) { FP_MARK(7); }
        mbar_wait(&full[st], (uint32_t)((c >> 1) & 1));
        if (c == nch0) { FP_MARK(8); }
        const T* Ks = ring + (size_t)(2 * st) * CR * D;
        const T* Vs = ring + (size_t)(2 * st + 1) * CR * D;
        // scores: LPR lanes per row (32 / LPR rows per warp at a time), lane sl
        // owns DPL contiguous dims whose q values sit in registers (qreg);
        // one vector load of the row slice, then a butterfly per head
        for (int r0 = warp * RPI; r0 < nr; r0 += kPW * RPI) {
            const int r = r0 + sub;
            const bool live = r < nr;
            double p[G];
#pragma unroll
            for (int h = 0; h < G; ++h) p[h] = 0.0;
            const T* kr = Ks + (live ? r : r0) * D + sl * DPL;
            double kv[DPL];
            load_row_slice<T, DPL>(kr, kv);
#pragma unroll
            for (int j = 0; j < DPL; ++j)
#pragma unroll
                for (int h = 0; h < G; ++h) p[h] += qreg[j][h] * kv[j];
#pragma unroll
            for (int h = 0; h < G; ++h) {
#pragma unroll
                for (int o = LPR / 2; o > 0; o >>= 1) p[h] += __shfl_xor_sync(0xffffffffu, p[h], o);
            }
            if (live && sl < G) {
                double v = p[0];
#pragma unroll
                for (int h = 1; h < G; ++h) v = sl == h ? p[h] : v;
                sc[r * G + sl] = v * isd;
            }
        }
        __syncthreads();
        if (c == nch0) { FP_MARK(9); }
        // warp h: the chunk's weights under the segment's running max
        for (int h = warp; h < G; h += kPW) {
            double m = -INFINITY;
            for (int r = lane; r < nr; r += 32) m = fmax(m, sc[r * G + h]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            const double m_old = s_m[h], m_new = fmax(m_old, m);
            double z = 0.0;
            for (int r = lane; r < nr; r += 32) {
                const double w = exp(sc[r * G + h] - m_new);
                sc[r * G + h] = w;
                z += w;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
            __syncwarp();  // every lane has read s_m[h] before lane 0 rewrites it
            if (lane == 0) {
                const double scale = m_old == -INFINITY ? 0.0 : exp(m_old - m_new);
                s_scale[h] = scale;
                s_z[h] = s_z[h] * scale + z;
                s_m[h] = m_new;
            }
        }
        __syncthreads();
        if (c == nch0) { FP_MARK(10); }
        if (warp < kOW) {  // sum_r w_r v_r with the rescaled running sums
#pragma unroll
            for (int h = 0; h < G; ++h) {
                const double sc_h = s_scale[h];
#pragma unroll
                for (int j = 0; j < DV; ++j) acc[h][j] *= sc_h;
            }
#pragma unroll 4
            for (int r = warp; r < nr; r += kOW) {
                double vv[DV];
#pragma unroll
                for (int j = 0; j < DV; ++j) vv[j] = elem_f64(Vs[r * D + lane * DV + j]);
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    const double w = sc[r * G + h];
#pragma unroll
                    for (int j = 0; j < DV; ++j) acc[h][j] += w * vv[j];
                }
            }
        }
        __syncthreads();  // the stage and sc are free
        if (c == nch0) { FP_MARK(11); }
        if (tid == 0 && c + 2 < nch) issue(c + 2);
        int sg_next = 3;
        if (c + 1 < nch) {
            int nr2;
            int64_t r2;
            chunk(c + 1, sg_next, r2, nr2);
        }
        if (sg_next != sg) {  // segment end: fixed-order reduction, normalize, norm
            if (warp < kOW) {
#pragma unroll
                for (int h = 0; h < G; ++h)
#pragma unroll
                    for (int j = 0; j < DV; ++j) {
                        red[((size_t)warp * G + h) * D + lane * DV + j] = acc[h][j];
                        acc[h][j] = 0.0;
                    }
            }
            __syncthreads();
            double* os = oseg + (size_t)sg * G * D;
            for (int i = tid; i < G * D; i += kPT) {
                double o = 0.0;
#pragma unroll
                for (int w = 0; w < kOW; ++w) o += red[(size_t)w * G * D + i];
                os[i] = o / s_z[i / D];
            }
            __syncthreads();
            for (int h = warp; h < G; h += kPW) {
                double x = 0.0;
                for (int d = lane; d < D; d += 32) x += os[h * D + d] * os[h * D + d];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                if (lane == 0) {
                    s_norm[sg][h] = sqrt(x);
                    s_lse[sg][h] = s_m[h] + log(s_z[h]);
                    s_m[h] = -INFINITY;
                    s_z[h] = 0.0;
                }
            }
            __syncthreads();
            FP_MARK(2 + sg);
        }
    }
    // merged default output (sink, local, decoded in order, merge_into) and its norm
    for (int h = warp; h < G; h += kPW) {
        double lse = 0.0, wsg[3] = {0.0, 0.0, 0.0};
        bool any = false;
        for (int sg = 0; sg < 3; ++sg) {
            if (seg_n[sg] == 0) continue;
            if (!any) {
                lse = s_lse[sg][h];
                wsg[sg] = 1.0;
                any = true;
                continue;
            }
            const double p = s_lse[sg][h];
            const double tot = lse > p ? lse + log1p(exp(p - lse)) : p + log1p(exp(lse - p));
            const double wa = exp(lse - tot), wb = exp(p - tot);
            for (int s2 = 0; s2 < sg; ++s2) wsg[s2] *= wa;
            wsg[sg] = wb;
            lse = tot;
        }
        double x = 0.0;
        for (int d = lane; d < D; d += 32) {
            double o = 0.0;
            for (int sg = 0; sg < 3; ++sg)
                if (seg_n[sg] > 0) o += wsg[sg] * oseg[((size_t)sg * G + h) * D + d];
            x += o * o;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) s_gn[h] = any ? sqrt(x) : 0.0;
    }
    // the 41 features of each head; feature 39 after the cluster max
    const int RS = 32 + 3 * D;
    for (int h = warp; h < G; h += kPW) {
        const int64_t head = bg * G + h;
        const double* r = rec + head * RS;
        const double* mk = r + 32;
        const double* mv = mk + D;
        const double* an = mv + D;
        double qn2 = 0.0, qk = 0.0, qa = 0.0, nmk = 0.0, nmv = 0.0;
#pragma unroll
        for (int d = lane; d < D; d += 32) {
            const double qd = qs[d * G + h];
            qn2 += qd * qd;
            qk += qd * mk[d];
            qa += qd * an[d];
            nmk += mk[d] * mk[d];
            nmv += mv[d] * mv[d];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            qn2 += __shfl_xor_sync(0xffffffffu, qn2, o);
            qk += __shfl_xor_sync(0xffffffffu, qk, o);
            qa += __shfl_xor_sync(0xffffffffu, qa, o);
            nmk += __shfl_xor_sync(0xffffffffu, nmk, o);
            nmv += __shfl_xor_sync(0xffffffffu, nmv, o);
        }
        if (lane == 0) {
            double* f = s_feat[h];
            const double qn = sqrt(qn2);
            const bool cpu_empty = r[5] != 0.0;
            f[0] = r[0];
            f[1] = r[1];
            f[2] = r[2];
            f[3] = r[3] + r[4] + (double)l_new;
            f[4] = r[6];
            f[5] = r[7];
            f[6] = sqrt(nmk);
            f[7] = sqrt(nmv);
            for (int i = 0; i < 4; ++i) {
                f[8 + i] = r[8 + i];
                f[12 + i] = r[12 + i];
                f[17 + i] = r[16 + i];
            }
            f[16] = (qn > 0.0 && !cpu_empty) ? qk / (qn * sqrt((double)D)) : 0.0;
            f[21] = seg_n[0] > 0 ? s_lse[0][h] : kEmptyLse;
            const double l_cpu = r[2];  // approx_lse_cpu (features.cpp:159-170)
            if (l_cpu == 0.0) f[22] = kEmptyLse;
            else if (qn == 0.0) f[22] = log(l_cpu);
            else f[22] = log(l_cpu) + qn * (qk / (qn * sqrt((double)D))) + 0.5 * qn * qn * r[17];
            f[23] = seg_n[1] > 0 ? s_lse[1][h] : kEmptyLse;
            f[24] = r[20];
            f[25] = r[21];
            f[26] = r[22];
            f[27] = seg_n[0] > 0 ? s_norm[0][h] : 0.0;
            f[28] = seg_n[1] > 0 ? s_norm[1][h] : 0.0;
            f[29] = r[23];
            f[30] = r[24];
            f[31] = r[25];
            f[32] = qn;
            f[33] = r[31];
            f[34] = (qn > 0.0 && r[31] > 0.0) ? qa / (qn * r[31]) : 0.0;
            for (int i = 0; i < 4; ++i) f[35 + i] = r[26 + i];
            f[40] = r[30];
        }
    }
    __syncthreads();
    FP_MARK(5);
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
    cluster.sync();  // the peers' reads are done before any CTA moves on and exits
    for (int i = tid; i < G * kF; i += kPT) feats[(bg * G + i / kF) * kF + i % kF] = s_feat[i / kF][i % kF];
    FP_MARK(6);
#ifdef FX_TRACE
    if (tid == 0 && blockIdx.y * gridDim.x + blockIdx.x < 1024)
        g_fp_trace[(blockIdx.y * gridDim.x + blockIdx.x) * 16 + 15] = clock64();
#endif
}

template <typename T, int G, int D>
void launch_ff(const fx_layout& L, const void* k, const void* v, int64_t l_new, const float* q,
               const double* rec, double* feats, cudaStream_t s) {
    const size_t smem = feat_smem_bytes<T, G, D>();
    FX_CUDA(cudaFuncSetAttribute(k_feat_fused<T, G, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)L.kv_heads, (unsigned)L.batch);
    cfg.blockDim = dim3(kPT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)L.kv_heads;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FX_CUDA(cudaLaunchKernelEx(&cfg, k_feat_fused<T, G, D>, L, k, v, l_new, q, rec, feats));
}

template <typename T, int D>
void launch_ff_g(const fx_layout& L, const void* k, const void* v, int64_t l_new, const float* q,
                 const double* rec, double* feats, cudaStream_t s) {
    switch (L.group_size) {
#define FX_FG(GG)                                                  \
    case GG:                                                       \
        launch_ff<T, GG, D>(L, k, v, l_new, q, rec, feats, s);     \
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

void launch_feat_fused(const fx_layout& L, const void* k, const void* v, int64_t l_new, const float* q,
                       const double* rec, double* feats, cudaStream_t s) {
    FX_REQUIRE(feat_fused_supported(L), FX_ERR_INVALID,
               "bad-shape: fused features need G in {1,2,4,7,8}, head_dim 64/128 and kv_heads <= 8");
    const bool bf = L.dtype == FX_BF16;
    if (L.head_dim == 128) {
        if (bf) launch_ff_g<__nv_bfloat16, 128>(L, k, v, l_new, q, rec, feats, s);
        else launch_ff_g<float, 128>(L, k, v, l_new, q, rec, feats, s);
    } else {
        if (bf) launch_ff_g<__nv_bfloat16, 64>(L, k, v, l_new, q, rec, feats, s);
        else launch_ff_g<float, 64>(L, k, v, l_new, q, rec, feats, s);
    }
    FX_CUDA(cudaGetLastError());
}

#ifdef FX_TRACE
extern "C" FX_API int fx_debug_fp_trace(long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_fp_trace, sizeof(long long) * n) == cudaSuccess ? 0 : -2;
}
#endif

}  // namespace fx
