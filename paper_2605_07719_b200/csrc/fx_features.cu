// fx_features.cu -- predictor inputs on the device (features.cpp:26-224).
//
// Prefill (once per layer, features.cpp:86-157): the KV-only fields of the
// PrefillStats record -- cpu-segment mean key / value vectors, moments of the
// cpu key / value row norms, mean sink row norms -- from two streaming passes
// over the cpu rows of every group (f64 sums, then central powers about the
// pass-1 mean, like compute_moments).  The anchor-side fields come from the
// label pipeline (fx_label.cu, k_pf_anchor).
//
// Decode (every step, features.cpp:172-224): one CTA per (b, g) attends each
// head's query over the sink, local and decoded rows only (the cpu segment is
// summarized by the record: approx_lse_cpu), writes the 41 features, and the
// default-KV output norm that feeds the cross-head maximum; a second small
// kernel writes that maximum (feature 39) for every head of the sequence.
#include <algorithm>

#include "fx_common.cuh"

namespace fx {
namespace {

constexpr int kFeat = 41;

__device__ double block_sum128(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += red[i];
    return s;
}
__device__ double block_max128(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = -INFINITY;
    for (int i = 0; i < nw; ++i) s = fmax(s, red[i]);
    return s;
}

// l2_norm of one stored row (matrix.hpp:80-84): sequential f64 sum of squares.
template <typename T>
__device__ double row_norm(const T* r, int D) {
    double s = 0.0;
    for (int d = 0; d < D; ++d) {
        const double x = (double)tofl(r[d]);
        s += x * x;
    }
    return sqrt(s);
}

// per-(b, g) accumulators: sum_k[D] sum_v[D] | nk nv sk sv | ck[3] cv[3]
struct GroupAcc {
    double* a;
    int D;
    __device__ double* sum_k(int64_t bg) const { return a + bg * (2 * D + 10); }
    __device__ double* sum_v(int64_t bg) const { return sum_k(bg) + D; }
    __device__ double* misc(int64_t bg) const { return sum_k(bg) + 2 * D; }
};

// pass 1: column sums over the cpu rows, row-norm sums over cpu and sink rows
template <typename T>
__global__ void __launch_bounds__(128) k_pfg_pass1(fx_layout L, const void* kp, const void* vp,
                                                   GroupAcc acc) {
    __shared__ double red[4];
    const int64_t bg = blockIdx.y;
    const int D = L.head_dim, t = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * 128, n = L.l_sink + L.l_cpu;
    const int nrow = (int)min((int64_t)128, n - r0);
    const T* K = static_cast<const T*>(kp) + (bg * L.l_cap + r0) * D;
    const T* V = static_cast<const T*>(vp) + (bg * L.l_cap + r0) * D;
    double nk = 0.0, nv = 0.0, sk = 0.0, sv = 0.0;
    if (t < nrow) {
        const double a = row_norm(K + (int64_t)t * D, D), b = row_norm(V + (int64_t)t * D, D);
        if (r0 + t < L.l_sink) {
            sk = a;
            sv = b;
        } else {
            nk = a;
            nv = b;
        }
    }
    double* m = acc.misc(bg);
    const double tk = block_sum128(nk, red), tv = block_sum128(nv, red);
    const double ts = block_sum128(sk, red), tw = block_sum128(sv, red);
    if (t == 0) {
        if (tk != 0.0) atomicAdd(m + 0, tk);
        if (tv != 0.0) atomicAdd(m + 1, tv);
        if (ts != 0.0) atomicAdd(m + 2, ts);
        if (tw != 0.0) atomicAdd(m + 3, tw);
    }
    if (t < D) {
        double ck = 0.0, cv = 0.0;
        for (int i = 0; i < nrow; ++i)
            if (r0 + i >= L.l_sink) {
                ck += (double)tofl(K[(int64_t)i * D + t]);
                cv += (double)tofl(V[(int64_t)i * D + t]);
            }
        if (ck != 0.0) atomicAdd(acc.sum_k(bg) + t, ck);
        if (cv != 0.0) atomicAdd(acc.sum_v(bg) + t, cv);
    }
}

// pass 2: central powers of the cpu row norms about the pass-1 means
template <typename T>
__global__ void __launch_bounds__(128) k_pfg_pass2(fx_layout L, const void* kp, const void* vp,
                                                   GroupAcc acc) {
    __shared__ double red[4];
    const int64_t bg = blockIdx.y;
    const int D = L.head_dim, t = threadIdx.x;
    const int64_t r0 = L.l_sink + (int64_t)blockIdx.x * 128;
    const int nrow = (int)min((int64_t)128, L.l_sink + L.l_cpu - r0);
    double* m = acc.misc(bg);
    const double mk = m[0] / (double)L.l_cpu, mv = m[1] / (double)L.l_cpu;
    double c[6] = {0, 0, 0, 0, 0, 0};
    if (t < nrow) {
        const T* K = static_cast<const T*>(kp) + (bg * L.l_cap + r0 + t) * D;
        const T* V = static_cast<const T*>(vp) + (bg * L.l_cap + r0 + t) * D;
        const double dk = row_norm(K, D) - mk, dv = row_norm(V, D) - mv;
        c[0] = dk * dk;
        c[1] = c[0] * dk;
        c[2] = c[0] * c[0];
        c[3] = dv * dv;
        c[4] = c[3] * dv;
        c[5] = c[3] * c[3];
    }
    for (int i = 0; i < 6; ++i) {
        const double s = block_sum128(c[i], red);
        if (t == 0 && s != 0.0) atomicAdd(m + 4 + i, s);
    }
}

// compute_moments from (mean, central power sums) (features.cpp:26-46)
__device__ void moments_of(double mean, double s2, double s3, double s4, double n, double* out) {
    const double m2 = s2 / n, m3 = s3 / n, m4 = s4 / n;
    out[0] = mean;
    out[1] = m2;
    out[2] = m2 > 0.0 ? m3 / pow(m2, 1.5) : 0.0;
    out[3] = m2 > 0.0 ? m4 / (m2 * m2) - 3.0 : 0.0;
}

// KV-only record fields for every head of the group
__global__ void __launch_bounds__(128) k_pfg_write(fx_layout L, GroupAcc acc, double* rec) {
    const int64_t bg = blockIdx.x;
    const int D = L.head_dim, G = L.group_size, t = threadIdx.x;
    const int RS = kStatsN + 3 * D;
    const double* m = acc.misc(bg);
    const double n = (double)L.l_cpu;
    for (int h = 0; h < G; ++h) {
        double* r = rec + (bg * G + h) * RS;
        if (t < D) {
            r[kStatsN + t] = L.l_cpu > 0 ? acc.sum_k(bg)[t] / n : 0.0;
            r[kStatsN + D + t] = L.l_cpu > 0 ? acc.sum_v(bg)[t] / n : 0.0;
        }
        if (t == 0) {
            r[6] = L.l_sink > 0 ? m[2] / (double)L.l_sink : 0.0;
            r[7] = L.l_sink > 0 ? m[3] / (double)L.l_sink : 0.0;
            if (L.l_cpu > 0) {
                moments_of(m[0] / n, m[4], m[5], m[6], n, r + 8);
                moments_of(m[1] / n, m[7], m[8], m[9], n, r + 12);
            } else {
                for (int i = 8; i < 16; ++i) r[i] = 0.0;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// decode features
// ---------------------------------------------------------------------------
// One CTA (256 threads) per (b, g), all G heads at once.  Each default
// segment (sink, local, decoded) streams through shared memory 64 rows at a
// time (K and V chunk as f32); scores for every (row, head) pair in f64,
// online softmax per (head, segment), sum e v per (head, dimension).  The
// segment partials give the sink / local summaries (segment_summary,
// features.cpp:66-77) and, LSE-merged, default_kv_attention's output norm
// (gpu_output_norm, features.cpp:81-84).  Sums associate differently from the
// reference's sequential loops (~1e-16 relative).
constexpr int kFT = 256, kFC = 64, kFMaxG = 8;

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float* f) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = bf16lo_to_f(w[i]);
        f[2 * i + 1] = bf16hi_to_f(w[i]);
    }
}
__device__ __forceinline__ void ld8(const float* p, float* f) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

// Chunk partials: one CTA per (64-row chunk of a default segment, group):
// m[h] = max score, z[h] = sum exp(s - m), o[h][d] = sum exp(s - m) v[d].
struct FeatChunks {
    int n_sink, n_local, n_new, n;  // chunks per segment, total per group
    double* m;                      // [n_bg][n][G]
    double* z;                      // [n_bg][n][G]
    double* o;                      // [n_bg][n][G][D]
};
__device__ __forceinline__ void chunk_seg(const FeatChunks& c, int ci, int* sg, int* k) {
    if (ci < c.n_sink) { *sg = 0; *k = ci; }
    else if (ci < c.n_sink + c.n_local) { *sg = 1; *k = ci - c.n_sink; }
    else { *sg = 2; *k = ci - c.n_sink - c.n_local; }
}

template <typename T>
__device__ __forceinline__ void unpack8(const T* p, float* f);
template <>
__device__ __forceinline__ void unpack8<__nv_bfloat16>(const __nv_bfloat16* p, float* f) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = bf16lo_to_f(w[i]);
        f[2 * i + 1] = bf16hi_to_f(w[i]);
    }
}
template <>
__device__ __forceinline__ void unpack8<float>(const float* p, float* f) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

// K and V of the chunk are staged raw (16-byte copies, rows padded by 16 bytes
// so the score loop's row-parallel 16-byte reads hit distinct banks); q is
// stored [D][G] in f64 so the G heads of one dimension are adjacent words.
template <typename T>
__global__ void __launch_bounds__(kFT) k_feat_chunk(fx_layout L, const void* kp, const void* vp,
                                                    int64_t l_new, const float* q, FeatChunks fc) {
    extern __shared__ __align__(16) unsigned char fsm[];
    const int D = L.head_dim, G = L.group_size, t = threadIdx.x;
    const int pitch = D + 16 / (int)sizeof(T);             // elements per staged row
    T* Ks = reinterpret_cast<T*>(fsm);                      // [kFC][pitch]
    T* Vs = Ks + kFC * pitch;                               // [kFC][pitch]
    double* qs = reinterpret_cast<double*>(Vs + kFC * pitch);  // [D][G]
    double* sc = qs + G * D;                                // [kFC][G] scores, then weights
    __shared__ double cm[kFMaxG];
    const int ci = blockIdx.x;
    const int64_t bg = blockIdx.y;
    int sg, k;
    chunk_seg(fc, ci, &sg, &k);
    const int64_t r0 = sg == 0 ? 0 : sg == 1 ? L.l_sink + L.l_cpu : L.l_sink + L.l_cpu + L.l_local;
    const int64_t sn = sg == 0 ? L.l_sink : sg == 1 ? L.l_local : l_new;
    const int64_t c0 = (int64_t)k * kFC;
    const int nr = (int)min((int64_t)kFC, sn - c0);
    const double isd = 1.0 / sqrt((double)D);
    const T* K = static_cast<const T*>(kp) + (bg * L.l_cap + r0 + c0) * D;
    const T* V = static_cast<const T*>(vp) + (bg * L.l_cap + r0 + c0) * D;
    for (int i = t; i < G * D; i += kFT) {
        const int h = i / D, d = i % D;
        qs[d * G + h] = (double)q[bg * G * D + i];
    }
    const int vpr = D * (int)sizeof(T) / 16;  // 16-byte vectors per row
    for (int i = t; i < nr * vpr; i += kFT) {
        const int r = i / vpr, c = i % vpr;
        const uint4 kx = __ldg(reinterpret_cast<const uint4*>(K + (int64_t)r * D) + c);
        const uint4 vx = __ldg(reinterpret_cast<const uint4*>(V + (int64_t)r * D) + c);
        *reinterpret_cast<uint4*>(Ks + r * pitch + c * (16 / (int)sizeof(T))) = kx;
        *reinterpret_cast<uint4*>(Vs + r * pitch + c * (16 / (int)sizeof(T))) = vx;
    }
    __syncthreads();
    for (int pr = t; pr < nr * G; pr += kFT) {  // one (row, head) score per thread
        const int r = pr / G, h = pr % G;
        const T* kr = Ks + r * pitch;
        double a = 0.0;
        for (int d0 = 0; d0 < D; d0 += 8) {
            float f[8];
            unpack8<T>(kr + d0, f);
#pragma unroll
            for (int u = 0; u < 8; ++u) a += qs[(d0 + u) * G + h] * (double)f[u];
        }
        sc[r * G + h] = a * isd;
    }
    __syncthreads();
    if (t < G) {
        double mx = -INFINITY;
        for (int r = 0; r < nr; ++r) mx = fmax(mx, sc[r * G + t]);
        cm[t] = mx;
    }
    __syncthreads();
    for (int pr = t; pr < nr * G; pr += kFT) sc[pr] = exp(sc[pr] - cm[pr % G]);
    __syncthreads();
    const int64_t slot = (bg * fc.n + ci) * G;
    if (t < G) {
        double z = 0.0;
        for (int r = 0; r < nr; ++r) z += sc[r * G + t];
        fc.m[slot + t] = cm[t];
        fc.z[slot + t] = z;
    }
    for (int i = t; i < G * D; i += kFT) {
        const int h = i / D, d = i % D;
        double a = 0.0;
        for (int r = 0; r < nr; ++r) a += sc[r * G + h] * (double)tofl(Vs[r * pitch + d]);
        fc.o[(slot + h) * D + d] = a;
    }
}

// Per group: merge the chunk partials of each segment, then the features.
__global__ void __launch_bounds__(kFT) k_feat(fx_layout L, int64_t l_new, const float* q,
                                              const double* rec, FeatChunks fc, double* feats,
                                              double* gpu_norm) {
    extern __shared__ __align__(16) unsigned char fsm[];
    const int D = L.head_dim, G = L.group_size, t = threadIdx.x;
    double* qs = reinterpret_cast<double*>(fsm);  // [G][D]
    double* part_o = qs + G * D;                  // [3][G][D] segment outputs (sum e v)
    double* cw = part_o + 3 * G * D;              // [n chunks][G] exp(m_chunk - m_segment)
    __shared__ double seg_m[3][kFMaxG], seg_z[3][kFMaxG];
    const int64_t bg = blockIdx.x;
    const int RS = kStatsN + 3 * D;
    for (int i = t; i < G * D; i += kFT) qs[i] = (double)q[bg * G * D + i];
    const int64_t seg_n[3] = {L.l_sink, L.l_local, l_new};
    const int first[3] = {0, fc.n_sink, fc.n_sink + fc.n_local};
    const int cnt[3] = {fc.n_sink, fc.n_local, fc.n_new};
    if (t < 3 * G) {  // segment max and denominator over its chunks
        const int sg = t / G, h = t % G;
        double m = -INFINITY;
        for (int c = 0; c < cnt[sg]; ++c) m = fmax(m, fc.m[(bg * fc.n + first[sg] + c) * G + h]);
        double z = 0.0;
        for (int c = 0; c < cnt[sg]; ++c) {
            const int64_t sl = (bg * fc.n + first[sg] + c) * G + h;
            z += fc.z[sl] * exp(fc.m[sl] - m);
        }
        seg_m[sg][h] = m;
        seg_z[sg][h] = z;
    }
    __syncthreads();
    for (int i = t; i < fc.n * G; i += kFT) {  // chunk weights, once per (chunk, head)
        const int c = i / G, h = i % G;
        const int sg = c < fc.n_sink ? 0 : c < fc.n_sink + fc.n_local ? 1 : 2;
        cw[i] = exp(fc.m[(bg * fc.n + c) * G + h] - seg_m[sg][h]);
    }
    __syncthreads();
    for (int i = t; i < 3 * G * D; i += kFT) {
        const int sg = i / (G * D), h = (i / D) % G, d = i % D;
        double a = 0.0;
        for (int c = first[sg]; c < first[sg] + cnt[sg]; ++c)
            a += fc.o[((bg * fc.n + c) * G + h) * D + d] * cw[c * G + h];
        part_o[i] = a;
    }
    __syncthreads();
    // per head (one warp each, no block barriers): segment summaries, merged
    // default norm, record-derived features
    const int lane = t & 31;
    for (int h = t >> 5; h < G; h += kFT / 32) {
        const int64_t head = bg * G + h;
        const double* r = rec + head * RS;
        const double* mk = r + kStatsN;
        const double* mv = mk + D;
        const double* an = mv + D;
        const double* qh = qs + h * D;
        double on[2], mz = -INFINITY;
        for (int sg = 0; sg < 3; ++sg) mz = seg_n[sg] > 0 ? fmax(mz, seg_m[sg][h]) : mz;
        double zt = 0.0, wsg[3];
        for (int sg = 0; sg < 3; ++sg) {
            wsg[sg] = seg_n[sg] > 0 ? exp(seg_m[sg][h] - mz) : 0.0;
            zt += wsg[sg] * seg_z[sg][h];
        }
        double x0 = 0.0, x1 = 0.0, xg = 0.0, qn2 = 0.0, qk = 0.0, qa = 0.0, nmk = 0.0, nmv = 0.0;
        for (int d = lane; d < D; d += 32) {
            const double o0 = seg_n[0] > 0 ? part_o[h * D + d] / seg_z[0][h] : 0.0;
            const double o1 = seg_n[1] > 0 ? part_o[G * D + h * D + d] / seg_z[1][h] : 0.0;
            double og = 0.0;
            for (int sg = 0; sg < 3; ++sg) og += wsg[sg] * part_o[sg * G * D + h * D + d];
            og = zt > 0.0 ? og / zt : 0.0;
            x0 += o0 * o0;
            x1 += o1 * o1;
            xg += og * og;
            qn2 += qh[d] * qh[d];
            qk += qh[d] * mk[d];
            qa += qh[d] * an[d];
            nmk += mk[d] * mk[d];
            nmv += mv[d] * mv[d];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            x0 += __shfl_xor_sync(0xffffffffu, x0, o);
            x1 += __shfl_xor_sync(0xffffffffu, x1, o);
            xg += __shfl_xor_sync(0xffffffffu, xg, o);
            qn2 += __shfl_xor_sync(0xffffffffu, qn2, o);
            qk += __shfl_xor_sync(0xffffffffu, qk, o);
            qa += __shfl_xor_sync(0xffffffffu, qa, o);
            nmk += __shfl_xor_sync(0xffffffffu, nmk, o);
            nmv += __shfl_xor_sync(0xffffffffu, nmv, o);
        }
        on[0] = sqrt(x0);
        on[1] = sqrt(x1);
        const double gn = sqrt(xg);
        if (lane == 0) {
            double* f = feats + head * kFeat;
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
            f[21] = seg_n[0] > 0 ? seg_m[0][h] + log(seg_z[0][h]) : kEmptyLseDev;
            // approx_lse_cpu (features.cpp:159-170)
            const double l_cpu = r[2];
            if (l_cpu == 0.0) f[22] = kEmptyLseDev;
            else if (qn == 0.0) f[22] = log(l_cpu);
            else {
                const double mu_q = qk / (qn * sqrt((double)D));
                f[22] = log(l_cpu) + qn * mu_q + 0.5 * qn * qn * r[17];
            }
            f[23] = seg_n[1] > 0 ? seg_m[1][h] + log(seg_z[1][h]) : kEmptyLseDev;
            f[24] = r[20];
            f[25] = r[21];
            f[26] = r[22];
            f[27] = seg_n[0] > 0 ? on[0] : 0.0;
            f[28] = seg_n[1] > 0 ? on[1] : 0.0;
            f[29] = r[23];
            f[30] = r[24];
            f[31] = r[25];
            f[32] = qn;
            f[33] = r[31];
            f[34] = (qn > 0.0 && r[31] > 0.0) ? qa / (qn * r[31]) : 0.0;
            for (int i = 0; i < 4; ++i) f[35 + i] = r[26 + i];
            f[40] = r[30];
            gpu_norm[head] = zt > 0.0 ? gn : 0.0;
        }
    }
}

// feature 39: max_h gpu_output_norm over the heads of sequence b
__global__ void k_feat_cross(int H, const double* gpu_norm, double* feats) {
    __shared__ double red[4];
    const int b = blockIdx.x;
    double m = 0.0;
    for (int h = threadIdx.x; h < H; h += blockDim.x) m = fmax(m, gpu_norm[(int64_t)b * H + h]);
    m = block_max128(m, red);
    for (int h = threadIdx.x; h < H; h += blockDim.x) feats[((int64_t)b * H + h) * kFeat + 39] = m;
}

}  // namespace

size_t prefill_group_scratch_bytes(const fx_layout& L) {
    return (size_t)L.batch * L.kv_heads * (2 * L.head_dim + 10) * sizeof(double);
}

void launch_prefill_group(const fx_layout& L, const void* k, const void* v, double* rec,
                          void* scratch, cudaStream_t s) {
    const int64_t n_bg = (int64_t)L.batch * L.kv_heads;
    GroupAcc acc{static_cast<double*>(scratch), L.head_dim};
    FX_CUDA(cudaMemsetAsync(scratch, 0, prefill_group_scratch_bytes(L), s));
    const bool bf = L.dtype == FX_BF16;
    if (L.l_sink + L.l_cpu > 0) {
        const dim3 g((unsigned)cdiv(L.l_sink + L.l_cpu, 128), (unsigned)n_bg);
        if (bf) k_pfg_pass1<__nv_bfloat16><<<g, 128, 0, s>>>(L, k, v, acc);
        else k_pfg_pass1<float><<<g, 128, 0, s>>>(L, k, v, acc);
        FX_CUDA(cudaGetLastError());
    }
    if (L.l_cpu > 0) {
        const dim3 g((unsigned)cdiv(L.l_cpu, 128), (unsigned)n_bg);
        if (bf) k_pfg_pass2<__nv_bfloat16><<<g, 128, 0, s>>>(L, k, v, acc);
        else k_pfg_pass2<float><<<g, 128, 0, s>>>(L, k, v, acc);
        FX_CUDA(cudaGetLastError());
    }
    k_pfg_write<<<(unsigned)n_bg, 128, 0, s>>>(L, acc, rec);
    FX_CUDA(cudaGetLastError());
}

size_t decode_features_scratch_bytes(const fx_layout& L, int64_t l_new) {
    const int64_t n_bg = (int64_t)L.batch * L.kv_heads;
    const int64_t n = cdiv(L.l_sink, kFC) + cdiv(L.l_local, kFC) + cdiv(l_new, kFC);
    return (size_t)(n_bg * n * L.group_size * (L.head_dim + 2) + n_bg * L.group_size + 64) * 8;
}

void launch_decode_features(const fx_layout& L, const void* k, const void* v, int64_t l_new,
                            const float* q, const double* rec, double* feats, void* scratch,
                            cudaStream_t s) {
    FX_REQUIRE(L.head_dim <= 256 && L.head_dim % 8 == 0 && L.group_size <= kFMaxG, FX_ERR_INVALID,
               "bad-shape: features need head_dim <= 256 (multiple of 8) and group_size <= 8");
    const int64_t n_bg = (int64_t)L.batch * L.kv_heads;
    const int D = L.head_dim, G = L.group_size;
    FeatChunks fc;
    fc.n_sink = (int)cdiv(L.l_sink, kFC);
    fc.n_local = (int)cdiv(L.l_local, kFC);
    fc.n_new = (int)cdiv(l_new, kFC);
    fc.n = fc.n_sink + fc.n_local + fc.n_new;
    double* w = static_cast<double*>(scratch);
    double* gpu_norm = w;
    fc.m = gpu_norm + n_bg * G;
    fc.z = fc.m + n_bg * fc.n * G;
    fc.o = fc.z + n_bg * fc.n * G;
    const bool bf = L.dtype == FX_BF16;
    if (fc.n > 0) {
        const size_t es = L.dtype == FX_BF16 ? 2 : 4;
        const size_t smem = 2 * (size_t)kFC * ((size_t)D * es + 16) + (size_t)G * D * 8 +
                            (size_t)kFC * G * 8 + 16;
        const dim3 grid((unsigned)fc.n, (unsigned)n_bg);
        if (bf) {
            FX_CUDA(cudaFuncSetAttribute(k_feat_chunk<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_feat_chunk<__nv_bfloat16><<<grid, kFT, smem, s>>>(L, k, v, l_new, q, fc);
        } else {
            FX_CUDA(cudaFuncSetAttribute(k_feat_chunk<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_feat_chunk<float><<<grid, kFT, smem, s>>>(L, k, v, l_new, q, fc);
        }
        FX_CUDA(cudaGetLastError());
    }
    const size_t smem2 = (size_t)G * D * 8 + (size_t)3 * G * D * 8 + (size_t)fc.n * G * 8 + 16;
    FX_CUDA(cudaFuncSetAttribute(k_feat, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    k_feat<<<(unsigned)n_bg, kFT, smem2, s>>>(L, l_new, q, rec, fc, feats, gpu_norm);
    FX_CUDA(cudaGetLastError());
    k_feat_cross<<<(unsigned)L.batch, 128, 0, s>>>(L.kv_heads * L.group_size, gpu_norm, feats);
    FX_CUDA(cudaGetLastError());
}

}  // namespace fx
