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
// One segment's attention summary for the query in qs: lse and output norm
// (segment_summary, features.cpp:66-77); scores of its rows in s (by row).
template <typename T>
__device__ void seg_summary(const T* K, const T* V, int64_t r0, int n, int D, const double* qs,
                            double* s, double* red, double isd, double* lse, double* onorm) {
    const int t = threadIdx.x;
    for (int i = t; i < n; i += blockDim.x) {
        const T* kr = K + (r0 + i) * D;
        double a = 0.0;
        for (int d = 0; d < D; ++d) a += qs[d] * (double)tofl(kr[d]);
        s[i] = a * isd;
    }
    __syncthreads();
    double mx = -INFINITY;
    for (int i = t; i < n; i += blockDim.x) mx = fmax(mx, s[i]);
    const double m = block_max128(mx, red);
    double z = 0.0;
    for (int i = t; i < n; i += blockDim.x) z += exp(s[i] - m);
    const double Z = block_sum128(z, red);
    double o = 0.0;
    if (t < D)
        for (int i = 0; i < n; ++i) o += exp(s[i] - m) * (double)tofl(V[(r0 + i) * D + t]);
    o = t < D ? o / Z : 0.0;
    *onorm = sqrt(block_sum128(o * o, red));
    *lse = m + log(Z);
}

template <typename T>
__global__ void __launch_bounds__(128) k_feat(fx_layout L, const void* kp, const void* vp,
                                              int64_t l_new, const float* q, const double* rec,
                                              double* feats, double* gpu_norm) {
    extern __shared__ double sm[];
    double* qs = sm;           // [D]
    double* s = qs + L.head_dim;  // [rows of the largest default segment]
    __shared__ double red[4];
    const int64_t bg = blockIdx.x;
    const int D = L.head_dim, G = L.group_size, t = threadIdx.x;
    const int RS = kStatsN + 3 * D;
    const double isd = 1.0 / sqrt((double)D);
    const T* K = static_cast<const T*>(kp) + bg * L.l_cap * D;
    const T* V = static_cast<const T*>(vp) + bg * L.l_cap * D;
    const int64_t o_loc = L.l_sink + L.l_cpu, o_new = o_loc + L.l_local;
    for (int h = 0; h < G; ++h) {
        const int64_t head = bg * G + h;
        const double* r = rec + head * RS;
        const double* mk = r + kStatsN;
        const double* mv = mk + D;
        const double* an = mv + D;
        const float* qh = q + head * D;
        if (t < D) qs[t] = (double)qh[t];
        __syncthreads();
        // sink / local summaries (segment_summary; empty -> kEmptyLse, 0)
        double lse_s = kEmptyLseDev, on_s = 0.0, lse_l = kEmptyLseDev, on_l = 0.0;
        if (L.l_sink > 0) seg_summary(K, V, 0, (int)L.l_sink, D, qs, s, red, isd, &lse_s, &on_s);
        if (L.l_local > 0) seg_summary(K, V, o_loc, (int)L.l_local, D, qs, s, red, isd, &lse_l, &on_l);
        // gpu_output_norm: default_kv_attention over sink, local, new merged
        // (a common max over the three segments; merge_into is exact algebra)
        const int n_def = (int)(L.l_sink + L.l_local + l_new);
        double gnorm = 0.0;
        if (n_def > 0) {
            for (int i = t; i < n_def; i += blockDim.x) {
                const int64_t row = i < L.l_sink ? i : o_loc + (i - L.l_sink);
                const T* kr = K + row * D;
                double a = 0.0;
                for (int d = 0; d < D; ++d) a += qs[d] * (double)tofl(kr[d]);
                s[i] = a * isd;
            }
            __syncthreads();
            double mx = -INFINITY;
            for (int i = t; i < n_def; i += blockDim.x) mx = fmax(mx, s[i]);
            const double m = block_max128(mx, red);
            double z = 0.0;
            for (int i = t; i < n_def; i += blockDim.x) z += exp(s[i] - m);
            const double Z = block_sum128(z, red);
            double o = 0.0;
            if (t < D)
                for (int i = 0; i < n_def; ++i) {
                    const int64_t row = i < L.l_sink ? i : o_loc + (i - L.l_sink);
                    o += exp(s[i] - m) * (double)tofl(V[row * D + t]);
                }
            o = t < D ? o / Z : 0.0;
            gnorm = sqrt(block_sum128(o * o, red));
        }
        (void)o_new;
        // query-side dot products (sequential order, matrix.hpp:74-84)
        if (t == 0) {
            double* f = feats + head * kFeat;
            double qn2 = 0.0, qk = 0.0, qa = 0.0;
            for (int d = 0; d < D; ++d) {
                qn2 += qs[d] * qs[d];
                qk += qs[d] * mk[d];
                qa += qs[d] * an[d];
            }
            const double qn = sqrt(qn2);
            double nmk = 0.0, nmv = 0.0;
            for (int d = 0; d < D; ++d) {
                nmk += mk[d] * mk[d];
                nmv += mv[d] * mv[d];
            }
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
            f[21] = lse_s;
            // approx_lse_cpu (features.cpp:159-170)
            const double l_cpu = r[2];
            if (l_cpu == 0.0) f[22] = kEmptyLseDev;
            else if (qn == 0.0) f[22] = log(l_cpu);
            else {
                const double mu_q = qk / (qn * sqrt((double)D));
                f[22] = log(l_cpu) + qn * mu_q + 0.5 * qn * qn * r[17];
            }
            f[23] = lse_l;
            f[24] = r[20];
            f[25] = r[21];
            f[26] = r[22];
            f[27] = on_s;
            f[28] = on_l;
            f[29] = r[23];
            f[30] = r[24];
            f[31] = r[25];
            f[32] = qn;
            f[33] = r[31];
            f[34] = (qn > 0.0 && r[31] > 0.0) ? qa / (qn * r[31]) : 0.0;
            for (int i = 0; i < 4; ++i) f[35 + i] = r[26 + i];
            f[40] = r[30];
            gpu_norm[head] = gnorm;
        }
        __syncthreads();
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

void launch_decode_features(const fx_layout& L, const void* k, const void* v, int64_t l_new,
                            const float* q, const double* rec, double* feats, double* gpu_norm,
                            cudaStream_t s) {
    FX_REQUIRE(L.head_dim <= 128, FX_ERR_INVALID, "bad-shape: features need head_dim <= 128");
    const int64_t n_def = L.l_sink + L.l_local + l_new;
    FX_REQUIRE(n_def <= 16384, FX_ERR_INVALID, "bad-shape: more than 16384 default rows");
    const int64_t n_bg = (int64_t)L.batch * L.kv_heads;
    const size_t smem = (size_t)(L.head_dim + std::max<int64_t>(n_def, 1)) * sizeof(double);
    const bool bf = L.dtype == FX_BF16;
    if (bf) {
        FX_CUDA(cudaFuncSetAttribute(k_feat<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_feat<__nv_bfloat16><<<(unsigned)n_bg, 128, smem, s>>>(L, k, v, l_new, q, rec, feats, gpu_norm);
    } else {
        FX_CUDA(cudaFuncSetAttribute(k_feat<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_feat<float><<<(unsigned)n_bg, 128, smem, s>>>(L, k, v, l_new, q, rec, feats, gpu_norm);
    }
    FX_CUDA(cudaGetLastError());
    k_feat_cross<<<(unsigned)L.batch, 128, 0, s>>>(L.kv_heads * L.group_size, gpu_norm, feats);
    FX_CUDA(cudaGetLastError());
}

}  // namespace fx
