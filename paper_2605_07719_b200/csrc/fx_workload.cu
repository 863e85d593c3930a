// fx_workload.cu -- the reference's synthetic workload generator
// (generate(spec), workload.cpp:154-308) with the bulk on the device.
//
// The reference draws every K and V element of a group from one SplitMix64
// stream (rng.hpp): element e = i*d + j takes the draws 4e+1 .. 4e+4 after the
// group stream's start (k: Box-Muller of draws 4e+1, 4e+2; v: 4e+3, 4e+4).
// SplitMix64 is a counter generator (state_n = state_0 + n*gamma), so the
// device fills [B][Hkv][L][D] in parallel, one thread per element pair.
// Everything that is O(d) per head -- archetype shuffle, local direction,
// needle / decoy directions and payload values, anchor and decode queries,
// decoded rows -- runs on the host in the reference's draw order (the stream
// is advanced past the bulk in O(1)) and reaches the device as an ordered
// patch list per group (row-range adds / sets / scales, applied in the
// reference's head order) plus the query and decoded-row arrays.
//
// Parity: host values are bit-identical to the reference (same libm, no
// contraction).  The bulk's Box-Muller uses CUDA's f64 log / cos / sqrt, which
// may differ from glibc in the last f64 ulp; after the f32 rounding an element
// can then differ by one f32 ulp, with probability ~1e-9 per element
// (tests/test_workload.py counts these against the compiled reference).
#include <algorithm>
#include <cmath>

#include <vector>

#include "fx_common.cuh"

namespace fx {
namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// SplitMix64 with the reference's fork / uniform / normal (rng.hpp).
struct Rng {
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() { return mix64(s += kGamma); }
    Rng fork(uint64_t stream) const {
        Rng r(s ^ (0xd1b54a32d192ed03ULL * (stream + 1)));
        r.next();
        return r;
    }
    double uniform() { return double(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double normal() {
        double u1 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);  // pi: std::numbers::pi
    }
    void skip(uint64_t n) { s += n * kGamma; }
};

double l2(const std::vector<float>& v) {
    double s = 0.0;
    for (float x : v) s += double(x) * double(x);
    return std::sqrt(s);
}
std::vector<float> unit_vec(Rng& r, size_t d) {
    std::vector<float> v(d);
    for (auto& x : v) x = float(r.normal());
    const double n = l2(v);
    for (auto& x : v) x = float(double(x) / n);
    return v;
}
std::vector<float> mix_direction(Rng& r, const std::vector<float>& base, double j) {
    const std::vector<float> n = unit_vec(r, base.size());
    const double a = std::sqrt(std::max(0.0, 1.0 - j * j));
    std::vector<float> v(base.size());
    for (size_t i = 0; i < v.size(); ++i) v[i] = float(a * base[i] + j * n[i]);
    const double nn = l2(v);
    for (auto& x : v) x = float(double(x) / nn);
    return v;
}
void scale_to(std::vector<float>& v, double target) {
    const double n = l2(v);
    for (auto& x : v) x = float(double(x) * target / n);
}

enum { kStreaming = 0, kRetrieval = 1, kSinkDecoy = 2, kDiffuse = 3 };
std::vector<int> layer_archetypes(const fx_workload_spec& sp, Rng& r) {
    const int h = sp.heads;
    auto count = [&](double f) { return int(std::lround(f * h)); };
    std::vector<int> a;
    for (int i = 0; i < count(sp.streaming_frac); ++i) a.push_back(kStreaming);
    for (int i = 0; i < count(sp.retrieval_frac); ++i) a.push_back(kRetrieval);
    for (int i = 0; i < count(sp.sink_frac); ++i) a.push_back(kSinkDecoy);
    while (int(a.size()) < h) a.push_back(kDiffuse);
    a.resize(size_t(h));
    for (size_t i = a.size(); i > 1; --i) std::swap(a[i - 1], a[r.next() % i]);  // Rng::shuffle
    return a;
}

// patches: op 0 = k[rows] += vec (float adds), 1 = v[rows] = data, 2 = v[rows] *= 0.1f
struct Patch {
    int32_t bg, op, r0, r1;
    int64_t data;  // offset into the patch data (floats)
};

__device__ __forceinline__ float box_muller(uint64_t a, uint64_t b) {
    double u1 = double(a >> 11) * 0x1.0p-53;
    const double u2 = double(b >> 11) * 0x1.0p-53;
    u1 = u1 > 0.0 ? u1 : 0x1.0p-53;  // the reference redraws on 0 (probability 2^-53)
    return float(sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2));
}

template <typename T>
__global__ void k_gen_bulk(int64_t rows, int D, int64_t l_cap, const uint64_t* __restrict__ state,
                           T* __restrict__ k, T* __restrict__ v) {
    const int64_t bg = blockIdx.y;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * D) return;
    const uint64_t s0 = state[bg];
    const uint64_t base = s0 + (uint64_t)(4 * e) * kGamma;
    const float kv = box_muller(mix64(base + 1 * kGamma), mix64(base + 2 * kGamma));
    const float vv = box_muller(mix64(base + 3 * kGamma), mix64(base + 4 * kGamma));
    const int64_t i = e / D, j = e % D;
    k[(bg * l_cap + i) * D + j] = (T)kv;
    v[(bg * l_cap + i) * D + j] = (T)vv;
}

// One CTA per group applies its patches in order (the reference's head order).
template <typename T>
__global__ void k_gen_patch(const Patch* __restrict__ patches, const int32_t* __restrict__ first,
                            const float* __restrict__ data, int D, int64_t l_cap, T* k, T* v) {
    const int bg = blockIdx.x;
    for (int p = first[bg]; p < first[bg + 1]; ++p) {
        const Patch P = patches[p];
        const int64_t n = (int64_t)(P.r1 - P.r0) * D;
        for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
            const int64_t i = P.r0 + e / D, j = e % D;
            const int64_t o = ((int64_t)bg * l_cap + i) * D + j;
            if (P.op == 0) k[o] = (T)((float)k[o] + data[P.data + j]);
            else if (P.op == 1) v[o] = (T)data[P.data + e];
            else v[o] = (T)((float)v[o] * 0.1f);
        }
        __syncthreads();
    }
}

}  // namespace

void generate_workload(const fx_layout& L, const fx_workload_spec& sp, const uint64_t* seeds,
                       const int32_t* layers, void* k, void* v, float* anchor_q, int32_t steps,
                       float* step_q, float* step_new_k, float* step_new_v, int32_t* archetypes,
                       void* scratch_alloc(size_t, void*), void* alloc_ctx, cudaStream_t s) {
    const int B = L.batch, Hkv = L.kv_heads, G = L.group_size, D = L.head_dim, H = Hkv * G;
    const size_t d = (size_t)D;
    const size_t l = (size_t)sp.context_len;
    const size_t l_cpu = l - (size_t)sp.sink_tokens - (size_t)sp.local_tokens;
    const size_t cpu0 = (size_t)sp.sink_tokens, local0 = cpu0 + l_cpu;
    const double qnorm = std::sqrt(double(d));
    std::vector<uint64_t> state((size_t)B * Hkv);
    std::vector<Patch> patches;
    std::vector<int32_t> first;
    std::vector<float> data;
    std::vector<float> hq((size_t)B * H * d), hsq((size_t)std::max(steps, 0) * B * H * d);
    std::vector<float> hnk((size_t)std::max(steps, 0) * B * Hkv * d), hnv(hnk.size());
    for (int b = 0; b < B; ++b) {
        Rng base(seeds[b]);
        Rng rng_l = base.fork((uint64_t)layers[b]);
        const std::vector<int> arch = layer_archetypes(sp, rng_l);
        if (archetypes)
            for (int h = 0; h < H; ++h) archetypes[(size_t)b * H + h] = arch[(size_t)h];
        for (int g = 0; g < Hkv; ++g) {
            const int bg = b * Hkv + g;
            first.push_back((int32_t)patches.size());
            Rng rng = rng_l.fork((uint64_t)g + 1000);
            state[(size_t)bg] = rng.s;
            rng.skip((uint64_t)4 * l * d);  // past the bulk K/V draws
            const int h0 = g * G;
            bool has_streaming = false;
            for (int hg = 0; hg < G; ++hg) has_streaming |= arch[(size_t)(h0 + hg)] == kStreaming;
            const std::vector<float> w_local = unit_vec(rng, d);
            auto add_k = [&](size_t r0, size_t r1, const std::vector<float>& vec) {
                patches.push_back({bg, 0, (int32_t)r0, (int32_t)r1, (int64_t)data.size()});
                data.insert(data.end(), vec.begin(), vec.end());
            };
            if (has_streaming) {
                std::vector<float> a(d);
                for (size_t j = 0; j < d; ++j) a[j] = float(sp.local_boost * w_local[j]);
                add_k(local0, l, a);
            }
            const size_t needle_slots = std::max<size_t>(1, l_cpu / 128);
            int retrieval_idx = 0;
            for (int hg = 0; hg < G; ++hg) {
                const int head = h0 + hg;
                Rng hrng = rng.fork((uint64_t)hg + 7);
                std::vector<float> q;
                switch (arch[(size_t)head]) {
                    case kStreaming:
                        q = mix_direction(hrng, w_local, sp.streaming_jitter);
                        break;
                    case kRetrieval: {
                        const std::vector<float> u = unit_vec(hrng, d);
                        const double alpha = sp.needle_strength * hrng.uniform(0.85, 1.15);
                        const double gamma = sp.payload_gain * hrng.uniform(0.85, 1.15);
                        for (int nn = 0; nn < sp.needles; ++nn) {
                            const int slot = retrieval_idx++;
                            size_t start = (size_t)slot % needle_slots * 128 +
                                           (size_t)slot / needle_slots * (size_t)sp.needle_tokens;
                            start = std::min(start, l_cpu - (size_t)sp.needle_tokens);
                            const size_t end = start + (size_t)sp.needle_tokens;
                            const std::vector<float> w_pay = unit_vec(hrng, d);
                            std::vector<float> a(d);
                            for (size_t j = 0; j < d; ++j) a[j] = float(alpha * u[j]);
                            add_k(cpu0 + start, cpu0 + end, a);
                            patches.push_back({bg, 1, (int32_t)(cpu0 + start), (int32_t)(cpu0 + end),
                                               (int64_t)data.size()});
                            for (size_t i = start; i < end; ++i)
                                for (size_t j = 0; j < d; ++j)
                                    data.push_back(float(gamma * w_pay[j] + 0.3 * hrng.normal()));
                        }
                        q = mix_direction(hrng, u, sp.query_jitter);
                        break;
                    }
                    case kSinkDecoy: {
                        const std::vector<float> u = unit_vec(hrng, d);
                        const size_t dstart = std::min<size_t>(128, l_cpu / 4);
                        const size_t pstart = std::min<size_t>(384, l_cpu - (size_t)sp.decoy_payload_tokens);
                        std::vector<float> a(d);
                        for (size_t j = 0; j < d; ++j) a[j] = float(sp.decoy_strength * u[j]);
                        add_k(cpu0 + dstart, cpu0 + dstart + (size_t)sp.decoy_tokens, a);
                        patches.push_back({bg, 2, (int32_t)(cpu0 + dstart),
                                           (int32_t)(cpu0 + dstart + (size_t)sp.decoy_tokens), 0});
                        const std::vector<float> w_pay = unit_vec(hrng, d);
                        for (size_t j = 0; j < d; ++j) a[j] = float(sp.decoy_payload_strength * u[j]);
                        add_k(cpu0 + pstart, cpu0 + pstart + (size_t)sp.decoy_payload_tokens, a);
                        patches.push_back({bg, 1, (int32_t)(cpu0 + pstart),
                                           (int32_t)(cpu0 + pstart + (size_t)sp.decoy_payload_tokens),
                                           (int64_t)data.size()});
                        for (size_t i = 0; i < (size_t)sp.decoy_payload_tokens; ++i)
                            for (size_t j = 0; j < d; ++j)
                                data.push_back(float(sp.payload_gain * w_pay[j] + 0.3 * hrng.normal()));
                        if (cpu0 > 0) patches.push_back({bg, 2, 0, (int32_t)cpu0, 0});
                        q = mix_direction(hrng, u, sp.query_jitter);
                        break;
                    }
                    default:
                        q = unit_vec(hrng, d);
                        break;
                }
                scale_to(q, qnorm);
                std::copy(q.begin(), q.end(), hq.begin() + ((size_t)b * H + head) * d);
            }
        }
        // decode trace: drifting queries plus one appended token per group
        Rng drng = rng_l.fork(0xdecull);
        std::vector<float> prev(hq.begin() + (size_t)b * H * d, hq.begin() + (size_t)(b + 1) * H * d);
        const double rho = sp.query_drift;
        for (int st = 0; st < steps; ++st) {
            std::vector<float> cur(H * d);
            for (int head = 0; head < H; ++head) {
                const std::vector<float> noise = unit_vec(drng, d);
                std::vector<float> q(d);
                for (size_t j = 0; j < d; ++j)
                    q[j] = float(rho * prev[head * d + j] + std::sqrt(1.0 - rho * rho) * qnorm * noise[j]);
                scale_to(q, qnorm);
                std::copy(q.begin(), q.end(), cur.begin() + head * d);
            }
            for (int g = 0; g < Hkv; ++g)
                for (size_t j = 0; j < d; ++j) {
                    const size_t o = (((size_t)st * B + b) * Hkv + g) * d + j;
                    hnk[o] = float(drng.normal());
                    hnv[o] = float(drng.normal());
                }
            std::copy(cur.begin(), cur.end(), hsq.begin() + ((size_t)st * B + b) * H * d);
            prev = cur;
        }
    }
    first.push_back((int32_t)patches.size());
    // device: bulk fill, then the ordered patches
    const size_t bytes_state = state.size() * 8, bytes_p = patches.size() * sizeof(Patch),
                 bytes_f = first.size() * 4, bytes_d = std::max<size_t>(data.size(), 1) * 4;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    char* w = static_cast<char*>(scratch_alloc(al(bytes_state) + al(bytes_p) + al(bytes_f) + al(bytes_d), alloc_ctx));
    uint64_t* d_state = reinterpret_cast<uint64_t*>(w);
    Patch* d_p = reinterpret_cast<Patch*>(w + al(bytes_state));
    int32_t* d_first = reinterpret_cast<int32_t*>(w + al(bytes_state) + al(bytes_p));
    float* d_data = reinterpret_cast<float*>(w + al(bytes_state) + al(bytes_p) + al(bytes_f));
    FX_CUDA(cudaMemcpyAsync(d_state, state.data(), bytes_state, cudaMemcpyHostToDevice, s));
    if (bytes_p) FX_CUDA(cudaMemcpyAsync(d_p, patches.data(), bytes_p, cudaMemcpyHostToDevice, s));
    FX_CUDA(cudaMemcpyAsync(d_first, first.data(), bytes_f, cudaMemcpyHostToDevice, s));
    if (!data.empty()) FX_CUDA(cudaMemcpyAsync(d_data, data.data(), data.size() * 4, cudaMemcpyHostToDevice, s));
    const int64_t rows = (int64_t)l;
    const dim3 g1((unsigned)cdiv(rows * D, 256), (unsigned)(B * Hkv));
    const dim3 g2((unsigned)(B * Hkv));
    if (L.dtype == FX_BF16) {
        k_gen_bulk<__nv_bfloat16><<<g1, 256, 0, s>>>(rows, D, L.l_cap, d_state, static_cast<__nv_bfloat16*>(k),
                                                    static_cast<__nv_bfloat16*>(v));
        FX_CUDA(cudaGetLastError());
        k_gen_patch<__nv_bfloat16><<<g2, 256, 0, s>>>(d_p, d_first, d_data, D, L.l_cap,
                                                     static_cast<__nv_bfloat16*>(k), static_cast<__nv_bfloat16*>(v));
    } else {
        k_gen_bulk<float><<<g1, 256, 0, s>>>(rows, D, L.l_cap, d_state, static_cast<float*>(k), static_cast<float*>(v));
        FX_CUDA(cudaGetLastError());
        k_gen_patch<float><<<g2, 256, 0, s>>>(d_p, d_first, d_data, D, L.l_cap, static_cast<float*>(k),
                                              static_cast<float*>(v));
    }
    FX_CUDA(cudaGetLastError());
    if (anchor_q) FX_CUDA(cudaMemcpyAsync(anchor_q, hq.data(), hq.size() * 4, cudaMemcpyHostToDevice, s));
    if (steps > 0) {
        if (step_q) FX_CUDA(cudaMemcpyAsync(step_q, hsq.data(), hsq.size() * 4, cudaMemcpyHostToDevice, s));
        if (step_new_k) FX_CUDA(cudaMemcpyAsync(step_new_k, hnk.data(), hnk.size() * 4, cudaMemcpyHostToDevice, s));
        if (step_new_v) FX_CUDA(cudaMemcpyAsync(step_new_v, hnv.data(), hnv.size() * 4, cudaMemcpyHostToDevice, s));
    }
    FX_CUDA(cudaStreamSynchronize(s));  // the host vectors die here
}

}  // namespace fx
