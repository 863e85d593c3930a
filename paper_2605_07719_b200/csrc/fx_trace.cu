// fx_trace.cu -- FXT1 workload traces (workload.cpp:311-433) to and from the
// device cache.  Format, all little-endian:
//   "FXT1" | version u32 (1) | input_hash u64 | seed u64
//   layers, heads, group_size, head_dim, context_len, sink, local, steps (u32)
//   per layer: per head  archetype u32, needle_count u32, (start u32, end u32)*
//              per group K [context_len x dim] f32, V [context_len x dim] f32
//              anchor queries [heads x dim] f32
//              per step  queries [heads x dim] f32, new K [groups x dim] f32,
//                        new V [groups x dim] f32
// A group's K (or V) in position order is exactly one cache row range
// [b][g][0, context_len) of the device layout, so it moves as one contiguous
// transfer (through an f32 staging buffer and a conversion for bf16 caches).
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fx_common.cuh"

namespace fx {
namespace {

constexpr char kMagic[4] = {'F', 'X', 'T', '1'};
constexpr uint32_t kVersion = 1;

struct File {
    std::FILE* f = nullptr;
    std::string path;
    File(const char* p, const char* mode) : path(p ? p : "") {
        f = p ? std::fopen(p, mode) : nullptr;
        FX_REQUIRE(f != nullptr, FX_ERR_INVALID, "io-error: cannot open " + path);
    }
    ~File() {
        if (f) std::fclose(f);
    }
    void read(void* dst, size_t n) {
        FX_REQUIRE(std::fread(dst, 1, n, f) == n, FX_ERR_INVALID, "corrupt-trace: truncated " + path);
    }
    void write(const void* src, size_t n) {
        FX_REQUIRE(std::fwrite(src, 1, n, f) == n, FX_ERR_INVALID, "io-error: short write to " + path);
    }
    void skip(int64_t n) {
        FX_REQUIRE(std::fseek(f, (long)n, SEEK_CUR) == 0, FX_ERR_INVALID, "corrupt-trace: truncated " + path);
    }
    uint32_t u32() {
        unsigned char b[4];
        read(b, 4);
        return (uint32_t)b[0] | (uint32_t)b[1] << 8 | (uint32_t)b[2] << 16 | (uint32_t)b[3] << 24;
    }
    uint64_t u64() {
        const uint64_t lo = u32();
        return lo | (uint64_t)u32() << 32;
    }
    void put32(uint32_t v) {
        const unsigned char b[4] = {(unsigned char)v, (unsigned char)(v >> 8), (unsigned char)(v >> 16),
                                    (unsigned char)(v >> 24)};
        write(b, 4);
    }
    void put64(uint64_t v) {
        put32((uint32_t)v);
        put32((uint32_t)(v >> 32));
    }
};

void read_header(File& f, fx_trace_info* h) {
    char m[4];
    f.read(m, 4);
    FX_REQUIRE(std::memcmp(m, kMagic, 4) == 0, FX_ERR_INVALID, "corrupt-trace: bad magic");
    FX_REQUIRE(f.u32() == kVersion, FX_ERR_INVALID, "corrupt-trace: bad version");
    h->input_hash = f.u64();
    h->seed = f.u64();
    int32_t* dims[8] = {&h->layers, &h->heads, &h->group_size, &h->head_dim, &h->context_len,
                        &h->sink_tokens, &h->local_tokens, &h->decode_steps};
    for (auto* p : dims) *p = (int32_t)f.u32();
    FX_REQUIRE(h->layers > 0 && h->heads > 0 && h->group_size > 0 && h->head_dim > 0 &&
                   h->context_len > h->sink_tokens + h->local_tokens && h->heads % h->group_size == 0,
               FX_ERR_INVALID, "corrupt-trace: implausible dimensions");
}

// host f32 rows -> device cache rows (dtype of the layout) via `stage`
void to_cache(const std::vector<float>& src, void* dst, int dtype, float* stage, cudaStream_t s) {
    const size_t n = src.size();
    if (dtype == FX_F32) {
        FX_CUDA(cudaMemcpyAsync(dst, src.data(), n * 4, cudaMemcpyHostToDevice, s));
    } else {
        FX_CUDA(cudaMemcpyAsync(stage, src.data(), n * 4, cudaMemcpyHostToDevice, s));
        launch_convert(stage, dst, dtype, n, s);
    }
    FX_CUDA(cudaStreamSynchronize(s));  // src is reused for the next block
}

}  // namespace

void trace_info(const char* path, fx_trace_info* info) {
    File f(path, "rb");
    read_header(f, info);
}

void trace_load(const char* path, int32_t layer, const fx_layout& L, int32_t b, void* k, void* v,
                float* anchor_q, float* step_q, float* new_k, float* new_v, int32_t* archetypes,
                void* scratch_alloc(size_t, void*), void* alloc_ctx, cudaStream_t s) {
    File f(path, "rb");
    fx_trace_info h;
    read_header(f, &h);
    const int64_t d = h.head_dim, l = h.context_len, H = h.heads, Hkv = h.heads / h.group_size;
    FX_REQUIRE(layer >= 0 && layer < h.layers, FX_ERR_INVALID, "bad-shape: layer not in the trace");
    FX_REQUIRE(L.kv_heads == Hkv && L.group_size == h.group_size && L.head_dim == h.head_dim &&
                   L.l_sink == h.sink_tokens && L.l_local == h.local_tokens &&
                   L.l_cpu == l - h.sink_tokens - h.local_tokens && L.l_cap >= l && b >= 0 && b < L.batch,
               FX_ERR_INVALID, "bad-shape: layout does not match the trace");
    const int64_t es = L.dtype == FX_BF16 ? 2 : 4;
    float* stage = L.dtype == FX_F32 ? nullptr : static_cast<float*>(scratch_alloc((size_t)l * d * 4, alloc_ctx));
    std::vector<float> buf;
    for (int32_t ly = 0; ly <= layer; ++ly) {
        const bool want = ly == layer;
        for (int64_t hh = 0; hh < H; ++hh) {
            const uint32_t a = f.u32(), n = f.u32();
            if (want && archetypes) archetypes[hh] = (int32_t)a;
            f.skip((int64_t)n * 8);
        }
        for (int64_t g = 0; g < Hkv; ++g)
            for (int t = 0; t < 2; ++t) {
                if (!want) {
                    f.skip(l * d * 4);
                    continue;
                }
                buf.resize((size_t)(l * d));
                f.read(buf.data(), buf.size() * 4);
                char* base = static_cast<char*>(t == 0 ? k : v);
                to_cache(buf, base + (((int64_t)b * Hkv + g) * L.l_cap) * d * es, L.dtype, stage, s);
            }
        auto block = [&](float* dst, int64_t n) {  // [n] f32 to a device pointer (or skip)
            if (!want || !dst) {
                f.skip(n * 4);
                return;
            }
            buf.resize((size_t)n);
            f.read(buf.data(), (size_t)n * 4);
            FX_CUDA(cudaMemcpyAsync(dst, buf.data(), (size_t)n * 4, cudaMemcpyHostToDevice, s));
            FX_CUDA(cudaStreamSynchronize(s));
        };
        block(anchor_q, H * d);
        for (int st = 0; st < h.decode_steps; ++st) {
            block(step_q ? step_q + (int64_t)st * H * d : nullptr, H * d);
            block(new_k ? new_k + (int64_t)st * Hkv * d : nullptr, Hkv * d);
            block(new_v ? new_v + (int64_t)st * Hkv * d : nullptr, Hkv * d);
        }
    }
}

void trace_save(const char* path, const fx_trace_info& h, const fx_layout& L, const int32_t* entries,
                const void* k, const void* v, const float* anchor_q, const float* step_q,
                const float* new_k, const float* new_v, const int32_t* archetypes,
                const int32_t* needle_count, const uint32_t* needles, cudaStream_t s) {
    const int64_t d = h.head_dim, l = h.context_len, H = h.heads, Hkv = h.heads / h.group_size;
    FX_REQUIRE(L.kv_heads == Hkv && L.group_size == h.group_size && L.head_dim == h.head_dim &&
                   L.l_sink == h.sink_tokens && L.l_local == h.local_tokens &&
                   L.l_cpu == l - h.sink_tokens - h.local_tokens && L.l_cap >= l,
               FX_ERR_INVALID, "bad-shape: layout does not match the trace header");
    File f(path, "wb");
    f.write(kMagic, 4);
    f.put32(kVersion);
    f.put64(h.input_hash);
    f.put64(h.seed);
    for (int32_t x : {h.layers, h.heads, h.group_size, h.head_dim, h.context_len, h.sink_tokens,
                      h.local_tokens, h.decode_steps})
        f.put32((uint32_t)x);
    const int64_t es = L.dtype == FX_BF16 ? 2 : 4;
    std::vector<unsigned char> raw((size_t)(l * d * es));
    std::vector<float> buf((size_t)(l * d));
    int64_t needle_off = 0;
    for (int32_t ly = 0; ly < h.layers; ++ly) {
        const int32_t b = entries[ly];
        FX_REQUIRE(b >= 0 && b < L.batch, FX_ERR_INVALID, "bad-shape: batch entry out of range");
        for (int64_t hh = 0; hh < H; ++hh) {
            const int64_t i = (int64_t)ly * H + hh;
            f.put32(archetypes ? (uint32_t)archetypes[i] : 3u);
            const uint32_t n = needle_count ? (uint32_t)needle_count[i] : 0u;
            f.put32(n);
            for (uint32_t j = 0; j < 2 * n; ++j) f.put32(needles[needle_off++]);
        }
        for (int64_t g = 0; g < Hkv; ++g)
            for (int t = 0; t < 2; ++t) {
                const char* base = static_cast<const char*>(t == 0 ? k : v);
                FX_CUDA(cudaMemcpyAsync(raw.data(), base + (((int64_t)b * Hkv + g) * L.l_cap) * d * es,
                                        raw.size(), cudaMemcpyDeviceToHost, s));
                FX_CUDA(cudaStreamSynchronize(s));
                if (L.dtype == FX_F32) {
                    std::memcpy(buf.data(), raw.data(), raw.size());
                } else {
                    const uint16_t* hbits = reinterpret_cast<const uint16_t*>(raw.data());
                    for (size_t e = 0; e < buf.size(); ++e) {
                        const uint32_t w = (uint32_t)hbits[e] << 16;
                        std::memcpy(&buf[e], &w, 4);
                    }
                }
                f.write(buf.data(), buf.size() * 4);
            }
        auto block = [&](const float* src, int64_t n) {
            std::vector<float> t((size_t)n, 0.0f);
            if (src) {
                FX_CUDA(cudaMemcpyAsync(t.data(), src, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
                FX_CUDA(cudaStreamSynchronize(s));
            }
            f.write(t.data(), t.size() * 4);
        };
        block(anchor_q ? anchor_q + (int64_t)ly * H * d : nullptr, H * d);
        for (int st = 0; st < h.decode_steps; ++st) {
            const int64_t o = (int64_t)ly * h.decode_steps + st;
            block(step_q ? step_q + o * H * d : nullptr, H * d);
            block(new_k ? new_k + o * Hkv * d : nullptr, Hkv * d);
            block(new_v ? new_v + o * Hkv * d : nullptr, Hkv * d);
        }
    }
}

}  // namespace fx
