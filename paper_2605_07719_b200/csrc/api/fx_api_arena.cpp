// Device-resident SegmentedKvCache copies (fx_api_arena.hpp).
#include "fx_api_arena.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "fluxattn/b200.hpp"

namespace fluxattn::b200 {
namespace {

constexpr int kLevels[4] = {16, 32, 64, 128};

std::size_t elem_bytes(int dtype) { return dtype == FX_BF16 ? 2 : 4; }
std::int64_t nblk(std::size_t rows, int blk) { return static_cast<std::int64_t>((rows + blk - 1) / blk); }
std::int64_t round16(std::int64_t x) { return (x + 15) / 16 * 16; }

void* dev_alloc(std::size_t bytes) {
    void* p = nullptr;
    check(fx_malloc(context(), bytes ? bytes : 1, &p));
    return p;
}
void dev_free(void* p) {
    if (p) fx_free(context(), p);
}

int kv_dtype() {
    const char* e = std::getenv("FLUXATTN_KV_DTYPE");
    return (e && std::string(e) == "bf16") ? FX_BF16 : FX_F32;
}
}  // namespace

Arena::Arena(const ArenaShape& shape, int dtype) : shape_(shape), dtype_(dtype) {}

Arena::~Arena() {
    try {
        dev_free(k_);
        dev_free(v_);
        for (void* m : meta_) dev_free(m);
        dev_free(absmax_);
        dev_free(scratch_);
    } catch (...) {
    }
}

void* Arena::scratch(std::size_t bytes) {
    if (bytes > scratch_bytes_) {
        dev_free(scratch_);
        scratch_ = nullptr;
        scratch_bytes_ = 0;
        scratch_ = dev_alloc(bytes);
        scratch_bytes_ = bytes;
    }
    return scratch_;
}

fx_layout Arena::slot_layout() const {
    fx_layout L{};
    L.batch = 1;
    L.kv_heads = 1;
    L.group_size = 1;
    L.head_dim = static_cast<std::int32_t>(shape_.dim);
    L.dtype = dtype_;
    L.l_sink = static_cast<std::int64_t>(shape_.sink);
    L.l_cpu = static_cast<std::int64_t>(shape_.cpu);
    L.l_local = static_cast<std::int64_t>(shape_.local);
    L.l_cap = l_cap_;
    return L;
}

fx_layout Arena::layout(int group_size) const {
    fx_layout L = slot_layout();
    L.batch = static_cast<std::int32_t>(owners_.size());
    L.group_size = group_size;
    return L;
}

fx_step_args Arena::step_args(std::int64_t l_new) const {
    fx_step_args a{};
    a.k = k_;
    a.v = v_;
    for (int i = 0; i < 4; ++i) a.meta[i] = meta_[i];
    a.absmax = absmax_;
    a.l_new = l_new;
    return a;
}

fx_step_args Arena::slot_args(int slot, std::int64_t l_new) const {
    const std::size_t es = elem_bytes(dtype_), D = shape_.dim;
    fx_step_args a = step_args(l_new);
    a.k = static_cast<const char*>(k_) + static_cast<std::size_t>(slot) * l_cap_ * D * es;
    a.v = static_cast<const char*>(v_) + static_cast<std::size_t>(slot) * l_cap_ * D * es;
    if (shape_.cpu > 0) {
        for (int i = 0; i < 4; ++i)
            a.meta[i] = static_cast<const char*>(meta_[i]) +
                        static_cast<std::size_t>(slot) * nblk(shape_.cpu, kLevels[i]) * 2 * D * es;
        a.absmax = absmax_ + static_cast<std::size_t>(slot) * D;
    }
    return a;
}

// Grow to `slots` slots of `l_cap` rows, keeping the resident rows.
void Arena::reserve(int slots, std::int64_t l_cap) {
    if (slots <= cap_slots_ && l_cap <= l_cap_) return;
    const int ncap = std::max(slots, std::max(4, cap_slots_ * 2));
    const std::int64_t ncap_rows = std::max(l_cap, l_cap_);
    const std::size_t es = elem_bytes(dtype_), D = shape_.dim;
    void* nk = dev_alloc(static_cast<std::size_t>(ncap) * ncap_rows * D * es);
    void* nv = dev_alloc(static_cast<std::size_t>(ncap) * ncap_rows * D * es);
    for (std::size_t s = 0; s < owners_.size(); ++s) {  // resident rows, slot by slot
        const std::size_t rows = shape_.sink + shape_.cpu + shape_.local + owners_[s].uploaded_new;
        check(fx_memcpy_d2d(context(), static_cast<char*>(nk) + s * ncap_rows * D * es,
                            static_cast<const char*>(k_) + s * l_cap_ * D * es, rows * D * es));
        check(fx_memcpy_d2d(context(), static_cast<char*>(nv) + s * ncap_rows * D * es,
                            static_cast<const char*>(v_) + s * l_cap_ * D * es, rows * D * es));
    }
    dev_free(k_);
    dev_free(v_);
    k_ = nk;
    v_ = nv;
    if (shape_.cpu > 0 && ncap > cap_slots_) {
        for (int i = 0; i < 4; ++i) {
            const std::size_t per = static_cast<std::size_t>(nblk(shape_.cpu, kLevels[i])) * 2 * D * es;
            void* nm = dev_alloc(static_cast<std::size_t>(ncap) * per);
            if (!owners_.empty()) check(fx_memcpy_d2d(context(), nm, meta_[i], owners_.size() * per));
            dev_free(meta_[i]);
            meta_[i] = nm;
        }
        float* na = static_cast<float*>(dev_alloc(static_cast<std::size_t>(ncap) * D * sizeof(float)));
        if (!owners_.empty())
            check(fx_memcpy_d2d(context(), na, absmax_, owners_.size() * D * sizeof(float)));
        dev_free(absmax_);
        absmax_ = na;
    }
    cap_slots_ = std::max(cap_slots_, ncap);
    l_cap_ = ncap_rows;
}

void Arena::upload_rows(int slot, std::int64_t row0, const float* k, const float* v, std::size_t rows) {
    if (rows == 0) return;
    const std::size_t es = elem_bytes(dtype_), D = shape_.dim, n = rows * D;
    char* kd = static_cast<char*>(k_) + (static_cast<std::size_t>(slot) * l_cap_ + row0) * D * es;
    char* vd = static_cast<char*>(v_) + (static_cast<std::size_t>(slot) * l_cap_ + row0) * D * es;
    if (dtype_ == FX_F32) {
        check(fx_memcpy_h2d(context(), kd, k, n * sizeof(float)));
        check(fx_memcpy_h2d(context(), vd, v, n * sizeof(float)));
        return;
    }
    float* st = thread_staging(n * sizeof(float));
    check(fx_memcpy_h2d(context(), st, k, n * sizeof(float)));
    check(fx_convert(context(), st, kd, FX_BF16, n));
    check(fx_memcpy_h2d(context(), st, v, n * sizeof(float)));
    check(fx_convert(context(), st, vd, FX_BF16, n));
}

void Arena::build_metadata(int slot) {
    if (shape_.cpu == 0) return;
    const fx_layout L = slot_layout();
    const fx_step_args a = slot_args(slot, 0);
    check(fx_build_metadata_levels(context(), &L, a.k, const_cast<void*>(a.meta[0]), const_cast<void*>(a.meta[1]),
                                   const_cast<void*>(a.meta[2]), const_cast<void*>(a.meta[3]),
                                   const_cast<float*>(a.absmax)));
}

void Arena::flush_pending() {
    std::size_t n = 0, row = 0;
    bool uniform = true;
    for (const Owner& o : owners_)
        if (o.pending) {
            if (n == 0) row = o.uploaded_new;
            uniform = uniform && o.uploaded_new == row;
            ++n;
        }
    if (n == 0) return;
    const std::size_t base = shape_.sink + shape_.cpu + shape_.local, D = shape_.dim;
    if (n == owners_.size() && uniform) {  // a decode step: one row per slot, one kernel
        std::vector<float> kn(n * D), vn(n * D);
        for (std::size_t s = 0; s < n; ++s) {
            const Owner& o = owners_[s];
            std::copy_n(o.cache->keys(Segment::New).row(o.uploaded_new).data(), D, kn.data() + s * D);
            std::copy_n(o.cache->values(Segment::New).row(o.uploaded_new).data(), D, vn.data() + s * D);
        }
        float* st = thread_staging(2 * n * D * sizeof(float));
        check(fx_memcpy_h2d(context(), st, kn.data(), n * D * sizeof(float)));
        check(fx_memcpy_h2d(context(), st + n * D, vn.data(), n * D * sizeof(float)));
        fx_layout L = layout(1);
        check(fx_append_kv(context(), &L, k_, v_, static_cast<std::int64_t>(base + row), st, st + n * D));
        for (Owner& o : owners_) {
            o.uploaded_new += 1;
            o.pending = false;
        }
        return;
    }
    for (std::size_t s = 0; s < owners_.size(); ++s) {
        Owner& o = owners_[s];
        if (!o.pending) continue;
        upload_rows(static_cast<int>(s), static_cast<std::int64_t>(base + o.uploaded_new),
                    o.cache->keys(Segment::New).row(o.uploaded_new).data(),
                    o.cache->values(Segment::New).row(o.uploaded_new).data(), 1);
        o.uploaded_new += 1;
        o.pending = false;
    }
}

int Arena::acquire(const SegmentedKvCache& cache, bool defer) {
    const std::size_t fresh = cache.len(Segment::New);
    const std::size_t base = shape_.sink + shape_.cpu + shape_.local;
    // rows to hold now, plus decode headroom (regrowth copies the slots)
    const std::int64_t need = round16(static_cast<std::int64_t>(base + fresh));
    const std::int64_t room = round16(need + std::max<std::int64_t>(256, need / 8));
    int slot;
    auto it = index_.find(&cache);
    if (it != index_.end()) {
        slot = it->second;
        Owner& o = owners_[static_cast<std::size_t>(slot)];
        if (o.generation == cache.generation() && fresh >= o.uploaded_new + (o.pending ? 1 : 0)) {
            if (o.pending && defer && fresh == o.uploaded_new + 1) return slot;
            o.pending = false;  // upload whatever is outstanding below
            if (need > l_cap_) reserve(cap_slots_, room);
            if (defer && fresh == o.uploaded_new + 1) {
                o.pending = true;
                return slot;
            }
            if (fresh > o.uploaded_new) {  // append_new since the last use: those rows only
                const Matrix& kn = cache.keys(Segment::New);
                const Matrix& vn = cache.values(Segment::New);
                const std::size_t D = shape_.dim;
                upload_rows(slot, static_cast<std::int64_t>(base + o.uploaded_new), kn.data() + o.uploaded_new * D,
                            vn.data() + o.uploaded_new * D, fresh - o.uploaded_new);
                o.uploaded_new = fresh;
            }
            return slot;
        }
    } else {
        slot = static_cast<int>(owners_.size());
        reserve(slot + 1, need > l_cap_ ? room : l_cap_);
        owners_.push_back({&cache, 0, 0});
        index_[&cache] = slot;
    }
    if (need > l_cap_) reserve(cap_slots_, room);
    std::int64_t row = 0;
    for (Segment s : kAllSegments) {  // position order sink | cpu | local | new (kv_cache.hpp:13-18)
        const Matrix& km = cache.keys(s);
        const Matrix& vm = cache.values(s);
        upload_rows(slot, row, km.data(), vm.data(), km.rows());
        row += static_cast<std::int64_t>(km.rows());
    }
    build_metadata(slot);
    owners_[static_cast<std::size_t>(slot)] = {&cache, cache.generation(), fresh};
    return slot;
}

ArenaShape shape_of(const SegmentedKvCache& cache) {
    return {cache.len(Segment::Sink), cache.len(Segment::Cpu), cache.len(Segment::Local), cache.dim()};
}

Arena& arena_for(const ArenaShape& shape) {
    context();  // the thread's context (and its arena map) exists first
    auto& slot = thread_arenas()[shape];
    if (!slot) slot = std::make_unique<Arena>(shape, kv_dtype());
    return *slot;
}

void release_device_caches() { thread_arenas().clear(); }

}  // namespace fluxattn::b200
