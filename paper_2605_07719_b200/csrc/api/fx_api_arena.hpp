// Device-resident copies of the reference's SegmentedKvCache objects for the
// C++ drop-in (no reference counterpart).
//
// The reference's caller keeps one cache per (layer, group) alive across
// decode steps and only appends one decoded row per step (pipeline.cpp:191-196,
// 406-408; kv_cache.hpp:68-73).  An Arena holds every cache of one segment
// shape in the batched device layout [slot][l_cap][D] (fx_layout batch = slot,
// kv_heads = 1), keyed by the cache's address and generation(): the first use
// uploads the segments and builds the four metadata levels on the device (the
// device analog of the caller's memo, pipeline.cpp:208-218); later uses upload
// only the New rows appended since.  execute_task / run / cache_attention /
// default_kv_attention then run on the resident rows.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <unordered_map>
#include <vector>

#include "fluxattn/kv_cache.hpp"
#include "fluxattn_b200.h"

namespace fluxattn::b200 {

struct ArenaShape {
    std::size_t sink, cpu, local, dim;
    bool operator<(const ArenaShape& o) const {
        if (sink != o.sink) return sink < o.sink;
        if (cpu != o.cpu) return cpu < o.cpu;
        if (local != o.local) return local < o.local;
        return dim < o.dim;
    }
};

class Arena {
public:
    Arena(const ArenaShape& shape, int dtype);
    ~Arena();
    Arena(const Arena&) = delete;
    Arena& operator=(const Arena&) = delete;

    // The cache's slot, with its rows up to date on the device.  defer: a
    // single newly appended row is left pending for flush_pending().
    int acquire(const SegmentedKvCache& cache, bool defer = false);
    // Uploads the deferred rows: one batched fx_append_kv when every slot has
    // exactly one pending row at the same position (a decode step), else row by row.
    void flush_pending();
    int slots() const { return static_cast<int>(owners_.size()); }
    // Layout over every slot for `l_new` decoded rows attended (rows per slot = l_cap).
    fx_layout layout(int group_size) const;
    // Step arguments with the arena's K / V / metadata / absmax filled in.
    fx_step_args step_args(std::int64_t l_new) const;
    // Single-slot view (batch 1) for the per-query calls.
    fx_layout slot_layout() const;
    fx_step_args slot_args(int slot, std::int64_t l_new) const;
    int dtype() const { return dtype_; }
    // Grow-only device scratch for per-call plans / queries / outputs.
    void* scratch(std::size_t bytes);
    const ArenaShape& shape() const { return shape_; }

private:
    struct Owner {
        const SegmentedKvCache* cache;
        std::uint64_t generation;
        std::size_t uploaded_new;
        bool pending = false;  // one deferred New row (uploaded_new + 1)
    };
    void reserve(int slots, std::int64_t l_cap);
    void upload_rows(int slot, std::int64_t row0, const float* k, const float* v, std::size_t rows);
    void build_metadata(int slot);

    ArenaShape shape_;
    int dtype_;
    std::int64_t l_cap_ = 0;
    int cap_slots_ = 0;
    void* k_ = nullptr;
    void* v_ = nullptr;
    void* meta_[4] = {nullptr, nullptr, nullptr, nullptr};
    float* absmax_ = nullptr;
    void* scratch_ = nullptr;
    std::size_t scratch_bytes_ = 0;
    std::vector<Owner> owners_;
    std::unordered_map<const SegmentedKvCache*, int> index_;
};

// The calling thread's arena for `shape` (one per shape per thread; KV dtype
// f32 unless FLUXATTN_KV_DTYPE=bf16).
Arena& arena_for(const ArenaShape& shape);
ArenaShape shape_of(const SegmentedKvCache& cache);
// Drops every device-resident cache of the calling thread.
void release_device_caches();
// (fx_api_context.cpp) the calling thread's arenas and f32 staging buffer
std::map<ArenaShape, std::unique_ptr<Arena>>& thread_arenas();
float* thread_staging(std::size_t bytes);

}  // namespace fluxattn::b200
