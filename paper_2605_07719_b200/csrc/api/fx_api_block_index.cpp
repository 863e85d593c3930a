// Reference block-index API (block_index.hpp) on the B200.
// Cites: /root/reference/proj/src/block_index.cpp:10-103.
#include <algorithm>
#include <stdexcept>

#include "../fx_selector_math.h"
#include "fluxattn/block_index.hpp"
#include "fx_api_common.hpp"

namespace fluxattn {
namespace {
using b200::check;
using b200::context;
using b200::DevMem;

// Device image [nblk][2][dim] (min row, max row) of host metadata.
std::vector<float> interleave(const BlockMetadata& m, std::size_t first, std::size_t count) {
    std::vector<float> out(count * 2 * m.dim);
    for (std::size_t b = 0; b < count; ++b) {
        std::copy_n(m.mins.data() + (first + b) * m.dim, m.dim, out.data() + (2 * b) * m.dim);
        std::copy_n(m.maxs.data() + (first + b) * m.dim, m.dim, out.data() + (2 * b + 1) * m.dim);
    }
    return out;
}
}  // namespace

BlockMetadata build_metadata(const Matrix& k_cpu, int block_size) {
    if (block_size <= 0) throw std::runtime_error("invalid-granularity: block size must be >= 1");
    BlockMetadata meta;
    meta.block_size = block_size;
    meta.source_len = k_cpu.rows();
    meta.dim = k_cpu.cols();
    meta.block_count = (k_cpu.rows() + static_cast<std::size_t>(block_size) - 1) / block_size;
    meta.mins.resize(meta.block_count * meta.dim);
    meta.maxs.resize(meta.block_count * meta.dim);
    if (meta.block_count == 0) return meta;
    DevMem dk(std::span<const float>(k_cpu.data(), k_cpu.size()));
    DevMem dm(meta.block_count * 2 * meta.dim * sizeof(float));
    check(fx_build_metadata(context(), dk.get(), FX_F32, static_cast<int64_t>(k_cpu.rows()),
                            static_cast<int32_t>(meta.dim), block_size, dm.get()));
    const auto h = dm.download<float>(meta.block_count * 2 * meta.dim);
    for (std::size_t b = 0; b < meta.block_count; ++b) {
        std::copy_n(h.data() + (2 * b) * meta.dim, meta.dim, meta.mins.data() + b * meta.dim);
        std::copy_n(h.data() + (2 * b + 1) * meta.dim, meta.dim, meta.maxs.data() + b * meta.dim);
    }
    return meta;
}

double block_score(std::span<const float> q, const BlockMetadata& meta, std::size_t block) {
    if (block >= meta.block_count) throw std::runtime_error("bad-block: block id out of range");
    const auto img = interleave(meta, block, 1);
    DevMem dm{std::span<const float>(img)}, dq(q), ds(sizeof(double));
    check(fx_block_scores(context(), dq.as<float>(), dm.get(), FX_F32, 1, static_cast<int32_t>(meta.dim),
                          ds.as<double>()));
    return ds.download<double>(1)[0];
}

SelectionResult topk_blocks(std::span<const float> q, const BlockMetadata& meta, std::size_t k) {
    SelectionResult sel;
    sel.block_size = meta.block_size;
    sel.source_len = meta.source_len;
    sel.clamped = k > meta.block_count;
    const std::size_t ke = std::min(k, meta.block_count);
    if (ke == 0) return sel;
    const auto img = interleave(meta, 0, meta.block_count);
    DevMem dm{std::span<const float>(img)}, dq(q), db(ke * sizeof(std::uint32_t));
    int64_t k_eff = 0;
    int32_t clamped = 0;
    check(fx_topk_blocks(context(), dq.as<float>(), dm.get(), FX_F32, static_cast<int64_t>(meta.block_count),
                         static_cast<int32_t>(meta.dim), static_cast<int64_t>(k), db.as<std::uint32_t>(),
                         &k_eff, &clamped));
    const auto ids = db.download<std::uint32_t>(static_cast<std::size_t>(k_eff));
    sel.blocks.assign(ids.begin(), ids.end());
    for (std::size_t b : sel.blocks)
        for (std::size_t t = meta.block_begin(b); t < meta.block_end(b); ++t) sel.token_indices.push_back(t);
    std::sort(sel.token_indices.begin(), sel.token_indices.end());
    sel.budget_realized =
        meta.source_len ? double(sel.token_indices.size()) / double(meta.source_len) : 0.0;
    return sel;
}

PartialOutput sparse_attention(std::span<const float> q, const SegmentedKvCache& cache,
                               const SelectionResult& sel) {
    if (sel.source_len != cache.len(Segment::Cpu))
        throw std::runtime_error("stale-selection: cpu segment length changed");
    if (sel.token_indices.empty()) return PartialOutput{};
    if (!all_finite(q)) throw std::runtime_error("non-finite: query");
    return detail::gathered_attention_unchecked(q, cache.keys(Segment::Cpu), cache.values(Segment::Cpu),
                                                sel.token_indices);
}

std::size_t blocks_for_budget(double budget, std::size_t l_cpu, int block_size) {
    return static_cast<std::size_t>(fx::sel::blocks_for_budget(budget, static_cast<int64_t>(l_cpu), block_size));
}

}  // namespace fluxattn
