// Reference attention API (attention.hpp) on the B200.
// Cites: /root/reference/proj/src/attention.cpp:10-164.
#include <cmath>
#include <stdexcept>

#include "fluxattn/attention.hpp"
#include "fx_api_common.hpp"

namespace fluxattn {
namespace {
using b200::check;
using b200::context;
using b200::DevMem;

// attention.cpp:10-20 input validation
void validate(std::span<const float> q, const Matrix& k, const Matrix& v) {
    if (k.rows() == 0 || v.rows() == 0) throw std::runtime_error("empty-context: attention over zero keys");
    if (k.rows() != v.rows()) throw std::runtime_error("bad-shape: K/V row count mismatch");
    if (q.size() != k.cols()) throw std::runtime_error("bad-shape: query width != key width");
    if (!all_finite(q) || !all_finite(k) || !all_finite(v))
        throw std::runtime_error("non-finite: attention input");
}

// Softmax attention of q over rows idx of (k, v) on the device.
PartialOutput device_attention(std::span<const float> q, const Matrix& k, const Matrix& v,
                               std::span<const std::uint32_t> idx) {
    PartialOutput out;
    if (idx.empty()) return out;
    const std::size_t dim = q.size();
    DevMem dq(q), dk(std::span<const float>(k.data(), k.size())),
        dv(std::span<const float>(v.data(), v.size())), di(idx);
    DevMem o(dim * sizeof(float)), lse(sizeof(float));
    check(fx_gathered_attention(context(), dq.as<float>(), dk.get(), dv.get(), FX_F32,
                                static_cast<int64_t>(k.rows()), static_cast<int32_t>(dim),
                                di.as<std::uint32_t>(), static_cast<int64_t>(idx.size()), o.as<float>(),
                                lse.as<float>()));
    const auto of = o.download<float>(dim);
    out.o.assign(of.begin(), of.end());
    out.lse = lse.download<float>(1)[0];
    out.tokens = idx.size();
    return out;
}

std::vector<std::uint32_t> iota_u32(std::size_t n) {
    std::vector<std::uint32_t> r(n);
    for (std::size_t i = 0; i < n; ++i) r[i] = static_cast<std::uint32_t>(i);
    return r;
}

// Stacked K/V of the chosen segments (position order) plus their row ids.
struct Stacked {
    Matrix k, v;
};
Stacked stack(const SegmentedKvCache& cache, std::initializer_list<Segment> segs) {
    Stacked s;
    for (Segment g : segs) {
        const Matrix& km = cache.keys(g);
        const Matrix& vm = cache.values(g);
        for (std::size_t r = 0; r < km.rows(); ++r) {
            s.k.append_row(km.row(r));
            s.v.append_row(vm.row(r));
        }
    }
    return s;
}
}  // namespace

namespace detail {

PartialOutput segment_attention_unchecked(std::span<const float> q, const Matrix& k, const Matrix& v) {
    const auto idx = iota_u32(k.rows());
    return device_attention(q, k, v, idx);
}

PartialOutput gathered_attention_unchecked(std::span<const float> q, const Matrix& k, const Matrix& v,
                                           std::span<const std::size_t> token_indices) {
    std::vector<std::uint32_t> idx(token_indices.begin(), token_indices.end());
    return device_attention(q, k, v, idx);
}

// attention.cpp:89-104 -- LSE merge on the device (fx_merge_partials).
void merge_into(PartialOutput& acc, const PartialOutput& part) {
    if (part.empty()) return;
    if (acc.empty()) {
        acc = part;
        return;
    }
    const std::size_t dim = acc.o.size();
    std::vector<float> o(2 * dim);
    for (std::size_t j = 0; j < dim; ++j) {
        o[j] = static_cast<float>(acc.o[j]);
        o[dim + j] = static_cast<float>(part.o[j]);
    }
    const float l[2] = {static_cast<float>(acc.lse), static_cast<float>(part.lse)};
    DevMem dop{std::span<const float>(o)}, dlp(std::span<const float>(l, 2));
    DevMem mo(dim * sizeof(float)), ml(sizeof(float));
    check(fx_merge_partials(context(), 2, static_cast<int32_t>(dim), dop.as<float>(), dlp.as<float>(),
                            mo.as<float>(), ml.as<float>()));
    const auto of = mo.download<float>(dim);
    acc.o.assign(of.begin(), of.end());
    acc.lse = ml.download<float>(1)[0];
    acc.tokens += part.tokens;
}

}  // namespace detail

std::vector<double> full_attention(std::span<const float> q, const Matrix& k, const Matrix& v) {
    validate(q, k, v);
    return detail::segment_attention_unchecked(q, k, v).o;
}

PartialOutput segment_attention(std::span<const float> q, const Matrix& k, const Matrix& v) {
    validate(q, k, v);
    return detail::segment_attention_unchecked(q, k, v);
}

PartialOutput combine_partials(std::span<const PartialOutput> parts) {
    std::vector<const PartialOutput*> live;
    for (const auto& p : parts)
        if (!p.empty()) live.push_back(&p);
    PartialOutput acc;
    if (live.empty()) return acc;
    if (live.size() == 1) return *live[0];
    const std::size_t dim = live[0]->o.size(), n = live.size();
    std::vector<float> o(n * dim), l(n);
    for (std::size_t i = 0; i < n; ++i) {
        for (std::size_t j = 0; j < dim; ++j) o[i * dim + j] = static_cast<float>(live[i]->o[j]);
        l[i] = static_cast<float>(live[i]->lse);
        acc.tokens += live[i]->tokens;
    }
    DevMem dop{std::span<const float>(o)}, dlp{std::span<const float>(l)};
    DevMem mo(dim * sizeof(float)), ml(sizeof(float));
    check(fx_merge_partials(context(), static_cast<int32_t>(n), static_cast<int32_t>(dim), dop.as<float>(),
                            dlp.as<float>(), mo.as<float>(), ml.as<float>()));
    const auto of = mo.download<float>(dim);
    acc.o.assign(of.begin(), of.end());
    acc.lse = ml.download<float>(1)[0];
    return acc;
}

std::vector<double> merge_partials(std::span<const PartialOutput> parts) {
    PartialOutput acc = combine_partials(parts);
    if (acc.empty()) throw std::runtime_error("empty-context: all partials empty");
    return std::move(acc.o);
}

// One softmax over every segment (equal to the reference's per-segment merge).
std::vector<double> cache_attention(std::span<const float> q, const SegmentedKvCache& cache) {
    Stacked s = stack(cache, {Segment::Sink, Segment::Cpu, Segment::Local, Segment::New});
    if (s.k.rows() == 0) throw std::runtime_error("empty-context: cache has no tokens");
    return detail::segment_attention_unchecked(q, s.k, s.v).o;
}

PartialOutput default_kv_attention(std::span<const float> q, const SegmentedKvCache& cache) {
    Stacked s = stack(cache, {Segment::Sink, Segment::Local, Segment::New});
    if (s.k.rows() == 0) return PartialOutput{};
    return detail::segment_attention_unchecked(q, s.k, s.v);
}

GroupView gqa_group_view(std::span<const HeadBinding> heads) {
    if (heads.empty()) throw std::runtime_error("empty-group: group view needs at least one head");
    GroupView g;
    g.cache = heads.front().cache;
    for (const auto& h : heads) {
        if (h.cache != g.cache) throw std::runtime_error("mixed-group: heads reference different caches");
        g.head_ids.push_back(h.head_id);
    }
    return g;
}

}  // namespace fluxattn
