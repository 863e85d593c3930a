// Reference attention API (attention.hpp) on the B200.
// Cites: /root/reference/proj/src/attention.cpp:10-164.
#include <cmath>
#include <stdexcept>

#include "fluxattn/attention.hpp"
#include "fx_api_arena.hpp"
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

// Attention of one query over the device-resident copy of `cache`
// (fx_api_arena.hpp): plan FULL = every cpu row plus the defaults
// (cache_attention), or blk 0 = the defaults only (default_kv_attention).
PartialOutput resident_attention(std::span<const float> q, const SegmentedKvCache& cache, bool with_cpu) {
    if (q.size() != cache.dim()) throw std::runtime_error("bad-shape: query width != key width");
    if (!all_finite(q)) throw std::runtime_error("non-finite: query");
    b200::Arena& ar = b200::arena_for(b200::shape_of(cache));
    const int slot = ar.acquire(cache);
    const std::size_t D = cache.dim();
    char* sc = static_cast<char*>(ar.scratch(4096 + 2 * D * sizeof(float)));
    int32_t* blk = reinterpret_cast<int32_t*>(sc);
    double* bud = reinterpret_cast<double*>(sc + 256);
    float* dq = reinterpret_cast<float*>(sc + 1024);
    float* dout = dq + D;
    float* dlse = reinterpret_cast<float*>(sc + 512);
    const fx_layout lay = ar.slot_layout();
    fx_step_args a = ar.slot_args(slot, static_cast<int64_t>(cache.len(Segment::New)));
    check(fx_memcpy_h2d(context(), dq, q.data(), D * sizeof(float)));
    a.q = dq;
    a.o = dout;
    a.lse = dlse;
    if (with_cpu) {
        a.plan_mode = FX_PLAN_FULL;
    } else {
        const int32_t zero = 0;
        const double none = 0.0;
        check(fx_memcpy_h2d(context(), blk, &zero, sizeof zero));
        check(fx_memcpy_h2d(context(), bud, &none, sizeof none));
        a.plan_mode = FX_PLAN_GIVEN;
        a.plan_blk = blk;
        a.plan_budgets = bud;
    }
    check(fx_decode_step(context(), &lay, &a));
    std::vector<float> o(D);
    float lse = 0.f;
    check(fx_memcpy_d2h(context(), o.data(), dout, D * sizeof(float)));
    check(fx_memcpy_d2h(context(), &lse, dlse, sizeof(float)));
    PartialOutput p;
    p.o.assign(o.begin(), o.end());
    p.lse = lse;
    p.tokens = cache.len(Segment::Sink) + cache.len(Segment::Local) + cache.len(Segment::New) +
               (with_cpu ? cache.len(Segment::Cpu) : 0);
    return p;
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

// attention.cpp:89-104 -- the reference's LSE merge of two partials, in
// double on the host (D + 1 values; a device round trip would cost more than
// the arithmetic and f32 would round the partials).
void merge_into(PartialOutput& acc, const PartialOutput& part) {
    if (part.empty()) return;
    if (acc.empty()) {
        acc = part;
        return;
    }
    const double lse_tot = acc.lse > part.lse ? acc.lse + std::log1p(std::exp(part.lse - acc.lse))
                                              : part.lse + std::log1p(std::exp(acc.lse - part.lse));
    const double wa = std::exp(acc.lse - lse_tot);
    const double wb = std::exp(part.lse - lse_tot);
    for (std::size_t j = 0; j < acc.o.size(); ++j) acc.o[j] = wa * acc.o[j] + wb * part.o[j];
    acc.lse = lse_tot;
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
    PartialOutput acc;
    for (const auto& p : parts) detail::merge_into(acc, p);  // attention.cpp:118-122
    return acc;
}

std::vector<double> merge_partials(std::span<const PartialOutput> parts) {
    PartialOutput acc = combine_partials(parts);
    if (acc.empty()) throw std::runtime_error("empty-context: all partials empty");
    return std::move(acc.o);
}

std::vector<double> cache_attention(std::span<const float> q, const SegmentedKvCache& cache) {
    if (cache.total_len() == 0) throw std::runtime_error("empty-context: cache has no tokens");
    return resident_attention(q, cache, true).o;
}

PartialOutput default_kv_attention(std::span<const float> q, const SegmentedKvCache& cache) {
    if (cache.len(Segment::Sink) + cache.len(Segment::Local) + cache.len(Segment::New) == 0)
        return PartialOutput{};
    return resident_attention(q, cache, false);
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
