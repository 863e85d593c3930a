// ref_shim.cpp -- C-ABI over the UNMODIFIED reference (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libfluxref.so).
//
// TEST INFRASTRUCTURE ONLY: used to pin the C restatement (fx_oracle.c), to
// generate golden vectors (tests/golden/make_golden.py) and, in bench.py, as
// the CPU baseline (`cpu_baseline.kind = "reference"` and `--impl
// reference`).  Nothing in the product path loads it.
//
// Every entry point returns 0 on success or -1 after storing the
// reference's exception text, readable through ref_last_error().
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "fluxattn/attention.hpp"
#include "fluxattn/block_index.hpp"
#include "fluxattn/budget_oracle.hpp"
#include "fluxattn/features.hpp"
#include "fluxattn/predictor.hpp"
#include "fluxattn/scheduler.hpp"
#include "fluxattn/selector.hpp"
#include "fluxattn/workload.hpp"

using namespace fluxattn;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

Matrix to_matrix(const float* p, std::size_t rows, std::size_t cols) {
    return Matrix(rows, cols, std::vector<float>(p, p + rows * cols));
}

BlockMetadata to_meta(const float* mins, const float* maxs, std::size_t nblk, std::size_t dim,
                      int blk, std::size_t source_len) {
    BlockMetadata m;
    m.block_size = blk;
    m.source_len = source_len;
    m.dim = dim;
    m.block_count = nblk;
    m.mins.assign(mins, mins + nblk * dim);
    m.maxs.assign(maxs, maxs + nblk * dim);
    return m;
}

// One group cache in the position layout sink | cpu | local | new.
SegmentedKvCache to_cache(const float* k, const float* v, std::size_t dim, std::size_t l_sink,
                          std::size_t l_cpu, std::size_t l_local, std::size_t l_new) {
    const std::size_t o_cpu = l_sink, o_loc = l_sink + l_cpu, o_new = o_loc + l_local;
    SegmentedKvCache c(to_matrix(k, l_sink, dim), to_matrix(v, l_sink, dim),
                       to_matrix(k + o_cpu * dim, l_cpu, dim), to_matrix(v + o_cpu * dim, l_cpu, dim),
                       to_matrix(k + o_loc * dim, l_local, dim),
                       to_matrix(v + o_loc * dim, l_local, dim));
    for (std::size_t i = 0; i < l_new; ++i)
        c.append_new(std::span<const float>(k + (o_new + i) * dim, dim),
                     std::span<const float>(v + (o_new + i) * dim, dim));
    return c;
}

void put_partial(const PartialOutput& p, std::size_t dim, double* o, double* lse,
                 std::uint64_t* tokens) {
    if (o) {
        if (p.o.size() == dim) std::memcpy(o, p.o.data(), dim * sizeof(double));
        else std::fill(o, o + dim, 0.0);
    }
    if (lse) *lse = p.lse;
    if (tokens) *tokens = p.tokens;
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_build_metadata(const float* k, std::size_t rows, std::size_t dim, int blk, float* mins,
                       float* maxs) {
    return guarded([&] {
        const BlockMetadata m = build_metadata(to_matrix(k, rows, dim), blk);
        std::memcpy(mins, m.mins.data(), m.mins.size() * sizeof(float));
        std::memcpy(maxs, m.maxs.data(), m.maxs.size() * sizeof(float));
    });
}

int ref_block_score(const float* q, const float* mins, const float* maxs, std::size_t nblk,
                    std::size_t dim, int blk, std::size_t source_len, std::size_t block,
                    double* out) {
    return guarded([&] {
        const BlockMetadata m = to_meta(mins, maxs, nblk, dim, blk, source_len);
        *out = block_score(std::span<const float>(q, dim), m, block);
    });
}

// blocks_out: [min(k,nblk)] selection order; tokens_out: [<= k*blk] ascending.
int ref_topk_blocks(const float* q, const float* mins, const float* maxs, std::size_t nblk,
                    std::size_t dim, int blk, std::size_t source_len, std::size_t k,
                    std::uint32_t* blocks_out, std::size_t* n_blocks, std::uint32_t* tokens_out,
                    std::size_t* n_tokens, int* clamped, double* budget_realized) {
    return guarded([&] {
        const BlockMetadata m = to_meta(mins, maxs, nblk, dim, blk, source_len);
        const SelectionResult s = topk_blocks(std::span<const float>(q, dim), m, k);
        *n_blocks = s.blocks.size();
        for (std::size_t i = 0; i < s.blocks.size(); ++i) blocks_out[i] = std::uint32_t(s.blocks[i]);
        *n_tokens = s.token_indices.size();
        if (tokens_out)
            for (std::size_t i = 0; i < s.token_indices.size(); ++i)
                tokens_out[i] = std::uint32_t(s.token_indices[i]);
        *clamped = s.clamped ? 1 : 0;
        *budget_realized = s.budget_realized;
    });
}

int ref_gathered_attention(const float* q, const float* k, const float* v, std::size_t rows,
                           std::size_t dim, const std::uint32_t* idx, std::size_t n, double* o,
                           double* lse, std::uint64_t* tokens) {
    return guarded([&] {
        const Matrix km = to_matrix(k, rows, dim), vm = to_matrix(v, rows, dim);
        std::vector<std::size_t> ids(idx, idx + n);
        put_partial(detail::gathered_attention_unchecked(std::span<const float>(q, dim), km, vm, ids),
                    dim, o, lse, tokens);
    });
}

int ref_segment_attention(const float* q, const float* k, const float* v, std::size_t rows,
                          std::size_t dim, double* o, double* lse) {
    return guarded([&] {
        put_partial(segment_attention(std::span<const float>(q, dim), to_matrix(k, rows, dim),
                                      to_matrix(v, rows, dim)),
                    dim, o, lse, nullptr);
    });
}

int ref_full_attention(const float* q, const float* k, const float* v, std::size_t rows,
                       std::size_t dim, double* o) {
    return guarded([&] {
        const auto r = full_attention(std::span<const float>(q, dim), to_matrix(k, rows, dim),
                                      to_matrix(v, rows, dim));
        std::memcpy(o, r.data(), dim * sizeof(double));
    });
}

int ref_merge_into(double* acc_o, double* acc_lse, std::uint64_t* acc_tokens, const double* o,
                   double lse, std::uint64_t tokens, std::size_t dim) {
    return guarded([&] {
        PartialOutput a, b;
        if (*acc_tokens) a.o.assign(acc_o, acc_o + dim);
        a.lse = *acc_lse;
        a.tokens = *acc_tokens;
        if (tokens) b.o.assign(o, o + dim);
        b.lse = lse;
        b.tokens = tokens;
        detail::merge_into(a, b);
        put_partial(a, dim, acc_o, acc_lse, acc_tokens);
    });
}

std::size_t ref_blocks_for_budget(double budget, std::size_t l_cpu, int blk) {
    return blocks_for_budget(budget, l_cpu, blk);
}

double ref_volume(int blk, std::size_t l_cpu, const double* budgets, int n) {
    return volume(blk, l_cpu, std::span<const double>(budgets, std::size_t(n)));
}

double ref_budget_at(double bgt0, double k, int streaming, int blk) {
    return budget_at(HeadProperties{bgt0, k, streaming != 0}, blk);
}

int ref_plan_group(const double* bgt0, const double* kslope, const int* streaming, int G,
                   std::size_t l_cpu, int* blk_out, double* budgets_out, double* volume_out,
                   double* cand_volumes, int* streaming_group) {
    return guarded([&] {
        std::vector<HeadProperties> props(std::size_t(std::max(G, 0)));
        for (int h = 0; h < G; ++h) props[std::size_t(h)] = {bgt0[h], kslope[h], streaming[h] != 0};
        const GroupPlan p = plan_group(0, props, l_cpu);
        *blk_out = p.block_size;
        *volume_out = p.volume;
        *streaming_group = p.streaming_group ? 1 : 0;
        for (std::size_t c = 0; c < 4; ++c) cand_volumes[c] = p.candidate_volumes[c];
        for (std::size_t h = 0; h < p.budgets.size(); ++h) budgets_out[h] = p.budgets[h];
    });
}

// execute_task on one group (scheduler.cpp:78-96). out_o: [G x dim].
int ref_execute_group(const float* k, const float* v, std::size_t dim, std::size_t l_sink,
                      std::size_t l_cpu, std::size_t l_local, std::size_t l_new,
                      const float* queries, int G, int blk, const double* budgets, double* out_o) {
    return guarded([&] {
        const SegmentedKvCache cache = to_cache(k, v, dim, l_sink, l_cpu, l_local, l_new);
        const BlockMetadata meta = build_metadata(cache.keys(Segment::Cpu), blk);
        SparseTask t;
        t.group_id = 0;
        t.plan.block_size = blk;
        t.plan.budgets.assign(budgets, budgets + G);
        t.l_cpu = l_cpu;
        t.head_count = G;
        t.cache = &cache;
        t.metadata = &meta;
        for (int h = 0; h < G; ++h)
            t.queries.emplace_back(queries + std::size_t(h) * dim, queries + std::size_t(h + 1) * dim);
        const TaskResult r = execute_task(t);
        for (int h = 0; h < G; ++h)
            std::memcpy(out_o + std::size_t(h) * dim, r.head_outputs[std::size_t(h)].data(),
                        dim * sizeof(double));
    });
}

// default_kv_attention (sink, local, new) for one head.
int ref_default_kv_attention(const float* k, const float* v, std::size_t dim, std::size_t l_sink,
                             std::size_t l_cpu, std::size_t l_local, std::size_t l_new,
                             const float* q, double* o, double* lse, std::uint64_t* tokens) {
    return guarded([&] {
        const SegmentedKvCache cache = to_cache(k, v, dim, l_sink, l_cpu, l_local, l_new);
        put_partial(default_kv_attention(std::span<const float>(q, dim), cache), dim, o, lse,
                    tokens);
    });
}

// ---------------------------------------------------------------------------
// CPU baseline: the reference's executed scheduler over a batch of groups.
// ---------------------------------------------------------------------------
struct RefBatch {
    std::vector<SegmentedKvCache> caches;
    std::vector<BlockMetadata> metas;
    std::vector<GroupPlan> plans;
    std::vector<std::vector<std::vector<float>>> queries;
    std::size_t dim = 0;
};

void* ref_batch_create() { return new RefBatch(); }
void ref_batch_destroy(void* h) { delete static_cast<RefBatch*>(h); }

// Adds one group task; metadata built at `blk` (memoized build, reported
// separately by the caller; pipeline.cpp:208-218).
int ref_batch_add(void* h, const float* k, const float* v, std::size_t dim, std::size_t l_sink,
                  std::size_t l_cpu, std::size_t l_local, std::size_t l_new, const float* queries,
                  int G, int blk, const double* budgets, double* meta_seconds) {
    return guarded([&] {
        auto* b = static_cast<RefBatch*>(h);
        b->dim = dim;
        b->caches.push_back(to_cache(k, v, dim, l_sink, l_cpu, l_local, l_new));
        const auto t0 = std::chrono::steady_clock::now();
        b->metas.push_back(build_metadata(b->caches.back().keys(Segment::Cpu), blk));
        const auto t1 = std::chrono::steady_clock::now();
        if (meta_seconds) *meta_seconds = std::chrono::duration<double>(t1 - t0).count();
        GroupPlan p;
        p.group_id = int(b->plans.size());
        p.block_size = blk;
        p.budgets.assign(budgets, budgets + G);
        p.volume = volume(blk, l_cpu, p.budgets);
        b->plans.push_back(p);
        std::vector<std::vector<float>> qs;
        for (int i = 0; i < G; ++i)
            qs.emplace_back(queries + std::size_t(i) * dim, queries + std::size_t(i + 1) * dim);
        b->queries.push_back(std::move(qs));
    });
}

// run(queue, profile, Executed) over all added groups with `host_workers`
// host threads (+1 accelerator-model thread, scheduler.cpp:219-279).
// Returns wall seconds of the run; out_o (optional) [n_groups x G x dim].
int ref_batch_run(void* h, int host_workers, double* seconds, double* out_o) {
    return guarded([&] {
        auto* b = static_cast<RefBatch*>(h);
        std::vector<SparseTask> tasks;
        for (std::size_t i = 0; i < b->plans.size(); ++i) {
            SparseTask t = make_task(b->plans[i], b->caches[i].len(Segment::Cpu), b->dim);
            t.cache = &b->caches[i];
            t.metadata = &b->metas[i];
            t.queries = b->queries[i];
            tasks.push_back(std::move(t));
        }
        TaskQueue q = enqueue_batch(std::move(tasks));
        WorkerProfile prof = WorkerProfile::standard(b->dim);
        prof.host_workers = host_workers;
        std::vector<TaskResult> results;
        const auto t0 = std::chrono::steady_clock::now();
        const ScheduleReport rep = run(q, prof, RunMode::Executed, &results);
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (rep.aborted) throw std::runtime_error("aborted: a task failed in the executed run");
        if (out_o) {
            for (std::size_t qi = 0; qi < results.size(); ++qi) {
                const int gid = results[qi].group_id;
                const auto& ho = results[qi].head_outputs;
                for (std::size_t hh = 0; hh < ho.size(); ++hh)
                    std::memcpy(out_o + (std::size_t(gid) * ho.size() + hh) * b->dim, ho[hh].data(),
                                b->dim * sizeof(double));
            }
        }
    });
}

// ---------------------------------------------------------------------------
// Synthetic workload (workload.cpp:154-308) for golden vectors.
// ---------------------------------------------------------------------------
void* ref_generate(const char* spec_json) {
    try {
        return new Workload(generate(WorkloadSpec::from_json(spec_json)));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_workload_destroy(void* h) { delete static_cast<Workload*>(h); }

// K/V of one group in position order, [context_len x dim] each.
int ref_workload_group_kv(void* h, int layer, int g, float* k, float* v) {
    return guarded([&] {
        const auto& c = static_cast<Workload*>(h)->layers.at(std::size_t(layer)).group_caches.at(
            std::size_t(g));
        std::size_t off = 0;
        for (auto s : {Segment::Sink, Segment::Cpu, Segment::Local}) {
            const Matrix& km = c.keys(s);
            const Matrix& vm = c.values(s);
            std::memcpy(k + off, km.data(), km.size() * sizeof(float));
            std::memcpy(v + off, vm.data(), vm.size() * sizeof(float));
            off += km.size();
        }
    });
}

// step < 0 -> anchor queries.  [heads x dim].
int ref_workload_queries(void* h, int layer, int step, float* out) {
    return guarded([&] {
        const auto& lw = static_cast<Workload*>(h)->layers.at(std::size_t(layer));
        const Matrix& m = step < 0 ? lw.anchor_queries : lw.step_queries.at(std::size_t(step));
        std::memcpy(out, m.data(), m.size() * sizeof(float));
    });
}

int ref_workload_new_kv(void* h, int layer, int step, float* k, float* v) {
    return guarded([&] {
        const auto& lw = static_cast<Workload*>(h)->layers.at(std::size_t(layer));
        const Matrix& km = lw.step_new_k.at(std::size_t(step));
        const Matrix& vm = lw.step_new_v.at(std::size_t(step));
        std::memcpy(k, km.data(), km.size() * sizeof(float));
        std::memcpy(v, vm.data(), vm.size() * sizeof(float));
    });
}

int ref_workload_archetype(void* h, int layer, int head) {
    return int(static_cast<Workload*>(h)->layers.at(std::size_t(layer)).heads.at(std::size_t(head))
                   .archetype);
}

// ---------------------------------------------------------------------------
// Predictor (predictor.cpp:161-185, 372-425).
// ---------------------------------------------------------------------------
void* ref_make_model(std::uint64_t seed) { return new PredictorModel(make_model(seed)); }
void* ref_load_model(const char* path) {
    try {
        return new PredictorModel(load_model(path));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_model_destroy(void* h) { delete static_cast<PredictorModel*>(h); }

// Copies layer weights/biases (f64) and the 41 (mu, sigma) pairs.
int ref_model_params(void* h, double* w1, double* b1, double* w2, double* b2, double* w3,
                     double* b3, double* mu, double* sigma) {
    return guarded([&] {
        const auto& m = *static_cast<PredictorModel*>(h);
        double* ws[3] = {w1, w2, w3};
        double* bs[3] = {b1, b2, b3};
        for (int i = 0; i < 3; ++i) {
            std::memcpy(ws[i], m.layers[std::size_t(i)].w.data(), m.layers[std::size_t(i)].w.size() * 8);
            std::memcpy(bs[i], m.layers[std::size_t(i)].b.data(), m.layers[std::size_t(i)].b.size() * 8);
        }
        std::memcpy(mu, m.norms.mu.data(), 41 * 8);
        std::memcpy(sigma, m.norms.sigma.data(), 41 * 8);
    });
}

int ref_model_set_norms(void* h, const double* mu, const double* sigma) {
    return guarded([&] {
        auto& m = *static_cast<PredictorModel*>(h);
        m.norms.mu.assign(mu, mu + 41);
        m.norms.sigma.assign(sigma, sigma + 41);
    });
}

int ref_save_model(void* h, const char* path) {
    return guarded([&] { save_model(*static_cast<PredictorModel*>(h), path); });
}

// out: {bgt0, k, s_prob}; z: raw logits.
int ref_predict(void* h, const double* raw, double* out, double* z) {
    return guarded([&] {
        const auto& m = *static_cast<PredictorModel*>(h);
        FeatureVector fv{};
        std::copy(raw, raw + 41, fv.begin());
        const Prediction p = predict(m, fv);
        out[0] = p.bgt0;
        out[1] = p.k;
        out[2] = p.s_prob;
        if (z) {
            const auto zz = forward_raw(m, normalize(fv, m.norms));
            std::copy(zz.begin(), zz.end(), z);
        }
    });
}

// ---------------------------------------------------------------------------
// output-aware budget oracle (budget_oracle.cpp) for one head of one group
// ---------------------------------------------------------------------------
int ref_cache_attention(const float* k, const float* v, std::size_t dim, std::size_t l_sink,
                        std::size_t l_cpu, std::size_t l_local, std::size_t l_new, const float* q,
                        double* o_full) {
    return guarded([&] {
        const SegmentedKvCache cache = to_cache(k, v, dim, l_sink, l_cpu, l_local, l_new);
        const auto o = cache_attention(std::span<const float>(q, dim), cache);
        std::copy(o.begin(), o.end(), o_full);
    });
}

int ref_min_budget(const float* k, const float* v, std::size_t dim, std::size_t l_sink,
                   std::size_t l_cpu, std::size_t l_local, std::size_t l_new, const float* q,
                   int blk, const double* o_full, double normalizer, double tau, double* budget,
                   std::uint64_t* blocks, int* saturated) {
    return guarded([&] {
        const SegmentedKvCache cache = to_cache(k, v, dim, l_sink, l_cpu, l_local, l_new);
        ErrorBudgetConfig cfg;
        cfg.tau = tau;
        const MinBudgetResult r = min_budget(std::span<const float>(q, dim), cache, blk,
                                             std::span<const double>(o_full, dim), normalizer, cfg);
        *budget = r.budget;
        *blocks = r.blocks;
        *saturated = r.saturated ? 1 : 0;
    });
}

int ref_label_streaming(const float* k, const float* v, std::size_t dim, std::size_t l_sink,
                        std::size_t l_cpu, std::size_t l_local, std::size_t l_new, const float* q,
                        const double* o_full, double normalizer, double tau, int* streaming) {
    return guarded([&] {
        const SegmentedKvCache cache = to_cache(k, v, dim, l_sink, l_cpu, l_local, l_new);
        ErrorBudgetConfig cfg;
        cfg.tau = tau;
        *streaming = label_streaming(std::span<const float>(q, dim), cache,
                                     std::span<const double>(o_full, dim), normalizer, cfg)
                         ? 1
                         : 0;
    });
}

int ref_fit_curve(const int* blks, const double* budgets, int n, double bgt0, int streaming,
                  double* k, double* free_intercept, double* max_abs_residual) {
    return guarded([&] {
        std::vector<std::pair<int, double>> pts;
        for (int i = 0; i < n; ++i) pts.emplace_back(blks[i], budgets[i]);
        const FitResult r = fit_curve(pts, bgt0, streaming != 0);
        *k = r.props.k;
        *free_intercept = r.free_intercept;
        *max_abs_residual = r.max_abs_residual;
    });
}

int ref_max_output_norm(const double* outs, std::size_t n, std::size_t dim, double* out) {
    return guarded([&] {
        std::vector<std::vector<double>> v(n);
        for (std::size_t h = 0; h < n; ++h) v[h].assign(outs + h * dim, outs + (h + 1) * dim);
        *out = max_output_norm(v);
    });
}

// ---------------------------------------------------------------------------
// features (features.cpp): prefill_stats on the cache without decoded rows,
// then decode_features on the cache with l_new decoded rows.  rec: the flat
// record of fx_oracle.c (FXO_STATS_N = 32 scalars, then mean_k, mean_v,
// anchor); feats: 41 values.
// ---------------------------------------------------------------------------
int ref_features(const float* k, const float* v, std::size_t dim, std::size_t l_sink,
                 std::size_t l_cpu, std::size_t l_local, std::size_t l_new, const float* anchor,
                 const double* budget4, double cross_anchor, int layer, int head, const float* q,
                 double cross_now, double* rec, double* feats) {
    return guarded([&] {
        const SegmentedKvCache pre = to_cache(k, v, dim, l_sink, l_cpu, l_local, 0);
        const std::array<double, 4> bf{budget4[0], budget4[1], budget4[2], budget4[3]};
        const PrefillStats st = prefill_stats(layer, head, pre, std::span<const float>(anchor, dim),
                                              bf, cross_anchor);
        std::fill(rec, rec + 32 + 3 * dim, 0.0);
        rec[0] = st.layer;
        rec[1] = st.head;
        rec[2] = double(st.l_cpu);
        rec[3] = double(st.l_sink);
        rec[4] = double(st.l_local);
        rec[5] = st.cpu_empty ? 1.0 : 0.0;
        rec[6] = st.sink_key_norm_mean;
        rec[7] = st.sink_value_norm_mean;
        const Moments* ms[3] = {&st.k_cpu_norms, &st.v_cpu_norms, &st.z_anchor};
        for (int i = 0; i < 3; ++i) {
            rec[8 + 4 * i] = ms[i]->mean;
            rec[9 + 4 * i] = ms[i]->var;
            rec[10 + 4 * i] = ms[i]->skew;
            rec[11 + 4 * i] = ms[i]->kurt;
        }
        rec[20] = st.lse_sink_anchor;
        rec[21] = st.lse_cpu_anchor;
        rec[22] = st.lse_local_anchor;
        rec[23] = st.out_sink_anchor_norm;
        rec[24] = st.out_cpu_anchor_norm;
        rec[25] = st.out_local_anchor_norm;
        for (int i = 0; i < 4; ++i) rec[26 + i] = st.budget_features[i];
        rec[30] = st.cross_head_max_anchor;
        rec[31] = l2_norm(std::span<const float>(st.anchor_query));
        for (std::size_t j = 0; j < dim; ++j) {
            rec[32 + j] = st.mean_k_cpu[j];
            rec[32 + dim + j] = st.mean_v_cpu[j];
            rec[32 + 2 * dim + j] = st.anchor_query[j];
        }
        const SegmentedKvCache cache = to_cache(k, v, dim, l_sink, l_cpu, l_local, l_new);
        const FeatureVector f = decode_features(std::span<const float>(q, dim), cache, st, cross_now);
        std::copy(f.begin(), f.end(), feats);
    });
}

double ref_gpu_output_norm(const float* k, const float* v, std::size_t dim, std::size_t l_sink,
                           std::size_t l_cpu, std::size_t l_local, std::size_t l_new, const float* q) {
    const SegmentedKvCache cache = to_cache(k, v, dim, l_sink, l_cpu, l_local, l_new);
    return gpu_output_norm(std::span<const float>(q, dim), cache);
}

// FXT1 traces (workload.cpp:311-433)
int ref_export_trace(void* h, const char* path, std::uint64_t input_hash) {
    return guarded([&] { export_trace(*static_cast<Workload*>(h), path, input_hash); });
}
void* ref_import_trace(const char* path) {
    try {
        return new Workload(import_trace(path, nullptr));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

} // extern "C"
