// Exercises the C++ drop-in through the reference's own headers/names only
// (as a reference caller would), checks the SPEC known answers in-process and
// writes inputs + outputs of randomized cases as JSON for tests/test_dropin.py
// to compare against the CPU oracle.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fluxattn/attention.hpp"
#include "fluxattn/block_index.hpp"
#include "fluxattn/scheduler.hpp"
#include "fluxattn/selector.hpp"

using namespace fluxattn;

static int g_fail = 0;
#define EXPECT(c)                                                            \
    do {                                                                     \
        if (!(c)) {                                                          \
            std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++g_fail;                                                        \
        }                                                                    \
    } while (0)

template <class F>
static bool throws_with(F&& f, const std::string& prefix) {
    try {
        f();
    } catch (const std::runtime_error& e) {
        return std::string(e.what()).rfind(prefix, 0) == 0;
    }
    return false;
}

struct Lcg {  // deterministic inputs (numpy reproduces them for the oracle side)
    unsigned long long s;
    float next() {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        return float(double((s >> 11) & ((1ull << 40) - 1)) / double(1ull << 40) * 2.0 - 1.0);
    }
};

static Matrix rand_matrix(Lcg& g, std::size_t r, std::size_t c) {
    Matrix m(r, c);
    for (std::size_t i = 0; i < r * c; ++i) m.data()[i] = g.next();
    return m;
}

static void dump_vec(FILE* f, const char* name, const std::vector<double>& v) {
    std::fprintf(f, "\"%s\": [", name);
    for (std::size_t i = 0; i < v.size(); ++i) std::fprintf(f, "%s%.17g", i ? "," : "", v[i]);
    std::fprintf(f, "]");
}

int main(int argc, char** argv) {
    const char* out_path = argc > 1 ? argv[1] : "dropin_out.json";
    // ---- SPEC.md known answers ----
    {
        Matrix k(1, 2, {1.f, 0.f}), v(1, 2, {3.f, 4.f});
        const std::vector<float> q{1.f, 0.f};
        auto o = full_attention(q, k, v);
        EXPECT(std::fabs(o[0] - 3) < 1e-6 && std::fabs(o[1] - 4) < 1e-6);
        Matrix k2(2, 2, {1.f, 1.f, 1.f, 1.f}), v2(2, 2, {1.f, 0.f, 0.f, 1.f});
        auto o2 = full_attention(q, k2, v2);
        EXPECT(std::fabs(o2[0] - 0.5) < 1e-6 && std::fabs(o2[1] - 0.5) < 1e-6);
        const std::vector<float> z{0.f, 0.f};
        EXPECT(std::fabs(segment_attention(z, k, v).lse) < 1e-6);
        EXPECT(std::fabs(segment_attention(z, k2, v2).lse - std::log(2.0)) < 1e-6);
        PartialOutput a{{1.0, 0.0}, 0.3, 1}, b{{0.0, 1.0}, 0.3, 1};
        const std::vector<PartialOutput> parts{a, b};
        auto m = merge_partials(parts);
        EXPECT(std::fabs(m[0] - 0.5) < 1e-6 && std::fabs(m[1] - 0.5) < 1e-6);
        EXPECT(throws_with([&] { merge_partials(std::vector<PartialOutput>{PartialOutput{}}); }, "empty-context"));
        EXPECT(throws_with([&] { full_attention(q, Matrix{}, Matrix{}); }, "empty-context"));
        EXPECT(throws_with([&] { build_metadata(k, 0); }, "invalid-granularity"));
        Lcg g{7};
        Matrix k33 = rand_matrix(g, 33, 4);
        auto meta = build_metadata(k33, 16);
        EXPECT(meta.block_count == 3 && meta.block_begin(2) == 32 && meta.block_end(2) == 33);
        auto meta1 = build_metadata(k33, 1);  // blk = 1: score == <q, k>
        const std::vector<float> q4{0.5f, -1.f, 0.25f, 2.f};
        EXPECT(block_score(q4, meta1, 5) == dot(q4, k33.row(5)));
        EXPECT(throws_with([&] { block_score(q4, meta1, 33); }, "bad-block"));
        auto sel = topk_blocks(q4, meta, 7);
        EXPECT(sel.clamped && sel.blocks.size() == 3 && sel.budget_realized == 1.0);
        const std::vector<double> bud{0.1};
        EXPECT(std::fabs(volume(16, 1024, bud) - 332.8) < 1e-9);
        const std::vector<HeadProperties> p1{{0.05, 0.0, false}};
        EXPECT(plan_group(0, p1, 1024).block_size == 128);
        const std::vector<HeadProperties> ps{{0.1, 0.0, true}, {0.2, 0.0, true}};
        auto sp = plan_group(3, ps, 1024);
        EXPECT(sp.streaming_group);
        EXPECT(throws_with([&] { priority(sp); }, "not-schedulable"));
        // ties: identical blocks -> lower ids first
        Matrix kt(64, 4);
        for (std::size_t i = 0; i < kt.size(); ++i) kt.data()[i] = 0.5f;
        auto st = topk_blocks(q4, build_metadata(kt, 16), 2);
        EXPECT(st.blocks.size() == 2 && st.blocks[0] == 0 && st.blocks[1] == 1);
    }
    // ---- randomized group tasks through run(Executed) ----
    FILE* f = std::fopen(out_path, "w");
    if (!f) return 2;
    std::fprintf(f, "{\"cases\": [\n");
    const int D = 64, G = 4;
    const std::size_t ls = 64, lc = 1500, ll = 256;
    Lcg g{42};
    std::vector<SegmentedKvCache> caches;
    std::vector<BlockMetadata> metas;
    std::vector<SparseTask> tasks;
    const int blks[4] = {16, 32, 64, 128};
    caches.reserve(4);
    metas.reserve(4);
    for (int t = 0; t < 4; ++t) {
        // one declarator list: draws happen in order (sink K, sink V, cpu K, ...)
        Matrix sk = rand_matrix(g, ls, D), sv = rand_matrix(g, ls, D), ck = rand_matrix(g, lc, D),
               cv = rand_matrix(g, lc, D), lk = rand_matrix(g, ll, D), lv = rand_matrix(g, ll, D);
        caches.emplace_back(std::move(sk), std::move(sv), std::move(ck), std::move(cv), std::move(lk),
                            std::move(lv));
        Matrix nk = rand_matrix(g, 2, D), nv = rand_matrix(g, 2, D);
        caches.back().append_new(nk.row(0), nv.row(0));
        caches.back().append_new(nk.row(1), nv.row(1));
    }
    for (int t = 0; t < 4; ++t) {
        metas.push_back(build_metadata(caches[t].keys(Segment::Cpu), blks[t]));
        GroupPlan plan;
        plan.group_id = 10 + t;
        plan.block_size = blks[t];
        plan.budgets = {0.05, 0.0, 0.2, 1.0};
        plan.volume = volume(blks[t], lc, plan.budgets) + t;  // distinct priorities
        SparseTask task = make_task(plan, lc, D);
        task.cache = &caches[t];
        task.metadata = &metas[t];
        for (int h = 0; h < G; ++h) {
            Matrix qq = rand_matrix(g, 1, D);
            task.queries.emplace_back(qq.data(), qq.data() + D);
        }
        tasks.push_back(std::move(task));
    }
    // per-head API results of task 0 (topk + sparse + defaults + merge)
    {
        const SparseTask& t0 = tasks[0];
        const auto& q = t0.queries[0];
        const std::size_t kb = blocks_for_budget(0.05, lc, 16);
        auto sel = topk_blocks(q, metas[0], kb);
        PartialOutput acc = default_kv_attention(q, caches[0]);
        detail::merge_into(acc, sparse_attention(q, caches[0], sel));
        std::vector<double> blocks(sel.blocks.begin(), sel.blocks.end());
        std::fprintf(f, "{\"kind\": \"per_head\", \"k\": %zu, ", kb);
        dump_vec(f, "blocks", blocks);
        std::fprintf(f, ", ");
        dump_vec(f, "o", acc.o);
        std::fprintf(f, "},\n");
    }
    TaskQueue queue = enqueue_batch(std::vector<SparseTask>(tasks));
    std::vector<TaskResult> results;
    ScheduleReport rep = run(queue, WorkerProfile::standard(D), RunMode::Executed, &results);
    EXPECT(!rep.aborted && results.size() == 4);
    // the batched extension returns the same outputs, in task order
    const std::vector<TaskResult> batched = execute_batch(std::span<const SparseTask>(queue.tasks()));
    EXPECT(batched.size() == results.size());
    for (std::size_t i = 0; i < batched.size(); ++i)
        for (std::size_t h = 0; h < batched[i].head_outputs.size(); ++h)
            EXPECT(batched[i].head_outputs[h] == results[i].head_outputs[h]);
    // the ops are pure and concurrently callable: four host
    // threads (each gets its own device context) run every task at once and
    // must reproduce the single-threaded execute_task bit for bit
    {
        std::vector<TaskResult> single;
        for (const SparseTask& t : queue.tasks()) single.push_back(execute_task(t));
        std::vector<std::vector<TaskResult>> per(4);
        std::vector<std::thread> th;
        for (int w = 0; w < 4; ++w)
            th.emplace_back([&, w] {
                for (int rep = 0; rep < 3; ++rep)
                    for (const SparseTask& t : queue.tasks()) per[w].push_back(execute_task(t));
            });
        for (auto& x : th) x.join();
        for (int w = 0; w < 4; ++w) {
            EXPECT(per[w].size() == 3 * single.size());
            for (std::size_t i = 0; i < per[w].size() && i < 3 * single.size(); ++i)
                EXPECT(per[w][i].head_outputs == single[i % single.size()].head_outputs);
        }
    }
    for (std::size_t i = 0; i < results.size(); ++i) {
        const SparseTask& t = queue.tasks()[i];
        EXPECT(results[i].group_id == t.group_id);
        std::fprintf(f, "{\"kind\": \"task\", \"group\": %d, \"order\": %zu, \"blk\": %d, \"heads\": [", t.group_id, i,
                     t.plan.block_size);
        for (int h = 0; h < G; ++h) {
            std::fprintf(f, "%s{", h ? "," : "");
            dump_vec(f, "o", results[i].head_outputs[static_cast<std::size_t>(h)]);
            std::fprintf(f, "}");
        }
        std::fprintf(f, "]}%s\n", i + 1 < results.size() ? "," : "");
    }
    std::fprintf(f, "]}\n");
    std::fclose(f);
    std::printf("dropin: %d failures\n", g_fail);
    return g_fail ? 1 : 0;
}
