// Reference task layer (scheduler.hpp) on the B200: the executed run is one
// batched device decode step over every task of the queue.
// Cites: /root/reference/proj/src/scheduler.cpp:11-287, 290-330.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <sstream>
#include <stdexcept>

#include "fluxattn/scheduler.hpp"
#include "fx_api_arena.hpp"
#include "fx_api_common.hpp"

namespace fluxattn {
namespace {
using b200::check;
using b200::context;
using b200::DevMem;

// Tasks batch into one device step when their caches share an arena shape,
// group size and decoded-row count.
struct Shape {
    std::size_t sink, cpu, local, fresh, dim;
    int heads;
    bool operator==(const Shape&) const = default;
};
Shape shape_of(const SparseTask& t) {
    const auto& c = *t.cache;
    return {c.len(Segment::Sink), c.len(Segment::Cpu), c.len(Segment::Local), c.len(Segment::New),
            c.dim(), static_cast<int>(t.queries.size())};
}

bool candidate_blk(int bs) {
    return std::find(kCandidateBlocks.begin(), kCandidateBlocks.end(), bs) != kCandidateBlocks.end();
}

// The reference's composition (scheduler.cpp:78-96) over the drop-in's own
// per-query device calls: for a block size outside the candidate set or
// metadata at another granularity than the plan -- exactly what the reference
// would select with task.metadata.
TaskResult execute_task_per_head(const SparseTask& task) {
    TaskResult res;
    res.group_id = task.group_id;
    const std::size_t l_cpu = task.cache->len(Segment::Cpu);
    for (std::size_t h = 0; h < task.queries.size(); ++h) {
        const auto& q = task.queries[h];
        PartialOutput acc = default_kv_attention(q, *task.cache);
        const std::size_t k = blocks_for_budget(task.plan.budgets.at(h), l_cpu, task.plan.block_size);
        if (k > 0) {
            const SelectionResult sel = topk_blocks(q, *task.metadata, k);
            detail::merge_into(acc, sparse_attention(q, *task.cache, sel));
        }
        res.head_outputs.push_back(std::move(acc.o));
    }
    return res;
}

// Executes `tasks` (same Shape, distinct caches) as one fx_decode_step over
// the device-resident caches of their arena: every arena slot is a batch
// entry (kv_heads = 1), plan given -- the task's blk and budgets, blk 0 and a
// zero query for slots without a task this step (their outputs are dropped).
void execute_batch(const std::vector<const SparseTask*>& tasks, std::vector<TaskResult*>& out) {
    const Shape s = shape_of(*tasks[0]);
    const std::size_t G = static_cast<std::size_t>(s.heads), D = s.dim;
    b200::Arena& ar = b200::arena_for(b200::shape_of(*tasks[0]->cache));
    std::vector<int> slot(tasks.size());
    for (std::size_t i = 0; i < tasks.size(); ++i) {
        const SparseTask& t = *tasks[i];
        for (std::size_t h = 0; h < G; ++h)
            if (t.queries[h].size() != D) throw std::runtime_error("bad-shape: query width != key width");
        if (t.plan.budgets.size() < G) throw std::runtime_error("bad-shape: plan has fewer budgets than heads");
        slot[i] = ar.acquire(*t.cache, /*defer=*/true);
    }
    ar.flush_pending();  // this step's appended rows: one batched append when they line up
    const std::size_t B = static_cast<std::size_t>(ar.slots());
    std::vector<int32_t> blk(B, 0);
    std::vector<double> bud(B * G, 0.0);
    std::vector<float> hq(B * G * D, 0.0f);
    for (std::size_t i = 0; i < tasks.size(); ++i) {
        const SparseTask& t = *tasks[i];
        const std::size_t b = static_cast<std::size_t>(slot[i]);
        bool any = false;
        for (std::size_t h = 0; h < G; ++h) {
            std::copy_n(t.queries[h].data(), D, hq.data() + (b * G + h) * D);
            bud[b * G + h] = t.plan.budgets[h];
            any |= blocks_for_budget(t.plan.budgets[h], s.cpu, t.plan.block_size) > 0;
        }
        // the reference selects on task.metadata and rejects a stale one (block_index.cpp:88)
        if (any && t.metadata->source_len != s.cpu)
            throw std::runtime_error("stale-selection: cpu segment length changed");
        blk[b] = s.cpu > 0 ? t.plan.block_size : 0;
    }
    const fx_layout lay = ar.layout(static_cast<int32_t>(G));
    // per-call device inputs / outputs in the arena's scratch: q | budgets | blk | o,
    // the inputs packed on the host and sent in one copy
    const auto al = [](std::size_t x) { return (x + 255) & ~std::size_t(255); };
    const std::size_t bq = al(hq.size() * sizeof(float)), bb = al(bud.size() * sizeof(double)),
                      bk = al(blk.size() * sizeof(int32_t)), bo = al(B * G * D * sizeof(float));
    char* sc = static_cast<char*>(ar.scratch(bq + bb + bk + bo));
    std::vector<char> packed(bq + bb + bk, 0);
    std::memcpy(packed.data(), hq.data(), hq.size() * sizeof(float));
    std::memcpy(packed.data() + bq, bud.data(), bud.size() * sizeof(double));
    std::memcpy(packed.data() + bq + bb, blk.data(), blk.size() * sizeof(int32_t));
    check(fx_memcpy_h2d(context(), sc, packed.data(), packed.size()));
    fx_step_args a = ar.step_args(static_cast<int64_t>(s.fresh));
    a.q = reinterpret_cast<const float*>(sc);
    a.plan_mode = FX_PLAN_GIVEN;
    a.plan_budgets = reinterpret_cast<double*>(sc + bq);
    a.plan_blk = reinterpret_cast<int32_t*>(sc + bq + bb);
    a.o = reinterpret_cast<float*>(sc + bq + bb + bk);
    check(fx_decode_step(context(), &lay, &a));
    std::vector<float> o(B * G * D);
    check(fx_memcpy_d2h(context(), o.data(), a.o, o.size() * sizeof(float)));
    for (std::size_t i = 0; i < tasks.size(); ++i) {
        const std::size_t b = static_cast<std::size_t>(slot[i]);
        out[i]->group_id = tasks[i]->group_id;
        out[i]->head_outputs.assign(G, std::vector<double>(D));
        for (std::size_t h = 0; h < G; ++h)
            std::copy_n(o.data() + (b * G + h) * D, D, out[i]->head_outputs[h].data());
    }
}

// Partitions tasks into device batches: the same Shape, each cache at most
// once per batch; tasks the batched step cannot express run per head.
// `finished` (optional) marks the tasks whose batch completed; on an
// exception `failing` holds the indices of the batch that threw.
void execute_all(const std::vector<const SparseTask*>& tasks, std::vector<TaskResult*>& out,
                 std::vector<bool>* finished = nullptr, std::vector<std::size_t>* failing = nullptr) {
    std::vector<bool> done(tasks.size(), false);
    for (std::size_t i = 0; i < tasks.size(); ++i) {
        const SparseTask& t = *tasks[i];
        if (failing) *failing = {i};
        if (!t.cache || !t.metadata) throw std::runtime_error("no-context: task has no executable payload");
        if (t.cache->len(Segment::Cpu) > 0 &&
            (!candidate_blk(t.plan.block_size) || t.metadata->block_size != t.plan.block_size)) {
            *out[i] = execute_task_per_head(t);
            done[i] = true;
            if (finished) (*finished)[i] = true;
        }
    }
    for (std::size_t i = 0; i < tasks.size(); ++i) {
        if (done[i]) continue;
        const Shape s = shape_of(*tasks[i]);
        std::vector<const SparseTask*> batch;
        std::vector<TaskResult*> res;
        std::vector<const SegmentedKvCache*> seen;
        std::vector<std::size_t> idx;
        for (std::size_t j = i; j < tasks.size(); ++j) {
            if (done[j] || !(shape_of(*tasks[j]) == s)) continue;
            if (std::find(seen.begin(), seen.end(), tasks[j]->cache) != seen.end()) continue;
            seen.push_back(tasks[j]->cache);
            batch.push_back(tasks[j]);
            res.push_back(out[j]);
            idx.push_back(j);
            done[j] = true;
        }
        if (failing) *failing = idx;
        execute_batch(batch, res);
        if (finished)
            for (std::size_t j : idx) (*finished)[j] = true;
    }
    if (failing) failing->clear();
}
}  // namespace

const char* policy_name(Policy p) {
    switch (p) {
        case Policy::Priority: return "priority";
        case Policy::NoParallel: return "no_parallel";
        case Policy::Uniform: return "uniform";
        case Policy::LengthBased: return "length";
    }
    return "?";
}

Policy parse_policy(const std::string& name) {
    for (Policy p : {Policy::Priority, Policy::NoParallel, Policy::Uniform, Policy::LengthBased})
        if (name == policy_name(p)) return p;
    throw std::runtime_error("bad-policy: " + name);
}

WorkerProfile WorkerProfile::standard(std::size_t head_dim) {
    WorkerProfile p;
    p.host_token_rate = 57e9 / double(p.host_workers) / (double(head_dim) * kBytesPerElement);
    return p;
}

SparseTask make_task(const GroupPlan& plan, std::size_t l_cpu, std::size_t head_dim) {
    if (plan.streaming_group) throw std::runtime_error("not-schedulable: streaming group");
    SparseTask t;
    t.group_id = plan.group_id;
    t.plan = plan;
    t.priority = priority(plan);
    t.l_cpu = l_cpu;
    t.head_count = static_cast<int>(plan.budgets.size());
    t.cost.token_units = plan.volume;
    t.cost.bytes_moved = plan.volume * double(head_dim) * kBytesPerElement;
    t.cost.flops = plan.volume * double(head_dim) * 2.0;
    return t;
}

TaskQueue::TaskQueue(std::vector<SparseTask> tasks) : tasks_(std::move(tasks)) {}

const SparseTask* TaskQueue::pop() {
    const std::size_t i = next_.fetch_add(1, std::memory_order_relaxed);
    return i < tasks_.size() ? &tasks_[i] : nullptr;
}

// Priority order: V(blk*) descending, group id ascending (scheduler.cpp:65-76).
TaskQueue enqueue_batch(std::vector<SparseTask> tasks) {
    std::vector<int> ids;
    ids.reserve(tasks.size());
    for (const auto& t : tasks) ids.push_back(t.group_id);
    std::sort(ids.begin(), ids.end());
    if (std::adjacent_find(ids.begin(), ids.end()) != ids.end())
        throw std::runtime_error("duplicate-task: group enqueued twice in one batch");
    std::stable_sort(tasks.begin(), tasks.end(), [](const SparseTask& a, const SparseTask& b) {
        return a.priority != b.priority ? a.priority > b.priority : a.group_id < b.group_id;
    });
    return TaskQueue(std::move(tasks));
}

TaskResult execute_task(const SparseTask& task) {
    if (task.cache == nullptr || task.metadata == nullptr)
        throw std::runtime_error("no-context: task has no executable payload");
    TaskResult r;
    std::vector<const SparseTask*> one{&task};
    std::vector<TaskResult*> out{&r};
    execute_all(one, out);
    return r;
}

std::vector<TaskResult> execute_batch(std::span<const SparseTask> tasks) {
    std::vector<TaskResult> res(tasks.size());
    std::vector<const SparseTask*> ptrs;
    std::vector<TaskResult*> out;
    for (std::size_t i = 0; i < tasks.size(); ++i) {
        ptrs.push_back(&tasks[i]);
        out.push_back(&res[i]);
    }
    execute_all(ptrs, out);
    return res;
}

ScheduleReport run(TaskQueue& queue, const WorkerProfile& workers, RunMode mode,
                   std::vector<TaskResult>* results) {
    if (mode == RunMode::Simulated)
        throw std::runtime_error("unsupported: simulated mode is the reference's A100+PCIe cost model");
    (void)workers;
    const auto& tasks = queue.tasks();
    std::vector<TaskResult> local;
    std::vector<TaskResult>& res = results ? *results : local;
    res.assign(tasks.size(), TaskResult{});
    ScheduleReport rep;
    rep.mode = RunMode::Executed;
    rep.policy = Policy::Priority;
    rep.workers.resize(1);
    rep.workers[0].accelerator = true;
    const auto t0 = std::chrono::steady_clock::now();
    // the whole queue as device steps (one per distinct task shape: one for a
    // decode step); a task counts as done only once its step has executed
    std::vector<bool> done(tasks.size(), false);
    std::vector<const SparseTask*> ptrs;
    std::vector<TaskResult*> out;
    for (std::size_t i = 0; i < tasks.size(); ++i) {
        ptrs.push_back(&tasks[i]);
        out.push_back(&res[i]);
    }
    std::vector<std::size_t> failing;
    try {
        execute_all(ptrs, out, &done, &failing);
    } catch (const std::exception&) {
        // the reference records the group whose task threw (scheduler.cpp:247-252);
        // a device step fails as a whole: every group of that step is reported
        for (std::size_t j : failing) rep.failed_groups.push_back(tasks[j].group_id);
        rep.aborted = true;
    }
    const double end = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rep.makespan = end;
    rep.workers[0].busy = end;
    int ndone = 0;
    for (std::size_t i = 0; i < tasks.size(); ++i) {
        if (!done[i]) continue;
        ++ndone;
        rep.events.push_back({static_cast<int>(i), tasks[i].group_id, 0, 0.0, end});
    }
    rep.workers[0].tasks = ndone;
    return rep;
}

ScheduleReport run_baseline(TaskQueue&, const WorkerProfile&, Policy) {
    throw std::runtime_error("unsupported: static baselines are the reference's cost-model ablations");
}

std::string ScheduleReport::to_json() const {
    std::ostringstream os;
    os.precision(17);
    os << "{\"mode\":\"" << (mode == RunMode::Simulated ? "sim" : "exec") << "\",\"policy\":\""
       << policy_name(policy) << "\",\"makespan\":" << makespan << ",\"aborted\":" << (aborted ? "true" : "false")
       << ",\"workers\":[";
    for (std::size_t i = 0; i < workers.size(); ++i)
        os << (i ? "," : "") << "{\"accelerator\":" << (workers[i].accelerator ? "true" : "false")
           << ",\"busy\":" << workers[i].busy << ",\"idle\":" << workers[i].idle << ",\"tasks\":" << workers[i].tasks
           << ",\"modeled_busy\":" << workers[i].modeled_busy << "}";
    os << "],\"tasks\":[";
    for (std::size_t i = 0; i < events.size(); ++i)
        os << (i ? "," : "") << "{\"task\":" << events[i].task_index << ",\"group\":" << events[i].group_id
           << ",\"worker\":" << events[i].worker << ",\"start\":" << events[i].start << ",\"end\":" << events[i].end
           << "}";
    os << "],\"failed_groups\":[";
    for (std::size_t i = 0; i < failed_groups.size(); ++i) os << (i ? "," : "") << failed_groups[i];
    os << "]}";
    return os.str();
}

std::string ScheduleReport::trace_csv() const {
    std::ostringstream os;
    os.precision(17);
    os << "task,group,worker,start,end\n";
    for (const auto& e : events) os << e.task_index << "," << e.group_id << "," << e.worker << "," << e.start << "," << e.end << "\n";
    return os.str();
}

}  // namespace fluxattn
