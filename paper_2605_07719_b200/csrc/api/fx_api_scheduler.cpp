// Reference task layer (scheduler.hpp) on the B200: the executed run is one
// batched device decode step over every task of the queue.
// Cites: /root/reference/proj/src/scheduler.cpp:11-287, 290-330.
#include <algorithm>
#include <chrono>
#include <sstream>
#include <stdexcept>

#include "fluxattn/scheduler.hpp"
#include "fx_api_common.hpp"

namespace fluxattn {
namespace {
using b200::check;
using b200::context;
using b200::DevMem;

// All tasks share one device layout when their segment shapes agree.
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

// Executes `tasks` (same Shape) as one fx_decode_step: batch = tasks, one KV
// group each, plan given (blk per task, budget per head).
void execute_batch(const std::vector<const SparseTask*>& tasks, std::vector<TaskResult*>& out) {
    const Shape s = shape_of(*tasks[0]);
    const std::size_t B = tasks.size(), G = static_cast<std::size_t>(s.heads), D = s.dim;
    const std::size_t rows = s.sink + s.cpu + s.local + s.fresh;
    fx_layout lay{};
    lay.batch = static_cast<int32_t>(B);
    lay.kv_heads = 1;
    lay.group_size = static_cast<int32_t>(G);
    lay.head_dim = static_cast<int32_t>(D);
    lay.dtype = FX_F32;
    lay.l_sink = static_cast<int64_t>(s.sink);
    lay.l_cpu = static_cast<int64_t>(s.cpu);
    lay.l_local = static_cast<int64_t>(s.local);
    lay.l_cap = static_cast<int64_t>(rows);
    std::vector<float> hk(B * rows * D), hv(B * rows * D), hq(B * G * D);
    std::vector<int32_t> blk(B);
    std::vector<double> bud(B * G, 0.0);
    for (std::size_t b = 0; b < B; ++b) {
        const SparseTask& t = *tasks[b];
        std::size_t r = 0;
        for (Segment g : {Segment::Sink, Segment::Cpu, Segment::Local, Segment::New}) {
            const Matrix& km = t.cache->keys(g);
            const Matrix& vm = t.cache->values(g);
            std::copy_n(km.data(), km.size(), hk.data() + (b * rows + r) * D);
            std::copy_n(vm.data(), vm.size(), hv.data() + (b * rows + r) * D);
            r += km.rows();
        }
        for (std::size_t h = 0; h < G; ++h) {
            if (t.queries[h].size() != D) throw std::runtime_error("bad-shape: query width != key width");
            std::copy_n(t.queries[h].data(), D, hq.data() + (b * G + h) * D);
            bud[b * G + h] = h < t.plan.budgets.size() ? t.plan.budgets[h] : 0.0;
        }
        const int bs = t.plan.block_size;
        if (s.cpu > 0 && std::find(kCandidateBlocks.begin(), kCandidateBlocks.end(), bs) == kCandidateBlocks.end())
            throw std::runtime_error("invalid-granularity: blk must be one of 16/32/64/128");
        blk[b] = bs;
    }
    DevMem dk{std::span<const float>(hk)}, dv{std::span<const float>(hv)}, dq{std::span<const float>(hq)};
    DevMem dblk{std::span<const int32_t>(blk)}, dbud{std::span<const double>(bud)};
    DevMem dabs(B * D * sizeof(float)), dout(B * G * D * sizeof(float));
    std::vector<std::unique_ptr<DevMem>> meta;
    fx_step_args a{};
    if (s.cpu > 0) {
        for (int blk_c : kCandidateBlocks)
            meta.push_back(std::make_unique<DevMem>(fx_meta_level_bytes(&lay, blk_c)));
        check(fx_build_metadata_levels(context(), &lay, dk.get(), meta[0]->get(), meta[1]->get(),
                                       meta[2]->get(), meta[3]->get(), dabs.as<float>()));
        for (int i = 0; i < 4; ++i) a.meta[i] = meta[static_cast<std::size_t>(i)]->get();
        a.absmax = dabs.as<float>();
    }
    a.k = dk.get();
    a.v = dv.get();
    a.l_new = static_cast<int64_t>(s.fresh);
    a.q = dq.as<float>();
    a.plan_mode = FX_PLAN_GIVEN;
    a.plan_blk = dblk.as<int32_t>();
    a.plan_budgets = dbud.as<double>();
    a.o = dout.as<float>();
    check(fx_decode_step(context(), &lay, &a));
    const auto o = dout.download<float>(B * G * D);
    for (std::size_t b = 0; b < B; ++b) {
        out[b]->group_id = tasks[b]->group_id;
        out[b]->head_outputs.assign(G, std::vector<double>(D));
        for (std::size_t h = 0; h < G; ++h)
            std::copy_n(o.data() + (b * G + h) * D, D, out[b]->head_outputs[h].data());
    }
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
    execute_batch(one, out);
    return r;
}

std::vector<TaskResult> execute_batch(std::span<const SparseTask> tasks) {
    std::vector<TaskResult> res(tasks.size());
    std::vector<bool> done(tasks.size(), false);
    for (std::size_t i = 0; i < tasks.size(); ++i) {
        if (done[i]) continue;
        if (!tasks[i].cache || !tasks[i].metadata)
            throw std::runtime_error("no-context: task has no executable payload");
        const Shape s = shape_of(tasks[i]);
        std::vector<const SparseTask*> batch;
        std::vector<TaskResult*> out;
        for (std::size_t j = i; j < tasks.size(); ++j) {
            if (done[j] || !tasks[j].cache || !tasks[j].metadata || !(shape_of(tasks[j]) == s)) continue;
            batch.push_back(&tasks[j]);
            out.push_back(&res[j]);
            done[j] = true;
        }
        execute_batch(batch, out);
    }
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
    // one device step per distinct task shape (one in practice: a decode step);
    // a task counts as done only once its batch has executed
    std::vector<bool> done(tasks.size(), false), claimed(tasks.size(), false);
    for (std::size_t i = 0; i < tasks.size(); ++i) {
        if (claimed[i]) continue;
        std::vector<std::size_t> idx;
        std::vector<const SparseTask*> batch;
        std::vector<TaskResult*> out;
        try {
            if (!tasks[i].cache || !tasks[i].metadata)
                throw std::runtime_error("no-context: task has no executable payload");
            const Shape s = shape_of(tasks[i]);
            for (std::size_t j = i; j < tasks.size(); ++j) {
                if (claimed[j] || !tasks[j].cache || !tasks[j].metadata || !(shape_of(tasks[j]) == s)) continue;
                idx.push_back(j);
                batch.push_back(&tasks[j]);
                out.push_back(&res[j]);
                claimed[j] = true;
            }
            execute_batch(batch, out);
            for (std::size_t j : idx) done[j] = true;
        } catch (const std::exception&) {
            // the reference records the group whose task threw (scheduler.cpp:247-252)
            if (idx.empty()) idx.push_back(i);
            for (std::size_t j : idx) {
                claimed[j] = true;
                rep.failed_groups.push_back(tasks[j].group_id);
            }
            rep.aborted = true;
            break;
        }
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
