// Reference selector API (selector.hpp) on the B200.
// Cites: /root/reference/proj/src/selector.cpp:9-52.
#include <stdexcept>

#include "../fx_selector_math.h"
#include "fluxattn/selector.hpp"
#include "fx_api_common.hpp"

namespace fluxattn {

double volume(int block_size, std::size_t l_cpu, std::span<const double> budgets) {
    double sum = 0.0;
    for (double b : budgets) sum = fx::sel::add(sum, fx::sel::clamp01(b));
    return fx::sel::volume_from_sum(block_size, static_cast<int64_t>(l_cpu), sum);
}

double budget_at(const HeadProperties& props, int block_size) {
    return fx::sel::budget_at(props.bgt0, props.k, props.streaming ? 1 : 0, block_size);
}

// plan_group runs on the device (the same kernel as the batched decode step).
GroupPlan plan_group(int group_id, std::span<const HeadProperties> props, std::size_t l_cpu) {
    if (props.empty()) throw std::runtime_error("empty-group: plan_group needs at least one head");
    using b200::DevMem;
    const std::size_t G = props.size();
    std::vector<double> b0(G), ks(G);
    std::vector<int32_t> st(G);
    for (std::size_t h = 0; h < G; ++h) {
        b0[h] = props[h].bgt0;
        ks[h] = props[h].k;
        st[h] = props[h].streaming ? 1 : 0;
    }
    DevMem db0{std::span<const double>(b0)}, dks{std::span<const double>(ks)}, dst{std::span<const int32_t>(st)};
    DevMem dblk(sizeof(int32_t)), dbud(G * sizeof(double)), dvol(sizeof(double)), dcand(4 * sizeof(double));
    b200::check(fx_plan_groups(b200::context(), 1, static_cast<int32_t>(G), static_cast<int64_t>(l_cpu),
                               db0.as<double>(), dks.as<double>(), dst.as<int32_t>(), dblk.as<int32_t>(),
                               dbud.as<double>(), dvol.as<double>(), dcand.as<double>(), nullptr));
    GroupPlan plan;
    plan.group_id = group_id;
    plan.block_size = dblk.download<int32_t>(1)[0];
    plan.streaming_group = plan.block_size == 0;
    if (plan.streaming_group) return plan;
    plan.budgets = dbud.download<double>(G);
    plan.volume = dvol.download<double>(1)[0];
    const auto c = dcand.download<double>(4);
    for (int i = 0; i < 4; ++i) plan.candidate_volumes[static_cast<std::size_t>(i)] = c[static_cast<std::size_t>(i)];
    return plan;
}

double priority(const GroupPlan& plan) {
    if (plan.streaming_group) throw std::runtime_error("not-schedulable: streaming group has no priority");
    return plan.volume;
}

}  // namespace fluxattn
