// fluxattn/selector.hpp -- drop-in declarations of the granularity-budget
// selector (/root/reference/proj/include/fluxattn/selector.hpp:12-39).
// plan_group runs on the B200 (fx_plan_groups); volume / budget_at evaluate the
// same single-source f64 arithmetic the device kernel uses
// (paper_2605_07719_b200/csrc/fx_selector_math.h).
#pragma once

#include <array>
#include <cstddef>
#include <span>
#include <vector>

#include "fluxattn/budget_oracle.hpp"

namespace fluxattn {

inline constexpr std::array<int, 4> kCandidateBlocks{16, 32, 64, 128};

struct GroupPlan {
    int group_id = 0;
    int block_size = 0;
    std::vector<double> budgets;  // per head; 0 for streaming heads
    double volume = 0.0;          // token-units at block_size (Eq. 3)
    bool streaming_group = false;
    std::array<double, 4> candidate_volumes{};
};

double volume(int block_size, std::size_t l_cpu, std::span<const double> budgets);
double budget_at(const HeadProperties& props, int block_size);
GroupPlan plan_group(int group_id, std::span<const HeadProperties> props, std::size_t l_cpu);
double priority(const GroupPlan& plan);

}  // namespace fluxattn
