// The reference's own decode loop (run_decode, pipeline.cpp:177-415) on a
// reference-generated workload, built twice by oracle/Makefile (target
// `dropin`): against the unmodified reference (pipeline_ref) and against this
// repo's include/ tree with the attention / block-index / selector / scheduler
// of libfluxattn_b200.so (pipeline_dropin, the reference's pipeline.cpp,
// features.cpp, budget_oracle.cpp, ... compiled unchanged).  Prints the decode
// report as JSON.  TEST INFRASTRUCTURE (tests/test_dropin.py).
//
// usage: pipeline_driver out.json context heads group_size head_dim layers steps
//                        fixed_blk fixed_bgt measure_deviation seed
//        fixed_blk 0 = the oracle property source (output-aware budgets).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>

#include "fluxattn/pipeline.hpp"
#include "fluxattn/workload.hpp"

using namespace fluxattn;

int main(int argc, char** argv) {
    if (argc < 12) {
        std::fprintf(stderr, "usage: %s out.json context heads G D layers steps blk bgt measure seed\n", argv[0]);
        return 2;
    }
    WorkloadSpec spec;
    spec.context_len = std::atoi(argv[2]);
    spec.heads = std::atoi(argv[3]);
    spec.group_size = std::atoi(argv[4]);
    spec.head_dim = std::atoi(argv[5]);
    spec.layers = std::atoi(argv[6]);
    spec.decode_steps = std::atoi(argv[7]);
    spec.seed = std::strtoull(argv[11], nullptr, 10);
    const int blk = std::atoi(argv[8]);
    const double bgt = std::atof(argv[9]);
    try {
        const Workload w = generate(spec);
        DecodeConfig cfg;
        cfg.mode = RunMode::Executed;
        cfg.profile = WorkerProfile::standard(static_cast<std::size_t>(spec.head_dim));
        cfg.measure_deviation = std::atoi(argv[10]) != 0;
        if (blk > 0) cfg.fixed = std::make_pair(blk, bgt);
        const auto t0 = std::chrono::steady_clock::now();
        const DecodeReport rep = run_decode(w, cfg);
        const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::ofstream f(argv[1]);
        f.precision(17);
        f << "{\"seconds\":" << sec << ",\"steps\":[";
        for (std::size_t i = 0; i < rep.steps.size(); ++i) {
            const StepReport& s = rep.steps[i];
            f << (i ? "," : "") << "{\"step\":" << s.step << ",\"makespan\":" << s.makespan
              << ",\"scheduled_tasks\":" << s.scheduled_tasks << ",\"streaming_groups\":" << s.streaming_groups
              << ",\"mean_allocated_budget\":" << s.mean_allocated_budget << ",\"total_volume\":" << s.total_volume
              << ",\"head_deviations\":[";
            for (std::size_t j = 0; j < s.head_deviations.size(); ++j) f << (j ? "," : "") << s.head_deviations[j];
            f << "]}";
        }
        f << "],\"plans\":[";
        for (std::size_t i = 0; i < rep.plans.size(); ++i) f << (i ? "," : "") << rep.plans[i].to_json();
        f << "]}\n";
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
