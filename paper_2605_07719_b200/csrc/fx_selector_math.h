// fx_selector_math.h -- single-source (host + device) arithmetic of the
// granularity-budget selector, used by the K5 kernel (fx_plan.cu) and by the
// C++ drop-in's scalar helpers, so both evaluate the identical operation
// sequence.  f64, round-to-nearest, no FMA contraction (the reference host
// build has none).
//   budget_at          selector.cpp:15-19   (Eq. 1)
//   volume             selector.cpp:9-13    (Eq. 3)
//   blocks_for_budget  block_index.cpp:96-103
#pragma once

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define FX_HD __host__ __device__ __forceinline__
#else
#define FX_HD inline
#endif

namespace fx {
namespace sel {

#if defined(__CUDA_ARCH__)
FX_HD double mul(double a, double b) { return __dmul_rn(a, b); }
FX_HD double add(double a, double b) { return __dadd_rn(a, b); }
FX_HD double sub(double a, double b) { return __dsub_rn(a, b); }
FX_HD double div(double a, double b) { return __ddiv_rn(a, b); }
#else
// Host: separate statements keep the compiler from contracting mul+add.
FX_HD double mul(double a, double b) {
    volatile double r = a * b;
    return r;
}
FX_HD double add(double a, double b) {
    volatile double r = a + b;
    return r;
}
FX_HD double sub(double a, double b) {
    volatile double r = a - b;
    return r;
}
FX_HD double div(double a, double b) {
    volatile double r = a / b;
    return r;
}
#endif

FX_HD double clamp01(double x) { return x < 0.0 ? 0.0 : (1.0 < x ? 1.0 : x); }

// log2 of the candidate granularities is exact
FX_HD double log2_blk(int blk) {
    return blk == 16 ? 4.0 : blk == 32 ? 5.0 : blk == 64 ? 6.0 : blk == 128 ? 7.0 : log2((double)blk);
}

FX_HD double budget_at(double bgt0, double k, int streaming, int blk) {
    if (streaming) return 0.0;
    const double kk = (k < 0.0) ? 0.0 : k;  // std::max(k, 0.0)
    return clamp01(add(bgt0, mul(kk, log2_blk(blk))));
}

// Eq. 3 given the already-clamped, head-order budget sum.
FX_HD double volume_from_sum(int blk, int64_t l_cpu, double clamped_sum) {
    const double L = (double)l_cpu;
    return add(div(mul(2.0, L), (double)blk), mul(mul(2.0, L), clamped_sum));
}

FX_HD int64_t blocks_for_budget(double budget, int64_t l_cpu, int blk) {
    if (!(budget > 0.0) || l_cpu == 0 || blk <= 0) return 0;
    const int64_t nblk = (l_cpu + blk - 1) / blk;
    const double raw = div(mul(budget, (double)l_cpu), (double)blk);
    const double c = ceil(sub(raw, 1e-12));
    int64_t k = c <= 0.0 ? 0 : (int64_t)c;
    if (k < 1) k = 1;
    return k < nblk ? k : nblk;
}

}  // namespace sel
}  // namespace fx
