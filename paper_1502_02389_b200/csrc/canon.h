// canon.h — the canonical decomposition constants of the lift kernels.
//
// These fix the ORDER of every floating-point addition (reading R5),
// so they are part of the numerical contract: changing one changes result bits
// (never correctness).  lift_workspace_bytes() is derived from them.
#pragma once

namespace lift {

// asum / dot (reduce.cuh)
constexpr int RED_T = 256;                        // lanes per chunk (= threads per CTA)
constexpr int RED_V = 8;                          // floats per vector slot (asVector^8)
#ifndef LIFT_RED_K
#define LIFT_RED_K 4     // 8192-element chunks: short per-CTA work, fine-grained balance
#endif
#ifndef LIFT_RED_G
#define LIFT_RED_G 256   // 2^21-element groups
#endif
constexpr int RED_K = LIFT_RED_K;                 // vectors per lane per chunk
constexpr long long RED_C = (long long)RED_T * RED_V * RED_K;  // elements per chunk
constexpr int RED_G = LIFT_RED_G;                 // chunks per group (level-1 fold)
static_assert(RED_G <= RED_T, "group fold uses one leaf per thread");

// gemv: rows of n >= GEMV_LONG_N = 65536 use exactly the dot order above (gemv_long.cuh);
// shorter rows the order defined in gemv.cuh: TR = gemv_tr_log2(n) threads per row
// (128 at n = 8192, 256 from n = 16384, down to 1 for short rows), thread t' owns the 8-float
// vectors t' + TR*k, 8 fp64 slot accumulators in ascending k, pairwise8, butterfly over
// the row's lanes, the row's TR/32 warp values pairwise (TR > 32).

}  // namespace lift
