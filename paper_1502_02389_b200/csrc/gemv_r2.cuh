// gemv_r2.cuh — gemv variant: each thread carries TWO rows (LIFT_VAR_GEMV_X = 4).
//
// gemv_kernel gives every thread one row; its x vectors (through L1) and their F2F
// conversions are paid once per row.  Here virtual row thread tp of two consecutive rows is
// one physical thread: each x vector is loaded and widened once and feeds both rows, so x
// costs half the loads, registers and XU conversions per A element.  Same canonical order
// (gemv.cuh: per row, thread tp's 8 slot accumulators over vectors tp + TR*k in ascending
// k, pairwise8, butterfly, TR/32 warp values pairwise) — bit-identical to gemv_kernel.
// Shapes: 2048 <= n, n % (8 TR GR2_B) == 0, 16-byte aligned rows; others use gemv_kernel.
#pragma once
#include "common.cuh"
#include "canon.h"
#include "gemv.cuh"

namespace lift {

#ifndef LIFT_GR2_B
#define LIFT_GR2_B 2      // vectors per row per thread in flight (x2 rows)
#endif
#ifndef LIFT_GR2_MINB
#define LIFT_GR2_MINB 5   // resident 128-thread CTAs per SM (register budget ~100)
#endif
constexpr int GR2_B = LIFT_GR2_B;

__host__ __device__ constexpr int gr2_threads(int trl) { return (1 << trl) < 128 ? 128 : (1 << trl); }

__host__ __device__ inline bool gr2_shape_ok(int64_t n) {
    if (n < 2048) return false;
    const int64_t tr = (int64_t)1 << gemv_tr_log2(n);
    return n % (8 * tr * GR2_B) == 0;
}

template <int TRL, int LW>
__global__ void __launch_bounds__(gr2_threads(TRL), LIFT_GR2_MINB) gemv_r2_kernel(GemvArgs a) {
    constexpr int TR = 1 << TRL;
    constexpr int T = gr2_threads(TRL);
    constexpr int G = T / TR;     // row pairs per block
    constexpr int RB = 2 * G;     // rows per block
    constexpr int B = GR2_B;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int tp = t & (TR - 1);
    const int g = t >> TRL;
    if (a.prefetch && tp < 2 && blockIdx.x < a.nblocks) {  // the block's rows (prefetch_l2)
        const int64_t row = (int64_t)blockIdx.x * RB + 2 * g + tp;
        if (row < a.m) prefetch_l2<4>(a.A + row * a.lda, a.n * 4);
    }
    pdl_wait();
    pdl_trigger();
    __shared__ double wv[2][2][T / 32];  // [block parity][row of the pair][warp]
    const int64_t nv = a.n / 8;
    int par = 0;
    for (int64_t blk = blockIdx.x; blk < a.nblocks; blk += gridDim.x, par ^= 1) {
        const int64_t r0 = blk * RB + 2 * g, r1 = r0 + 1;
        const float* p0 = a.A + (r0 < a.m ? r0 : a.m - 1) * a.lda;  // dead rows re-read a live one
        const float* p1 = a.A + (r1 < a.m ? r1 : a.m - 1) * a.lda;
        double acc0[8], acc1[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc0[e] = acc1[e] = 0.0;
        for (int64_t k = 0; k * TR < nv; k += B) {
            f8 a0[B], a1[B], xv[B];
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const int64_t q = tp + (k + b) * TR;
                a0[b] = ld_slot<LW>(p0 + 8 * q);
                a1[b] = ld_slot<LW>(p1 + 8 * q);
                xv[b] = ld_x<LW>(a.x + 8 * q);
            }
#pragma unroll
            for (int b = 0; b < B; ++b)
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const double xd = (double)xv[b].v[e];  // one widening feeds both rows
                    acc0[e] = __fma_rn((double)a0[b].v[e], xd, acc0[e]);
                    acc1[e] = __fma_rn((double)a1[b].v[e], xd, acc1[e]);
                }
        }
        const double v0 = warp_pairwise(pairwise8(acc0));
        const double v1 = warp_pairwise(pairwise8(acc1));
        if (lane == 0) {
            wv[par][0][warp] = v0;
            wv[par][1][warp] = v1;
        }
        __syncthreads();
        if (tp < 2) {  // thread 0 of the row group folds row 0, thread 1 row 1
            const int64_t row = tp == 0 ? r0 : r1;
            const double* w = wv[par][tp] + (warp & ~((TR >> 5) - 1));  // the group's first warp
            double d;
            if constexpr (TRL == 8) d = pairwise8(w);
            else if constexpr (TRL == 7) d = __dadd_rn(__dadd_rn(w[0], w[1]), __dadd_rn(w[2], w[3]));
            else if constexpr (TRL == 6) d = __dadd_rn(w[0], w[1]);
            else d = w[0];
            if (row < a.m) {
                const double yb = __dmul_rn((double)a.beta, (double)a.y[row]);  // scal(b, y)
                a.y_out[row] = __double2float_rn(__fma_rn((double)a.alpha, d, yb));
            }
        }
    }
}

}  // namespace lift
