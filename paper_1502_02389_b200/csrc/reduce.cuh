// reduce.cuh — R1..R4: the fused single-pass map-reduce for asum and dot.
//
//   asum(x)   = reduce(add, 0) o map(abs, x)
//   dot(x, y) = reduce(add, 0) o map(mult) o zip(x, y)
//
// The kernel realises the end point of the paper's Fig. 4 derivation,
//   reduce(+,0) o join o map(reduce-seq(lambda acc,a. acc + abs(a), 0)) o split^C,
// with the device-specific structure of Fig. 7a/7b re-designed for B200:
//
//  R2 split^C + reorder-stride: the input is cut into canonical chunks
//     of RED_C = 2^15 elements.  Inside a chunk, lane t of RED_T = 256 owns the
//     8-float vectors t, t+256, t+512, ... (reorder-stride with s = 256), so a warp
//     reads 32 consecutive 32-byte vectors per instruction (LDG.256, coalesced).
//     Chunks go to CTAs grid-stride (map-workgroup).
//  R1 fused reduce-seq o map-seq (rule 5f): each lane keeps 8
//     accumulators (one per vector slot e) and folds acc_e = acc_e + |x| (asum) or
//     acc_e = fma(x, y, acc_e) (dot) over its 16 vectors in ascending order — no
//     intermediate array.
//  R3 toLocal + iterate(split-2 reduce): lane value = fixed pairwise
//     fold of its 8 accumulators in fp64; warp butterfly (xor 1,2,4,8,16); then the
//     8 warp values pairwise through shared memory -> one fp64 CHUNK PARTIAL.
//  R4 the outermost reduce-seq o join, single pass, no second launch: a
//     two-level last-block-done.  The CTA that finishes the last chunk of a group of
//     RED_G = 64 chunks folds that group's partials (pairwise); the CTA that
//     finishes the last group folds the group partials (pairwise, zero-padded to a
//     power of two) and writes the fp32 result (rounded once) and/or the fp64
//     partial.  Tickets are reset to 0 by the CTAs that consume them.
//
// Determinism: every addition above happens in an order that is a pure function of
// n (chunk, lane, slot, group indices) — never of the grid size, the SM count,
// the load width or the CTA finishing order.  Results are bit-identical run to run
// and across grid sizes.  Together the chunk/group/final folds form the pairwise
// tree over chunk partials zero-padded to a power of two, so shards whose size is a
// power-of-two number of groups compose bit-exactly (reading R5).
#pragma once
#include "common.cuh"
#include "canon.h"

namespace lift {

// The fused per-element step (rule 5f).  Acc is the per-lane accumulator type: fp32
// (the paper-era choice; overflows to Inf if a 16-term lane run exceeds FLT_MAX) or
// fp64 (exact products, no overflow for any finite fp32 input; the default — see
// DESIGN.md reading R13 and the measured cost in profiles/).
template <class Acc>
struct AsumOp {
    using acc_t = Acc;
    static constexpr bool kTwoInputs = false;
    __device__ __forceinline__ static Acc step(Acc acc, float a, float) {
        if constexpr (sizeof(Acc) == 8) return __dadd_rn(acc, fabs((double)a));
        else return __fadd_rn(acc, fabsf(a));  // abs then add, fused
    }
};
template <class Acc>
struct DotOp {
    using acc_t = Acc;
    static constexpr bool kTwoInputs = true;
    __device__ __forceinline__ static Acc step(Acc acc, float a, float b) {
        if constexpr (sizeof(Acc) == 8) return __fma_rn((double)a, (double)b, acc);  // exact product
        else return __fmaf_rn(a, b, acc);  // mult then add, one rounding
    }
};

struct ReduceArgs {
    int64_t n;
    const float* x;
    const float* y;
    int64_t nc;          // chunks
    int64_t ng;          // groups
    unsigned* tick;      // ng group tickets + 1 global ticket (zero on entry and exit)
    double* chunk_part;  // nc
    double* group_part;  // ng
    float* out_f32;      // may be null
    double* out_f64;     // may be null
};

// Pairwise fold of 256 per-thread values (warp butterfly, then 8 warps pairwise).
// Result valid in thread 0.  `wbuf` holds 8 doubles in shared memory.
__device__ __forceinline__ double cta_pairwise256(double v, double* wbuf) {
    v = warp_pairwise(v);
    if ((threadIdx.x & 31) == 0) wbuf[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0) r = pairwise8(wbuf);
    __syncthreads();  // wbuf may be reused after this
    return r;
}

template <class Op, int LW, int B0>
__device__ __forceinline__ void chunk_body_full(const float* xc, const float* yc,
                                                typename Op::acc_t* acc) {
    constexpr int B = B0 < RED_K ? B0 : RED_K;
    static_assert(RED_K % B == 0, "load batch must divide RED_K");
    const int t = threadIdx.x;
#pragma unroll
    for (int k0 = 0; k0 < RED_K; k0 += B) {
        f8 xv[B];
        f8 yv[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            xv[b] = ld_slot<LW>(xc + (int64_t)RED_V * (t + (k0 + b) * RED_T));
            if constexpr (Op::kTwoInputs)
                yv[b] = ld_slot<LW>(yc + (int64_t)RED_V * (t + (k0 + b) * RED_T));
        }
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
            for (int e = 0; e < RED_V; ++e)
                acc[e] = Op::step(acc[e], xv[b].v[e], Op::kTwoInputs ? yv[b].v[e] : 0.f);
    }
}

// Partial last chunk: same order, elements >= n skipped.  Skipping equals adding
// +0 exactly (the accumulators start at +0 and can never become -0 in RN).
template <class Op>
__device__ __forceinline__ void chunk_body_tail(const float* xc, const float* yc, int64_t len,
                                                typename Op::acc_t* acc) {
    const int t = threadIdx.x;
    for (int k = 0; k < RED_K; ++k) {
#pragma unroll
        for (int e = 0; e < RED_V; ++e) {
            const int64_t j = (int64_t)RED_V * (t + k * RED_T) + e;
            if (j < len) acc[e] = Op::step(acc[e], xc[j], Op::kTwoInputs ? yc[j] : 0.f);
        }
    }
}

template <class Op, int LW, int B>
__global__ void __launch_bounds__(RED_T) reduce_kernel(ReduceArgs a) {
    __shared__ double wbuf[RED_T / 32];
    __shared__ int s_last_chunk, s_last_group;
    const int t = threadIdx.x;

    for (int64_t c = blockIdx.x; c < a.nc; c += gridDim.x) {
        // ---- R1/R2: fused per-lane fold over the chunk ---------------------------
        const int64_t base = c * RED_C;
        const float* xc = a.x + base;
        const float* yc = Op::kTwoInputs ? a.y + base : nullptr;
        typename Op::acc_t acc[RED_V];
#pragma unroll
        for (int e = 0; e < RED_V; ++e) acc[e] = 0;
        if (base + RED_C <= a.n) chunk_body_full<Op, LW, B>(xc, yc, acc);
        else chunk_body_tail<Op>(xc, yc, a.n - base, acc);

        // ---- R3: lane -> warp -> CTA, fixed pairwise, fp64 -----------------------
        double lane8[RED_V];
#pragma unroll
        for (int e = 0; e < RED_V; ++e) lane8[e] = (double)acc[e];
        const double part = cta_pairwise256(pairwise8(lane8), wbuf);

        // ---- R4 level 1: publish the chunk partial, group ticket -----------------
        const int64_t g = c / RED_G;
        if (t == 0) {
            a.chunk_part[c] = part;
            __threadfence();
            const int64_t gcount = min((int64_t)RED_G, a.nc - g * RED_G);
            const unsigned old = atomicAdd(&a.tick[g], 1u);
            s_last_chunk = (old == (unsigned)(gcount - 1));
        }
        __syncthreads();
        if (!s_last_chunk) continue;  // uniform across the CTA

        // This CTA finished the group's last chunk: fold the group (pairwise over
        // RED_G leaves; RED_G <= RED_T so one leaf per thread, missing ones = 0).
        __threadfence();
        const int64_t leaf = g * RED_G + t;
        double v = (t < RED_G && leaf < a.nc) ? __ldcg(&a.chunk_part[leaf]) : 0.0;
        const double gpart = cta_pairwise256(v, wbuf);
        if (t == 0) {
            a.group_part[g] = gpart;
            a.tick[g] = 0u;  // reset for the next call (workspace contract)
            __threadfence();
            const unsigned old = atomicAdd(&a.tick[a.ng], 1u);
            s_last_group = (old == (unsigned)(a.ng - 1));
        }
        __syncthreads();
        if (!s_last_group) continue;

        // ---- R4 level 2: final fold over all group partials ----------------------
        __threadfence();
        int64_t p2 = 1;
        while (p2 < a.ng) p2 <<= 1;
        double tv;
        if (p2 <= RED_T) {
            tv = (t < a.ng) ? __ldcg(&a.group_part[t]) : 0.0;
        } else {
            // Thread t folds the aligned block [t*blk, (t+1)*blk) pairwise with a
            // binary-counter stack, so the overall fold is the pairwise tree.
            const int64_t blk = p2 / RED_T;
            double stk[40];
            int top = 0;
            for (int64_t i = 0; i < blk; ++i) {
                const int64_t li = (int64_t)t * blk + i;
                double w = (li < a.ng) ? __ldcg(&a.group_part[li]) : 0.0;
                for (int64_t cnt = i; cnt & 1; cnt >>= 1) w = __dadd_rn(stk[--top], w);
                stk[top++] = w;
            }
            tv = stk[0];
        }
        const double total = cta_pairwise256(tv, wbuf);
        if (t == 0) {
            if (a.out_f64) *a.out_f64 = total;
            if (a.out_f32) *a.out_f32 = __double2float_rn(total);
            a.tick[a.ng] = 0u;
        }
    }
}

}  // namespace lift
