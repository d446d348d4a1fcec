// gemv_long.cuh — gemv rows of n >= GEMV_LONG_N columns (G2 for long rows).
//
// For long rows the canonical order of a row's dot is EXACTLY the stand-alone dot's
// (reduce.cuh, reading R5): chunks of RED_C = 8192 columns; in a chunk lane t of 256
// owns the 8-float vectors t + 256k (k < RED_K), 8 fp64 slot accumulators, pairwise8,
// warp butterfly, the 8 warp values pairwise -> chunk partial; chunk partials pairwise in
// groups of RED_G (zero-padded to a power of two), group partials pairwise (zero-padded).
// So gemv(A, x, y, a, b)_i = fp32(fma(a, dot64(A_i, x), b * y_i)) with dot64 bit-identical
// to lift_dot_partial(A_i, x) — tested.
//
// Two kernels compute that order:
//  * gemv_long_kernel: one 256-thread CTA per row (grid-stride over rows), chunk by
//    chunk; thread 0 folds the chunk partials on binary-counter stacks (the pairwise tree
//    of aligned power-of-two blocks).  Enough rows keep every SM busy.
//  * gemv_split_kernel (few rows, workspace given): one CTA per (row, chunk), the
//    reduction kernel's single-pass two-level last-block-done per row (per-row tickets),
//    and the row's final CTA runs the epilogue.  A 1 x 2^24 gemv becomes 2048 CTAs
//    instead of one.
#pragma once
#include "gemv.cuh"
#include "reduce.cuh"

namespace lift {

constexpr int64_t GEMV_LONG_N = 1 << 16;  // canonical: rows this long use the dot order

// Pairwise tree of `count` leaves pushed one by one (binary-counter stack), closed by
// zero leaves up to the next power of two: equals warp_fold_leaves over the same leaves.
struct PairStack {
    double s[24];
    int top = 0;
    int64_t n = 0;
    __device__ __forceinline__ void push(double w) {
        for (int64_t c = n; c & 1; c >>= 1) w = __dadd_rn(s[--top], w);
        s[top++] = w;
        ++n;
    }
    __device__ __forceinline__ double close() {
        int64_t p2 = 1;
        while (p2 < n) p2 <<= 1;
        while (n < p2) push(0.0);
        const double r = s[0];
        top = 0;
        n = 0;
        return r;
    }
};

__device__ __forceinline__ void gemv_row_out(const GemvArgs& a, int64_t row, double d, bool peers) {
    const double yb = __dmul_rn((double)a.beta, (double)a.y[row]);  // scal(b, y): exact
    const float out = __double2float_rn(__fma_rn((double)a.alpha, d, yb));
    if (peers) {
        for (int q = 0; q < a.p; ++q) a.y_peers[q][a.row0 + row] = out;
    } else {
        a.y_out[row] = out;
    }
}

template <int LW, bool PEERS>
__global__ void __launch_bounds__(RED_T, 4) gemv_long_kernel(GemvArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ double wbuf[2][RED_T / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t nc = (a.n + RED_C - 1) / RED_C;
    const int64_t ng = (nc + RED_G - 1) / RED_G;
    int par = 0;
    for (int64_t row = blockIdx.x; row < a.m; row += gridDim.x) {
        const float* rp = a.A + row * a.lda;
        PairStack cs, gs;  // meaningful in thread 0 only
        double gp = 0.0;
        for (int64_t c = 0; c < nc; ++c, par ^= 1) {
            const int64_t base = c * RED_C;
            double acc[RED_V];
#pragma unroll
            for (int e = 0; e < RED_V; ++e) acc[e] = 0.0;
            if (base + RED_C <= a.n) chunk_body_full<DotOp<double>, LW, 4>(rp + base, a.x + base, acc);
            else chunk_body_tail<DotOp<double>>(rp + base, a.x + base, a.n - base, acc);
            const double v = warp_pairwise(pairwise8(acc));
            if (lane == 0) wbuf[par][warp] = v;
            __syncthreads();
            if (t == 0) {
                cs.push(pairwise8(wbuf[par]));
                if ((c + 1) % RED_G == 0 || c + 1 == nc) {
                    gp = cs.close();
                    if (ng > 1) gs.push(gp);
                }
            }
        }
        if (t == 0) gemv_row_out(a, row, ng > 1 ? gs.close() : gp, PEERS);
    }
    if constexpr (PEERS) {  // once per CTA, after its rows
        __syncthreads();  // every row store of this CTA precedes its count
        if (warp == 0) {
            const int64_t mine = blockIdx.x < a.m ? (a.m - 1 - blockIdx.x) / gridDim.x + 1 : 0;
            gemv_cta_done(a, mine);
        }
    }
}

// Split path workspace (W bytes, zero-filled once): [chunk partials f64 m x nc]
// [group partials f64 m x ng] ... [tickets u32 m x (ng + 1): the last gemv_ws_ticket_region(W)
// bytes].  As for the reductions, the ticket region depends on W only, and every ticket
// is reset to 0 by the CTA that consumes it, so one buffer serves every (m, n) it fits.
__host__ __device__ constexpr size_t gemv_ws_ticket_region(size_t w) {
    return (w / 3) & ~(size_t)15;
}

struct GemvSplitArgs {
    GemvArgs g;
    int64_t nc, ng;
    double* chunk_part;  // m x nc
    double* group_part;  // m x ng
    unsigned* tick;      // m x (ng + 1)
};

template <int LW>
__global__ void __launch_bounds__(RED_T, DotOp<double>::kMinBlocks) gemv_split_kernel(GemvSplitArgs s) {
    pdl_wait();
    pdl_trigger();
    const GemvArgs& a = s.g;
    __shared__ double wbuf[RED_T / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t total = a.m * s.nc;
    for (int64_t id = blockIdx.x; id < total; id += gridDim.x) {
        const int64_t row = id / s.nc, c = id - row * s.nc;
        const int64_t base = c * RED_C;
        const float* rp = a.A + row * a.lda;
        double acc[RED_V];
#pragma unroll
        for (int e = 0; e < RED_V; ++e) acc[e] = 0.0;
        if (base + RED_C <= a.n) chunk_body_full<DotOp<double>, LW, 4>(rp + base, a.x + base, acc);
        else chunk_body_tail<DotOp<double>>(rp + base, a.x + base, a.n - base, acc);
        const double v = warp_pairwise(pairwise8(acc));
        if (lane == 0) wbuf[warp] = v;
        __syncthreads();
        if (warp == 0) {
            double* cp = s.chunk_part + row * s.nc;
            double* gpart = s.group_part + row * s.ng;
            unsigned* tk = s.tick + row * (s.ng + 1);
            const int64_t g = c / RED_G;
            unsigned last = 0;
            if (lane == 0) {
                cp[c] = pairwise8(wbuf);
                const int64_t gcount = min((int64_t)RED_G, s.nc - g * RED_G);
                last = (ticket_acq_rel(&tk[g]) == (unsigned)(gcount - 1));
            }
            if (__shfl_sync(0xffffffffu, last, 0)) {
                ticket_acquired(&tk[g]);
                const int64_t g0 = g * RED_G;
                const double gv = warp_fold_leaves(cp + g0, min((int64_t)RED_G, s.nc - g0));
                if (s.ng == 1) {
                    if (lane == 0) {
                        tk[0] = 0u;
                        gemv_row_out(a, row, gv, false);
                    }
                } else {
                    last = 0;
                    if (lane == 0) {
                        gpart[g] = gv;
                        tk[g] = 0u;  // reset for the next call (workspace contract)
                        last = (ticket_acq_rel(&tk[s.ng]) == (unsigned)(s.ng - 1));
                    }
                    if (__shfl_sync(0xffffffffu, last, 0)) {
                        ticket_acquired(&tk[s.ng]);
                        const double d = warp_fold_leaves(gpart, s.ng);
                        if (lane == 0) {
                            tk[s.ng] = 0u;
                            gemv_row_out(a, row, d, false);
                        }
                    }
                }
            }
        }
        __syncthreads();  // wbuf is reused by the next (row, chunk)
    }
}

}  // namespace lift
