// gemv.cuh — G1..G3: y_out = alpha * A x + beta * y.
//
//   gemv(A, x, y, a, b):  z = map(scal(a) o dot(x), A)
//                         map(add) o zip(z, scal(b, y))
//
// A is row-major with leading dimension lda (map(..., A) maps over rows, P:815;
// DESIGN.md reading R8).  "The dot-product from gemv might be implemented in a
// totally different way from the stand-alone dot-product" — and it is:
//
//  G1 toLocal(x): x is staged once per resident CTA (per column panel of
//     up to GEMV_PMAX columns) by the TMA bulk-copy engine (cp.async.bulk -> UBLKCP,
//     an mbarrier counts the bytes) through a small fp32 staging buffer, and widened
//     to fp64 in a slot-major shared layout xs[e][q] = x[8q + e], so the per-lane
//     reads below are conflict-free LDS.64.  x is reused by every row the CTA folds.
//  G2 per-row dot, exact products, fp64 accumulation.  A WARP OWNS WHOLE ROWS (no
//     cross-warp combine per row): lane l owns the 8-float vectors l, l+32, l+64, ...
//     of a row (reorder-stride, s = 32; coalesced 256-bit LDG), 8 fp64 accumulators
//     per row and lane fold acc_e = fma(A_ij, x_j, acc_e) in ascending vector order
//     (A_ij * x_j is exact in fp64, so each step rounds once); lane value = pairwise
//     fold of the 8 accumulators, then the warp butterfly xor 1..16.  A warp carries
//     GEMV_R rows at once (each x slot read from shared memory feeds GEMV_R rows) and
//     keeps GEMV_U k-steps of loads in flight per row.
//  G3 fused epilogue (rule 5f map-map fusion): y_out_i = fp32(fma(alpha, d_i,
//     beta * y_i)) in fp64, rounded once (reading R10).  y_out may alias y.
//
// Scheduling: one CTA per block of (warps x GEMV_R) rows is launched; resident CTAs
// steal the not-yet-launched blocks with Cluster Launch Control, so x is staged once
// per resident CTA while the hardware balances rows across SMs.
//
// The order of every addition is a function of n only (not of m, the grid, the
// row-to-warp assignment, the load width or the panel count, since panels are
// multiples of 256 columns), so a row's bits are the same however rows are sharded.
//
// (A split-K variant — 8 warps per row, A rows streamed through a TMA ring by a
// producer warp — was built and measured: 5.4-5.6 TB/s at 8192x16384 but only
// 4.1-4.6 TB/s at 8192x8192, bounded by the per-row cross-warp combine; see
// profiles/.  Whole rows per warp won at the bench size.)
#pragma once
#include "common.cuh"
#include "canon.h"

namespace lift {

#ifndef LIFT_GEMV_R
#define LIFT_GEMV_R 2  // rows per warp
#endif
#ifndef LIFT_GEMV_U
#define LIFT_GEMV_U 4  // k-steps of loads in flight per row
#endif
constexpr int GEMV_R = LIFT_GEMV_R;
constexpr int GEMV_U = LIFT_GEMV_U;
constexpr int GEMV_PMAX = 16384;             // max x-panel columns staged in shared memory
#ifndef LIFT_GEMV_XSTG
#define LIFT_GEMV_XSTG 4096
#endif
constexpr int GEMV_XSTG = LIFT_GEMV_XSTG;     // fp32 staging buffer (floats) for the bulk copy
constexpr int GEMV_SMEM_LIMIT = 227 * 1024;  // opt-in dynamic shared memory per CTA

struct GemvArgs {
    int64_t m, n, lda;
    float alpha, beta;
    const float* A;
    const float* x;
    const float* y;
    float* y_out;
    int P;          // panel columns (multiple of 256, <= GEMV_PMAX)
    int xs_stride;  // doubles per slot row of xs (= P/8 + 1, padding breaks bank conflicts)
    // NEXT-1 fused all-gather of y (null y_peers: plain local y_out)
    float* const* y_peers;  // p pointers: every rank's full-length y (IPC-mapped)
    int64_t row0;           // global row of local row 0
    void* const* xpeers;    // p exchange buffers (flags + block counters)
    int p, rank;
    unsigned long long epoch;
    int* error;
    int64_t nblocks;        // row blocks of this launch
};

__host__ __device__ constexpr size_t gemv_smem_bytes(int P) {
    return 64 /*barriers*/ + (size_t)GEMV_XSTG * 4 /*fp32 stage*/ +
           (size_t)8 * (P / 8 + 1) * 8 /*fp64 slot-major x*/;
}

// Stage x[c0, c0+pc) into xs (fp64, slot-major).  Called by the whole CTA.
template <int NT>
__device__ __forceinline__ void gemv_stage_x(const GemvArgs& a, int64_t c0, int pc,
                                             uint64_t* bar, float* xstage, double* xs,
                                             uint32_t& phase) {
    const int t = threadIdx.x;
    for (int p0 = 0; p0 < pc; p0 += GEMV_XSTG) {
        const int len = min(GEMV_XSTG, pc - p0);
        const float* src = a.x + c0 + p0;
        const bool aligned = ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
        const int nbulk = aligned ? (len & ~3) : 0;  // elements moved by the TMA bulk copy
        if (t == 0 && nbulk > 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive_expect_tx(bar, (uint32_t)nbulk * 4u);
            bulk_g2s(xstage, src, (uint32_t)nbulk * 4u, bar);
        }
        for (int j = nbulk + t; j < len; j += NT) xstage[j] = __ldg(src + j);
        __syncthreads();
        if (nbulk > 0) {
            mbar_wait(bar, phase);
            phase ^= 1u;
        }
        for (int j = t; j < len; j += NT) {
            const int jj = p0 + j;
            xs[(jj & 7) * a.xs_stride + (jj >> 3)] = (double)xstage[j];
        }
        __syncthreads();  // xstage is reused by the next piece
    }
    // zero the padding slots of the last vector (columns pc .. round_up(pc, 8))
    for (int jj = pc + t; jj < ((pc + 7) & ~7); jj += NT)
        xs[(jj & 7) * a.xs_stride + (jj >> 3)] = 0.0;
    __syncthreads();
}

// Fold panel columns [c0, c0+pc) of rows `rows[0..R)` into acc (lane-owned vectors).
template <int R, int U, int LW>
__device__ __forceinline__ void gemv_panel(const GemvArgs& a, const int64_t* rows, int64_t c0,
                                           int pc, const double* xs, double (&acc)[R][8]) {
    const int lane = threadIdx.x & 31;
    const int kfull = pc / 256;  // k-steps where all 32 lanes hold a full vector
    const float* rowp[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rowp[r] = a.A + rows[r] * a.lda + c0;

    int k = 0;
    for (; k + U <= kfull; k += U) {
        f8 av[U][R];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int r = 0; r < R; ++r)
                av[u][r] = ld_slot<LW>(rowp[r] + 8 * (lane + 32 * (k + u)));
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int q = lane + 32 * (k + u);
            double xv[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) xv[e] = xs[e * a.xs_stride + q];
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    acc[r][e] = __fma_rn((double)av[u][r].v[e], xv[e], acc[r][e]);
        }
    }
    for (; k < kfull; ++k) {
        const int q = lane + 32 * k;
        f8 av[R];
#pragma unroll
        for (int r = 0; r < R; ++r) av[r] = ld_slot<LW>(rowp[r] + 8 * q);
        double xv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) xv[e] = xs[e * a.xs_stride + q];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[r][e] = __fma_rn((double)av[r].v[e], xv[e], acc[r][e]);
    }
    if (kfull * 256 < pc) {  // ragged last k-step: same order, columns >= pc skipped
        const int q = lane + 32 * kfull;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int j = 8 * q + e;
            if (j < pc) {
                const double xj = xs[e * a.xs_stride + q];
#pragma unroll
                for (int r = 0; r < R; ++r)
                    acc[r][e] = __fma_rn((double)__ldg(rowp[r] + j), xj, acc[r][e]);
            }
        }
    }
}

template <int R>
__device__ __forceinline__ void gemv_epilogue(const GemvArgs& a, const int64_t* rows, int nvalid,
                                              double (&acc)[R][8]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const double d = warp_pairwise(pairwise8(acc[r]));
        if (lane == r && r < nvalid) {
            const double w = __dmul_rn((double)a.beta, (double)a.y[rows[r]]);  // scal(b, y): exact
            const float out = __double2float_rn(__fma_rn((double)a.alpha, d, w));
            if (a.y_peers) {  // fused all-gather: the row lands in every rank's full y
                for (int q = 0; q < a.p; ++q) a.y_peers[q][a.row0 + rows[r]] = out;
            } else {
                a.y_out[rows[r]] = out;
            }
        }
    }
}

// NEXT-1 fused all-gather: after each row block the CTA counts it in this rank's
// exchange buffer; the CTA that completes the LAST block publishes the rank's flag into
// every peer's buffer (system-scope release; the row stores were fenced at system scope
// before each count) and waits for all p flags, so the kernel ends only when every
// rank's rows have landed in this rank's y — stream-ordered consumers can read it.
__device__ __forceinline__ void gemv_block_done(const GemvArgs& a) {
    const int lane = threadIdx.x & 31;
    const int bank = (int)(a.epoch & 1ull);
    unsigned last = 0;
    if (lane == 0) {
        __threadfence_system();  // this block's row stores before its count
        unsigned long long* cnt = xchg_counter(a.xpeers[a.rank], a.p, bank);
        last = (atomicAdd(cnt, 1ull) == (unsigned long long)(a.nblocks - 1));
        if (last) {
            __threadfence_system();
            *cnt = 0ull;  // reset for epoch + 2 (this bank's next use)
        }
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return;
    bool ok = true;
    if (lane < a.p) {
        XchgSlot* dst = reinterpret_cast<XchgSlot*>(a.xpeers[lane]) + bank * a.p + a.rank;
        st_release_sys(&dst->flag, a.epoch);
        ok = xchg_wait_flag(a.xpeers[a.rank], bank * a.p, lane, a.epoch);
    }
    if (!__all_sync(0xffffffffu, ok) && lane == 0 && a.error) *a.error = 1;
}

// MULTI = false: n <= P, x staged once per CTA.  MULTI = true: n > P, x re-staged per
// panel for every row block.
template <int NT, int R, int U, int LW, bool MULTI>
// minBlocks = 2 for 256 threads (two CTAs per SM) gives ptxas a 128-register budget, which
// it spends on issuing all GEMV_U x GEMV_R 256-bit loads of a step up front (measured).
__global__ void __launch_bounds__(NT, (NT <= 256 ? 2 : 1)) gemv_kernel(GemvArgs a) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint64_t* clc_bar = reinterpret_cast<uint64_t*>(smem + 8);
    uint4* clc_resp = reinterpret_cast<uint4*>(smem + 16);
    float* xstage = reinterpret_cast<float*>(smem + 64);
    double* xs = reinterpret_cast<double*>(smem + 64 + (size_t)GEMV_XSTG * 4);
    const int warp = threadIdx.x >> 5;
    uint32_t phase = 0;
    Clc clc{clc_resp, clc_bar, 0};
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(clc_bar, 1);
    }
    __syncthreads();
    if constexpr (!MULTI) gemv_stage_x<NT>(a, 0, (int)a.n, bar, xstage, xs, phase);

    constexpr int64_t rows_per_block = (int64_t)(NT / 32) * R;
    int64_t blk = blockIdx.x;
    while (true) {
#ifndef LIFT_GEMV_NOCLC
        if (threadIdx.x == 0) clc_try_cancel(clc);  // steal the next block while we work
#endif
        const int64_t r0 = blk * rows_per_block + (int64_t)warp * R;
        int64_t rows[R];
#pragma unroll
        for (int r = 0; r < R; ++r) rows[r] = min(r0 + r, a.m - 1);
        double acc[R][8];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[r][e] = 0.0;
        if constexpr (!MULTI) {
            if (r0 < a.m) gemv_panel<R, U, LW>(a, rows, 0, (int)a.n, xs, acc);
        } else {
            for (int64_t c0 = 0; c0 < a.n; c0 += a.P) {
                const int pc = (int)min((int64_t)a.P, a.n - c0);
                gemv_stage_x<NT>(a, c0, pc, bar, xstage, xs, phase);
                if (r0 < a.m) gemv_panel<R, U, LW>(a, rows, c0, pc, xs, acc);
                __syncthreads();  // all warps done with xs before the next panel
            }
        }
        if (r0 < a.m) gemv_epilogue<R>(a, rows, (int)min((int64_t)R, a.m - r0), acc);
        int64_t next;
#ifndef LIFT_GEMV_NOCLC
        const bool more = clc_fetch(clc, next);
#else
        const bool more = false;
        next = 0;
#endif
        __syncthreads();  // everyone has read the response before it is reused
        if (a.y_peers && warp == 0) gemv_block_done(a);  // after the barrier: rows stored
        if (!more) break;
        blk = next;
    }
}

}  // namespace lift
