// gemv.cuh — G1..G3: y_out = alpha * A x + beta * y.
//
//   gemv(A, x, y, a, b):  z = map(scal(a) o dot(x), A)
//                         map(add) o zip(z, scal(b, y))
//
// A is row-major with leading dimension lda (map(..., A) maps over rows, P:815;
// DESIGN.md reading R8).  "The dot-product from gemv might be implemented in a
// totally different way from the stand-alone dot-product" — and it is.
//
// Canonical order of a row's dot (a function of n only — never of m, the grid, the
// row-to-CTA assignment, the load path or the pointer alignment):
//   * the row is cut into chunks of CW = min(8192, round_up(n, 1024)) columns;
//   * inside a chunk, warp w in [0,8) owns the segment [w*CW/8, (w+1)*CW/8);
//   * inside a segment, lane l owns the 4-float vectors l, l+32, l+64, ...
//     (reorder-stride with s = 32: a warp reads 512 contiguous bytes per step);
//   * each lane folds 4 fp64 accumulators acc_e = fma(A_ij, x_j, acc_e) (A_ij * x_j is
//     exact in fp64, so each step rounds once) over its vectors, chunk by chunk;
//     columns >= n are skipped;
//   * lane value = (acc0 + acc1) + (acc2 + acc3); warp value = butterfly xor 1..16;
//     row value d = pairwise fold of the 8 warp values;
//   * epilogue (rule 5f map-map fusion): y_out_i = fp32(fma(alpha, d, beta*y_i))
//     in fp64, rounded once (reading R10).
//
// Two kernels implement exactly this order:
//  gemv_tma  (A 16-B aligned, lda % 4 == 0, n % 4 == 0, n <= GEMV_NMAX_TMA) —
//    G1 toLocal(x): x is staged once per CTA by the TMA bulk-copy engine
//       (cp.async.bulk -> UBLKCP) and widened to fp64 in a slot-major shared layout
//       xs[e][q] = x[4q+e] (conflict-free LDS.64);
//    G2 A streamed through a ring of shared-memory stages by cp.async.bulk, one row
//       chunk per stage: a producer warp fills, 8 consumer warps fold their segments
//       (full/empty mbarriers; bytes in flight cost no registers); rows are units
//       handed out by Cluster Launch Control (hardware work stealing), so x is staged
//       once per resident CTA while every SM keeps pulling rows until none are left;
//    G3 the last warp to finish a row folds the 8 warp values and writes y_out.
//  gemv_ldg  (any alignment / lda / n) — the same order with direct loads (x read
//    through L1 and widened per use), one row per CTA step, CLC-scheduled.
#pragma once
#include "common.cuh"
#include "canon.h"

namespace lift {

constexpr int GEMV_WARPS = 8;                 // consumer warps (= column segments)
constexpr int GEMV_CW_MAX = 8192;             // chunk width cap (columns)
constexpr int GEMV_NMAX_TMA = 16384;          // x (fp64) must fit in shared memory
constexpr int GEMV_SMAX = 6;                  // max ring stages
constexpr int GEMV_SMEM_LIMIT = 227 * 1024;   // opt-in dynamic shared memory per CTA
constexpr int GEMV_CTRL_BYTES = 1024;         // control block at the start of smem
#ifndef LIFT_GEMV_RU
#define LIFT_GEMV_RU 2   // rows per CLC work unit (gemv_tma)
#endif
#ifndef LIFT_GEMV_CLC_DEPTH
#define LIFT_GEMV_CLC_DEPTH 3  // CLC steal requests kept in flight
#endif
constexpr int GEMV_RU = LIFT_GEMV_RU;
constexpr int GEMV_CLC_DEPTH = LIFT_GEMV_CLC_DEPTH;

struct GemvArgs {
    int64_t m, n, lda;
    float alpha, beta;
    const float* A;
    const float* x;
    const float* y;
    float* y_out;
    int cw;         // chunk width (columns), multiple of 1024
    int nchunks;    // chunks per row
    int xs_stride;  // doubles per slot row of xs (ceil(n/4) + 1 pad)
    int stages;     // ring stages (gemv_tma)
};

__host__ __device__ inline int gemv_chunk_width(int64_t n) {
    int64_t r = ((n > 0 ? n : 1) + 1023) / 1024 * 1024;
    return (int)(r < GEMV_CW_MAX ? r : GEMV_CW_MAX);
}
__host__ __device__ inline size_t gemv_xs_bytes(int xs_stride) { return (size_t)4 * xs_stride * 8; }
__host__ __device__ inline size_t gemv_stage_bytes(int cw) { return (size_t)cw * 4; }

struct GemvCtrl {              // lives in the first GEMV_CTRL_BYTES of shared memory
    uint64_t full[GEMV_SMAX];
    uint64_t empty[GEMV_SMAX];
    uint64_t xbar;
    uint64_t clc_bar[GEMV_CLC_DEPTH];
    uint4 clc_resp[GEMV_CLC_DEPTH];
    int64_t meta_row[GEMV_SMAX];    // row of the chunk in a stage; -1 = no more work
    int meta_chunk[GEMV_SMAX];
    double rowpart[8][GEMV_WARPS];  // warp values of up to 8 rows in flight
    int rowcnt[8];
};
static_assert(sizeof(GemvCtrl) <= GEMV_CTRL_BYTES, "gemv control block too large");

__device__ __forceinline__ double pairwise4(const double* v) {
    return __dadd_rn(__dadd_rn(v[0], v[1]), __dadd_rn(v[2], v[3]));
}

// Row value and epilogue from the 8 warp values (fixed pairwise order); yrow = y[row]
// (loaded early by the caller so the epilogue never waits on global memory).
__device__ __forceinline__ void gemv_finish_row(const GemvArgs& a, int64_t row, const double* wv,
                                                float yrow) {
    const double d = pairwise8(wv);
    const double w = __dmul_rn((double)a.beta, (double)yrow);  // scal(b, y): exact
    a.y_out[row] = __double2float_rn(__fma_rn((double)a.alpha, d, w));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------------- gemv_tma
// Fold warp w's segment of one chunk (row columns [c0, c0+cw), valid < n) from the
// shared stage `sa` into acc; xs is the fp64 slot-major copy of x.
__device__ __forceinline__ void gemv_fold_stage(const GemvArgs& a, const float* sa, int64_t c0,
                                                const double* xs, double (&acc)[4]) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int sw = a.cw / GEMV_WARPS;  // segment width (multiple of 128)
    const int seg0 = w * sw;
    const int64_t valid = a.n - c0;
    const int nv = sw / 128;           // 4-float vectors per lane
    const int q0 = (int)(c0 >> 2);
    if (seg0 + sw <= valid) {
#pragma unroll 4
        for (int k = 0; k < nv; ++k) {
            const int col = seg0 + 4 * (lane + 32 * k);
            const float4 v = *reinterpret_cast<const float4*>(sa + col);
            const int q = q0 + (col >> 2);
            acc[0] = __fma_rn((double)v.x, xs[0 * a.xs_stride + q], acc[0]);
            acc[1] = __fma_rn((double)v.y, xs[1 * a.xs_stride + q], acc[1]);
            acc[2] = __fma_rn((double)v.z, xs[2 * a.xs_stride + q], acc[2]);
            acc[3] = __fma_rn((double)v.w, xs[3 * a.xs_stride + q], acc[3]);
        }
    } else {
        for (int k = 0; k < nv; ++k) {
            const int col = seg0 + 4 * (lane + 32 * k);
            const int q = q0 + (col >> 2);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (col + e < valid)
                    acc[e] = __fma_rn((double)sa[col + e], xs[e * a.xs_stride + q], acc[e]);
        }
    }
}

__global__ void __launch_bounds__((GEMV_WARPS + 1) * 32, 1) gemv_tma_kernel(GemvArgs a) {
    extern __shared__ __align__(1024) unsigned char smem[];
    GemvCtrl& C = *reinterpret_cast<GemvCtrl*>(smem);
    double* xs = reinterpret_cast<double*>(smem + GEMV_CTRL_BYTES);
    float* ring = reinterpret_cast<float*>(smem + GEMV_CTRL_BYTES + gemv_xs_bytes(a.xs_stride));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int S = a.stages;
    const size_t stage_floats = (size_t)a.cw;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&C.full[s], 1);
            mbar_init(&C.empty[s], GEMV_WARPS);
        }
        mbar_init(&C.xbar, 1);
        for (int q = 0; q < GEMV_CLC_DEPTH; ++q) mbar_init(&C.clc_bar[q], 1);
        for (int r = 0; r < 8; ++r) C.rowcnt[r] = 0;
    }
    __syncthreads();

    // ---- G1: stage x (fp32, by TMA, through the still-idle ring), widen to fp64 -----
    {
        float* xstage = ring;
        const int n = (int)a.n;  // n % 4 == 0 and x is 16-B aligned on this path
        if (tid == 0) {
            mbar_arrive_expect_tx(&C.xbar, (uint32_t)n * 4u);
            bulk_g2s(xstage, a.x, (uint32_t)n * 4u, &C.xbar);
        }
        mbar_wait(&C.xbar, 0);
        for (int j = tid; j < n; j += blockDim.x)
            xs[(j & 3) * a.xs_stride + (j >> 2)] = (double)xstage[j];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // ring -> TMA again
        __syncthreads();
    }

    if (warp == GEMV_WARPS) {
        // ============ producer: one lane streams row chunks, steals units by CLC ======
        // A unit is GEMV_RU consecutive rows.  GEMV_CLC_DEPTH steal requests stay in
        // flight (one response buffer + mbarrier each) so the CLC round trip hides
        // behind several units of streaming.  Requests are only issued before a failure
        // has been observed; after one, the outstanding ones are drained and we stop.
        if (lane == 0) {
            Clc clc[GEMV_CLC_DEPTH];
            for (int q = 0; q < GEMV_CLC_DEPTH; ++q) {
                clc[q] = Clc{&C.clc_resp[q], &C.clc_bar[q], 0};
                clc_try_cancel(clc[q]);
            }
            int64_t unit = blockIdx.x;
            uint32_t it = 0;
            int q = 0;
            while (true) {
                const int64_t r_end = min((unit + 1) * GEMV_RU, a.m);
                for (int64_t row = unit * GEMV_RU; row < r_end; ++row) {
                    for (int c = 0; c < a.nchunks; ++c) {
                        const int s = (int)(it % S);
                        const uint32_t k = it / S;
                        if (k > 0) mbar_wait(&C.empty[s], (k - 1) & 1);
                        const int64_t c0 = (int64_t)c * a.cw;
                        const uint32_t bytes = (uint32_t)min((int64_t)a.cw, a.n - c0) * 4u;
                        C.meta_row[s] = row;
                        C.meta_chunk[s] = c;
                        mbar_arrive_expect_tx(&C.full[s], bytes);
                        bulk_g2s(ring + (size_t)s * stage_floats, a.A + row * a.lda + c0, bytes,
                                 &C.full[s]);
                        ++it;
                    }
                }
                int64_t next;
                if (!clc_fetch(clc[q], next)) {
                    for (int d = 1; d < GEMV_CLC_DEPTH; ++d) {  // drain the others
                        int64_t ignored;
                        clc_fetch(clc[(q + d) % GEMV_CLC_DEPTH], ignored);
                    }
                    break;
                }
                clc_try_cancel(clc[q]);  // re-arm this slot
                q = (q + 1) % GEMV_CLC_DEPTH;
                unit = next;
            }
            const int s = (int)(it % S);  // termination token
            const uint32_t k = it / S;
            if (k > 0) mbar_wait(&C.empty[s], (k - 1) & 1);
            C.meta_row[s] = -1;
            mbar_arrive(&C.full[s]);
        }
        return;
    }

    // ==================== consumers: 8 warps, one column segment each ================
    // Single-chunk rows (n <= 8192) with a full segment: this warp's x values never
    // change, so they live in registers (nv <= 8 vectors x 4 fp64) and the per-row
    // shared-memory traffic is A only.
    const int sw = a.cw / GEMV_WARPS, nv = sw / 128;
    const bool xreg = a.nchunks == 1 && (int64_t)(warp + 1) * sw <= a.n;
    double xr[8][4];
    if (xreg) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < nv) {
                const int q = (warp * sw) / 4 + lane + 32 * k;
#pragma unroll
                for (int e = 0; e < 4; ++e) xr[k][e] = xs[e * a.xs_stride + q];
            }
    }
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    uint32_t it = 0;
    int rowslot = 0;
    float yrow = 0.f;
    while (true) {
        const int s = (int)(it % S);
        mbar_wait(&C.full[s], (it / S) & 1);
        const int64_t row = C.meta_row[s];
        if (row < 0) break;
        const int c = C.meta_chunk[s];
        if (c == 0 && lane == 0) yrow = __ldg(a.y + row);  // prefetch for the epilogue
        if (xreg) {  // same order as gemv_fold_stage, x from registers
            const float* sa = ring + (size_t)s * stage_floats + warp * sw;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < nv) {
                    const float4 v = *reinterpret_cast<const float4*>(sa + 4 * (lane + 32 * k));
                    acc[0] = __fma_rn((double)v.x, xr[k][0], acc[0]);
                    acc[1] = __fma_rn((double)v.y, xr[k][1], acc[1]);
                    acc[2] = __fma_rn((double)v.z, xr[k][2], acc[2]);
                    acc[3] = __fma_rn((double)v.w, xr[k][3], acc[3]);
                }
        } else {
            gemv_fold_stage(a, ring + (size_t)s * stage_floats, (int64_t)c * a.cw, xs, acc);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&C.empty[s]);
        ++it;
        if (c == a.nchunks - 1) {  // this warp's share of the row is complete
            const double wv = warp_pairwise(pairwise4(acc));
            acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
            if (lane == 0) {
                C.rowpart[rowslot][warp] = wv;
                __threadfence_block();
                if (atomicAdd(&C.rowcnt[rowslot], 1) == GEMV_WARPS - 1) {  // last warp: G3
                    __threadfence_block();
                    double v8[GEMV_WARPS];
#pragma unroll
                    for (int w = 0; w < GEMV_WARPS; ++w)
                        v8[w] = *((volatile double*)&C.rowpart[rowslot][w]);
                    C.rowcnt[rowslot] = 0;
                    gemv_finish_row(a, row, v8, yrow);
                }
            }
            rowslot = (rowslot + 1) & 7;
        }
    }
}

// ---------------------------------------------------------------------- gemv_ldg
// Same order with direct loads; one row per CTA step; rows scheduled by CLC.
template <int LW>  // 4: float4 A loads (A 16-B aligned, lda % 4 == 0); 1: scalar
__global__ void __launch_bounds__(GEMV_WARPS * 32) gemv_ldg_kernel(GemvArgs a) {
    __shared__ double wv[GEMV_WARPS];
    __shared__ __align__(16) uint4 clc_resp;
    __shared__ __align__(8) uint64_t clc_bar;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    Clc clc{&clc_resp, &clc_bar, 0};
    if (threadIdx.x == 0) mbar_init(&clc_bar, 1);
    __syncthreads();
    const int sw = a.cw / GEMV_WARPS, nv = sw / 128;
    int64_t row = blockIdx.x;
    while (true) {
        float yrow = 0.f;
        if (threadIdx.x == 0) {
            clc_try_cancel(clc);
            yrow = __ldg(a.y + row);
        }
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const float* ar = a.A + row * a.lda;
        for (int c = 0; c < a.nchunks; ++c) {
            const int64_t c0 = (int64_t)c * a.cw;
            const int64_t valid = a.n - c0;
            for (int k = 0; k < nv; ++k) {
                const int col = w * sw + 4 * (lane + 32 * k);
                if (LW == 4 && col + 4 <= valid) {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(ar + c0 + col));
                    const float* xp = a.x + c0 + col;
                    acc[0] = __fma_rn((double)v.x, (double)__ldg(xp + 0), acc[0]);
                    acc[1] = __fma_rn((double)v.y, (double)__ldg(xp + 1), acc[1]);
                    acc[2] = __fma_rn((double)v.z, (double)__ldg(xp + 2), acc[2]);
                    acc[3] = __fma_rn((double)v.w, (double)__ldg(xp + 3), acc[3]);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (col + e < valid)
                            acc[e] = __fma_rn((double)__ldg(ar + c0 + col + e),
                                              (double)__ldg(a.x + c0 + col + e), acc[e]);
                }
            }
        }
        const double v = warp_pairwise(pairwise4(acc));
        if (lane == 0) wv[w] = v;
        __syncthreads();
        if (threadIdx.x == 0) gemv_finish_row(a, row, wv, yrow);
        int64_t next;
        const bool more = clc_fetch(clc, next);
        __syncthreads();  // wv and the CLC response are reused next step
        if (!more) break;
        row = next;
    }
}

}  // namespace lift
