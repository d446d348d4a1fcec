// gemv_xs.cuh — G1 toLocal(x) for gemv rows whose columns split evenly over the row's
// threads (n % (8 TR) == 0, 2048 <= n <= GXS_NMAX): x staged ONCE per resident CTA in
// shared memory, already widened to fp64 (local memory for
// "frequently accessed data"; x is reused by every row), and A streamed
// through a per-thread register ring that runs ACROSS row blocks.
//
// Same canonical order as gemv.cuh (a function of n only; results are bit-identical to
// gemv_kernel's): TR = 2^gemv_tr_log2(n) threads per row, thread t' < TR owns the 8-float
// vectors t' + TR*k (k < K = n / (8 TR)), 8 fp64 slot accumulators folded in ascending k,
// pairwise8, butterfly over the row's lanes, the row's TR/32 warp values pairwise, fused
// epilogue.  What changes is the data movement:
//
//  * gemv_kernel reads x through L1 for every row: those loads hold registers next to the
//    A loads (ptxas then issues a thread's A loads in two waves) and each x element is
//    widened (F2F) again per row.  Timing experiments (LIFT_GEMV_EXPT) put
//    the x loads at ~2.2 us and the x conversions at ~1 us of 42.5 us at 8192^2.
//  * Here x lives in shared memory as fp64: xs[j][q] = (x[8q+2j], x[8q+2j+1]) (double2,
//    j = 0..3), so the 32 lanes of a warp read 32 consecutive 16-byte entries per LDS.128
//    (conflict-free) and no register waits on global memory for x.
//  * Persistent CTAs take row blocks by Cluster Launch Control stealing (common.cuh Clc):
//    the grid covers every block; resident CTAs cancel not-yet-launched ones and take
//    their block, so x is staged once per resident CTA while rows stay dynamically
//    balanced across SMs.
//  * A ring of P vectors per thread is refilled P vectors ahead in the flat sequence
//    (block, k): while a thread folds the last P vectors of a row, the first P vectors of
//    its NEXT block are already in flight, so the row's reduction, barrier and epilogue
//    overlap the next block's loads (a persistent CTA otherwise drains its loads at every
//    block boundary).  The next block is known early: its try_cancel is issued at the
//    start of the current block and fetched before the current block's last round.
//  * One CTA barrier per row block; it also orders every thread's read of the CLC
//    response before the next try_cancel.
#pragma once
#include "common.cuh"
#include "canon.h"
#include "gemv.cuh"

namespace lift {

#ifndef LIFT_GXS_T
#define LIFT_GXS_T 256   // threads per CTA
#endif
#ifndef LIFT_GXS_P
#define LIFT_GXS_P 4     // A vectors per thread in flight (ring depth; launch shape only)
#endif
#ifndef LIFT_GXS_MINB
#define LIFT_GXS_MINB 3  // resident CTAs per SM (3 x (64 KiB x + 256 threads) at n = 8192)
#endif
constexpr int GXS_T = LIFT_GXS_T;
constexpr int GXS_P = LIFT_GXS_P;
constexpr int GXS_NMIN = 2048;           // narrower rows: gemv_kernel (x is tiny, L1 serves it)
constexpr int64_t GXS_NMAX = 3 * 8192;   // fp64 x (8 B/column) must fit in shared memory
constexpr int GXS_HDR = 64 + 2 * (GXS_T / 32) * 8;  // CLC barrier + response, warp values

__host__ __device__ constexpr size_t gxs_smem_bytes(int64_t n) {
    return (size_t)GXS_HDR + (size_t)n * 8;  // x as fp64
}

// Whether the staged, pipelined kernel handles n: every row thread owns K full vectors,
// K a multiple of the ring depth.
__host__ __device__ inline bool gxs_shape_ok(int64_t n) {
    if (n < GXS_NMIN || n > GXS_NMAX) return false;
    const int64_t tr = (int64_t)1 << gemv_tr_log2(n);
    return n % (8 * tr) == 0 && (n / (8 * tr)) % GXS_P == 0;
}

template <int LW>
__device__ __forceinline__ void gxs_fold(const f8& av, const double2* xs, int64_t nv, int64_t q,
                                         double (&acc)[8]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const double2 xv = xs[j * nv + q];
        acc[2 * j] = __fma_rn((double)av.v[2 * j], xv.x, acc[2 * j]);
        acc[2 * j + 1] = __fma_rn((double)av.v[2 * j + 1], xv.y, acc[2 * j + 1]);
    }
}

template <int TRL, int LW, bool PEERS>
__global__ void __launch_bounds__(GXS_T, LIFT_GXS_MINB) gemv_xs_kernel(GemvArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* clc_bar = reinterpret_cast<uint64_t*>(smem);
    uint4* clc_resp = reinterpret_cast<uint4*>(smem + 16);
    double(*wv)[GXS_T / 32] = reinterpret_cast<double(*)[GXS_T / 32]>(smem + 64);
    double2* xs = reinterpret_cast<double2*>(smem + GXS_HDR);
    constexpr int TR = 1 << TRL;
    constexpr int RP = GXS_T / TR;  // rows per block
    constexpr int P = GXS_P;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int tp = t & (TR - 1);
    const int64_t nv = a.n / 8;
    const int K = (int)(nv / TR);  // vectors per thread per row (a multiple of P)
    Clc clc{clc_resp, clc_bar, 0};
    if (t == 0) mbar_init(clc_bar, 1);

    if ((t & ((1 << TRL) - 1)) == 0) {  // the first block's rows (common.cuh prefetch_l2)
        const int64_t r = (int64_t)blockIdx.x * RP + (t >> TRL);
        if (r < a.m) prefetch_l2<4>(a.A + r * a.lda, a.n * 4);
    }
    pdl_wait();  // x, A, y may be the previous kernel's output
    pdl_trigger();
    // ---- G1: x -> fp64 shared memory, once per resident CTA -------------------------
    {
        double* xd = reinterpret_cast<double*>(xs);
        for (int64_t j = t; j < a.n; j += GXS_T) {
            const int64_t q = j >> 3;
            const int e = (int)(j & 7);
            xd[2 * ((e >> 1) * nv + q) + (e & 1)] = (double)__ldg(a.x + j);
        }
    }
    __syncthreads();  // x staged; the CLC barrier initialised

    int64_t blk = blockIdx.x;
    const int rsub = t >> TRL;  // this thread's row within a block
    auto row_ptr = [&](int64_t b) {
        const int64_t r = b * RP + rsub;
        return a.A + (r < a.m ? r : a.m - 1) * a.lda;  // dead rows re-read a live one
    };
    if (t == 0) clc_try_cancel(clc);
    const float* rp = row_ptr(blk);
    f8 ring[P];
#pragma unroll
    for (int j = 0; j < P; ++j) ring[j] = ld_slot<LW>(rp + 8 * (tp + (int64_t)TR * j));

    int par = 0;
    int64_t my_blocks = 0;
    while (true) {
        double acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.0;
        int64_t next = 0;
        bool more = false;
        const float* rpn = rp;
        const int fetch_round = K > P ? P : 0;  // learn the next block one round in
        for (int k0 = 0; k0 < K; k0 += P) {
            const bool last_round = k0 + P == K;
            if (k0 == fetch_round) {  // the next block: L2-prefetch its rows now, and its
                more = clc_fetch(clc, next);  // first ring loads go out before this row's tree
                if (more) {
                    rpn = row_ptr(next);
                    if (tp == 0) prefetch_l2<4>(rpn, a.n * 4);
                }
            }
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const f8 av = ring[j];
                if (!last_round) ring[j] = ld_slot<LW>(rp + 8 * (tp + (int64_t)TR * (k0 + P + j)));
                else if (more) ring[j] = ld_slot<LW>(rpn + 8 * (tp + (int64_t)TR * j));
                gxs_fold<LW>(av, xs, nv, tp + (int64_t)TR * (k0 + j), acc);
            }
        }
        // ---- reduction over the row's TR threads (gemv.cuh's tree) -------------------
        const double v = warp_pairwise(pairwise8(acc));
        if (lane == 0) wv[par][warp] = v;
        __syncthreads();  // warp values visible; every thread has read the CLC response
        if (t == 0 && more) clc_try_cancel(clc);  // the block after next
        const int64_t row = blk * RP + rsub;
        if (tp == 0 && row < a.m) {
            const double* w = wv[par] + warp;  // the row's TR/32 warps start at `warp`
            double d;
            if constexpr (TRL == 8) d = pairwise8(w);
            else if constexpr (TRL == 7) d = __dadd_rn(__dadd_rn(w[0], w[1]), __dadd_rn(w[2], w[3]));
            else if constexpr (TRL == 6) d = __dadd_rn(w[0], w[1]);
            else d = w[0];
            const double yb = __dmul_rn((double)a.beta, (double)a.y[row]);  // scal(b, y): exact
            const float out = __double2float_rn(__fma_rn((double)a.alpha, d, yb));
            if constexpr (PEERS) {  // fused all-gather: the row lands in every rank's full y
                for (int q = 0; q < a.p; ++q) a.y_peers[q][a.row0 + row] = out;
            } else {
                a.y_out[row] = out;
            }
        }
        ++my_blocks;
        if (!more) break;
        blk = next;
        rp = rpn;
        par ^= 1;
    }
    if constexpr (PEERS) {
        // One system fence and one count per CTA (not per block): every row this CTA
        // stored precedes its count; the CTA completing the count publishes the rank.
        __syncthreads();
        if (warp == 0) gemv_cta_done(a, my_blocks);
    }
}

}  // namespace lift
