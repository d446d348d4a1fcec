// gemv_tma.cuh — G1 + G2 with the TMA engine: x staged once per CTA in shared memory as
// fp64 (toLocal) and the rows of A streamed by cp.async.bulk into a
// shared-memory ring, so the bytes in flight live in shared memory, not in registers.
//
// Why: a streaming kernel's bandwidth is bounded by the bytes it keeps in flight per SM
// (Little's law).  gemv_kernel holds its in-flight A vectors in registers next to the x
// vectors it reads through L1, so ptxas issues a thread's A loads in two waves (measured,
// removing the x loads alone lifts 8192^2 from 42.5 to 40.3 us).  Here one
// producer warp keeps up to GTM_S x 16 KiB of A in flight per SM regardless of registers.
//
// Same canonical order as gemv.cuh (results bit-identical to gemv_kernel):
// TR = 2^gemv_tr_log2(n) threads per row, thread t' owns vectors t' + TR*k (k < K),
// 8 fp64 slot accumulators in ascending k, pairwise8, warp butterfly, the row's TR/32 warp
// values pairwise, fused epilogue fp32(fma(alpha, d, beta*y)).  Requires n % (8 TR) == 0,
// 16-byte aligned rows (lda % 4 == 0) and 2048 <= n <= GTM_NMAX.
//
// Roles (persistent CTA, one per SM, Cluster Launch Control stealing of row blocks):
//  * producer warp (one elected lane): for each block and k-step j, waits for ring stage s
//    to be empty, records the block id in the stage header, and bulk-copies the block's
//    RB row segments A[row][8 TR j, 8 TR (j+1)) (RB x 32 TR bytes = 16 KiB) into the stage,
//    completing the stage's `full` mbarrier by transaction bytes.  After the last block it
//    publishes a sentinel stage (block id -1).
//  * GTM_CW consumer warps: thread c = (row group g, virtual row thread tp); each thread
//    carries GTM_R rows of its group (x read once from shared memory feeds GTM_R rows).
//    Per stage: wait `full`, fold its vector of each row, release the stage (`empty`, one
//    arrive per warp).  After the K-th stage of a block: warp butterfly, one named barrier
//    over the consumer warps, the row's warp values pairwise, epilogue.
#pragma once
#include "common.cuh"
#include "canon.h"
#include "gemv.cuh"

namespace lift {

#ifndef LIFT_GTM_S
#define LIFT_GTM_S 8     // ring stages of 16 KiB
#endif
#ifndef LIFT_GTM_R
#define LIFT_GTM_R 2     // rows per consumer thread
#endif
#ifndef LIFT_GTM_CW
#define LIFT_GTM_CW 8    // consumer warps
#endif
constexpr int GTM_S = LIFT_GTM_S;
constexpr int GTM_R = LIFT_GTM_R;
constexpr int GTM_CW = LIFT_GTM_CW;
constexpr int GTM_CT = GTM_CW * 32;          // consumer threads
constexpr int GTM_T = GTM_CT + 32;           // + one producer warp
constexpr int GTM_STAGE = 16384;             // bytes per ring stage
constexpr int64_t GTM_NMAX = 16384;          // fp64 x (128 KiB) + ring must fit
// header: [0,8) CLC mbarrier, [16,32) CLC response, [64, 64+8S) full[], [.., +8S) empty[],
// then S block ids (int64), then warp values [2][R][CW] doubles
constexpr int GTM_HDR_RAW = 64 + 3 * 8 * GTM_S + 2 * GTM_R * GTM_CW * 8;
constexpr int GTM_HDR = (GTM_HDR_RAW + 127) & ~127;

// ring stages that fit next to x (at most GTM_S): 8 at n = 8192, 6 at n = 16384
__host__ __device__ constexpr int gtm_stages(int64_t n, size_t smem_optin) {
    const int64_t room =
        ((int64_t)smem_optin - GTM_HDR - n * 8 - (LIFT_TREE == 2 ? 8192 : 0)) / GTM_STAGE;
    return (int)(room < GTM_S ? room : GTM_S);
}
__host__ __device__ constexpr size_t gtm_smem_bytes(int64_t n, int nst) {
    return (size_t)GTM_HDR + (size_t)n * 8 + (size_t)nst * GTM_STAGE;
}

__host__ __device__ inline bool gtm_shape_ok(int64_t n) {
    if (n < 2048 || n > GTM_NMAX) return false;
    const int64_t tr = (int64_t)1 << gemv_tr_log2(n);
    return n % (8 * tr) == 0 && GTM_CT % tr == 0;
}

template <int TRL, bool PEERS>
__global__ void __launch_bounds__(GTM_T, 1) gemv_tma_kernel(GemvArgs a, int nst) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int TR = 1 << TRL;
    constexpr int G = GTM_CT / TR;             // row groups among the consumer threads
    constexpr int RB = G * GTM_R;              // rows per block
    constexpr int SEG = TR * 32;               // bytes of one row per k-step (TR x 8 floats)
    static_assert(RB * SEG == GTM_STAGE, "a stage holds one k-step of a block");
    uint64_t* clc_bar = reinterpret_cast<uint64_t*>(smem);
    uint4* clc_resp = reinterpret_cast<uint4*>(smem + 16);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 64);
    uint64_t* empty = full + GTM_S;
    int64_t* hdr = reinterpret_cast<int64_t*>(empty + GTM_S);
    double* wv = reinterpret_cast<double*>(hdr + GTM_S);  // [2][R][CW]
    double2* xs = reinterpret_cast<double2*>(smem + GTM_HDR);
    unsigned char* ring = smem + GTM_HDR + (size_t)a.n * 8;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t nv = a.n / 8;
    const int K = (int)(nv / TR);  // k-steps per row block

    if (t == 0) {
        mbar_init(clc_bar, 1);
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], GTM_CT);  // every consumer thread releases the stage
        }
    }
    pdl_wait();  // x, A, y may be the previous kernel's output
    pdl_trigger();
    {  // G1: x -> fp64 shared memory (xs[j][q] = x[8q+2j .. 8q+2j+1]), once per CTA
        double* xd = reinterpret_cast<double*>(xs);
        for (int64_t j = t; j < a.n; j += GTM_T) {
            const int64_t q = j >> 3;
            const int e = (int)(j & 7);
            xd[2 * ((e >> 1) * nv + q) + (e & 1)] = (double)__ldg(a.x + j);
        }
    }
    __syncthreads();

    if (warp == GTM_CW) {  // ---------------------------------------------------- producer
        if (lane == 0) {
            Clc clc{clc_resp, clc_bar, 0};
            int64_t blk = blockIdx.x;
            int s = 0;
            uint32_t ph = 0;
            clc_try_cancel(clc);
            while (true) {
                for (int j = 0; j < K; ++j) {
                    mbar_wait(&empty[s], ph ^ 1u);
                    hdr[s] = blk;
                    mbar_arrive_expect_tx(&full[s], (uint32_t)GTM_STAGE);
                    unsigned char* dst = ring + (size_t)s * GTM_STAGE;
#pragma unroll 1
                    for (int rr = 0; rr < RB; ++rr) {
                        int64_t row = blk * RB + rr;
                        row = row < a.m ? row : a.m - 1;  // dead rows re-read a live one
                        bulk_g2s(dst + rr * SEG, a.A + row * a.lda + (int64_t)j * 8 * TR, SEG,
                                 &full[s]);
                    }
                    if (++s == nst) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                int64_t next;
                if (!clc_fetch(clc, next)) break;
                blk = next;
                clc_try_cancel(clc);
            }
            mbar_wait(&empty[s], ph ^ 1u);  // sentinel: no more blocks
            hdr[s] = -1;
            mbar_arrive(&full[s]);
        }
        return;
    }

    // ---------------------------------------------------------------------- consumers
    const int c = t;                 // consumer thread
    const int g = c >> TRL;          // row group
    const int tp = c & (TR - 1);     // virtual row thread
    int s = 0;
    uint32_t ph = 0;
    int par = 0;
    int64_t my_blocks = 0;
    while (true) {
        double acc[GTM_R][8];
#pragma unroll
        for (int r = 0; r < GTM_R; ++r)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[r][e] = 0.0;
        int64_t blk = -1;
        for (int j = 0; j < K; ++j) {
            mbar_wait(&full[s], ph);
            blk = hdr[s];
            if (blk < 0) break;
            const unsigned char* st = ring + (size_t)s * GTM_STAGE;
            const int64_t q = tp + (int64_t)TR * j;
            double2 xv[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) xv[jj] = xs[jj * nv + q];
#pragma unroll
            for (int r = 0; r < GTM_R; ++r) {
                const float4* ap = reinterpret_cast<const float4*>(st + (g * GTM_R + r) * SEG + tp * 32);
                const float4 a0 = ap[0], a1 = ap[1];
                const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    acc[r][2 * jj] = __fma_rn((double)av[2 * jj], xv[jj].x, acc[r][2 * jj]);
                    acc[r][2 * jj + 1] = __fma_rn((double)av[2 * jj + 1], xv[jj].y, acc[r][2 * jj + 1]);
                }
            }
            // each consumer thread releases the stage after its own reads of it (the arrive
            // orders them before the producer's next bulk copy into the stage; one arrive per
            // warp after __syncwarp was equivalent but not visible to compute-sanitizer racecheck)
            mbar_arrive(&empty[s]);
            if (++s == nst) {
                s = 0;
                ph ^= 1u;
            }
        }
        if (blk < 0) break;
        // ---- reduction over each row's TR threads (gemv.cuh's tree) ------------------
#pragma unroll
        for (int r = 0; r < GTM_R; ++r) {
            const double v = warp_pairwise(pairwise8(acc[r]));
            if (lane == 0) wv[(par * GTM_R + r) * GTM_CW + warp] = v;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(GTM_CT) : "memory");  // consumers only
        if (tp == 0) {
#pragma unroll
            for (int r = 0; r < GTM_R; ++r) {
                const int64_t row = blk * RB + g * GTM_R + r;
                if (row >= a.m) continue;
                const double* w = wv + (par * GTM_R + r) * GTM_CW + warp;  // the row's warps
                double d;
                if constexpr (TRL == 8) d = pairwise8(w);
                else if constexpr (TRL == 7) d = __dadd_rn(__dadd_rn(w[0], w[1]), __dadd_rn(w[2], w[3]));
                else if constexpr (TRL == 6) d = __dadd_rn(w[0], w[1]);
                else d = w[0];
                const double yb = __dmul_rn((double)a.beta, (double)a.y[row]);  // scal(b, y)
                const float out = __double2float_rn(__fma_rn((double)a.alpha, d, yb));
                if constexpr (PEERS) {
                    for (int qq = 0; qq < a.p; ++qq) a.y_peers[qq][a.row0 + row] = out;
                } else {
                    a.y_out[row] = out;
                }
            }
        }
        ++my_blocks;
        par ^= 1;
    }
    if constexpr (PEERS) {
        asm volatile("bar.sync 1, %0;" ::"r"(GTM_CT) : "memory");  // the CTA's rows stored
        if (warp == 0) gemv_cta_done(a, my_blocks);
    }
}

}  // namespace lift
