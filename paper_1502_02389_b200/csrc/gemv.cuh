// gemv.cuh — G1..G3: y_out = alpha * A x + beta * y.
//
//   gemv(A, x, y, a, b):  z = map(scal(a) o dot(x), A)
//                         map(add) o zip(z, scal(b, y))
//
// A is row-major with leading dimension lda (map(..., A) maps over rows, P:815;
// DESIGN.md reading R8).  "The dot-product from gemv might be implemented in a
// totally different way from the stand-alone dot-product"; here it is the
// reduction kernel's shape applied per row — m independent dots, one CTA holding
// 256/TR rows, hardware-scheduled:
//
//  G1 toLocal(x): x is read through the SM's L1 (ld.global.nc with an
//     evict_last hint), where every CTA resident on the SM shares one copy — x is
//     32-64 KiB at the paper's sizes, so after the first row it is an L1
//     hit; A streams past L1 (L1::no_allocate).
//  G2 per-row dot, exact products, fp64 accumulation, in a canonical order that
//     depends on n only (reading R5/R13): TR = threads per row = the largest power of two
//     in [1, 256] with v*TR <= ceil(n/8), v = 8 for n >= 2048 else 4 (else 1); thread t' < TR owns the 8-float
//     vectors t' + TR*k (reorder-stride, s = TR; coalesced 256-bit LDG) and folds them
//     into 8 fp64 slot accumulators, acc_e = fma(A_ij, x_j, acc_e) in ascending k
//     (A_ij * x_j is exact in fp64, so each step rounds once); the partial last vector
//     (n % 8 != 0) is the last vector of its owner; thread value = pairwise fold of the
//     8 accumulators; butterfly over the row's lanes (xor 1..min(TR,32)/2); for TR > 32
//     the row's TR/32 warp values pairwise.
//     Each thread loads GEMV_B = 4 vectors of A per batch (32 KiB per CTA).
//  G3 fused epilogue (rule 5f map-map fusion): y_out_i = fp32(fma(alpha, d_i,
//     beta * y_i)) in fp64, rounded once (reading R10).  y_out may alias y.
//
// Why a CTA (or half of one) per row rather than one warp per row: a whole 32 KiB row is
// an ~11 us task for a single warp at its share of HBM bandwidth, so the last wave of
// rows left SMs idle (the time stepped by ~9 us per extra wave, scripts/gemv_msweep.py);
// 128-256 threads finish a row in a few us, and the hardware balances many CTAs per slot.
//
// The order of every addition is a function of n only (not of m, the grid, the load
// width or alignment), so a row's bits are the same however rows are sharded.
#pragma once
#include "common.cuh"
#include "canon.h"

namespace lift {

#ifndef LIFT_GEMV_B
#define LIFT_GEMV_B 4     // vectors per thread in flight (launch shape only, not the order)
#endif
#ifndef LIFT_GEMV_EXPT
#define LIFT_GEMV_EXPT 0  // timing experiments only (scripts/gpu_r2_gemv.sh); never the product
#endif
#ifndef LIFT_GEMV_MINB
#define LIFT_GEMV_MINB 4  // resident CTAs per SM: 64 registers, ~128 KiB of A in flight per SM
#endif
constexpr int GEMV_T = 256;  // threads per CTA
constexpr int GEMV_B = LIFT_GEMV_B;
constexpr int GEMV_MINB = LIFT_GEMV_MINB;
// canonical: TR = the largest power of two <= 256 with v * TR <= ceil(n/8), v = 8 vectors
// per thread for rows of >= 2048 floats, 4 below (measured: v = 8 at n = 8192 42.8 vs
// 44.1 us; v = 4 at n = 1001 18.7 vs 21.9 us)

struct GemvArgs {
    int64_t m, n, lda;
    float alpha, beta;
    const float* A;
    const float* x;
    const float* y;
    float* y_out;
    int64_t nblocks;  // row blocks (of 256/TR rows) of this launch
    int prefetch;     // L2-prefetch each block's rows at CTA start (many waves of blocks)
    int64_t resident;     // first-wave stagger (common.cuh): CTAs resident at once
    unsigned stagger_ns;  //   and ns per first-wave CTA index (0: none)
    // NEXT-1 fused all-gather of y (null y_peers: plain local y_out)
    float* const* y_peers;  // p pointers: every rank's full-length y (IPC-mapped)
    int64_t row0;           // global row of local row 0
    void* const* xpeers;    // p exchange buffers (flags + block counters)
    int p, rank;
    unsigned long long epoch;
    int* error;
};

// log2 of the threads per row for n columns (canonical: a function of n only).
__host__ __device__ constexpr int gemv_tr_log2(int64_t n) {
    const int64_t nvc = (n + 7) / 8;
    const int64_t v = nvc >= 256 ? 8 : 4;
    int l = 8;
    while (l > 0 && nvc < (v << l)) --l;
    return l;
}

// fp32 -> fp64 by integer ops (ALU pipe) — exact for normal numbers only (not 0, subnormal,
// Inf, NaN); timing experiments (LIFT_GEMV_EXPT) only.
__device__ __forceinline__ double f2d_bits(float f) {
    const unsigned u = __float_as_uint(f);
    const unsigned hi = (((u >> 3) & 0x0FFFFFFFu) | (u & 0x80000000u)) + 0x38000000u;
    return __hiloint2double((int)hi, (int)(u << 29));
}

// x through L1: one copy per SM serves every resident CTA (G1).
template <int LW>
__device__ __forceinline__ f8 ld_x(const float* p) {
    if constexpr (LW == 8) {
        f8 r;
        asm("ld.global.nc.L1::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
              "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
            : "l"(p));
        return r;
    } else if constexpr (LW == 4) {
        f8 r;
        const float4 u = __ldg(reinterpret_cast<const float4*>(p));
        const float4 w = __ldg(reinterpret_cast<const float4*>(p) + 1);
        r.v[0] = u.x; r.v[1] = u.y; r.v[2] = u.z; r.v[3] = u.w;
        r.v[4] = w.x; r.v[5] = w.y; r.v[6] = w.z; r.v[7] = w.w;
        return r;
    } else {
        f8 r;
#pragma unroll
        for (int e = 0; e < 8; ++e) r.v[e] = __ldg(p + e);
        return r;
    }
}

// NEXT-1 fused all-gather: every CTA adds the number of row blocks it finished to this
// rank's counter (`red.release.gpu`: fire-and-forget, so no CTA holds its slot waiting for
// an atomic's reply — with a returning atomic per CTA the 8192^2 gemv ran 40% slower, and
// a per-CTA __threadfence_system cost as much, scripts/xchg_p1.py).  The release orders
// the CTA's row stores — local and remote, by any of its threads before the barrier that
// precedes the call — before its count.  ONE CTA, the last of the grid (the last to be
// scheduled, so it waits least; any other CTA can still run, so waiting cannot deadlock),
// acquires the counter until every block is counted, resets it, publishes the rank's
// flag into every peer's buffer (system-scope release: cumulative, so it carries every
// counted CTA's stores) and waits for all p flags: the kernel ends only when every rank's
// rows have landed in this rank's y.  Called by warp 0 after a CTA barrier.
__device__ __forceinline__ void gemv_cta_done(const GemvArgs& a, int64_t count) {
    const int lane = threadIdx.x & 31;
    const int bank = (int)(a.epoch & 1ull);
    unsigned long long* cnt = xchg_counter(a.xpeers[a.rank], a.p, bank);
    if (lane == 0 && count > 0)
        asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(cnt),
                     "l"((unsigned long long)count)
                     : "memory");
    if (blockIdx.x != gridDim.x - 1) return;
    bool ok = true;
    if (lane == 0) {  // bounded wait (~10 s), like the flag wait
        unsigned long long v, spins = 0;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
            if (v >= (unsigned long long)a.nblocks) break;
            __nanosleep(64);
            if (++spins > (1ull << 27)) {
                ok = false;
                break;
            }
        }
        *cnt = 0ull;  // reset for epoch + 2 (its next use is a later kernel)
    }
    __syncwarp();  // lane 0's acquire before every lane's release below
    if (lane < a.p) {
        XchgSlot* dst = reinterpret_cast<XchgSlot*>(a.xpeers[lane]) + bank * a.p + a.rank;
        st_release_sys(&dst->flag, a.epoch);
        ok = xchg_wait_flag(a.xpeers[a.rank], bank * a.p, lane, a.epoch) && ok;
    }
    if (!__all_sync(0xffffffffu, ok) && lane == 0 && a.error) *a.error = 1;
}

// TRL = log2(threads per row) = gemv_tr_log2(n); LW = load width class of A, lda and x;
// PEERS = the NEXT-1 fused all-gather (its code in the block loop costs the plain kernel
// ~20% through worse load scheduling, so it is a separate instantiation).
// One row's slot accumulators (thread tp of TR): the canonical order of gemv.cuh.
// XS (LIFT_VAR_GEMV_X = 5): x was bulk-copied into shared memory (xsm, fp32) by the TMA
// engine at CTA start; the first batch's A loads go out before the wait for it.
__device__ __forceinline__ f8 ld_x_smem(const float* xsm, int64_t q) {
    const float4 u = reinterpret_cast<const float4*>(xsm)[2 * q];
    const float4 w = reinterpret_cast<const float4*>(xsm)[2 * q + 1];
    f8 r;
    r.v[0] = u.x; r.v[1] = u.y; r.v[2] = u.z; r.v[3] = u.w;
    r.v[4] = w.x; r.v[5] = w.y; r.v[6] = w.z; r.v[7] = w.w;
    return r;
}

template <int TRL, int LW, bool XS = false>
__device__ __forceinline__ void gemv_row_acc(const GemvArgs& a, const float* rp, int tp, int lane,
                                             int64_t nv, int tailn, double (&acc)[8],
                                             const float* xsm = nullptr, uint64_t* xbar = nullptr,
                                             bool* xready = nullptr) {
    constexpr int TR = 1 << TRL;
    constexpr int B = (LW == 2 || LW == 3) ? 2 : GEMV_B;  // realigned rows: 2 (4 spills; measured)
    const int d = (LW == 2 || LW == 3) ? (int)((reinterpret_cast<uintptr_t>(rp) >> 2) & 7) : 0;
    // LW 2: rows realigned, x 32-byte aligned; LW 3: rows and x realigned
    constexpr bool RA = LW == 2 || LW == 3;
    constexpr int LX = RA ? 8 : LW;
    const int dxo = LW == 3 ? (int)((reinterpret_cast<uintptr_t>(a.x) >> 2) & 7) : 0;
    int64_t k = 0;
    if constexpr (XS && !RA) {  // x from shared memory (loaded just in time, LDS)
        for (; (k + B) * TR <= nv; k += B) {
            f8 av[B];
#pragma unroll
            for (int b = 0; b < B; ++b) av[b] = ld_slot<LW>(rp + 8 * (tp + (k + b) * TR));
            if (!*xready) {
                mbar_wait(xbar, 0);
                *xready = true;
            }
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const f8 xv = ld_x_smem(xsm, tp + (k + b) * TR);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    acc[e] = __fma_rn((double)av[b].v[e], (double)xv.v[e], acc[e]);
            }
        }
    }
    for (; (k + B) * TR <= nv; k += B) {  // full batches: every vector in range
        f8 av[B], xv[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int64_t q = tp + (k + b) * TR;
            av[b] = RA ? ld_realigned(rp + 8 * q, d, q > 0 && 8 * q - d + 16 <= a.n)
                       : ld_slot<RA ? 8 : LW>(rp + 8 * q);
            xv[b] = LW == 3 ? ld_realigned(a.x + 8 * q, dxo, q > 0 && 8 * q - dxo + 16 <= a.n)
                            : ld_x<LX>(a.x + 8 * q);
        }
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
            for (int e = 0; e < 8; ++e) {
#if LIFT_GEMV_EXPT == 1  // TIMING EXPERIMENT ONLY (wrong results): no x conversion
                acc[e] = __dadd_rn((double)av[b].v[e], acc[e]) + (double)__int_as_float(__float_as_int(xv[b].v[e]) & 0);
#elif LIFT_GEMV_EXPT == 2  // TIMING EXPERIMENT: both widened by integer ops (normal numbers only)
                acc[e] = __fma_rn(f2d_bits(av[b].v[e]), f2d_bits(xv[b].v[e]), acc[e]);
#elif LIFT_GEMV_EXPT == 3  // TIMING EXPERIMENT: x widened by integer ops (normal numbers only)
                acc[e] = __fma_rn((double)av[b].v[e], f2d_bits(xv[b].v[e]), acc[e]);
#elif LIFT_GEMV_EXPT == 4  // TIMING EXPERIMENT: x loaded but not converted
                acc[e] = __dadd_rn((double)av[b].v[e], acc[e]) + (xv[b].v[e] == 1234.5f ? 1.0 : 0.0);
#elif LIFT_GEMV_EXPT == 6  // TIMING EXPERIMENT: x not loaded but converted (computed value)
                acc[e] = __fma_rn((double)av[b].v[e],
                                  (double)__int_as_float(0x3f800000 + (int)(k + b) * 8 + e + tp), acc[e]);
#else
                acc[e] = __fma_rn((double)av[b].v[e], (double)xv[b].v[e], acc[e]);
#endif
            }
    }
    if (k * TR < nv) {  // last batch: vectors >= nv are masked to +0 x +0
        f8 av[B], xv[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int64_t q0 = tp + (k + b) * TR;
            const bool in = q0 < nv;
            const int64_t q = in ? q0 : nv - 1;  // a valid address; the value is masked
            av[b] = RA ? ld_realigned(rp + 8 * q, d, q > 0 && 8 * q - d + 16 <= a.n)
                       : ld_slot<RA ? 8 : LW>(rp + 8 * q);
            xv[b] = LW == 3 ? ld_realigned(a.x + 8 * q, dxo, q > 0 && 8 * q - dxo + 16 <= a.n)
                            : ld_x<LX>(a.x + 8 * q);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                av[b].v[e] = in ? av[b].v[e] : 0.f;
                xv[b].v[e] = in ? xv[b].v[e] : 0.f;
            }
        }
        // adding +0 never changes an accumulator that started at +0 (RN: +0 + -0 = +0),
        // so the masked slots leave the order of the real terms untouched
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
            for (int e = 0; e < 8; ++e)
                acc[e] = __fma_rn((double)av[b].v[e], (double)xv[b].v[e], acc[e]);
    }
    if (tailn && tp == (int)(nv & (TR - 1))) {  // the partial last vector, by its owner
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (e < tailn)
                acc[e] = __fma_rn((double)__ldg(rp + 8 * nv + e), (double)__ldg(a.x + 8 * nv + e),
                                  acc[e]);
    }
}

template <int TRL, int LW, bool PEERS, bool XS = false>
__global__ void __launch_bounds__(GEMV_T, GEMV_MINB) gemv_kernel(GemvArgs a) {
    constexpr int RPB = GEMV_T >> TRL;  // rows per block
    // With many waves of blocks, the TMA prefetch puts a block's whole rows in flight at
    // once, more than the threads' register-bound load waves hold (8192^2: 43.2 -> 41.2 us);
    // when every block is resident at once it only duplicates the loads (1024 x 8192: 8.1 ->
    // 9.8 us), so the launcher enables it for >= 4 waves (scripts/gpu_r2_ab.sh)
    if (a.prefetch && threadIdx.x < RPB && blockIdx.x < a.nblocks) {  // this CTA's first rows
        const int64_t row = (int64_t)blockIdx.x * RPB + threadIdx.x;
        if (row < a.m) prefetch_l2<4>(a.A + row * a.lda, a.n * 4);
    }
    pdl_wait();
    pdl_trigger();
    first_wave_stagger(a.resident, a.stagger_ns);
    constexpr int TR = 1 << TRL;
    constexpr int RP = GEMV_T / TR;  // rows per block
    __shared__ double wv[2][GEMV_T / 32];  // warp values, double-buffered by block parity
    __shared__ float* ypeer[PEERS ? 32 : 1];  // NEXT-1: the p peer y pointers, loaded once
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    extern __shared__ __align__(128) unsigned char gemv_dsm[];
    __shared__ __align__(8) uint64_t xbar;
    bool xready = false;
    if constexpr (XS) {  // x -> shared memory by one TMA bulk copy (n % 4 == 0, 16-B aligned)
        if (t == 0) {
            mbar_init(&xbar, 1);
            mbar_arrive_expect_tx(&xbar, (uint32_t)(a.n * 4));
            bulk_g2s(gemv_dsm, a.x, (uint32_t)(a.n * 4), &xbar);
        }
        __syncthreads();  // the barrier initialised before anyone waits on it
    }
    if constexpr (PEERS) {  // off the row path: a row store then needs no pointer load
        if (t < a.p) ypeer[t] = a.y_peers[t];
        __syncthreads();
    }
    const int tp = t & (TR - 1);  // thread within its row
    const int64_t nv = a.n / 8;   // full vectors per row
    const int tailn = (int)(a.n & 7);
    int par = 0;
    for (int64_t blk = blockIdx.x; blk < a.nblocks; blk += gridDim.x, par ^= 1) {
        const int64_t row = blk * RP + (t >> TRL);
        const bool live = row < a.m;
        const float* rp = a.A + (live ? row : a.m - 1) * a.lda;  // dead rows re-read a live one
        double acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.0;
        gemv_row_acc<TRL, LW, XS>(a, rp, tp, lane, nv, tailn, acc,
                                  reinterpret_cast<const float*>(gemv_dsm), &xbar, &xready);
        double d;
        if constexpr (TR < 32) {
            // rows narrower than a warp: butterfly over the row's TR lanes only (xor stays
            // inside the aligned lane group), no shared memory, no barrier
            d = pairwise8(acc);
#pragma unroll
            for (int o = 1; o < TR; o <<= 1) d = __dadd_rn(d, __shfl_xor_sync(0xffffffffu, d, o));
        } else {
            const double v = warp_pairwise(pairwise8(acc));
            if (lane == 0) wv[par][warp] = v;
            __syncthreads();
            d = 0.0;
            if (tp == 0) {  // the row's TR/32 warps start at this thread's warp
                const double* w = wv[par] + warp;
                if constexpr (TRL == 8) d = pairwise8(w);
                else if constexpr (TRL == 7) d = __dadd_rn(__dadd_rn(w[0], w[1]), __dadd_rn(w[2], w[3]));
                else if constexpr (TRL == 6) d = __dadd_rn(w[0], w[1]);
                else d = w[0];
            }
        }
        if (tp == 0 && live) {
            const double yb = __dmul_rn((double)a.beta, (double)a.y[row]);  // scal(b, y): exact
            const float out = __double2float_rn(__fma_rn((double)a.alpha, d, yb));
            if constexpr (PEERS) {  // fused all-gather: the row lands in every rank's full y
                for (int q = 0; q < a.p; ++q) ypeer[q][a.row0 + row] = out;
            } else {
                a.y_out[row] = out;
            }
        }
    }
    if constexpr (PEERS) {  // once per CTA, after its blocks (the loop stays the plain kernel's)
        __syncthreads();  // every row store of this CTA precedes its count
        if (warp == 0) {
            const int64_t mine = blockIdx.x < a.nblocks
                                     ? (a.nblocks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
            gemv_cta_done(a, mine);
        }
    }
}

}  // namespace lift
