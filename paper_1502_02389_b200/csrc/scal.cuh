// scal.cuh — S1: y = alpha * x, the paper's scal(a, x) = map(mult(a), x)
// (PAPER.md P:793).
//
// The paper lowers it as join o map-workgroup(asScalar o map-local(vect-4(mul3)) o
// asVector-4) o split-1024 (Fig. 3b; Fig. 3c).  On B200 the
// same structure becomes a grid-stride loop over tiles of SCAL_T x SCAL_U slots of
// 8 floats: map-workgroup -> CTAs over tiles, map-local -> threads over slots,
// asVector-8 -> one 256-bit LDG/STG per slot.  Unlike Fig. 3c's
// `i < len/1024` loop (which drops the tail), any n >= 0 and any 4-byte alignment
// are handled: a scalar head brings x to the vector alignment, a scalar tail
// finishes the last < 8 elements; both run in CTA 0 of the same launch.
// Every element is RN(alpha * x_i), so the result is bit-exact regardless of LW.
#pragma once
#include "common.cuh"

namespace lift {

// Tile = 1024 threads x 1 slot (32 KiB in, 32 KiB out), two CTAs per SM: ~64 KiB of
// loads in flight per SM.  Measured (scripts/ab.py, 2^28): 256 x 4 (8 CTAs, 256 KiB in
// flight) 313.9 us, 256 x 1 308.9, 512 x 1 307.7, 1024 x 1 303.9 (7.07 TB/s); capping
// resident CTAs below full thread occupancy costs more (1024 x 1 at one CTA/SM: 447 us).
// A read+write stream runs best with fewer bytes queued per SM.
#ifndef LIFT_SCAL_T
#define LIFT_SCAL_T 1024
#endif
#ifndef LIFT_SCAL_U
#define LIFT_SCAL_U 1
#endif
constexpr int SCAL_T = LIFT_SCAL_T;  // threads per CTA
constexpr int SCAL_U = LIFT_SCAL_U;  // 8-float slots per thread per tile

template <int LW, bool ALIAS>
__device__ __forceinline__ f8 scal_load(const float* p) {
    if constexpr (LW == 8 && ALIAS) return ld_v8(p);  // x == y: stay off the .nc path
    else if constexpr (ALIAS) {
        f8 r;
#pragma unroll
        for (int e = 0; e < 8; ++e) r.v[e] = p[e];
        return r;
    } else return ld_slot<LW>(p);
}

// head: elements [0, head) ; body: nslots slots of 8 starting at element `head` ;
// tail: elements [head + 8*nslots, head + 8*nslots + tail).
template <int LW, bool ALIAS>
__global__ void __launch_bounds__(SCAL_T) scal_kernel(int64_t nslots, int head, int tail,
                                                      float alpha, const float* x, float* y,
                                                      int prefetch, int64_t resident = 0,
                                                      unsigned stagger_ns = 0) {
    // the first wave's tiles, L2-prefetched before the wait (common.cuh prefetch_l2)
    if (prefetch && threadIdx.x == 0 && in_first_wave(2048 / SCAL_T)) {
        const int64_t s0 = (int64_t)blockIdx.x * SCAL_T * SCAL_U;
        const int64_t ns = nslots - s0 < (int64_t)SCAL_T * SCAL_U ? nslots - s0 : (int64_t)SCAL_T * SCAL_U;
        if (ns > 0) prefetch_l2<1>(x + head + 8 * s0, ns * 32);
    }
    pdl_wait();
    pdl_trigger();
    first_wave_stagger(resident, stagger_ns);  // common.cuh
    const int t = threadIdx.x;
    if (blockIdx.x == 0) {
        if (t < head) y[t] = alpha * x[t];
        const int64_t tb = head + 8 * nslots;
        if (t >= 32 && t < 32 + tail) y[tb + (t - 32)] = alpha * x[tb + (t - 32)];
    }
    const float* xb = x + head;
    float* yb = y + head;
    constexpr int64_t TILE = (int64_t)SCAL_T * SCAL_U;
    for (int64_t s0 = (int64_t)blockIdx.x * TILE; s0 < nslots; s0 += (int64_t)gridDim.x * TILE) {
        if (s0 + TILE <= nslots) {
            f8 v[SCAL_U];
#pragma unroll
            for (int u = 0; u < SCAL_U; ++u)
                v[u] = scal_load<LW, ALIAS>(xb + 8 * (s0 + u * SCAL_T + t));
#pragma unroll
            for (int u = 0; u < SCAL_U; ++u) {
#pragma unroll
                for (int e = 0; e < 8; ++e) v[u].v[e] = __fmul_rn(alpha, v[u].v[e]);
                st_slot<LW>(yb + 8 * (s0 + u * SCAL_T + t), v[u]);
            }
        } else {
#pragma unroll
            for (int u = 0; u < SCAL_U; ++u) {
                const int64_t s = s0 + u * SCAL_T + t;
                if (s < nslots) {
                    f8 v = scal_load<LW, ALIAS>(xb + 8 * s);
#pragma unroll
                    for (int e = 0; e < 8; ++e) v.v[e] = __fmul_rn(alpha, v.v[e]);
                    st_slot<LW>(yb + 8 * s, v);
                }
            }
        }
    }
}

// NEXT-4 load axis, TMA bulk variant (compile-time LIFT_SCAL_TMA = 1; scripts/tune.py):
// per tile the TMA engine copies SCAL_TMA_TILE floats of x into shared memory (one
// mbarrier completes by bytes), the CTA scales them in place, and one bulk store writes the
// tile to y.  Same RN(alpha * x_i) per element, so the same bits.  Needs x and y 16-byte
// aligned after the head (the launcher's 128-/256-bit classes).
#ifndef LIFT_SCAL_TMA
#define LIFT_SCAL_TMA 0
#endif
constexpr int SCAL_TMA_T = 256;
constexpr int SCAL_TMA_TILE = 8192;  // floats (32 KiB) per tile

__global__ void __launch_bounds__(SCAL_TMA_T) scal_tma_kernel(int64_t nslots, int head, int tail,
                                                               float alpha, const float* x, float* y) {
    __shared__ __align__(128) float buf[SCAL_TMA_TILE];
    __shared__ __align__(8) uint64_t bar;
    pdl_wait();
    pdl_trigger();
    const int t = threadIdx.x;
    if (t == 0) mbar_init(&bar, 1);
    if (blockIdx.x == 0) {
        if (t < head) y[t] = alpha * x[t];
        const int64_t tb = head + 8 * nslots;
        if (t >= 32 && t < 32 + tail) y[tb + (t - 32)] = alpha * x[tb + (t - 32)];
    }
    __syncthreads();
    const float* xb = x + head;
    float* yb = y + head;
    const int64_t nf = 8 * nslots;
    uint32_t phase = 0;
    for (int64_t f0 = (int64_t)blockIdx.x * SCAL_TMA_TILE; f0 < nf;
         f0 += (int64_t)gridDim.x * SCAL_TMA_TILE, phase ^= 1u) {
        const int len = (int)(nf - f0 < SCAL_TMA_TILE ? nf - f0 : SCAL_TMA_TILE);  // multiple of 8
        if (t == 0) {
            mbar_arrive_expect_tx(&bar, (uint32_t)len * 4u);
            bulk_g2s(buf, xb + f0, (uint32_t)len * 4u, &bar);
        }
        mbar_wait(&bar, phase);
        for (int i = 4 * t; i < len; i += 4 * SCAL_TMA_T) {
            float4 v = *reinterpret_cast<float4*>(buf + i);
            v.x = __fmul_rn(alpha, v.x);
            v.y = __fmul_rn(alpha, v.y);
            v.z = __fmul_rn(alpha, v.z);
            v.w = __fmul_rn(alpha, v.w);
            *reinterpret_cast<float4*>(buf + i) = v;
        }
        fence_proxy_async_smem();  // the generic writes before the async-proxy read
        __syncthreads();
        if (t == 0) {
            bulk_s2g(yb + f0, buf, (uint32_t)len * 4u);
            bulk_commit_and_wait_read();  // buf is reused (or released) only after the read
        }
        __syncthreads();
    }
}

}  // namespace lift
