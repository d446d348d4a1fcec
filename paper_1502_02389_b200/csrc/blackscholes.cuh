// blackscholes.cuh — NEXT-3 row: the paper's BlackScholes benchmark (Fig. 9,
// PAPER.md P:829-835), a pure map:
//
//     BSComputation(s) = d1 = compD1(s); d2 = compD2(d1, s)
//                        return { compCall(d1, d2, s), compPut(d1, d2, s) }
//     blackScholes(s)  = map(BSComputation, s)
//
// The helper bodies are "not shown"; reading R22 takes the standard
// closed form for European options without dividends, strike K, rate r, volatility v,
// maturity T fixed per call (the paper maps over the stock prices only):
//     d1 = (ln(s/K) + (r + v^2/2) T) / (v sqrt T),  d2 = d1 - v sqrt T
//     call = s N(d1) - K e^{-rT} N(d2),   put = K e^{-rT} N(-d2) - s N(-d1)
//     N(x) = erfc(-x/sqrt 2) / 2
// fp32 storage and arithmetic (the paper's 4-byte elements).  N comes from one
// tail evaluation per d: with e = N(-|d|) (small, relatively accurate), N(d) and N(-d)
// are e and 1 - e (>= 1/2, so nothing cancels).  The tail is the Abramowitz-Stegun
// 26.2.17 polynomial (|error| < 7.5e-8, the CND of the NVIDIA SDK BlackScholes the
// paper compares with) and log/exp/rcp use the MUFU unit; DESIGN.md reading
// R22 bounds the price error well inside the 1e-6 (s + K) test tolerance.
//
// B200 mapping: like scal — one CTA per tile, 8 consecutive prices per thread from
// one 256-bit load, two 256-bit stores (call, put); the per-price transcendental
// chain is independent across the 8, which gives the MUFU/FMA pipes ILP.  12 bytes
// move per price, and the SFU/FMA work per price is ~40 instructions, so at the
// paper's 4M prices this map is instruction-bound rather than HBM-bound (profiles/).
#pragma once
#include "common.cuh"

namespace lift {

constexpr int BS_T = 256;  // threads per CTA
constexpr int BS_U = 1;    // 8-price slots per thread per tile

// Per-call constants, computed once on the host in fp64 and rounded to fp32
// (lift_blackscholes), so no thread spends issue slots re-deriving them.  With
// ln s = ln2 * log2 s:  d1 = log2(s) * d1_scale + d1_bias  (one FFMA after the MUFU).
struct BsConst {
    float d1_scale;  // ln2 / (v sqrt T)
    float d1_bias;   // ((r + v^2/2) T - ln K) / (v sqrt T)
    float vsqrt;     // v sqrt T
    float disc;      // K e^{-rT}
};

// MUFU approximations with flush-to-zero: the arguments here are never subnormal
// (s >= 1e-38 is normal; exp underflow to 0 is the correct limit), so the subnormal
// rescaling the non-ftz forms add is pure issue overhead.
__device__ __forceinline__ float ex2_ftz(float a) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}
__device__ __forceinline__ float lg2_ftz(float a) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}
__device__ __forceinline__ float rcp_ftz(float a) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}

// N(-x) for x >= 0, the small tail: Abramowitz-Stegun 26.2.17,
//     N(-x) = phi(x) (b1 t + b2 t^2 + ... + b5 t^5),  t = 1 / (1 + p x),
// |error| < 7.5e-8 — the CND of the NVIDIA SDK BlackScholes the paper compares with
// (P:1112).  phi's 1/sqrt(2 pi) is folded into the coefficients c_i = b_i / sqrt(2 pi).
__device__ __forceinline__ float norm_tail(float x) {
    constexpr float kP = 0.2316419f;
    constexpr double kRsqrt2Pi = 0.39894228040143267794;
    constexpr float c1 = (float)(0.319381530 * kRsqrt2Pi), c2 = (float)(-0.356563782 * kRsqrt2Pi),
                    c3 = (float)(1.781477937 * kRsqrt2Pi), c4 = (float)(-1.821255978 * kRsqrt2Pi),
                    c5 = (float)(1.330274429 * kRsqrt2Pi);
    constexpr float kHalfLog2e = -0.72134752044448170368f;  // exp(-x^2/2) = 2^(k x^2)
    const float t = rcp_ftz(__fmaf_rn(kP, x, 1.0f));
    const float poly = t * __fmaf_rn(t, __fmaf_rn(t, __fmaf_rn(t, __fmaf_rn(t, c5, c4), c3), c2), c1);
    return ex2_ftz(kHalfLog2e * x * x) * poly;
}

// N(d) and N(-d) from a single tail evaluation (see the header comment).
__device__ __forceinline__ void norm_cdf_pair(float d, float& n_pos, float& n_neg) {
    const float tail = norm_tail(fabsf(d));  // N(-|d|)
    const float body = 1.0f - tail;          // N(|d|)
    n_pos = d >= 0.f ? body : tail;          // N(d)
    n_neg = d >= 0.f ? tail : body;          // N(-d)
}

// One BSComputation.  An error e in ln s shifts d1 and d2 alike, and to
// first order the prices do not move (s phi(d1) = K e^{-rT} phi(d2)), so the MUFU
// log2 suffices (reading R22).
__device__ __forceinline__ void bs_one(float S, const BsConst& c, float& call, float& put) {
    const float d1 = __fmaf_rn(lg2_ftz(S), c.d1_scale, c.d1_bias);  // compD1
    const float d2 = d1 - c.vsqrt;                                   // compD2
    float n_d1, n_md1, n_d2, n_md2;
    norm_cdf_pair(d1, n_d1, n_md1);
    norm_cdf_pair(d2, n_d2, n_md2);
    call = __fmaf_rn(S, n_d1, -c.disc * n_d2);   // compCall
    put = __fmaf_rn(c.disc, n_md2, -S * n_md1);  // compPut
}

// head / body (nslots x 8 prices, LW-wide accesses) / tail, as in scal.cuh.
template <int LW>
__global__ void __launch_bounds__(BS_T) blackscholes_kernel(int64_t nslots, int head, int tail,
                                                            const float* s, float* call,
                                                            float* put, BsConst c) {
    pdl_wait();
    pdl_trigger();
    const int t = threadIdx.x;
    if (blockIdx.x == 0) {
        const int64_t tb = head + 8 * nslots;
        if (t < head) bs_one(s[t], c, call[t], put[t]);
        if (t >= 32 && t < 32 + tail) bs_one(s[tb + t - 32], c, call[tb + t - 32], put[tb + t - 32]);
    }
    const float* sb = s + head;
    float* cb = call + head;
    float* pb = put + head;
    constexpr int64_t TILE = (int64_t)BS_T * BS_U;
    for (int64_t s0 = (int64_t)blockIdx.x * TILE; s0 < nslots; s0 += (int64_t)gridDim.x * TILE) {
#pragma unroll
        for (int u = 0; u < BS_U; ++u) {
            const int64_t slot = s0 + u * BS_T + t;
            if (slot < nslots) {
                const f8 v = ld_slot<LW>(sb + 8 * slot);
                f8 oc, op;
#pragma unroll
                for (int e = 0; e < 8; ++e) bs_one(v.v[e], c, oc.v[e], op.v[e]);
                if constexpr (LW == 8) {
                    st_v8(cb + 8 * slot, oc);
                    st_v8(pb + 8 * slot, op);
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        cb[8 * slot + e] = oc.v[e];
                        pb[8 * slot + e] = op.v[e];
                    }
                }
            }
        }
    }
}

}  // namespace lift
