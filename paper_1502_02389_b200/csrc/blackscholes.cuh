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
// fp32 storage and arithmetic (the paper's 4-byte elements) with the IEEE-
// accurate libdevice logf/expf/erfcf/sqrtf (no fast math).  One erfcf per d: with
// e = erfc(|d|/sqrt 2) (the small tail, relatively accurate), N(-|d|) = e/2 and
// N(|d|) = 1 - e/2 (>= 1/2, so 1 - e/2 loses nothing) — both tails stay accurate
// with half the erfcf calls of evaluating N(d) and N(-d) separately.
//
// B200 mapping: like scal — one CTA per tile, 8 consecutive prices per thread from
// one 256-bit load, two 256-bit stores (call, put); the per-price transcendental
// chain is independent across the 8, which gives the MUFU/FMA pipes ILP.  12 bytes
// move per price, and the SFU/FMA work per price is ~100+ instructions, so at the
// paper's 4M prices this map is instruction-bound rather than HBM-bound (profiles/).
#pragma once
#include "common.cuh"

namespace lift {

constexpr int BS_T = 256;  // threads per CTA
constexpr int BS_U = 1;    // 8-price slots per thread per tile

struct BsParams {
    float K, r, v, T;
};

struct BsConst {
    float invK, drift_T, vsqrt, inv_vsqrt, disc;
};

__device__ __forceinline__ BsConst bs_const(const BsParams& p) {
    BsConst c;
    const float sqrtT = sqrtf(p.T);
    c.invK = 1.0f / p.K;
    c.drift_T = (p.r + 0.5f * p.v * p.v) * p.T;
    c.vsqrt = p.v * sqrtT;
    c.inv_vsqrt = 1.0f / c.vsqrt;
    c.disc = p.K * expf(-p.r * p.T);
    return c;
}

// N(d) and N(-d) from a single erfcf (see the header comment).
__device__ __forceinline__ void norm_cdf_pair(float d, float& n_pos, float& n_neg) {
    constexpr float kRsqrt2 = 0.70710678118654752440f;
    const float half_tail = 0.5f * erfcf(fabsf(d) * kRsqrt2);  // N(-|d|)
    const float body = 1.0f - half_tail;                        // N(|d|)
    n_pos = d >= 0.f ? body : half_tail;                        // N(d)
    n_neg = d >= 0.f ? half_tail : body;                        // N(-d)
}

// One BSComputation.
__device__ __forceinline__ void bs_one(float S, const BsConst& c, const BsParams& p, float& call,
                                       float& put) {
    const float d1 = (logf(S * c.invK) + c.drift_T) * c.inv_vsqrt;  // compD1
    const float d2 = d1 - c.vsqrt;                                  // compD2
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
                                                            float* put, BsParams p) {
    const BsConst c = bs_const(p);
    const int t = threadIdx.x;
    if (blockIdx.x == 0) {
        const int64_t tb = head + 8 * nslots;
        if (t < head) bs_one(s[t], c, p, call[t], put[t]);
        if (t >= 32 && t < 32 + tail) bs_one(s[tb + t - 32], c, p, call[tb + t - 32], put[tb + t - 32]);
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
                for (int e = 0; e < 8; ++e) bs_one(v.v[e], c, p, oc.v[e], op.v[e]);
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
