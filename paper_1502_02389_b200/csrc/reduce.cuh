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
//     of RED_C = RED_T * 8 * RED_K elements (8192).  Inside a chunk, lane t of RED_T = 256 owns the
//     8-float vectors t, t+256, t+512, ... (reorder-stride with s = 256), so a warp
//     reads 32 consecutive 32-byte vectors per instruction (LDG.256, coalesced).
//     Chunks go to CTAs grid-stride (map-workgroup).
//  R1 fused reduce-seq o map-seq (rule 5f): each lane keeps 8
//     accumulators (one per vector slot e) and folds acc_e = acc_e + |x| (asum) or
//     acc_e = fma(x, y, acc_e) (dot) over its RED_K vectors in ascending order — no
//     intermediate array.
//  R3 toLocal + iterate(split-2 reduce): lane value = fixed pairwise
//     fold of its 8 accumulators in fp64; warp butterfly (xor 1,2,4,8,16); then the
//     8 warp values pairwise through shared memory -> one fp64 CHUNK PARTIAL.  One
//     CTA barrier per chunk; everything after it runs in warp 0 only.
//  R4 the outermost reduce-seq o join, single pass, no second launch: a
//     two-level last-block-done.  The CTA that finishes the last chunk of a group of
//     RED_G chunks folds that group's partials (pairwise); the CTA that finishes the
//     last group folds the group partials (pairwise, zero-padded to a power of two)
//     and writes the fp32 result (rounded once) and/or the fp64 partial.  Tickets
//     are reset to 0 by the CTAs that consume them.
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

#ifndef LIFT_DOT_MINB
#define LIFT_DOT_MINB 4  // resident CTAs per SM the dot kernel is compiled for (registers)
#endif
#ifndef LIFT_ASUM_MINB
#define LIFT_ASUM_MINB 6  // the same for asum
#endif
#ifndef LIFT_RED_RMINB
#define LIFT_RED_RMINB 4  // resident CTAs per SM for the realigned (LW 2) reductions
#endif
#ifndef LIFT_RED_RB
#define LIFT_RED_RB 2
#endif
#ifndef LIFT_RED_FLAT
#define LIFT_RED_FLAT 1  // one ticket level + whole-CTA fold for 256 < nc <= 2048 (mid sizes)
#endif
#ifndef LIFT_RED_EXPT
#define LIFT_RED_EXPT 0  // timing experiments only (never the product)
#endif
#ifndef LIFT_RED_TMA
#define LIFT_RED_TMA 0  // NEXT-4 (tune.py): chunks arrive by TMA bulk copy into shared memory
#endif
#ifndef LIFT_RED_TMA
#define LIFT_RED_TMA 0  // NEXT-4 (tune.py): chunks arrive by TMA bulk copy into shared memory
#endif
#ifndef LIFT_SC_FENCE
#define LIFT_SC_FENCE 0
#endif

// The fused per-element step (rule 5f).  Acc is the per-lane accumulator type.
//  * asum uses fp32 accumulators over its RED_K = 4-term runs (|x| is exact, so only
//    4-term rounding) — no fp32->fp64 conversion per element.  A run can only
//    overflow if terms approach FLT_MAX/4; then the chunk is recomputed with fp64
//    accumulators (see reduce_kernel), so results never differ from the fp64 fold by
//    more than rounding and Inf/NaN inputs still propagate.
//  * dot uses fp64 accumulators with exact products (an fp32 product could overflow
//    or lose bits to underflow); reading R13.
template <class Acc>
struct AsumOp {
    using acc_t = Acc;
    template <class A2>
    using rebind = AsumOp<A2>;
    static constexpr bool kTwoInputs = false;
    static constexpr bool kMapStore = false;
    static constexpr int kMinBlocks = LIFT_ASUM_MINB;
    __device__ __forceinline__ static Acc step(Acc acc, float a, float) {
        if constexpr (sizeof(Acc) == 8) return __dadd_rn(acc, fabs((double)a));
        else return __fadd_rn(acc, fabsf(a));  // abs then add, fused
    }
};
template <class Acc>
struct DotOp {
    using acc_t = Acc;
    template <class A2>
    using rebind = DotOp<A2>;
    static constexpr bool kTwoInputs = true;
    static constexpr bool kMapStore = false;
    static constexpr int kMinBlocks = LIFT_DOT_MINB;
    __device__ __forceinline__ static Acc step(Acc acc, float a, float b) {
        if constexpr (sizeof(Acc) == 8) return __fma_rn((double)a, (double)b, acc);  // exact product
        else return __fmaf_rn(a, b, acc);  // mult then add, one rounding
    }
};

// NEXT-2 — cross-op fusion by rule 5f: asum(scal(a, x)).
//   map(f) o map(g) -> map(f o g) and reduce-seq(f) o map-seq(g) -> one fold, so
//   y = scal(a, x) is written AND asum(y) is folded in the same pass over x: 8 bytes
//   per element instead of scal's 8 plus asum's 4.  The fold consumes exactly the
//   stored y values in asum's canonical order, so the result is bit-identical to
//   lift_asum(lift_scal(x)).
template <class Acc>
struct ScalAsumOp {
    using acc_t = Acc;
    template <class A2>
    using rebind = ScalAsumOp<A2>;
    static constexpr bool kTwoInputs = false;
    static constexpr bool kMapStore = true;
    static constexpr int kMinBlocks = 4;
    __device__ __forceinline__ static float map(float a, float alpha) { return __fmul_rn(alpha, a); }
    __device__ __forceinline__ static Acc step(Acc acc, float m, float) {
        return AsumOp<Acc>::step(acc, m, 0.f);
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
    float alpha;         // kMapStore ops: the map's scalar
    float* map_out;      // kMapStore ops: where the mapped values are stored (n floats)
    // NEXT-1 fused cross-GPU combine (null peers: plain single-GPU result)
    void* const* peers;  // p exchange buffers, peers[rank] = this rank's own
    int p, rank;
    unsigned long long epoch;  // > 0, increasing per call on the same buffers
    int* error;                // set to 1 if the peers did not arrive in time
    int prefetch;              // L2-prefetch the CTA's first chunk before the PDL wait
    int64_t resident;          // first-wave stagger (common.cuh): CTAs resident at once
    unsigned stagger_ns;       //   and ns per first-wave CTA index (0: none)
};

// ---- NEXT-1: the outermost reduce across GPUs, inside the kernel -------------------
// Exchange buffer (per rank, lift_xchg_bytes): two banks (epoch parity) of p slots of
// {double value; u64 flag}.  The final CTA of every rank stores its fp64 partial into
// slot `rank` of every peer's buffer (NVLink P2P stores to IPC-mapped memory), then
// raises the slot's flag to `epoch` with a system-scope release; it then waits for all
// p flags of its own buffer (acquire) and folds the p values pairwise in rank order
// (zero-padded to 32 — the same tree as lift_combine), so every rank gets the same
// bits with no separate collective launch.  Two banks suffice: a peer can be at most
// one call ahead, since finishing call e needs this rank's call-e publish.
// Warp 0 of the finishing CTA: publish `total`, gather all ranks', fold, write out.
__device__ __forceinline__ void xchg_combine(const ReduceArgs& a, double total) {
    const int lane = threadIdx.x & 31;
    const int bank = (int)(a.epoch & 1ull) * a.p;
    if (lane < a.p) {
        XchgSlot* dst = reinterpret_cast<XchgSlot*>(a.peers[lane]) + bank + a.rank;
        dst->value = total;
        st_release_sys(&dst->flag, a.epoch);  // the release orders the value store before it
    }
    double v = 0.0;
    bool ok = true;
    if (lane < a.p) {  // bounded spin (~10 s): a missing peer must not hang the GPU
        ok = xchg_wait_flag(a.peers[a.rank], bank, lane, a.epoch);
        XchgSlot* own = reinterpret_cast<XchgSlot*>(a.peers[a.rank]) + bank + lane;
        v = ok ? ld_relaxed_sys_f64(&own->value) : 0.0;
    }
    const bool all_ok = __all_sync(0xffffffffu, ok);
    const double sum = warp_pairwise(v);  // pairwise over ranks, zero-padded to 32
    if (lane == 0) {
        const double r = all_ok ? sum : __longlong_as_double(0x7ff8000000000000ll);  // NaN
        if (!all_ok && a.error) *a.error = 1;
        if (a.out_f64) *a.out_f64 = r;
        if (a.out_f32) *a.out_f32 = __double2float_rn(r);
    }
}

// Last-block-done tickets.  Lane 0 publishes a partial with a plain store and takes a
// ticket with an acq_rel atomic (release: its store before the ticket; acquire: every
// earlier ticket holder's store before what follows); the warp barrier then orders the
// other lanes' leaf loads after lane 0's acquire.  (LIFT_SC_FENCE: the __threadfence
// pair instead, for A/B runs.)
__device__ __forceinline__ unsigned ticket_acq_rel(unsigned* t) {
#if LIFT_SC_FENCE == 1
    __threadfence();
    return atomicAdd(t, 1u);
#elif LIFT_SC_FENCE == 2  // (A/B) release-only ticket; the last CTA acquires separately
    unsigned old;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(t) : "memory");
    return old;
#else
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(t) : "memory");
    return old;
#endif
}
__device__ __forceinline__ void ticket_acquired(const unsigned* t) {
#if LIFT_SC_FENCE == 1
    (void)t;
    __threadfence();
#elif LIFT_SC_FENCE == 2
    if ((threadIdx.x & 31) == 0) {  // acquire: synchronizes with every release on the ticket
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(t) : "memory");
    }
    __syncwarp();
#else
    (void)t;
    __syncwarp();
#endif
}

// Warp-level pairwise fold of `nleaf` fp64 leaves read from global memory (L2),
// zero-padded to a power of two p2: lane l folds the aligned block [l*blk, (l+1)*blk)
// (blk = max(1, p2/32)) with a binary-counter stack — the pairwise tree restricted to
// that block — and the butterfly joins the 32 blocks.  Any such decomposition into
// aligned power-of-two blocks yields exactly THE pairwise tree over the leaves.
__device__ __forceinline__ double warp_fold_leaves(const double* leaves, int64_t nleaf) {
    const int lane = threadIdx.x & 31;
    int64_t p2 = 1;
    while (p2 < nleaf) p2 <<= 1;
    const int64_t blk = p2 > 32 ? p2 / 32 : 1;
    const int64_t l0 = (int64_t)lane * blk;
    double v;
    if (blk == 1) {
        v = (lane < nleaf) ? __ldcg(leaves + lane) : 0.0;
    } else if (blk <= 8) {
        // all of the lane's leaves in flight at once (one L2 round trip), then the
        // pairwise tree over them
        double w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = (i < blk && l0 + i < nleaf) ? __ldcg(leaves + l0 + i) : 0.0;
        if (blk == 2) v = __dadd_rn(w[0], w[1]);
        else if (blk == 4) v = __dadd_rn(__dadd_rn(w[0], w[1]), __dadd_rn(w[2], w[3]));
        else v = pairwise8(w);
    } else {
        // batches of 8 leaves (8 loads in flight), each batch's subtree pushed on a
        // binary-counter stack: the pairwise tree over aligned batches of 8 leaves
        double stk[40];
        int top = 0;
        for (int64_t b = 0; b < blk / 8; ++b) {
            double w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int64_t li = l0 + 8 * b + i;
                w[i] = (li < nleaf) ? __ldcg(leaves + li) : 0.0;
            }
            double s = pairwise8(w);
            for (int64_t cnt = b; cnt & 1; cnt >>= 1) s = __dadd_rn(stk[--top], s);
            stk[top++] = s;
        }
        v = stk[0];
    }
    return warp_pairwise(v);
}

// n == 0 on one rank of an all-reduce: it still has to publish (a zero) and combine.
__global__ void xchg_only_kernel(ReduceArgs a) {
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x < 32) xchg_combine(a, 0.0);
}

// LW == 2: operands at any 4-byte alignment (slices at odd float offsets), read as
// 32-byte-aligned blocks and shifted (common.cuh ld_realigned); never with a map store.
template <class Op, int LW, int B0>
__device__ __forceinline__ void chunk_body_full(const float* xc, const float* yc,
                                                typename Op::acc_t* acc, float alpha = 0.f,
                                                float* mo = nullptr, int64_t base = 0,
                                                int64_t n = 0) {
    constexpr int BL = LW == 2 ? LIFT_RED_RB : B0;  // realigned: fewer vectors held (registers)
    constexpr int B = BL < RED_K ? BL : RED_K;
    static_assert(RED_K % B == 0, "load batch must divide RED_K");
    static_assert(LW != 2 || !Op::kMapStore, "no realigned map stores");
    const int t = threadIdx.x;
    // LW == 2: offsets past a 32-byte boundary (uniform); base, n: this chunk's first global
    // element and the operand length, for ld_realigned's inside-the-operand test
    const int dx = LW == 2 ? (int)((reinterpret_cast<uintptr_t>(xc) >> 2) & 7) : 0;
    const int dy = (LW == 2 && Op::kTwoInputs) ? (int)((reinterpret_cast<uintptr_t>(yc) >> 2) & 7) : 0;
#pragma unroll
    for (int k0 = 0; k0 < RED_K; k0 += B) {
        f8 xv[B];
        f8 yv[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int64_t q = t + (k0 + b) * RED_T;
            if constexpr (LW == 2) {
                const int64_t j = base + (int64_t)RED_V * q;  // global index of the vector
                xv[b] = ld_realigned(xc + (int64_t)RED_V * q, dx, j >= dx && j - dx + 16 <= n);
                if constexpr (Op::kTwoInputs)
                    yv[b] = ld_realigned(yc + (int64_t)RED_V * q, dy, j >= dy && j - dy + 16 <= n);
            } else {
                xv[b] = ld_slot<LW>(xc + (int64_t)RED_V * q);
                if constexpr (Op::kTwoInputs) yv[b] = ld_slot<LW>(yc + (int64_t)RED_V * q);
            }
        }
        if constexpr (Op::kMapStore) {
#pragma unroll
            for (int b = 0; b < B; ++b) {
#pragma unroll
                for (int e = 0; e < RED_V; ++e) xv[b].v[e] = Op::map(xv[b].v[e], alpha);
                st_slot<LW>(mo + (int64_t)RED_V * (t + (k0 + b) * RED_T), xv[b]);
            }
        }
#pragma unroll
        for (int b = 0; b < B; ++b)
#pragma unroll
            for (int e = 0; e < RED_V; ++e)
                acc[e] = Op::step(acc[e], xv[b].v[e], Op::kTwoInputs ? yv[b].v[e] : 0.f);
    }
}

// NEXT-4 load axis, TMA bulk variant (compile-time LIFT_RED_TMA = 1; scripts/tune.py): the
// chunk's x (and y) arrive in shared memory by one bulk copy each (an mbarrier completes by
// bytes); lanes then read their vectors t + 256k from shared memory — the same values in
// the same order, so the same bits.  Full, 16-byte-aligned chunks only.
template <class Op>
__device__ __forceinline__ void chunk_body_tma(const float* xc, const float* yc,
                                               typename Op::acc_t* acc, uint64_t* bar,
                                               uint32_t& phase) {
    extern __shared__ __align__(128) unsigned char red_smem[];
    float* xs = reinterpret_cast<float*>(red_smem);
    float* ys = xs + RED_C;
    const int t = threadIdx.x;
    if (t == 0) {
        mbar_arrive_expect_tx(bar, (uint32_t)(RED_C * 4 * (Op::kTwoInputs ? 2 : 1)));
        bulk_g2s(xs, xc, RED_C * 4, bar);
        if constexpr (Op::kTwoInputs) bulk_g2s(ys, yc, RED_C * 4, bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
#pragma unroll
    for (int k = 0; k < RED_K; ++k) {
        const int q = t + k * RED_T;
        const float4 a0 = reinterpret_cast<const float4*>(xs)[2 * q];
        const float4 a1 = reinterpret_cast<const float4*>(xs)[2 * q + 1];
        const float xv[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        float yv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if constexpr (Op::kTwoInputs) {
            const float4 b0 = reinterpret_cast<const float4*>(ys)[2 * q];
            const float4 b1 = reinterpret_cast<const float4*>(ys)[2 * q + 1];
            yv[0] = b0.x; yv[1] = b0.y; yv[2] = b0.z; yv[3] = b0.w;
            yv[4] = b1.x; yv[5] = b1.y; yv[6] = b1.z; yv[7] = b1.w;
        }
#pragma unroll
        for (int e = 0; e < RED_V; ++e) acc[e] = Op::step(acc[e], xv[e], yv[e]);
    }
}

// Partial last chunk: same order, elements >= n skipped.  Skipping equals adding
// +0 exactly (the accumulators start at +0 and can never become -0 in RN).
template <class Op>
__device__ __forceinline__ void chunk_body_tail(const float* xc, const float* yc, int64_t len,
                                                typename Op::acc_t* acc, float alpha = 0.f,
                                                float* mo = nullptr) {
    const int t = threadIdx.x;
    for (int k = 0; k < RED_K; ++k) {
#pragma unroll
        for (int e = 0; e < RED_V; ++e) {
            const int64_t j = (int64_t)RED_V * (t + k * RED_T) + e;
            if (j < len) {
                float v = xc[j];
                if constexpr (Op::kMapStore) {
                    v = Op::map(v, alpha);
                    mo[j] = v;
                }
                acc[e] = Op::step(acc[e], v, Op::kTwoInputs ? yc[j] : 0.f);
            }
        }
    }
}

// Resident CTAs per SM the register budget must allow (ptxas trades registers for how
// many loads it issues up front).  Measured: asum 6 (all 4 loads up front, 40 regs),
// dot 4 (all 8 loads up front); minBlocks 1 collapses occupancy (-40%).
#ifdef LIFT_TRACE
// Diagnostic builds only (-DLIFT_TRACE; never the product .so): per-chunk CTA
// [start, end] globaltimer stamps and SM id, read back with lift_trace_read().
__device__ unsigned long long g_trace[3 * 65536];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// R3 + R4 for chunk c whose per-lane accumulators are `acc`: lane -> warp (butterfly)
// -> CTA (8 warps pairwise) -> fp64 chunk partial; then warp 0 alone publishes it and
// runs the two-level last-block-done.  Exactly one CTA barrier on the common path.
template <class Op, int LW, int B>
__device__ __forceinline__ void chunk_finish(const ReduceArgs& a, int64_t c,
                                             const typename Op::acc_t* acc, double (*wbuf)[8],
                                             int parity) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t base = c * RED_C;
    double lane8[RED_V];
    bool bad = false;
#pragma unroll
    for (int e = 0; e < RED_V; ++e) {
        lane8[e] = (double)acc[e];
        if constexpr (sizeof(acc[0]) == 4) bad |= !isfinite(acc[e]);
    }
    double wv = warp_pairwise(pairwise8(lane8));
    if (lane == 0) wbuf[parity][warp] = wv;
    bool redo = false;
    if constexpr (sizeof(acc[0]) == 4) redo = __syncthreads_or(bad);  // the one barrier
    else __syncthreads();
    if constexpr (sizeof(acc[0]) == 4) {
        if (redo) {  // rare: an fp32 run overflowed (or the chunk holds Inf/NaN)
            const float* xc = a.x + base;
            const float* yc = Op::kTwoInputs ? a.y + base : nullptr;
            const bool full = base + RED_C <= a.n;
            double acc64[RED_V];
#pragma unroll
            for (int e = 0; e < RED_V; ++e) acc64[e] = 0.0;
            if constexpr (Op::kMapStore) {
                // refold this thread's own stored map values
                chunk_body_tail<AsumOp<double>>(a.map_out + base, nullptr,
                                                min((int64_t)RED_C, a.n - base), acc64);
            } else {
                using Op64 = typename Op::template rebind<double>;
                if (full) chunk_body_full<Op64, LW, B>(xc, yc, acc64, 0.f, nullptr, base, a.n);
                else chunk_body_tail<Op64>(xc, yc, a.n - base, acc64);
            }
            wv = warp_pairwise(pairwise8(acc64));
            if (lane == 0) wbuf[parity][warp] = wv;  // nobody reads wbuf before the barrier
            __syncthreads();
        }
    }
#ifdef LIFT_TRACE
    if (t == 0 && c < 65536) g_trace[3 * c + 1] = gtimer();
#endif
#if LIFT_RED_FLAT
    // Mid sizes (256 < nc <= 2048 chunks, one chunk per CTA): ONE ticket level and the whole
    // last CTA folds every chunk partial — blk = p2(nc)/256 leaves per thread, warp
    // butterfly, 8 warp values pairwise: the pairwise tree over the chunk partials
    // zero-padded to p2(nc), i.e. exactly the two-level tree (p2(ceil(nc/256)) * 256 =
    // p2(nc)), so the same bits with two dependent L2 round trips instead of four.  The
    // cost: every CTA's warps wait for the ticket at a second CTA barrier.
    if (a.nc > RED_G && a.nc <= 8 * RED_G && gridDim.x == a.nc && !a.peers) {
        __shared__ unsigned flat_last;
        if (t == 0) {
            a.chunk_part[c] = pairwise8(wbuf[parity]);
            flat_last = ticket_acq_rel(&a.tick[0]) == (unsigned)(a.nc - 1);
        }
        __syncthreads();  // thread 0's acquire (and the verdict) ordered before every thread
        if (!flat_last) return;
        int64_t p2 = 1;
        while (p2 < a.nc) p2 <<= 1;
        const int blk = (int)(p2 / RED_T);  // 2, 4 or 8
        double w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t li = (int64_t)t * blk + i;
            w[i] = (i < blk && li < a.nc) ? __ldcg(a.chunk_part + li) : 0.0;
        }
        double v = blk == 2 ? __dadd_rn(w[0], w[1])
                 : blk == 4 ? __dadd_rn(__dadd_rn(w[0], w[1]), __dadd_rn(w[2], w[3]))
                            : pairwise8(w);
        v = warp_pairwise(v);
        if (lane == 0) wbuf[parity ^ 1][warp] = v;
        __syncthreads();
        if (t == 0) {
            const double total = pairwise8(wbuf[parity ^ 1]);
            a.tick[0] = 0u;
            if (a.out_f64) *a.out_f64 = total;
            if (a.out_f32) *a.out_f32 = __double2float_rn(total);
#ifdef LIFT_TRACE
            g_trace[3 * 65535] = gtimer();  // timeline marker: the final result store (flat path)
            g_trace[3 * 65535 + 1] = (unsigned long long)c;
#endif
        }
        return;
    }
#endif
    if (warp != 0) return;

    // ---- R4, warp 0 only: publish the chunk partial, group ticket ----------------
    const int64_t g = c / RED_G;
    unsigned last = 0;
    if (lane == 0) {
        a.chunk_part[c] = pairwise8(wbuf[parity]);
        const int64_t gcount = min((int64_t)RED_G, a.nc - g * RED_G);
#if LIFT_RED_EXPT == 1  // TIMING EXPERIMENT ONLY (wrong results): no CTA waits for a ticket
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&a.tick[g]) : "memory");
        (void)gcount;
        last = 0;
        if (c == 0 && lane == 0) *a.out_f32 = 0.f;
#else
        last = (ticket_acq_rel(&a.tick[g]) == (unsigned)(gcount - 1));
#endif
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return;

    // Last chunk of group g: fold the group's RED_G chunk partials (pairwise).
    ticket_acquired(&a.tick[g]);
    const int64_t g0 = g * RED_G;
    const double gpart = warp_fold_leaves(a.chunk_part + g0, min((int64_t)RED_G, a.nc - g0));
    if (a.ng == 1) {  // one group: the pairwise fold over one leaf is the leaf itself
        if (lane == 0) a.tick[0] = 0u;
        if (a.peers) {
            xchg_combine(a, gpart);
        } else if (lane == 0) {
            if (a.out_f64) *a.out_f64 = gpart;
            if (a.out_f32) *a.out_f32 = __double2float_rn(gpart);
        }
        return;
    }
    last = 0;
    if (lane == 0) {
        a.group_part[g] = gpart;
        a.tick[g] = 0u;  // reset for the next call (workspace contract)
        last = (ticket_acq_rel(&a.tick[a.ng]) == (unsigned)(a.ng - 1));
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return;

    // Last group: final pairwise fold over the group partials, round once.
    ticket_acquired(&a.tick[a.ng]);
    const double total = warp_fold_leaves(a.group_part, a.ng);
    if (lane == 0) a.tick[a.ng] = 0u;
    if (a.peers) {
        xchg_combine(a, total);
    } else if (lane == 0) {
        if (a.out_f64) *a.out_f64 = total;
        if (a.out_f32) *a.out_f32 = __double2float_rn(total);
    }
#ifdef LIFT_TRACE
    if (lane == 0) {  // timeline marker: the final result store (two-level path)
        g_trace[3 * 65535] = gtimer();
        g_trace[3 * 65535 + 1] = (unsigned long long)c;
    }
#endif
}

__device__ __forceinline__ void trace_start(int64_t c) {
#ifdef LIFT_TRACE
    if (threadIdx.x == 0 && c < 65536) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_trace[3 * c] = gtimer();
        g_trace[3 * c + 2] = smid;
    }
#else
    (void)c;
#endif
}

// One CTA per chunk, hardware-scheduled (the default).
template <class Op, int LW, int B, bool DESC = false>
__global__ void __launch_bounds__(RED_T, LW == 2 ? LIFT_RED_RMINB : Op::kMinBlocks) reduce_kernel(ReduceArgs a) {
    // the CTA's first chunk, L2-prefetched before the wait (common.cuh prefetch_l2); the
    // launcher enables it for the fused map+store ops (LIFT_VAR_PREFETCH)
    if (a.prefetch && threadIdx.x == 0 && blockIdx.x < a.nc) {
        const int64_t b0 = (DESC ? a.nc - 1 - (int64_t)blockIdx.x : (int64_t)blockIdx.x) * RED_C;
        const int64_t len = (a.n - b0 < RED_C ? a.n - b0 : RED_C) * 4;
        prefetch_l2<2>(a.x + b0, len);
        if constexpr (Op::kTwoInputs) prefetch_l2<2>(a.y + b0, len);
    }
    pdl_wait();
    pdl_trigger();
    first_wave_stagger(a.resident, a.stagger_ns);  // common.cuh
    __shared__ double wbuf[2][RED_T / 32];  // double-buffered by chunk parity
    constexpr bool kTma = LIFT_RED_TMA && LW >= 4 && !Op::kMapStore;
    __shared__ uint64_t tma_bar;
    uint32_t tma_phase = 0;
    if constexpr (kTma) {
        if (threadIdx.x == 0) mbar_init(&tma_bar, 1);
        __syncthreads();
    }
    int parity = 0;
    // Temporal order of the chunks (never the summation order: partials are stored and
    // folded by chunk INDEX, so the bits are the same either way).  Descending lets a
    // reduction that follows a map over the same vector (scal, then asum of its input)
    // start where the map ended — on the tail the map just left in the 126 MB L2.
    const int64_t cstep = DESC ? -(int64_t)gridDim.x : (int64_t)gridDim.x;
    for (int64_t c = DESC ? a.nc - 1 - blockIdx.x : blockIdx.x; DESC ? c >= 0 : c < a.nc;
         c += cstep, parity ^= 1) {
        trace_start(c);
        // ---- R1/R2: fused per-lane fold over the chunk ---------------------------
        const int64_t base = c * RED_C;
        const float* xc = a.x + base;
        const float* yc = Op::kTwoInputs ? a.y + base : nullptr;
        typename Op::acc_t acc[RED_V];
#pragma unroll
        for (int e = 0; e < RED_V; ++e) acc[e] = 0;
        float* mo = Op::kMapStore ? a.map_out + base : nullptr;
        if (kTma && base + RED_C <= a.n) chunk_body_tma<Op>(xc, yc, acc, &tma_bar, tma_phase);
        else if (base + RED_C <= a.n) chunk_body_full<Op, LW, B>(xc, yc, acc, a.alpha, mo, base, a.n);
        else chunk_body_tail<Op>(xc, yc, a.n - base, acc, a.alpha, mo);
        chunk_finish<Op, LW, B>(a, c, acc, wbuf, parity);
    }
}

}  // namespace lift
