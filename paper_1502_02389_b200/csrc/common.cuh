// common.cuh — sm_100a building blocks shared by the lift kernels.
//
// The paper's low-level OpenCL patterns (Table 2) become
// these B200 mechanisms:
//   asVector^8 / vect^8  -> 256-bit LDG/STG (LDG.E.ENL2.256,
//                                                  sm_100-only; 8 fp32 per lane)
//   toLocal                   -> gemv's x: the SM's L1 (one copy
//                                                  serves every resident CTA; gemv.cuh)
//   iterate^k(split-2 reduce) in local memory    -> __shfl_xor butterfly
//   reduce-seq                -> a per-thread register fold
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lift {

struct f8 {
    float v[8];
};

// 256-bit read-only streaming load (no L1 allocation): one asVector^8 element.
__device__ __forceinline__ f8 ld_nc_v8(const float* p) {
    f8 r;
    asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
          "=f"(r.v[6]), "=f"(r.v[7])
        : "l"(p));
    return r;
}

// Coherent (non-.nc) 256-bit load: used when the input may alias the output.
__device__ __forceinline__ f8 ld_v8(const float* p) {
    f8 r;
    asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                   "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p)
                 : "memory");
    return r;
}

__device__ __forceinline__ void st_v8(float* p, const f8& r) {
    asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "f"(r.v[0]), "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]),
                 "f"(r.v[6]), "f"(r.v[7])
                 : "memory");
}

// Load one 8-float slot with the widest access the alignment class allows.
// LW = 8: one 256-bit load; LW = 4: two 128-bit loads; LW = 1: eight scalar loads.
// All three return the same values, so the arithmetic order never depends on LW.
template <int LW>
__device__ __forceinline__ f8 ld_slot(const float* p) {
    if constexpr (LW == 8) {
        return ld_nc_v8(p);
    } else if constexpr (LW == 4) {
        f8 r;
        float4 a = __ldg(reinterpret_cast<const float4*>(p));
        float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
        r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
        r.v[4] = b.x; r.v[5] = b.y; r.v[6] = b.z; r.v[7] = b.w;
        return r;
    } else {
        f8 r;
#pragma unroll
        for (int e = 0; e < 8; ++e) r.v[e] = __ldg(p + e);
        return r;
    }
}

// Store one 8-float slot with the widest access the alignment class allows.
template <int LW>
__device__ __forceinline__ void st_slot(float* p, const f8& v) {
    if constexpr (LW == 8) {
        st_v8(p, v);
    } else if constexpr (LW == 4) {
        reinterpret_cast<float4*>(p)[0] = make_float4(v.v[0], v.v[1], v.v[2], v.v[3]);
        reinterpret_cast<float4*>(p)[1] = make_float4(v.v[4], v.v[5], v.v[6], v.v[7]);
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) p[e] = v.v[e];
    }
}

// Fixed pairwise fold of 8 fp64 values: ((v0+v1)+(v2+v3))+((v4+v5)+(v6+v7)).
__device__ __forceinline__ double pairwise8(const double* v) {
    return __dadd_rn(__dadd_rn(__dadd_rn(v[0], v[1]), __dadd_rn(v[2], v[3])),
                     __dadd_rn(__dadd_rn(v[4], v[5]), __dadd_rn(v[6], v[7])));
}

// Warp butterfly with xor distances 1,2,4,8,16: a pairwise tree over lanes in
// ascending adjacent pairs (IEEE addition is commutative, so lanes i and i^d get
// bit-identical sums).  Every lane ends with the warp total.
//
// NEXT-4 tree axis (compile-time, scripts/tune.py): LIFT_TREE = 2 builds the same tree as
// the paper's Fig. 7a/7b lowering, toLocal + iterate^5(split-2 reduce) in shared memory
// with a warp barrier per level: level s keeps b[i] = b[2i] + b[2i+1] for i < s — the
// same adjacent pairs, so the same bits as the butterfly.
#ifndef LIFT_TREE
#define LIFT_TREE 1  // 1: shuffle butterfly, 2: shared-memory tree
#endif
__device__ __forceinline__ double warp_pairwise(double v) {
#if LIFT_TREE == 2
    __shared__ double tree_buf[32][32];  // one row per warp of the CTA (<= 1024 threads)
    const int lane = threadIdx.x & 31;
    double* b = tree_buf[threadIdx.x >> 5];
    b[lane] = v;
    __syncwarp();
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        double t = 0.0;
        if (lane < s) t = __dadd_rn(b[2 * lane], b[2 * lane + 1]);
        __syncwarp();
        if (lane < s) b[lane] = t;
        __syncwarp();
    }
    const double r = b[0];
    __syncwarp();
    return r;
#else
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
#endif
}

// LW == 2 (gemv rows, asum/dot operands): data at any 4-byte alignment (odd n with
// lda = n, offset views).  A lane loads the 32-byte-aligned block holding the start of its vector and
// the following block (through L1, where it is usually the next lane's block) and shifts
// by d = the row's offset in floats past a 32-byte boundary.  The values, hence the
// order, are those of any other load width.  (Taking the next block from lane + 1 by
// shuffle measured slower: 72.9 vs 63.2 us at 8192 x 8191.)
template <int D>
__device__ __forceinline__ f8 realign(const f8& own, const f8& nxt) {
    f8 v;
#pragma unroll
    for (int e = 0; e < 8; ++e) v.v[e] = (e + D < 8) ? own.v[e + D] : nxt.v[e + D - 8];
    return v;
}

__device__ __forceinline__ f8 ld_l1_v8(const float* p) {  // read-only, L1-allocating
    f8 r;
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
          "=f"(r.v[6]), "=f"(r.v[7])
        : "l"(p));
    return r;
}

// The 8 floats at p (4-byte aligned; d = floats past the 32-byte boundary, uniform per row
// or operand).  `inner`: both 32-byte blocks around them lie inside the operand, so they
// are read whole (the second one is usually already in L1: the next lane's) and shifted;
// otherwise — the operand's first and last vectors — the 8 floats are read one by one, so
// no byte outside the operand is ever touched.
__device__ __forceinline__ f8 ld_realigned(const float* p, int d, bool inner) {
    if (d == 0) return ld_l1_v8(p);
    if (!inner) {
        f8 r;
#pragma unroll
        for (int e = 0; e < 8; ++e) r.v[e] = __ldg(p + e);
        return r;
    }
    const f8 own = ld_l1_v8(p - d), nxt = ld_l1_v8(p - d + 8);
    switch (d) {
        case 1: return realign<1>(own, nxt);
        case 2: return realign<2>(own, nxt);
        case 3: return realign<3>(own, nxt);
        case 4: return realign<4>(own, nxt);
        case 5: return realign<5>(own, nxt);
        case 6: return realign<6>(own, nxt);
        default: return realign<7>(own, nxt);
    }
}

// ---- Programmatic dependent launch (sm_90+) ------------------------------------------
// Every lift kernel is launched with programmatic stream serialization (lift.cu,
// launch()), so its CTAs may be scheduled while the previous kernel on the stream still
// drains.  pdl_wait() blocks until that kernel has completed and its memory is visible;
// it is the first statement of every kernel, before any global access, which makes the
// early start safe whatever the previous kernel was (a no-op when launched without the
// attribute).  pdl_trigger() lets the NEXT kernel's CTAs be scheduled once every CTA of
// this one has started (they then wait in their own pdl_wait()).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// L2 prefetch of [p, p + bytes) by the TMA engine (one instruction, no registers, no
// completion to wait for).  Issued BEFORE pdl_wait() by the first CTAs of a kernel, it
// overlaps their first DRAM round trip with the previous kernel's tail: L2 is the point of
// coherence, so prefetching data the previous kernel may still write is harmless (its
// stores update the L2 line; nothing is read into registers or L1 before the wait).
// p must be 16-byte aligned; bytes is rounded down to a multiple of 16.
#ifndef LIFT_PREFETCH
#define LIFT_PREFETCH 7  // bit mask: 1 scal, 2 reductions, 4 gemv
#endif
// Only CTAs of the first resident wave (blockIdx < SMs x resident CTAs per SM) can start
// while the previous kernel still drains; later CTAs would only duplicate their own loads.
__device__ __forceinline__ bool in_first_wave(int per_sm) {
    unsigned nsm;
    asm("mov.u32 %0, %%nsmid;" : "=r"(nsm));
    return blockIdx.x < nsm * (unsigned)per_sm;
}
// First-wave stagger.  The CTAs of a launch's first resident wave start together (the PDL
// wait releases them at once) and issue all their loads at once; with the DRAM queues shared
// fairly, they then also FINISH together (per-CTA trace, asum 2^24: 888 CTAs end within ~1 us
// of each other), and the next wave's first loads meet an idle memory pipe for a DRAM
// latency.  So CTA b < resident of the first wave starts its loads b x ns_per_cta after its
// own start (lane 0 of every warp spins on %globaltimer; the other lanes wait at the warp
// barrier): the wave's requests spread over about the time DRAM needs to serve them, its
// CTAs retire staggered and the next wave streams in behind them.  Timing only: nothing
// about what is computed depends on it.
__device__ __forceinline__ void first_wave_stagger(int64_t resident, unsigned ns_per_cta) {
    if (ns_per_cta && (int64_t)blockIdx.x < resident && blockIdx.x > 0 && (threadIdx.x & 31) == 0) {
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        const unsigned long long until = t0 + (unsigned long long)blockIdx.x * ns_per_cta;
        do asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); while (t < until);
    }
    __syncwarp();
}

template <int WHO>
__device__ __forceinline__ void prefetch_l2(const void* p, int64_t bytes) {
#if LIFT_PREFETCH
    if constexpr ((LIFT_PREFETCH & WHO) == 0) return;
    bytes &= ~(int64_t)15;
    if (bytes <= 0 || (reinterpret_cast<uintptr_t>(p) & 15)) return;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((uint32_t)bytes)
                 : "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- mbarrier + Cluster Launch Control (sm_100): hardware work stealing ---------------
// A resident CTA cancels a not-yet-launched CTA of the same grid and takes over its
// blockIdx (SASS UGETNEXTWORKID).  This gives persistent CTAs (per-CTA setup such as
// gemv's x staging paid once per resident CTA) with the dynamic load balance of a
// one-CTA-per-unit grid (per-SM bandwidth differs, so static splits finish unevenly).
// Protocol: thread 0 issues clc_try_cancel before the current unit's work; after the
// work every thread calls clc_fetch; a __syncthreads must separate clc_fetch from the
// next clc_try_cancel (the response buffer is reused).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
            "selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// TMA bulk copies (cp.async.bulk -> SASS UBLKCP): global -> shared completes `bar` by
// transaction bytes; shared -> global is tracked by the issuing thread's bulk groups.
// Addresses and sizes must be multiples of 16 bytes.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst_smem)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src_smem)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit_and_wait_read() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

struct Clc {
    uint4* resp;    // 16-byte response, shared memory
    uint64_t* bar;  // mbarrier (count 1), shared memory
    uint32_t phase;
};

__device__ __forceinline__ void clc_try_cancel(const Clc& c) {
    mbar_arrive_expect_tx(c.bar, 16);
    asm volatile(
        "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 "
        "[%0], [%1];" ::"r"(smem_u32(c.resp)),
        "r"(smem_u32(c.bar))
        : "memory");
}

// Returns true and the stolen CTA's blockIdx.x in `next`, or false (no work left).
__device__ __forceinline__ bool clc_fetch(Clc& c, int64_t& next) {
    mbar_wait(c.bar, c.phase);
    c.phase ^= 1u;
    uint32_t ok, cx;
    asm volatile(
        "{ .reg .b128 r; .reg .pred p; ld.shared.b128 r, [%2]; "
        "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r; selp.u32 %0, 1, 0, p; "
        "clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, r; }"
        : "=r"(ok), "=r"(cx)
        : "r"(smem_u32(c.resp))
        : "memory");
    next = cx;
    // order this generic read of the response before the next try_cancel's async write
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    return ok != 0;
}

// ---- NEXT-1 peer-memory exchange primitives (reduce.cuh, gemv.cuh) -----------------
// Exchange buffer of one rank: [2 banks x p slots of XchgSlot][2 u64 counters].
struct XchgSlot {
    double value;
    unsigned long long flag;
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double ld_relaxed_sys_f64(const double* p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long* xchg_counter(void* buf, int p, int bank) {
    return reinterpret_cast<unsigned long long*>(reinterpret_cast<XchgSlot*>(buf) + 2 * p) + bank;
}

// Lane q < p: wait until slot q of this rank's bank carries `epoch` (bounded ~10 s).
// Returns false on timeout.
__device__ __forceinline__ bool xchg_wait_flag(void* own_buf, int bank_base, int q,
                                               unsigned long long epoch) {
    XchgSlot* own = reinterpret_cast<XchgSlot*>(own_buf) + bank_base + q;
    unsigned long long spins = 0;
    while (ld_acquire_sys(&own->flag) != epoch) {
        __nanosleep(128);
        if (++spins > (1ull << 26)) return false;
    }
    return true;
}

}  // namespace lift
