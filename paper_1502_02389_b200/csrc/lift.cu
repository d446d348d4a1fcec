// lift.cu — the C ABI of liblift.so (include/lift.h): argument checks, launch
// configuration and the cross-rank combine kernel.  Every step of the hot path runs
// in the kernels of scal.cuh, reduce.cuh and gemv.cuh; this file only validates and
// launches (no host arithmetic on the data, no CPU fallback).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/lift.h"
#include "canon.h"
#include "common.cuh"
#include "blackscholes.cuh"
#include "gemv.cuh"
#include "gemv_xs.cuh"
#include "gemv_tma.cuh"
#include "gemv_r2.cuh"
#include "reduce.cuh"
#include "gemv_long.cuh"
#include "scal.cuh"

#ifndef LIFT_ASUM_B
#define LIFT_ASUM_B 8  // 256-bit loads in flight per lane (asum)
#endif
#ifndef LIFT_DOT_B
#define LIFT_DOT_B 4   // vector pairs in flight per lane (dot)
#endif
#ifndef LIFT_ASUM_ACC
#define LIFT_ASUM_ACC float   // per-lane accumulators (canonical order, reading R13)
#endif
#ifndef LIFT_DOT_ACC
#define LIFT_DOT_ACC double
#endif

namespace lift {

// X1: outermost reduce over p per-rank fp64 partials, pairwise (zero-padded to 2^k).
__global__ void combine_kernel(int p, const double* __restrict__ partials, float* result) {
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int64_t p2 = 1;
    while (p2 < p) p2 <<= 1;
    double stk[40];
    int top = 0;
    for (int64_t i = 0; i < p2; ++i) {
        double w = (i < p) ? partials[i] : 0.0;
        for (int64_t cnt = i; cnt & 1; cnt >>= 1) w = __dadd_rn(stk[--top], w);
        stk[top++] = w;
    }
    *result = __double2float_rn(stk[0]);
}

namespace {

std::atomic<int> g_grid_limit{0};
std::atomic<int> g_var[LIFT_VAR_COUNT];  // NEXT-4 runtime variants (0 = tuned default)

inline int var(lift_variant k) { return g_var[k].load(std::memory_order_relaxed); }

// LIFT_VAR_LOAD_WIDTH: cap a load class (8 = 256-bit, 4 = 128-bit, 1 = scalar).
inline int cap_lw(int lw) {
    const int c = var(LIFT_VAR_LOAD_WIDTH);
    return c == 0 ? lw : (lw < c ? lw : c);
}
inline bool lw_capped() { const int c = var(LIFT_VAR_LOAD_WIDTH); return c != 0 && c != 8; }

std::atomic<int> g_sms[64];  // per-device SM count cache (0 = not yet queried)
std::mutex g_mu;

struct OccEntry {
    const void* fn;
    int dev;
    size_t smem;
    int blocks;
};
OccEntry g_occ[256];
int g_nocc = 0;

int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

int sm_count(int dev) {
    if (dev < 0 || dev >= 64) return 148;
    int s = g_sms[dev].load(std::memory_order_relaxed);
    if (s == 0) {
        cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
        if (s <= 0) s = 148;
        g_sms[dev].store(s, std::memory_order_relaxed);
    }
    return s;
}

// Resident CTAs per SM for `fn` (cached).  Also raises the dynamic smem limit.
int occupancy(const void* fn, int threads, size_t smem) {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_mu);
    for (int i = 0; i < g_nocc; ++i)
        if (g_occ[i].fn == fn && g_occ[i].dev == dev && g_occ[i].smem == smem)
            return g_occ[i].blocks;
    // The attribute is a per-function maximum: set it to the device's opt-in maximum, so
    // launches with any dynamic smem size (other n) stay valid whatever the call order.
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, fn);
    if (smem + fa.sharedSizeBytes > 48 * 1024) {  // opt-in maximum minus the static smem
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        const int room = optin - (int)fa.sharedSizeBytes;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             room > (int)smem ? room : (int)smem);
    }
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, threads, smem) != cudaSuccess ||
        b < 1)
        b = 1;
    if (g_nocc < 256) g_occ[g_nocc++] = OccEntry{fn, dev, smem, b};
    return b;
}

#ifndef LIFT_PERSISTENT
#define LIFT_PERSISTENT 0  // 1: grid capped at resident CTAs (grid-stride); 0: one CTA per unit
#endif
// `stealing`: the kernel takes further units by Cluster Launch Control instead of a
// grid-stride loop, so its grid must cover all units (the test grid cap cannot apply).
int64_t grid_for(int64_t work_ctas, const void* fn, int threads, size_t smem, bool persistent,
                 bool stealing = false) {
    const int dev = current_device();
    int64_t g = work_ctas;
    const int64_t resident = (int64_t)sm_count(dev) * occupancy(fn, threads, smem);  // also sets smem attr
    if (persistent && resident < g) g = resident;
    if (g > 0x7fffffffLL) g = 0x7fffffffLL;
    const int lim = g_grid_limit.load();
    if (!stealing && lim > 0 && g > lim) g = lim;
    return g < 1 ? 1 : g;
}

inline bool misaligned4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3) != 0; }
inline int align_class(uintptr_t a) { return (a & 31) == 0 ? 8 : ((a & 15) == 0 ? 4 : 1); }

#ifndef LIFT_PDL
#define LIFT_PDL 1  // launch with programmatic stream serialization (common.cuh pdl_wait)
#endif

// Launch `k` on `s`; with LIFT_PDL the launch may overlap the previous kernel's drain
// (every lift kernel starts with pdl_wait()).
template <typename... KArgs, typename... Args>
void launch(void (*k)(KArgs...), int64_t grid, int block, size_t smem, cudaStream_t s,
            Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = LIFT_PDL ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

thread_local cudaError_t g_last_cuda = cudaSuccess;  // the last failed launch of this thread

lift_status launched() {
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return LIFT_OK;
    g_last_cuda = e;
    return LIFT_ERR_CUDA;
}

// Workspace layout for a buffer of W bytes (W floored to 16):
//   [chunk partials f64 x nc][group partials f64 x ng] ... [tickets u32, last R(W) bytes]
// The ticket region depends on W ONLY, so every call made on the same buffer (with the
// same ws_bytes) agrees where the tickets live, and no call's partials ever overlap any
// call's tickets — the tickets stay zero across calls of different n (the contract's
// "zero-fill once").  R(W) holds W/512 + 2 tickets, enough for the largest n that fits.
inline size_t ticket_region(size_t wf) { return ((wf / 512 + 2) * 4 + 15) & ~(size_t)15; }

struct WsLayout {
    int64_t nc, ng;
    size_t partial_bytes;
};
WsLayout ws_layout(int64_t n) {
    WsLayout L;
    L.nc = (n + RED_C - 1) / RED_C;
    L.ng = (L.nc + RED_G - 1) / RED_G;
    L.partial_bytes = 8 * (size_t)(L.nc + L.ng);
    return L;
}
bool ws_fits(const WsLayout& L, size_t wbytes) {
    const size_t wf = wbytes & ~(size_t)15;
    const size_t r = ticket_region(wf);
    return wf >= r && wf - r >= L.partial_bytes && (size_t)(L.ng + 1) * 4 <= r;
}
size_t ws_bytes_for(int64_t n) {
    const WsLayout L = ws_layout(n);
    size_t w = (L.partial_bytes + L.partial_bytes / 127 + 32 + 15) & ~(size_t)15;
    while (!ws_fits(L, w)) w += 16;
    return w;
}

struct XchgArgs {  // NEXT-1: in-kernel cross-GPU combine (all null: single GPU)
    void* const* peers = nullptr;
    int p = 1, rank = 0;
    unsigned long long epoch = 0;
    int* error = nullptr;
};

#ifndef LIFT_REDUCE_REALIGN
#define LIFT_REDUCE_REALIGN 1  // 4-byte-aligned asum/dot operands: realigned 256-bit loads
#endif

// One launch of reduce_kernel (the 128-/256-bit classes; DESC: chunks visited in
// descending order, reduce.cuh).
// First-wave stagger (common.cuh first_wave_stagger): LIFT_VAR_STAGGER = 0 auto
// (LIFT_STAGGER_NS ns per 32 KiB a CTA reads where `auto_on`), 1 off, v >= 2: v ns per
// 32 KiB.  Applies when every unit has its own CTA and the units outnumber the resident CTA
// slots.  Measured (scripts/gpu_r2_stagger.sh, 0 / 2 / 3 / 4 / 6 ns): asum 2^24 14.6 -> 13.6,
// dot 2^24 23.8 -> 22.7, asum 2^28 149.8 -> 148.9, dot 2^26 77.0 -> 76.4, gemv 8192^2 (x in
// shared memory) 40.6 -> 39.8 us; the gemv x-through-L1 path lost (8192 x 16384 78.2 -> 78.7,
// 4096^2 14.2 -> 14.3), so auto leaves it off there.
#ifndef LIFT_STAGGER_NS
#define LIFT_STAGGER_NS 2
#endif
struct Stagger {
    int64_t resident = 0;
    unsigned ns = 0;
};
inline Stagger stagger_for(int64_t grid, int64_t units, const void* fn, int threads, size_t smem,
                           int64_t bytes_per_cta, bool auto_on = true) {
    Stagger st;
    const int v = var(LIFT_VAR_STAGGER);
    const int64_t per32k = v == 0 ? (auto_on ? LIFT_STAGGER_NS : 0) : v == 1 ? 0 : v;
    if (per32k == 0 || grid != units) return st;
    const int64_t r = (int64_t)sm_count(current_device()) * occupancy(fn, threads, smem);
    if (r >= units) return st;
    st.resident = r;
    st.ns = (unsigned)((per32k * bytes_per_cta + 16384) / 32768);
    return st;
}

template <class Op, int LW, int B, bool DESC>
lift_status reduce_go(ReduceArgs a, int64_t nc, cudaStream_t stream) {
    const size_t tsm = (LIFT_RED_TMA && !Op::kMapStore) ? (size_t)RED_C * 4 * (Op::kTwoInputs ? 2 : 1) : 0;
    const void* fn = (const void*)reduce_kernel<Op, LW, B, DESC>;
    const int64_t grid = grid_for(nc, fn, RED_T, tsm, LIFT_PERSISTENT);
    const Stagger st = stagger_for(grid, nc, fn, RED_T, tsm, (int64_t)RED_C * 4 * (Op::kTwoInputs ? 2 : 1));
    a.resident = st.resident;
    a.stagger_ns = st.ns;
    launch(reduce_kernel<Op, LW, B, DESC>, grid, RED_T, tsm, stream, a);
    return launched();
}

template <class Op, int B>
lift_status reduce_launch(int64_t n, const float* x, const float* y, float* out32, double* out64,
                          void* ws, size_t ws_bytes, cudaStream_t stream, float alpha = 0.f,
                          float* map_out = nullptr, const XchgArgs& xa = XchgArgs()) {
    if (n < 0) return LIFT_ERR_INVALID_VALUE;
    if (!out32 && !out64) return LIFT_ERR_NULL_POINTER;
    if (n > 0 && (!x || (Op::kTwoInputs && !y) || !ws || (Op::kMapStore && !map_out)))
        return LIFT_ERR_NULL_POINTER;
    if (Op::kMapStore && misaligned4(map_out)) return LIFT_ERR_INVALID_VALUE;
    if (misaligned4(x) || (Op::kTwoInputs && misaligned4(y)) || misaligned4(out32) ||
        (reinterpret_cast<uintptr_t>(out64) & 7))
        return LIFT_ERR_INVALID_VALUE;
    if (n == 0 && xa.peers) {  // still publish (+0) and combine with the other ranks
        ReduceArgs a{};
        a.out_f32 = out32;
        a.out_f64 = out64;
        a.peers = xa.peers;
        a.p = xa.p;
        a.rank = xa.rank;
        a.epoch = xa.epoch;
        a.error = xa.error;
        launch(xchg_only_kernel, 1, 32, 0, stream, a);
        return launched();
    }
    if (n == 0) {  // reduce over an empty array yields z = +0; no map
        if (out32 && cudaMemsetAsync(out32, 0, sizeof(float), stream) != cudaSuccess)
            return LIFT_ERR_CUDA;
        if (out64 && cudaMemsetAsync(out64, 0, sizeof(double), stream) != cudaSuccess)
            return LIFT_ERR_CUDA;
        return LIFT_OK;
    }
    const WsLayout L = ws_layout(n);
    if (!ws_fits(L, ws_bytes) || (reinterpret_cast<uintptr_t>(ws) & 15)) return LIFT_ERR_WORKSPACE;
    const size_t wf = ws_bytes & ~(size_t)15;

    ReduceArgs a{};
    a.n = n;
    a.x = x;
    a.y = y;
    a.nc = L.nc;
    a.ng = L.ng;
    a.tick = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + wf - ticket_region(wf));
    a.chunk_part = reinterpret_cast<double*>(ws);
    a.group_part = a.chunk_part + L.nc;
    a.out_f32 = out32;
    a.out_f64 = out64;
    a.alpha = alpha;
    a.map_out = map_out;
    a.peers = xa.peers;
    a.p = xa.p;
    a.rank = xa.rank;
    a.epoch = xa.epoch;
    a.error = xa.error;
    {
        const int pf = var(LIFT_VAR_PREFETCH);
        a.prefetch = pf == 2 || (pf == 0 && Op::kMapStore);
    }
    const int ord = var(LIFT_VAR_ORDER);
    const bool desc = ord == 2 || (ord == 0 && !Op::kMapStore);

    uintptr_t al = reinterpret_cast<uintptr_t>(x);
    if (Op::kTwoInputs) al |= reinterpret_cast<uintptr_t>(y);
    if (Op::kMapStore) al |= reinterpret_cast<uintptr_t>(map_out);
    int lw = align_class(al);
    if constexpr (!Op::kMapStore) {
        // realigned 256-bit blocks (common.cuh); not when the variant caps the width
        if (lw == 1 && LIFT_REDUCE_REALIGN && !lw_capped()) lw = 2;
    }
    lw = lw == 2 ? 2 : cap_lw(lw);
    if (desc && lw == 8) return reduce_go<Op, 8, B, true>(a, L.nc, stream);
    if (desc && lw == 4) return reduce_go<Op, 4, B, true>(a, L.nc, stream);
    const void* fn = lw == 8 ? (const void*)reduce_kernel<Op, 8, B>
                   : lw == 4 ? (const void*)reduce_kernel<Op, 4, B>
                   : lw == 2 ? (const void*)reduce_kernel<Op, Op::kMapStore ? 1 : 2, B>
                             : (const void*)reduce_kernel<Op, 1, B>;
    // NEXT-4 TMA variant: the chunk buffers are dynamic shared memory
    const size_t tsm = (LIFT_RED_TMA && lw >= 4 && !Op::kMapStore)
                           ? (size_t)RED_C * 4 * (Op::kTwoInputs ? 2 : 1) : 0;
    const int64_t grid = grid_for(L.nc, fn, RED_T, tsm, LIFT_PERSISTENT);
    const Stagger st = stagger_for(grid, L.nc, fn, RED_T, tsm, (int64_t)RED_C * 4 * (Op::kTwoInputs ? 2 : 1));
    a.resident = st.resident;
    a.stagger_ns = st.ns;
    if (lw == 8) launch(reduce_kernel<Op, 8, B>, grid, RED_T, tsm, stream, a);
    else if (lw == 4) launch(reduce_kernel<Op, 4, B>, grid, RED_T, tsm, stream, a);
    else if (lw == 2) launch(reduce_kernel<Op, Op::kMapStore ? 1 : 2, B>, grid, RED_T, 0, stream, a);
    else launch(reduce_kernel<Op, 1, B>, grid, RED_T, 0, stream, a);
    return launched();
}

#ifndef LIFT_SCAL_SMEM
#define LIFT_SCAL_SMEM 0  // (A/B knob) dynamic smem reserved per CTA: caps resident CTAs per SM
#endif

template <int LW, bool ALIAS>
void scal_go(int64_t grid, int64_t nslots, int head, int tail, float alpha, const float* x,
             float* y, cudaStream_t s) {
    const int pf = var(LIFT_VAR_PREFETCH);
    constexpr int64_t TILE = (int64_t)SCAL_T * SCAL_U;  // slots per tile
    const Stagger st = stagger_for(grid, (nslots + TILE - 1) / TILE, (const void*)scal_kernel<LW, ALIAS>,
                                   SCAL_T, LIFT_SCAL_SMEM, TILE * 64, false);
    launch(scal_kernel<LW, ALIAS>, grid, SCAL_T, LIFT_SCAL_SMEM, s, nslots, head, tail, alpha, x, y,
           pf == 1 ? 0 : 1, st.resident, st.ns);
}

template <int LW>
const void* scal_fn(bool alias) {
    return alias ? (const void*)scal_kernel<LW, true> : (const void*)scal_kernel<LW, false>;
}

#ifndef LIFT_GEMV_REALIGN
#define LIFT_GEMV_REALIGN 1  // misaligned rows: realigned 256-bit loads + lane shuffles
#endif

template <int TRL, int LW, bool PEERS>
lift_status gemv_go(GemvArgs a, cudaStream_t s) {
    constexpr int64_t rp = GEMV_T >> TRL;  // rows per block
    a.nblocks = (a.m + rp - 1) / rp;
    const void* fn = (const void*)gemv_kernel<TRL, LW, PEERS>;
    const int64_t grid = grid_for(a.nblocks, fn, GEMV_T, 0, LIFT_PERSISTENT);
    const int dev = current_device();
    const int pf = var(LIFT_VAR_PREFETCH);
    a.prefetch = pf == 2 || (pf == 0 && a.nblocks >= 4 * (int64_t)sm_count(dev) * occupancy(fn, GEMV_T, 0));
    const Stagger st = stagger_for(grid, a.nblocks, fn, GEMV_T, 0, rp * a.n * 4, false);
    a.resident = st.resident;
    a.stagger_ns = st.ns;
    launch(gemv_kernel<TRL, LW, PEERS>, grid, GEMV_T, 0, s, a);
    return launched();
}

template <int TRL, int LW>
lift_status gxsm_go(GemvArgs a, cudaStream_t s) {
    constexpr int64_t rp = GEMV_T >> TRL;  // rows per block
    a.nblocks = (a.m + rp - 1) / rp;
    const size_t smem = (size_t)a.n * 4;
    const void* fn = (const void*)gemv_kernel<TRL, LW, false, true>;
    const int64_t grid = grid_for(a.nblocks, fn, GEMV_T, smem, LIFT_PERSISTENT);
    const int pf = var(LIFT_VAR_PREFETCH);
    a.prefetch = pf == 2 || (pf == 0 && a.nblocks >= 4 * (int64_t)sm_count(current_device()) *
                                                         occupancy(fn, GEMV_T, smem));
    const Stagger st = stagger_for(grid, a.nblocks, fn, GEMV_T, smem, rp * a.n * 4);
    a.resident = st.resident;
    a.stagger_ns = st.ns;
    launch(gemv_kernel<TRL, LW, false, true>, grid, GEMV_T, smem, s, a);
    return launched();
}

template <int TRL, bool PEERS>
lift_status gemv_lw(const GemvArgs& a, int lw, cudaStream_t s) {
    if (lw == 2) return gemv_go<TRL, 2, PEERS>(a, s);
    if (lw == 3) return gemv_go<TRL, 3, PEERS>(a, s);
    return lw == 8 ? gemv_go<TRL, 8, PEERS>(a, s)
         : lw == 4 ? gemv_go<TRL, 4, PEERS>(a, s) : gemv_go<TRL, 1, PEERS>(a, s);
}

template <bool PEERS>
lift_status gemv_trl(const GemvArgs& a, int lw, cudaStream_t s) {
    switch (gemv_tr_log2(a.n)) {  // threads per row: part of the canonical order (n only)
        case 8: return gemv_lw<8, PEERS>(a, lw, s);
        case 7: return gemv_lw<7, PEERS>(a, lw, s);
        case 6: return gemv_lw<6, PEERS>(a, lw, s);
        case 5: return gemv_lw<5, PEERS>(a, lw, s);
        case 4: return gemv_lw<4, PEERS>(a, lw, s);
        case 3: return gemv_lw<3, PEERS>(a, lw, s);
        case 2: return gemv_lw<2, PEERS>(a, lw, s);
        case 1: return gemv_lw<1, PEERS>(a, lw, s);
        default: return gemv_lw<0, PEERS>(a, lw, s);
    }
}

#ifndef LIFT_GXS_AUTO
#define LIFT_GXS_AUTO 0  // auto never picks the staged-x kernel: slower at every measured shape
#endif                   // (DESIGN.md §6); LIFT_VAR_GEMV_X = 2 selects it
inline bool gxs_auto(int64_t, int64_t) { return LIFT_GXS_AUTO != 0; }

template <int TRL, int LW, bool PEERS>
lift_status gxs_go(GemvArgs a, cudaStream_t s) {
    constexpr int64_t rp = GXS_T >> TRL;  // rows per block
    a.nblocks = (a.m + rp - 1) / rp;
    const size_t smem = gxs_smem_bytes(a.n);
    const void* fn = (const void*)gemv_xs_kernel<TRL, LW, PEERS>;
    // CLC stealing: the grid covers every block (resident CTAs take the rest)
    const int64_t grid = grid_for(a.nblocks, fn, GXS_T, smem, false, true);
    launch(gemv_xs_kernel<TRL, LW, PEERS>, grid, GXS_T, smem, s, a);
    return launched();
}

template <int TRL, bool PEERS>
lift_status gtm_go(GemvArgs a, int nst, cudaStream_t s) {
    constexpr int64_t rb = (GTM_CT >> TRL) * GTM_R;  // rows per block
    a.nblocks = (a.m + rb - 1) / rb;
    const size_t smem = gtm_smem_bytes(a.n, nst);
    const void* fn = (const void*)gemv_tma_kernel<TRL, PEERS>;
    const int64_t grid = grid_for(a.nblocks, fn, GTM_T, smem, false, true);
    launch(gemv_tma_kernel<TRL, PEERS>, grid, GTM_T, smem, s, a, nst);
    return launched();
}

template <bool PEERS>
lift_status gtm_trl(const GemvArgs& a, int nst, cudaStream_t s) {
    switch (gemv_tr_log2(a.n)) {  // n >= 2048: 32..256 threads per row
        case 8: return gtm_go<8, PEERS>(a, nst, s);
        case 7: return gtm_go<7, PEERS>(a, nst, s);
        case 6: return gtm_go<6, PEERS>(a, nst, s);
        default: return gtm_go<5, PEERS>(a, nst, s);
    }
}

template <int TRL, int LW>
lift_status gr2_go(GemvArgs a, cudaStream_t s) {
    constexpr int T = gr2_threads(TRL);
    constexpr int64_t rb = 2 * (T >> TRL);  // rows per block
    a.nblocks = (a.m + rb - 1) / rb;
    const void* fn = (const void*)gemv_r2_kernel<TRL, LW>;
    const int64_t grid = grid_for(a.nblocks, fn, T, 0, LIFT_PERSISTENT);
    const int pf = var(LIFT_VAR_PREFETCH);
    a.prefetch = pf == 2 || (pf == 0 && a.nblocks >= 4 * (int64_t)sm_count(current_device()) *
                                                         occupancy(fn, T, 0));
    launch(gemv_r2_kernel<TRL, LW>, grid, T, 0, s, a);
    return launched();
}

lift_status gr2_trl(const GemvArgs& a, int lw, cudaStream_t s) {
    switch (gemv_tr_log2(a.n)) {  // n >= 2048: 32..256 threads per row
        case 8: return lw == 8 ? gr2_go<8, 8>(a, s) : gr2_go<8, 4>(a, s);
        case 7: return lw == 8 ? gr2_go<7, 8>(a, s) : gr2_go<7, 4>(a, s);
        case 6: return lw == 8 ? gr2_go<6, 8>(a, s) : gr2_go<6, 4>(a, s);
        default: return lw == 8 ? gr2_go<5, 8>(a, s) : gr2_go<5, 4>(a, s);
    }
}

int smem_optin(int dev) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
}

template <bool PEERS>
lift_status gxs_trl(const GemvArgs& a, int lw, cudaStream_t s) {
    switch (gemv_tr_log2(a.n)) {  // n >= GXS_NMIN: 32..256 threads per row
        case 8: return lw == 8 ? gxs_go<8, 8, PEERS>(a, s) : gxs_go<8, 4, PEERS>(a, s);
        case 7: return lw == 8 ? gxs_go<7, 8, PEERS>(a, s) : gxs_go<7, 4, PEERS>(a, s);
        case 6: return lw == 8 ? gxs_go<6, 8, PEERS>(a, s) : gxs_go<6, 4, PEERS>(a, s);
        default: return lw == 8 ? gxs_go<5, 8, PEERS>(a, s) : gxs_go<5, 4, PEERS>(a, s);
    }
}

// Split-path workspace bytes for (m, n): partials + a ticket region of a third of W.
size_t gemv_ws_bytes_for(int64_t m, int64_t n) {
    if (n < GEMV_LONG_N || m <= 0) return 0;
    const int64_t nc = (n + RED_C - 1) / RED_C, ng = (nc + RED_G - 1) / RED_G;
    const size_t part = 8 * (size_t)m * (size_t)(nc + ng);
    const size_t tick = 4 * (size_t)m * (size_t)(ng + 1);
    size_t w = (part + part / 2 + 64 + 15) & ~(size_t)15;
    while (w - gemv_ws_ticket_region(w) < part || gemv_ws_ticket_region(w) < tick) w += 16;
    return w;
}

template <int LW>
lift_status gemv_split_go(const GemvArgs& a, void* ws, size_t ws_bytes, cudaStream_t s) {
    GemvSplitArgs sa{};
    sa.g = a;
    sa.nc = (a.n + RED_C - 1) / RED_C;
    sa.ng = (sa.nc + RED_G - 1) / RED_G;
    const size_t wf = ws_bytes & ~(size_t)15;
    sa.chunk_part = static_cast<double*>(ws);
    sa.group_part = sa.chunk_part + a.m * sa.nc;
    sa.tick = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + wf - gemv_ws_ticket_region(wf));
    const int64_t grid = grid_for(a.m * sa.nc, (const void*)gemv_split_kernel<LW>, RED_T, 0,
                                  LIFT_PERSISTENT);
    launch(gemv_split_kernel<LW>, grid, RED_T, 0, s, sa);
    return launched();
}

template <int LW, bool PEERS>
lift_status gemv_long_go(GemvArgs a, cudaStream_t s) {
    a.nblocks = a.m;
    const int64_t grid = grid_for(a.m, (const void*)gemv_long_kernel<LW, PEERS>, RED_T, 0,
                                  LIFT_PERSISTENT);
    launch(gemv_long_kernel<LW, PEERS>, grid, RED_T, 0, s, a);
    return launched();
}

lift_status gemv_launch(const GemvArgs& a, cudaStream_t s, void* ws = nullptr,
                        size_t ws_bytes = 0) {
    // the widest load class that A's rows (base + lda) and x all allow; the order of the
    // arithmetic does not depend on it (gemv.cuh)
    const uintptr_t al = reinterpret_cast<uintptr_t>(a.A) | reinterpret_cast<uintptr_t>(a.x);
    int lw = cap_lw(((al & 31) == 0 && a.lda % 8 == 0) ? 8 : ((al & 15) == 0 && a.lda % 4 == 0) ? 4 : 1);
    if (a.n >= GEMV_LONG_N) {  // long rows: the stand-alone dot's order (gemv_long.cuh)
        // few rows cannot fill the GPU with one CTA each: split them over (row, chunk)
        // CTAs when the caller gave a workspace large enough
        const bool split = !a.y_peers && ws && (reinterpret_cast<uintptr_t>(ws) & 15) == 0 &&
                           a.m < 4 * (int64_t)sm_count(current_device()) &&
                           ws_bytes >= gemv_ws_bytes_for(a.m, a.n);
        if (split)
            return lw == 8 ? gemv_split_go<8>(a, ws, ws_bytes, s)
                 : lw == 4 ? gemv_split_go<4>(a, ws, ws_bytes, s) : gemv_split_go<1>(a, ws, ws_bytes, s);
        if (a.y_peers)
            return lw == 8 ? gemv_long_go<8, true>(a, s)
                 : lw == 4 ? gemv_long_go<4, true>(a, s) : gemv_long_go<1, true>(a, s);
        return lw == 8 ? gemv_long_go<8, false>(a, s)
             : lw == 4 ? gemv_long_go<4, false>(a, s) : gemv_long_go<1, false>(a, s);
    }
    // G1 toLocal(x): rows of GXS_NMIN..GXS_NMAX columns that split evenly over their
    // threads, aligned, and enough of them to amortise one x staging per resident CTA
    // (gemv_xs.cuh)
    const int gx = var(LIFT_VAR_GEMV_X);
    if (gx == 4 && lw >= 4 && !a.y_peers && gr2_shape_ok(a.n))  // two rows per thread
        return gr2_trl(a, lw, s);
    // x bulk-copied into shared memory per CTA (gemv_kernel XS): with many waves of blocks
    // the first batch's four A loads go out at once (x holds no registers across the DRAM
    // wait): 8192^2 42.3 -> 40.7 us, 16384 x 8192 79.6 -> 76.8 us; with few waves the extra
    // x traffic per CTA costs more than it saves (4096^2 13.6 -> 14.2 us), so auto requires
    // >= 4 waves
    bool xs = gx == 5;
    if (gx == 0 && lw >= 4 && !a.y_peers && a.n >= 2048 && a.n <= 12288 && a.n % 4 == 0) {
        const int trl = gemv_tr_log2(a.n);
        const int64_t nb = (a.m + (GEMV_T >> trl) - 1) / (GEMV_T >> trl);
        xs = nb >= 4 * (int64_t)sm_count(current_device()) * GEMV_MINB;
    }
    if (xs && lw >= 4 && !a.y_peers && a.n >= 1024 && a.n <= 12288 && a.n % 4 == 0) {
        switch (gemv_tr_log2(a.n)) {  // x bulk-copied into shared memory per CTA
            case 8: return lw == 8 ? gxsm_go<8, 8>(a, s) : gxsm_go<8, 4>(a, s);
            case 7: return lw == 8 ? gxsm_go<7, 8>(a, s) : gxsm_go<7, 4>(a, s);
            case 6: return lw == 8 ? gxsm_go<6, 8>(a, s) : gxsm_go<6, 4>(a, s);
            default: return lw == 8 ? gxsm_go<5, 8>(a, s) : gxsm_go<5, 4>(a, s);
        }
    }
    if (gx == 3 && lw >= 4 && gtm_shape_ok(a.n)) {  // TMA ring (gemv_tma.cuh)
        const int nst = gtm_stages(a.n, (size_t)smem_optin(current_device()));
        if (nst >= 2) return a.y_peers ? gtm_trl<true>(a, nst, s) : gtm_trl<false>(a, nst, s);
    }
    if (lw >= 4 && gxs_shape_ok(a.n) && (gx == 2 || (gx == 0 && gxs_auto(a.m, a.n))))
        return a.y_peers ? gxs_trl<true>(a, lw, s) : gxs_trl<false>(a, lw, s);
    // rows and/or x at arbitrary 4-byte alignment: realigned 256-bit loads (common.cuh);
    // 2 = rows only (x 32-byte aligned), 3 = rows and x
    if (lw == 1 && LIFT_GEMV_REALIGN && !lw_capped())
        lw = (reinterpret_cast<uintptr_t>(a.x) & 31) == 0 ? 2 : 3;
    return a.y_peers ? gemv_trl<true>(a, lw, s) : gemv_trl<false>(a, lw, s);
}

}  // namespace
}  // namespace lift

using namespace lift;

extern "C" {

int lift_abi_version(void) { return LIFT_ABI_VERSION; }

int64_t lift_reduce_chunk_elems(void) { return RED_C; }
int lift_reduce_group_chunks(void) { return RED_G; }

const char* lift_status_string(lift_status s) {
    switch (s) {
        case LIFT_OK: return "LIFT_OK";
        case LIFT_ERR_INVALID_VALUE: return "LIFT_ERR_INVALID_VALUE: bad length, stride or alignment";
        case LIFT_ERR_NULL_POINTER: return "LIFT_ERR_NULL_POINTER: required pointer is NULL";
        case LIFT_ERR_WORKSPACE: return "LIFT_ERR_WORKSPACE: workspace too small or misaligned";
        case LIFT_ERR_CUDA: return "LIFT_ERR_CUDA: kernel launch failed";
    }
    return "LIFT_ERR_UNKNOWN";
}

const char* lift_last_cuda_error(void) {
    return g_last_cuda == cudaSuccess ? "no error" : cudaGetErrorString(g_last_cuda);
}

size_t lift_workspace_bytes(int64_t n) { return ws_bytes_for(n < 0 ? 0 : n); }

lift_status lift_workspace_check(const void* ws, size_t ws_bytes, lift_stream_t stream) {
    if (!ws) return LIFT_ERR_NULL_POINTER;
    if (reinterpret_cast<uintptr_t>(ws) & 15) return LIFT_ERR_INVALID_VALUE;
    const size_t wf = ws_bytes & ~(size_t)15;
    const size_t r = ticket_region(wf);
    if (wf < r) return LIFT_ERR_WORKSPACE;
    std::vector<unsigned> h(r / 4);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(h.data(), static_cast<const char*>(ws) + (wf - r), r,
                                    cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        g_last_cuda = e;
        return LIFT_ERR_CUDA;
    }
    for (unsigned v : h)
        if (v) return LIFT_ERR_WORKSPACE;
    return LIFT_OK;
}

lift_status lift_set_variant(lift_variant knob, int value) {
    if ((int)knob < 0 || (int)knob >= LIFT_VAR_COUNT) return LIFT_ERR_INVALID_VALUE;
    bool ok = false;
    switch (knob) {
        case LIFT_VAR_LOAD_WIDTH: ok = value == 0 || value == 1 || value == 4 || value == 8; break;
        case LIFT_VAR_GEMV_X: ok = value >= 0 && value <= 5; break;
        case LIFT_VAR_PREFETCH: ok = value >= 0 && value <= 2; break;
        case LIFT_VAR_ORDER: ok = value >= 0 && value <= 2; break;
        case LIFT_VAR_STAGGER: ok = value >= 0 && value <= 64; break;
        default: break;
    }
    if (!ok) return LIFT_ERR_INVALID_VALUE;
    g_var[knob].store(value);
    return LIFT_OK;
}

int lift_get_variant(lift_variant knob) {
    if ((int)knob < 0 || (int)knob >= LIFT_VAR_COUNT) return -1;
    return var(knob);
}

lift_status lift_debug_set_grid_limit(int max_ctas) {
    if (max_ctas < 0) return LIFT_ERR_INVALID_VALUE;
    g_grid_limit.store(max_ctas);
    return LIFT_OK;
}

lift_status lift_scal(int64_t n, float alpha, const float* x, float* y, lift_stream_t stream) {
    if (n < 0) return LIFT_ERR_INVALID_VALUE;
    if (n == 0) return LIFT_OK;
    if (!x || !y) return LIFT_ERR_NULL_POINTER;
    if (misaligned4(x) || misaligned4(y)) return LIFT_ERR_INVALID_VALUE;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const uintptr_t ax = reinterpret_cast<uintptr_t>(x), ay = reinterpret_cast<uintptr_t>(y);
    const int lw = cap_lw(align_class(ax - ay));  // relative phase of x and y
    const uintptr_t boundary = (uintptr_t)lw * 4;
    int64_t head = (int64_t)(((boundary - (ax % boundary)) % boundary) / 4);
    if (head > n) head = n;
    const int64_t body = n - head;
    const int64_t nslots = body / 8;
    const int tail = (int)(body % 8);
    const bool alias = (x == y);
    const void* fn = lw == 8 ? scal_fn<8>(alias) : lw == 4 ? scal_fn<4>(alias) : scal_fn<1>(alias);
    if (LIFT_SCAL_TMA && lw >= 4) {  // NEXT-4 TMA bulk variant (compile-time)
        const int64_t tiles = (8 * nslots + SCAL_TMA_TILE - 1) / SCAL_TMA_TILE;
        const int64_t grid = grid_for(tiles, (const void*)scal_tma_kernel, SCAL_TMA_T, 0, false);
        launch(scal_tma_kernel, grid, SCAL_TMA_T, 0, s, nslots, (int)head, tail, alpha, x, y);
        return launched();
    }
    const int64_t tile = (int64_t)SCAL_T * SCAL_U;
    const int64_t grid = grid_for((nslots + tile - 1) / tile, fn, SCAL_T, LIFT_SCAL_SMEM, LIFT_PERSISTENT);
    if (lw == 8) alias ? scal_go<8, true>(grid, nslots, (int)head, tail, alpha, x, y, s)
                       : scal_go<8, false>(grid, nslots, (int)head, tail, alpha, x, y, s);
    else if (lw == 4) alias ? scal_go<4, true>(grid, nslots, (int)head, tail, alpha, x, y, s)
                            : scal_go<4, false>(grid, nslots, (int)head, tail, alpha, x, y, s);
    else alias ? scal_go<1, true>(grid, nslots, (int)head, tail, alpha, x, y, s)
               : scal_go<1, false>(grid, nslots, (int)head, tail, alpha, x, y, s);
    return launched();
}

lift_status lift_asum(int64_t n, const float* x, float* result, void* ws, size_t ws_bytes,
                      lift_stream_t stream) {
    if (!result) return LIFT_ERR_NULL_POINTER;
    return reduce_launch<AsumOp<LIFT_ASUM_ACC>, LIFT_ASUM_B>(n, x, nullptr, result, nullptr, ws, ws_bytes,
                                              reinterpret_cast<cudaStream_t>(stream));
}

lift_status lift_dot(int64_t n, const float* x, const float* y, float* result, void* ws,
                     size_t ws_bytes, lift_stream_t stream) {
    if (!result) return LIFT_ERR_NULL_POINTER;
    return reduce_launch<DotOp<LIFT_DOT_ACC>, LIFT_DOT_B>(n, x, y, result, nullptr, ws, ws_bytes,
                                            reinterpret_cast<cudaStream_t>(stream));
}

lift_status lift_asum_partial(int64_t n, const float* x, double* partial, void* ws,
                              size_t ws_bytes, lift_stream_t stream) {
    if (!partial) return LIFT_ERR_NULL_POINTER;
    return reduce_launch<AsumOp<LIFT_ASUM_ACC>, LIFT_ASUM_B>(n, x, nullptr, nullptr, partial, ws, ws_bytes,
                                              reinterpret_cast<cudaStream_t>(stream));
}

lift_status lift_dot_partial(int64_t n, const float* x, const float* y, double* partial,
                             void* ws, size_t ws_bytes, lift_stream_t stream) {
    if (!partial) return LIFT_ERR_NULL_POINTER;
    return reduce_launch<DotOp<LIFT_DOT_ACC>, LIFT_DOT_B>(n, x, y, nullptr, partial, ws, ws_bytes,
                                            reinterpret_cast<cudaStream_t>(stream));
}

lift_status lift_scal_asum(int64_t n, float alpha, const float* x, float* y, float* result,
                           void* ws, size_t ws_bytes, lift_stream_t stream) {
    if (!result) return LIFT_ERR_NULL_POINTER;
    if (n > 0 && x && y && x == y) return LIFT_ERR_INVALID_VALUE;  // x is read on the .nc path
    return reduce_launch<ScalAsumOp<LIFT_ASUM_ACC>, LIFT_ASUM_B>(
        n, x, nullptr, result, nullptr, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), alpha,
        y);
}

size_t lift_xchg_bytes(int p) {
    return p < 1 ? 0 : (size_t)2 * p * sizeof(XchgSlot) + 2 * sizeof(unsigned long long);
}

lift_status lift_xchg_create(int p, void** buf) {
    if (p < 1 || p > 32) return LIFT_ERR_INVALID_VALUE;
    if (!buf) return LIFT_ERR_NULL_POINTER;
    void* d = nullptr;
    if (cudaMalloc(&d, lift_xchg_bytes(p)) != cudaSuccess) return LIFT_ERR_CUDA;
    if (cudaMemset(d, 0, lift_xchg_bytes(p)) != cudaSuccess) {
        cudaFree(d);
        return LIFT_ERR_CUDA;
    }
    *buf = d;
    return LIFT_OK;
}

lift_status lift_ipc_alloc(size_t bytes, void** buf) {
    if (!buf) return LIFT_ERR_NULL_POINTER;
    if (bytes == 0) return LIFT_ERR_INVALID_VALUE;
    void* d = nullptr;
    if (cudaMalloc(&d, bytes) != cudaSuccess) return LIFT_ERR_CUDA;
    *buf = d;
    return LIFT_OK;
}

lift_status lift_xchg_destroy(void* buf) {
    if (!buf) return LIFT_OK;
    return cudaFree(buf) == cudaSuccess ? LIFT_OK : LIFT_ERR_CUDA;
}

lift_status lift_ipc_get_handle(const void* buf, void* handle) {
    if (!buf || !handle) return LIFT_ERR_NULL_POINTER;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, const_cast<void*>(buf)) != cudaSuccess) return LIFT_ERR_CUDA;
    static_assert(sizeof(h) == LIFT_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(handle, &h, sizeof(h));
    return LIFT_OK;
}

lift_status lift_ipc_open_handle(const void* handle, void** ptr) {
    if (!handle || !ptr) return LIFT_ERR_NULL_POINTER;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    if (cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return LIFT_ERR_CUDA;
    return LIFT_OK;
}

lift_status lift_ipc_close_handle(void* ptr) {
    if (!ptr) return LIFT_OK;
    return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? LIFT_OK : LIFT_ERR_CUDA;
}

static lift_status xchg_check(void* const* peers, int p, int rank, unsigned long long epoch,
                              XchgArgs& xa, int* error) {
    if (p < 1 || p > 32 || rank < 0 || rank >= p || epoch == 0) return LIFT_ERR_INVALID_VALUE;
    if (!peers) return LIFT_ERR_NULL_POINTER;
    xa.peers = peers;
    xa.p = p;
    xa.rank = rank;
    xa.epoch = epoch;
    xa.error = error;
    return LIFT_OK;
}

lift_status lift_asum_allreduce(int64_t n, const float* x, float* result, void* ws,
                                size_t ws_bytes, void* const* peers, int p, int rank,
                                unsigned long long epoch, int* error, lift_stream_t stream) {
    if (!result) return LIFT_ERR_NULL_POINTER;
    XchgArgs xa;
    const lift_status st = xchg_check(peers, p, rank, epoch, xa, error);
    if (st != LIFT_OK) return st;
    return reduce_launch<AsumOp<LIFT_ASUM_ACC>, LIFT_ASUM_B>(
        n, x, nullptr, result, nullptr, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), 0.f,
        nullptr, xa);
}

lift_status lift_dot_allreduce(int64_t n, const float* x, const float* y, float* result,
                               void* ws, size_t ws_bytes, void* const* peers, int p, int rank,
                               unsigned long long epoch, int* error, lift_stream_t stream) {
    if (!result) return LIFT_ERR_NULL_POINTER;
    XchgArgs xa;
    const lift_status st = xchg_check(peers, p, rank, epoch, xa, error);
    if (st != LIFT_OK) return st;
    return reduce_launch<DotOp<LIFT_DOT_ACC>, LIFT_DOT_B>(
        n, x, y, result, nullptr, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream), 0.f,
        nullptr, xa);
}

lift_status lift_combine(int p, const double* partials, float* result, lift_stream_t stream) {
    if (p < 1) return LIFT_ERR_INVALID_VALUE;
    if (!partials || !result) return LIFT_ERR_NULL_POINTER;
    if ((reinterpret_cast<uintptr_t>(partials) & 7) || misaligned4(result))
        return LIFT_ERR_INVALID_VALUE;
    launch(combine_kernel, 1, 32, 0, reinterpret_cast<cudaStream_t>(stream), p, partials, result);
    return launched();
}

lift_status lift_gemv_allgather(int64_t m, int64_t n, float alpha, const float* A, int64_t lda,
                                const float* x, float beta, const float* y, float* const* y_peers,
                                int64_t row0, void* const* xpeers, int p, int rank,
                                unsigned long long epoch, int* error, lift_stream_t stream) {
    if (m < 0 || n < 0 || row0 < 0) return LIFT_ERR_INVALID_VALUE;
    if (lda < (n > 1 ? n : 1)) return LIFT_ERR_INVALID_VALUE;
    if (p < 1 || p > 32 || rank < 0 || rank >= p || epoch == 0) return LIFT_ERR_INVALID_VALUE;
    if (!y_peers || !xpeers) return LIFT_ERR_NULL_POINTER;
    if (m == 0) return LIFT_ERR_INVALID_VALUE;  // every rank must contribute >= 1 row
    if (!y || (n > 0 && (!A || !x))) return LIFT_ERR_NULL_POINTER;
    if (misaligned4(A) || misaligned4(x) || misaligned4(y)) return LIFT_ERR_INVALID_VALUE;
    GemvArgs a{};
    a.m = m;
    a.n = n;
    a.lda = lda;
    a.alpha = alpha;
    a.beta = beta;
    a.A = A;
    a.x = x;
    a.y = y;
    a.y_out = nullptr;
    a.y_peers = y_peers;
    a.row0 = row0;
    a.xpeers = xpeers;
    a.p = p;
    a.rank = rank;
    a.epoch = epoch;
    a.error = error;
    return gemv_launch(a, reinterpret_cast<cudaStream_t>(stream));
}

lift_status lift_gemv(int64_t m, int64_t n, float alpha, const float* A, int64_t lda,
                      const float* x, float beta, const float* y, float* y_out,
                      lift_stream_t stream) {
    if (m < 0 || n < 0) return LIFT_ERR_INVALID_VALUE;
    if (lda < (n > 1 ? n : 1)) return LIFT_ERR_INVALID_VALUE;
    if (m == 0) return LIFT_OK;
    if (!y || !y_out || (n > 0 && (!A || !x))) return LIFT_ERR_NULL_POINTER;
    if (misaligned4(A) || misaligned4(x) || misaligned4(y) || misaligned4(y_out))
        return LIFT_ERR_INVALID_VALUE;
    GemvArgs a{};
    a.m = m;
    a.n = n;
    a.lda = lda;
    a.alpha = alpha;
    a.beta = beta;
    a.A = A;
    a.x = x;
    a.y = y;
    a.y_out = y_out;
    return gemv_launch(a, reinterpret_cast<cudaStream_t>(stream));
}

lift_status lift_gemv_ws(int64_t m, int64_t n, float alpha, const float* A, int64_t lda,
                         const float* x, float beta, const float* y, float* y_out, void* ws,
                         size_t ws_bytes, lift_stream_t stream) {
    if (m < 0 || n < 0) return LIFT_ERR_INVALID_VALUE;
    if (lda < (n > 1 ? n : 1)) return LIFT_ERR_INVALID_VALUE;
    if (m == 0) return LIFT_OK;
    if (!y || !y_out || (n > 0 && (!A || !x))) return LIFT_ERR_NULL_POINTER;
    if (misaligned4(A) || misaligned4(x) || misaligned4(y) || misaligned4(y_out))
        return LIFT_ERR_INVALID_VALUE;
    GemvArgs a{};
    a.m = m;
    a.n = n;
    a.lda = lda;
    a.alpha = alpha;
    a.beta = beta;
    a.A = A;
    a.x = x;
    a.y = y;
    a.y_out = y_out;
    return gemv_launch(a, reinterpret_cast<cudaStream_t>(stream), ws, ws_bytes);
}

size_t lift_gemv_workspace_bytes(int64_t m, int64_t n) {
    // the split path is only taken for rows too few to fill the GPU (gemv_launch)
    if (m >= 4 * (int64_t)sm_count(current_device())) return 0;
    return gemv_ws_bytes_for(m, n);
}

lift_status lift_blackscholes(int64_t n, const float* s, float K, float r, float v, float T,
                              float* call, float* put, lift_stream_t stream) {
    if (n < 0) return LIFT_ERR_INVALID_VALUE;
    if (!(K > 0.f) || !(v > 0.f) || !(T > 0.f) || !isfinite(r) || !isfinite(K) ||
        !isfinite(v) || !isfinite(T))
        return LIFT_ERR_INVALID_VALUE;
    if (n == 0) return LIFT_OK;
    if (!s || !call || !put) return LIFT_ERR_NULL_POINTER;
    if (misaligned4(s) || misaligned4(call) || misaligned4(put)) return LIFT_ERR_INVALID_VALUE;
    const uintptr_t as = reinterpret_cast<uintptr_t>(s), ac = reinterpret_cast<uintptr_t>(call),
                    ap = reinterpret_cast<uintptr_t>(put);
    // vector path needs s, call and put in the same 32-byte phase (then a common head)
    const bool same = ((as - ac) & 31) == 0 && ((as - ap) & 31) == 0;
    int64_t head = same ? (int64_t)(((32 - (as & 31)) & 31) / 4) : 0;
    if (head > n) head = n;
    const int64_t body = n - head;
    const int64_t nslots = body / 8;
    const int tail = (int)(body % 8);
    const double vs = (double)v * sqrt((double)T);
    const BsConst p{(float)(M_LN2 / vs),
                    (float)((((double)r + 0.5 * (double)v * v) * T - log((double)K)) / vs),
                    (float)vs, (float)(K * exp(-(double)r * T))};
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t tile = (int64_t)BS_T * BS_U;
    if (same) {
        const int64_t grid = grid_for((nslots + tile - 1) / tile, (const void*)blackscholes_kernel<8>,
                                      BS_T, 0, false);
        launch(blackscholes_kernel<8>, grid, BS_T, 0, st, nslots, (int)head, tail, s, call, put, p);
    } else {
        const int64_t grid = grid_for((nslots + tile - 1) / tile, (const void*)blackscholes_kernel<1>,
                                      BS_T, 0, false);
        launch(blackscholes_kernel<1>, grid, BS_T, 0, st, nslots, (int)head, tail, s, call, put, p);
    }
    return launched();
}

#ifdef LIFT_TRACE
int lift_trace_read(void* host, size_t bytes) {
    return cudaMemcpyFromSymbol(host, lift::g_trace, bytes) == cudaSuccess ? 0 : 4;
}
#endif

}  // extern "C"
