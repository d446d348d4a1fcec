/* lift.h — C ABI of liblift.so: the B200 (sm_100a) hot path of Steuwer, Fensch &
 * Dubach, "Patterns and Rewrite Rules for Systematic Code Generation"
 * (arXiv 1502.02389; /root/reference/PAPER.md cited as P:<line>).
 *
 * The four BLAS compositions of the paper's Fig. 8:
 *     scal(a, x)          = map(mult(a), x)
 *     asum(x)             = reduce(add, 0) o map(abs, x)
 *     dot(x, y)           = reduce(add, 0) o map(mult) o zip(x, y)
 *     gemv(A, x, y, a, b) = map(add) o zip(map(scal(a) o dot(x), A),
 *                                          scal(b, y))
 *   with abs(x) = if (x < 0) -x else x, add = +, mult = * (P:789-790),
 *   and gemv computing "y = alpha A x + beta y".
 *
 * General contract (every entry point):
 *  - Storage is fp32 (reading R1 in DESIGN.md: the paper's elements are 4 bytes,
 *    P:1077-1080).  All array pointers are DEVICE pointers of the stream's device (the
 *    current device for a NULL stream; the call switches to that device for its
 *    duration), at least 4-byte aligned; wider alignment only enables wider loads and
 *    never changes a result bit.
 *  - Every compute call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *    default stream): it validates its arguments on the host, enqueues exactly one
 *    kernel (none for empty work; a cudaMemsetAsync for an empty reduction) and
 *    returns.  It never synchronises, never allocates and never touches host copies of
 *    the data.  The exceptions are the one-time setup calls of the NEXT-1 exchange
 *    (lift_xchg_create/destroy, lift_ipc_*), which allocate, map or free synchronously,
 *    and the off-hot-path check lift_workspace_check, which waits for its stream.
 *    Results are stream-ordered in device
 *    memory; read them after your own sync.  A reduction's result is a 1-element
 *    device array, following the paper's "primitives are arrays of length 1"
 *     and reduce's type T[] -> T[1].
 *  - The caller owns every buffer, including the workspace and the exchange buffers
 *    (which lift_xchg_create allocates on the caller's behalf).  The library keeps no
 *    device memory and no mutable state except a per-device cache of the SM count
 *    and kernel occupancies, the process-global NEXT-4 strategy knobs
 *    (lift_set_variant; none changes a result bit) and the test hook
 *    lift_debug_set_grid_limit.
 *  - Errors are returned synchronously and nothing is launched:
 *      LIFT_ERR_INVALID_VALUE  n, m < 0; lda < max(1, n); p < 1; a pointer that is
 *                              not 4-byte aligned;
 *      LIFT_ERR_NULL_POINTER   a required pointer is NULL while the length is > 0;
 *      LIFT_ERR_WORKSPACE      ws too small for n (see lift_workspace_bytes) or ws not
 *                              16-B aligned;
 *      LIFT_ERR_CUDA           the launch itself failed (cudaGetLastError).
 *    Faults inside a kernel surface at the caller's next synchronisation.
 *  - Determinism: every floating-point addition happens in an order that depends
 *    only on the lengths (reading R5), so results are bit-identical run to
 *    run, across grid sizes, SM counts and pointer alignments.
 *  - Thread safety: all calls are reentrant.  A workspace must not be used by two
 *    calls that can run concurrently (use one per stream).
 */
#ifndef LIFT_H_
#define LIFT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same object as cudaStream_t / CUstream (an opaque driver stream handle). */
typedef struct CUstream_st* lift_stream_t;

typedef enum {
    LIFT_OK = 0,
    LIFT_ERR_INVALID_VALUE = 1,
    LIFT_ERR_NULL_POINTER = 2,
    LIFT_ERR_WORKSPACE = 3,
    LIFT_ERR_CUDA = 4
} lift_status;

/* ABI version of this header (bumped on any signature or contract change). */
#define LIFT_ABI_VERSION 1
int lift_abi_version(void);

/* The canonical decomposition that fixes the summation order of asum/dot (DESIGN.md
 * reading R5): chunks of lift_reduce_chunk_elems() elements, folded in groups of
 * lift_reduce_group_chunks() chunks.  Shards that are a power-of-two number of groups
 * combine (lift_combine) to the same bits as the unsharded call. */
int64_t lift_reduce_chunk_elems(void);
int lift_reduce_group_chunks(void);

/* Static, NUL-terminated description of a status code. */
const char* lift_status_string(lift_status s);
/* The CUDA error behind the calling thread's last LIFT_ERR_CUDA (cudaGetErrorString), or
 * "no error".  Static string; host only. */
const char* lift_last_cuda_error(void);

/* Bytes of workspace lift_asum / lift_dot / *_partial need for length n (a multiple of
 * 16).  The workspace holds the single-pass reduction's chunk/group partials (from its
 * start) and its last-block-done tickets (in a tail region whose size depends only on
 * ws_bytes).  The caller ZERO-FILLS it ONCE after allocation and then always passes the
 * SAME ws_bytes with that buffer; every call leaves the tickets at zero again, so one
 * buffer serves any n with lift_workspace_bytes(n) <= ws_bytes, indefinitely.  Two calls
 * in flight on one workspace, or a buffer that was not zero-filled, break this contract
 * (use one workspace per stream; the Python binding allocates one per (device, stream)).
 * A kernel that faults leaves the CUDA context unusable — every later launch then fails
 * with LIFT_ERR_CUDA — so stale tickets of an aborted call are never consumed.  (An
 * in-kernel guard that detects live foreign tickets was built and measured: it cost the
 * reductions 2-20%, and is not part of the product.) */
size_t lift_workspace_bytes(int64_t n);

/* Host-side check of that contract, off the hot path: waits for `stream`, copies the
 *   workspace's ticket region (its last bytes, a function of ws_bytes only) to the host and
 *   returns LIFT_OK if every ticket is zero, LIFT_ERR_WORKSPACE if any is not (a call was
 *   aborted, two calls overlapped on the buffer, or it was never zero-filled — zero-fill it
 *   again before the next call), LIFT_ERR_CUDA if the copy fails.  ws_bytes as passed to the
 *   reductions; ws must be 16-byte aligned (else LIFT_ERR_INVALID_VALUE). */
lift_status lift_workspace_check(const void* ws, size_t ws_bytes, lift_stream_t stream);

/* S1 — scal: y[i] = RN_fp32(alpha * x[i]) for 0 <= i < n.
 *   x: n floats in; y: n floats out; y == x (in place) is allowed, any other overlap
 *   is undefined.  n == 0 launches nothing.  Bit-exact by construction. */
lift_status lift_scal(int64_t n, float alpha, const float* x, float* y, lift_stream_t stream);

/* R1-R4 — asum: *result = RN_fp32(sum_i |x[i]|), n == 0 -> +0.0f (z = 0,
 *   P:794).  Single kernel, single pass (fused map+reduce, Fig. 4 (8)), with
 *   an fp64 cross-CTA fold.  x: n floats in; result: 1 float out (device);
 *   ws: lift_workspace_bytes(n) bytes (see above). */
lift_status lift_asum(int64_t n, const float* x, float* result, void* ws, size_t ws_bytes,
                      lift_stream_t stream);

/* R1-R4 — dot: *result = RN_fp32(sum_i x[i]*y[i]), n == 0 -> +0.0f.
 *   zip requires equal lengths, so one n describes both x and y. */
lift_status lift_dot(int64_t n, const float* x, const float* y, float* result, void* ws,
                     size_t ws_bytes, lift_stream_t stream);

/* Sharding helpers: the same reductions, but the un-rounded fp64 total is written to
 *   *partial (1 double, device) instead of an fp32 result.  Used per rank before the
 *   cross-GPU combine (X1). */
lift_status lift_asum_partial(int64_t n, const float* x, double* partial, void* ws,
                              size_t ws_bytes, lift_stream_t stream);
lift_status lift_dot_partial(int64_t n, const float* x, const float* y, double* partial,
                             void* ws, size_t ws_bytes, lift_stream_t stream);

/* NEXT-2 — fused scal + asum (rule 5f across ops): in ONE pass over x,
 *   y[i] = RN_fp32(alpha * x[i]) and *result = asum(y) — bit-identical to lift_scal
 *   followed by lift_asum on y (same canonical fold of the same values), but x is read
 *   once and y is not read back: 8 instead of 12 bytes per element.  y must not
 *   overlap x (x == y -> LIFT_ERR_INVALID_VALUE).  Workspace as for lift_asum. */
lift_status lift_scal_asum(int64_t n, float alpha, const float* x, float* y, float* result,
                           void* ws, size_t ws_bytes, lift_stream_t stream);

/* NEXT-1 — fused cross-GPU combine over peer memory (NVLink P2P stores).
 *   Each rank owns an EXCHANGE BUFFER of lift_xchg_bytes(p) bytes (lift_xchg_create:
 *   cudaMalloc'd and zeroed; the caller owns it and frees it with lift_xchg_destroy).
 *   Ranks share buffers with CUDA IPC (lift_ipc_get_handle / lift_ipc_open_handle; the
 *   64-byte handles travel over any host channel) and pass `peers`, a DEVICE array of p
 *   device pointers with peers[rank] = the own buffer, the others IPC-mapped.
 *   lift_*_allreduce run the single-pass reduction; its final CTA stores the fp64
 *   partial into slot `rank` of every peer's buffer, raises the slot flag to `epoch`
 *   (system-scope release), waits for all p flags of its own buffer and folds the p
 *   partials pairwise in rank order: every rank gets the SAME fp32 bits, equal to
 *   lift_combine over the gathered *_partial results — with no separate collective.
 *   p in [1, 32]; epoch > 0 and EXACTLY previous + 1 per call on the same exchange
 *   buffers (two banks alternate by epoch parity; a peer can be at most one call ahead,
 *   so consecutive calls must land in different banks); all p ranks must make the
 *   matching call with the same epoch.  The
 *   wait is bounded (~10 s): on timeout *result = NaN and *error (device int, may be
 *   NULL) is set to 1.  Workspace as for lift_asum. */
#define LIFT_IPC_HANDLE_BYTES 64
size_t lift_xchg_bytes(int p);
lift_status lift_xchg_create(int p, void** buf);
/* cudaMalloc'd buffer for IPC sharing (a base pointer, as cudaIpcGetMemHandle needs);
 * free with lift_xchg_destroy. */
lift_status lift_ipc_alloc(size_t bytes, void** buf);
lift_status lift_xchg_destroy(void* buf);
lift_status lift_ipc_get_handle(const void* buf, void* handle);
lift_status lift_ipc_open_handle(const void* handle, void** ptr);
lift_status lift_ipc_close_handle(void* ptr);
lift_status lift_asum_allreduce(int64_t n, const float* x, float* result, void* ws,
                                size_t ws_bytes, void* const* peers, int p, int rank,
                                unsigned long long epoch, int* error, lift_stream_t stream);
lift_status lift_dot_allreduce(int64_t n, const float* x, const float* y, float* result,
                               void* ws, size_t ws_bytes, void* const* peers, int p, int rank,
                               unsigned long long epoch, int* error, lift_stream_t stream);

/* NEXT-1 — gemv with the all-gather of y fused in: rank `rank` owns rows
 *   [row0, row0 + m) of the global A; each finished row is stored straight into every
 *   rank's full-length y (y_peers: DEVICE array of p pointers, IPC-mapped, from
 *   lift_ipc_alloc), and the CTA that finishes the rank's last row block publishes the
 *   rank's flag into every exchange buffer (xpeers, as for lift_*_allreduce, including
 *   the same epoch rule) and waits for all p flags.  When the kernel ends, this rank's
 *   y holds every rank's rows — bit-identical to lift_gemv + an all-gather.  m >= 1 on
 *   every rank; y_out is implied (y_peers[rank] + row0).  A peer one call ahead stores
 *   its next rows while this rank may still read this call's y, so callers alternate two
 *   y buffers by epoch parity (dist.PeerExchange does).  On a peer timeout the error word
 *   is set and the missing rows are left unwritten. */
lift_status lift_gemv_allgather(int64_t m, int64_t n, float alpha, const float* A, int64_t lda,
                                const float* x, float beta, const float* y,
                                float* const* y_peers, int64_t row0, void* const* xpeers,
                                int p, int rank, unsigned long long epoch, int* error,
                                lift_stream_t stream);

/* X1 — combine: *result = RN_fp32(pairwise_sum(partials[0..p))), the outermost
 *   reduce over per-rank partials in a fixed pairwise order (zero-padded to a power
 *   of two), so every rank that calls it on the gathered partials gets the same bits.
 *   partials: p doubles (device); result: 1 float (device); p >= 1. */
lift_status lift_combine(int p, const double* partials, float* result, lift_stream_t stream);

/* G1-G3 — gemv:
 *   y_out[i] = RN_fp32( alpha * (sum_j A[i*lda + j] * x[j]) + beta * y[i] ),  0 <= i < m,
 *   the dot in fp64 with exact products, the epilogue fma'd in fp64 and rounded once.
 *   A: m x n row-major, leading dimension lda >= max(1, n) (map over rows);
 *   x: n floats; y: m floats; y_out: m floats (y_out == y allowed).
 *   Literal semantics (reading R11): A, x and y are always read, so NaN/Inf propagate
 *   even when alpha or beta is 0 (no BLAS quick return).  m == 0 launches nothing;
 *   n == 0 gives y_out = RN_fp32(beta * y). */
lift_status lift_gemv(int64_t m, int64_t n, float alpha, const float* A, int64_t lda,
                      const float* x, float beta, const float* y, float* y_out,
                      lift_stream_t stream);

/* gemv with a workspace (same result bits as lift_gemv for every input).
 *   Rows of n >= 65536 columns are summed in the stand-alone dot's canonical order
 *   (y_out[i] uses exactly lift_dot_partial(A_i, x) in fp64).  When such rows are too few
 *   to occupy the GPU with one CTA each (m < 4 x SMs), ws lets the call spread each row's
 *   8192-column chunks over many CTAs with a per-row single-pass last-block-done.
 *   ws: device buffer of ws_bytes >= lift_gemv_workspace_bytes(m, n), 16-byte aligned,
 *   zero-filled ONCE by the caller (the kernels leave their tickets at zero); one
 *   buffer per stream, reusable for any (m, n) it fits.  ws may be NULL or smaller: the
 *   call then uses one CTA per row (same bits, fewer CTAs).  Other arguments and errors
 *   as lift_gemv. */
lift_status lift_gemv_ws(int64_t m, int64_t n, float alpha, const float* A, int64_t lda,
                         const float* x, float beta, const float* y, float* y_out, void* ws,
                         size_t ws_bytes, lift_stream_t stream);
/* Workspace bytes for lift_gemv_ws's split path at (m, n); 0 when no split would be used:
 *   rows shorter than 65536 columns, or m >= 4 x the current device's SM count (one CTA
 *   per row then fills the GPU). */
size_t lift_gemv_workspace_bytes(int64_t m, int64_t n);

/* NEXT-3 — BlackScholes (Fig. 9): map(BSComputation, s) over n stock prices.
 *   call[i] = s_i N(d1) - K e^{-rT} N(d2),  put[i] = K e^{-rT} N(-d2) - s_i N(-d1),
 *   d1 = (ln(s_i/K) + (r + v^2/2) T) / (v sqrt T),  d2 = d1 - v sqrt T,  N = normal CDF
 *   (closed form; the paper does not print the helpers, P:825 — DESIGN.md reading R22).
 *   s: n floats in (prices > 0); call, put: n floats out (SoA).  fp32 arithmetic: N(-|d|)
 *   by the Abramowitz-Stegun 26.2.17 polynomial (|error| < 7.5e-8), log2/exp2/rcp by the
 *   hardware approximations (reading R22); per-option error <= 5e-7 (s + K)
 *   against the fp64 oracle.  K, v, T must be > 0 and finite, r finite, else
 *   LIFT_ERR_INVALID_VALUE.  n == 0 launches nothing. */
lift_status lift_blackscholes(int64_t n, const float* s, float K, float r, float v, float T,
                              float* call, float* put, lift_stream_t stream);

/* NEXT-4 — device-specific strategy variants, the analogs of the paper's per-device
 *   lowerings (Fig. 7a/7b: tree in local memory or not, vector width, split
 *   sizes), selectable at run time.  Every variant computes the SAME canonical order, so
 *   none changes a result bit (tested); they only change how data moves.  Process-global;
 *   value 0 = the tuned default.  Unknown knob or value: LIFT_ERR_INVALID_VALUE.
 *     LIFT_VAR_LOAD_WIDTH  cap on the global load/store width: 0 auto (the widest the
 *                          alignment allows: LDG/STG.256), 1 scalar, 4 = 128-bit, 8 = 256-bit
 *     LIFT_VAR_GEMV_X      gemv rows of 2048..24576 columns: 0 auto (5 when the launch has
 *                          >= 4 waves of row blocks and n <= 12288, else 1), 1 x read through
 *                          L1 and widened per use, 5 x bulk-copied (TMA) into shared memory
 *                          per CTA as fp32 and read from there, 2 x staged once per CTA as fp64 in shared
 *                          memory + a register ring of A (persistent CTAs, Cluster Launch
 *                          Control stealing), 3 the same x staging + a TMA ring of A row
 *                          segments fed by a producer warp (n <= 16384), 4 two rows per
 *                          thread: each x vector loaded and widened once for both
 *     LIFT_VAR_PREFETCH    TMA L2 prefetch of a CTA's first unit at its start, before the PDL
 *                          wait (overlaps the previous kernel's tail): 0 auto (scal: first
 *                          wave; fused map+reduce: on; asum/dot: off; gemv: when the launch
 *                          has >= 4 waves of row blocks), 1 off everywhere, 2 on everywhere
 *     LIFT_VAR_ORDER       temporal order in which asum/dot visit their chunks (the summation
 *                          order is by chunk index either way): 0 auto (descending, so a
 *                          reduction after a map over the same vector starts on the tail the
 *                          map left in L2; the fused map+reduce ascending), 1 ascending,
 *                          2 descending
 *     LIFT_VAR_STAGGER     first-wave stagger (asum/dot/fused map+reduce, gemv): when a launch
 *                          has more units than resident CTA slots, CTA b of the first wave
 *                          delays its loads by b x (v ns per 32 KiB it reads), so the wave
 *                          retires staggered instead of together: 0 auto (2 ns per 32 KiB;
 *                          for gemv only with x in shared memory), 1 off, 2..64 that many ns
 *                          per 32 KiB
 *   (The other Fig. 7 axes — shared-memory tree vs shuffle butterfly, TMA bulk loads, chunk
 *   size — are compile-time variants searched by scripts/tune.py.) */
typedef enum {
    LIFT_VAR_LOAD_WIDTH = 0,
    LIFT_VAR_GEMV_X = 1,
    LIFT_VAR_PREFETCH = 2,
    LIFT_VAR_ORDER = 3,
    LIFT_VAR_STAGGER = 4,
    LIFT_VAR_COUNT = 5
} lift_variant;
lift_status lift_set_variant(lift_variant knob, int value);
int lift_get_variant(lift_variant knob);

/* TEST HOOK: cap the number of CTAs any subsequent launch may use (0 = no cap,
 *   the default).  Used by the determinism tests to show results do not depend on
 *   the grid.  Process-global; not for production use. */
lift_status lift_debug_set_grid_limit(int max_ctas);

#ifdef __cplusplus
}
#endif

#endif /* LIFT_H_ */
