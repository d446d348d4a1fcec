/* oracle.c — the CPU oracle for the paper's BLAS compositions.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load or call this code.
 * The product path (paper_1502_02389_b200/) never imports it, and this file
 * shares no code, header, helper or constant with the CUDA path.
 *
 * Source: Steuwer, Fensch, Dubach, "Patterns and Rewrite Rules for Systematic
 * Code Generation" (arXiv 1502.02389) = /root/reference/PAPER.md, cited P:<line>.
 *
 * Each function is the paper's PLAIN DEFINITION written out (the method reaches
 * the same result up to the reassociation that P:368 licenses):
 *     P:789  add(x, y)  = x + y
 *     P:790  mult(x, y) = x * y
 *     P:791  abs(x)     = if (x < 0) -x else x
 *     P:793  scal(a, x) = map(mult(a), x)
 *     P:794  asum(x)    = reduce(add, 0) o map(abs, x)
 *     P:795  dot(x, y)  = reduce(add, 0) o map(mult) o zip(x, y)
 *     P:796-798 gemv(A, x, y, a, b) = map(add) o zip(z, scal(b, y)),
 *                                     z = map(scal(a) o dot(x), A)
 *
 * Arithmetic: fp64 throughout (reading R1).  Inputs are fp32, so
 * (double)x*(double)y and (double)a*(double)x are EXACT (24+24 < 53 bits) and
 * abs is exact; the only error is the summation.  reduce(add, 0) is a left
 * fold from z = 0 (P:305, P:332 reduce-seq "an accumulation variable is
 * initialized with z") with Neumaier's (Kahan-Babuska) compensation, which —
 * unlike plain Kahan — survives [2^60, 1, -2^60] (reading R15).
 * Compile with -O2 -fno-fast-math -ffp-contract=off: fast-math deletes the
 * compensation.
 *
 * Pins (tests/test_oracle.py): SPEC worked examples, closed forms (asum of
 * +-c, dot(x,1)=sum x, gemv(I)=ax+by), exact rational brute force for N<=64,
 * math.fsum for larger N, compensation-alive cases.  No function here is
 * "parity unpinned".
 */
#include <math.h>
#include <stdint.h>

/* One Neumaier step: (s, c) += v.  The compensated value is s + c. */
static inline void neumaier_add(double *s, double *c, double v) {
    double t = *s + v;
    if (fabs(*s) >= fabs(v))
        *c += (*s - t) + v;
    else
        *c += (v - t) + *s;
    *s = t;
}

/* The compensated value s + c.  If the running sum is +-Inf the compensation
 * term is Inf - Inf = NaN and meaningless; the plain fold's value is s itself. */
double oracle_finish(const double *state) {
    return isinf(state[0]) ? state[0] : state[0] + state[1];
}

/* P:791 abs(x) = if (x < 0) -x else x — written literally (reading R3: -0.0
 * stays -0.0 and NaN passes through; the sum is unaffected because z = +0). */
static inline double paper_abs(double x) { return (x < 0) ? -x : x; }

/* P:793 scal(a, x) = map(mult(a), x): y_i = a * x_i, exact in fp64.
 * The caller rounds to fp32 once for bit-exact comparison (RN(a*x_i)). */
void oracle_scal(int64_t n, float a, const float *x, double *y) {
    for (int64_t i = 0; i < n; ++i) y[i] = (double)a * (double)x[i];
}

/* Streaming form of P:794 asum: folds n more elements into state[0..1] =
 * (s, c).  Start from state = {0, 0} (z = 0); the value is state[0]+state[1]. */
void oracle_asum_acc(int64_t n, const float *x, double *state) {
    double s = state[0], c = state[1];
    for (int64_t i = 0; i < n; ++i) neumaier_add(&s, &c, paper_abs((double)x[i]));
    state[0] = s;
    state[1] = c;
}

/* P:794 asum(x) = reduce(add, 0) o map(abs, x). n = 0 gives +0 (z = 0). */
double oracle_asum(int64_t n, const float *x) {
    double st[2] = {0.0, 0.0};
    oracle_asum_acc(n, x, st);
    return oracle_finish(st);
}

/* Streaming form of P:795 dot (zip requires equal lengths). */
void oracle_dot_acc(int64_t n, const float *x, const float *y, double *state) {
    double s = state[0], c = state[1];
    for (int64_t i = 0; i < n; ++i) neumaier_add(&s, &c, (double)x[i] * (double)y[i]);
    state[0] = s;
    state[1] = c;
}

/* P:795 dot(x, y) = reduce(add, 0) o map(mult) o zip(x, y). */
double oracle_dot(int64_t n, const float *x, const float *y) {
    double st[2] = {0.0, 0.0};
    oracle_dot_acc(n, x, y, st);
    return oracle_finish(st);
}

/* P:796-798 gemv, with P:814 "y = aAx + by" and reading R8: A is row-major,
 * element (i, j) at A[i*lda + j] — map(..., A) maps over ROWS.
 *   z_i   = a * dot(A_i, x)                    (scal(a) o dot(x))
 *   out_i = add(z_i, b * y_i)                  (map(add) o zip(z, scal(b,y)))
 * Each product is rounded once in fp64 in the paper's order; the caller rounds
 * out_i to fp32 once.  m = 0 writes nothing; n = 0 gives out_i = 0 + b*y_i. */
void oracle_gemv(int64_t m, int64_t n, float a, const float *A, int64_t lda,
                 const float *x, float b, const float *y, double *out) {
    for (int64_t i = 0; i < m; ++i) {
        double st[2] = {0.0, 0.0};
        oracle_dot_acc(n, A + i * lda, x, st);
        double d = oracle_finish(st);
        double z = (double)a * d;
        double w = (double)b * (double)y[i];
        out[i] = z + w;
    }
}

/* ---------------------------------------------------------------- BlackScholes
 * NEXT-3 row.  Fig. 9:
 *     BSComputation(s) = d1 = compD1(s); d2 = compD2(d1, s)
 *                        return { compCall(d1, d2, s), compPut(d1, d2, s) }
 *     blackScholes(s)  = map(BSComputation, s)
 * The helper bodies are "not shown" — reading R22: the standard closed-form
 * Black-Scholes price of European options without dividends, with strike K, rate r,
 * volatility v and maturity T fixed (the paper maps over the stock prices s only):
 *     d1 = (ln(s/K) + (r + v^2/2) T) / (v sqrt(T)),   d2 = d1 - v sqrt(T)
 *     call = s N(d1) - K e^{-rT} N(d2),   put = K e^{-rT} N(-d2) - s N(-d1)
 *     N(x) = erfc(-x / sqrt(2)) / 2            (standard normal CDF)
 * fp64 with the C library's erfc/log/exp/sqrt.  Pins: textbook values, put-call
 * parity, the v -> 0 and s -> 0 limits (tests/test_oracle_bs.py). */
static inline double norm_cdf(double x) { return 0.5 * erfc(-x / sqrt(2.0)); }

void oracle_blackscholes(int64_t n, const float *s, double K, double r, double v, double T,
                         double *call, double *put) {
    const double vsqrt = v * sqrt(T);
    const double disc = K * exp(-r * T);
    for (int64_t i = 0; i < n; ++i) {
        const double S = (double)s[i];
        const double d1 = (log(S / K) + (r + 0.5 * v * v) * T) / vsqrt;  /* compD1 */
        const double d2 = d1 - vsqrt;                                    /* compD2 */
        call[i] = S * norm_cdf(d1) - disc * norm_cdf(d2);                /* compCall */
        put[i] = disc * norm_cdf(-d2) - S * norm_cdf(-d1);               /* compPut */
    }
}
