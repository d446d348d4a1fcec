"""Pins for the CPU oracle (oracle/), independent of the oracle itself.

Each test checks the oracle against something the paper or mathematics fixes:
worked examples (tests/golden/), closed forms, exact rational brute force
(fractions.Fraction), the correctly-rounded math.fsum, and invariants — chosen so a
dropped term, wrong sign, wrong index or transposed operand fails at least one.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")
U64 = 2.0 ** -53


def _cases():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["op"])
def test_spec_worked_examples(case):
    op = case["op"]
    if op == "scal":
        got = oracle.scal(case["alpha"], case["x"])
        assert got.tolist() == case["expect"]
    elif op == "asum":
        assert oracle.asum(case["x"]) == case["expect"]
    elif op == "dot":
        assert oracle.dot(case["x"], case["y"]) == case["expect"]
    elif op == "reduce":
        assert oracle.dot(case["x"], np.ones(len(case["x"]))) == case["expect"]
    elif op == "gemv":
        got = oracle.gemv(case["A"], case["x"], case["y"], case["alpha"], case["beta"])
        assert got.tolist() == case["expect"]


def test_empty_inputs_give_z():
    # reduce(add, 0) over [] is z = 0
    assert oracle.asum(np.zeros(0, np.float32)) == 0.0
    assert oracle.dot(np.zeros(0, np.float32), np.zeros(0, np.float32)) == 0.0
    # gemv with n = 0: out = 0 + beta*y
    out = oracle.gemv(np.zeros((3, 0), np.float32), np.zeros(0), [1.0, -2.0, 4.0], 1.5, 0.5)
    assert out.tolist() == [0.5, -1.0, 2.0]
    assert oracle.gemv(np.zeros((0, 4), np.float32), np.ones(4), [], 1.0, 1.0).size == 0


@pytest.mark.parametrize("n", [1, 7, 1000, 1 << 20])
@pytest.mark.parametrize("k", [0, 3, 23])
def test_asum_plus_minus_c_closed_form(n, k):
    # BASELINE north star: asum of a +-c vector equals N*c exactly.
    rng = np.random.default_rng(n * 31 + k)
    c = 2.0 ** -k
    x = (np.where(rng.random(n) < 0.5, -c, c)).astype(np.float32)
    assert oracle.asum(x) == n * c


def test_dot_with_ones_is_sum():
    # BASELINE north star: dot(x, 1) equals sum(x); checked against math.fsum,
    # which is correctly rounded (an independent algorithm).
    for seed, n in [(1, 10), (2, 4097), (3, 1 << 18)]:
        x = np.random.default_rng(seed).uniform(-1, 1, n).astype(np.float32)
        got = oracle.dot(x, np.ones(n, np.float32))
        ref = math.fsum(x.astype(np.float64).tolist())
        assert abs(got - ref) <= 2 * U64 * abs(ref) + 1e-300
        assert np.float32(got) == np.float32(ref)


@pytest.mark.parametrize("seed", range(20))
def test_brute_force_exact_rationals_small(seed):
    # N <= 64: exact sums with fractions.Fraction.
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 65))
    x = rng.uniform(-1, 1, n).astype(np.float32)
    y = rng.uniform(-3, 3, n).astype(np.float32)
    ex_asum = sum(abs(Fraction(float(v))) for v in x)
    ex_dot = sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x, y))
    terms = sum(abs(Fraction(float(a)) * Fraction(float(b))) for a, b in zip(x, y))
    assert abs(Fraction(oracle.asum(x)) - ex_asum) <= Fraction(2 * U64) * ex_asum
    assert abs(Fraction(oracle.dot(x, y)) - ex_dot) <= Fraction(2 * U64) * terms
    assert np.float32(oracle.asum(x)) == np.float32(float(ex_asum))
    assert np.float32(oracle.dot(x, y)) == np.float32(float(ex_dot))


@pytest.mark.parametrize("n", [1 << 12, 1 << 20])
def test_fsum_large(n):
    rng = np.random.default_rng(n)
    x = rng.uniform(-1, 1, n).astype(np.float32)
    y = rng.uniform(0, 2, n).astype(np.float32)
    prods = (x.astype(np.float64) * y.astype(np.float64)).tolist()  # exact in fp64
    ref = math.fsum(prods)
    scale = math.fsum(abs(p) for p in prods)
    assert abs(oracle.dot(x, y) - ref) <= 2 * U64 * scale
    ref_a = math.fsum(abs(float(v)) for v in x)
    assert abs(oracle.asum(x) - ref_a) <= 2 * U64 * ref_a


def test_compensation_alive():
    # Neumaier survives cancellation that defeats plain and Kahan summation
    # (reading R15).
    x = np.array([2.0 ** 60, 1.0, -(2.0 ** 60)], np.float32)
    assert oracle.dot(x, np.ones(3, np.float32)) == 1.0
    x = np.array([1.0] + [2.0 ** -53] * 1024, np.float32)
    assert oracle.dot(x, np.ones(x.size, np.float32)) == 1.0 + 2.0 ** -43


def test_asum_abs_semantics():
    x = np.array([-1.5, 2.0, -0.0, 0.0, -3.25], np.float32)
    assert oracle.asum(x) == 6.75
    assert oracle.asum(-x) == oracle.asum(x)          # abs is even
    assert math.copysign(1.0, oracle.asum(np.array([-0.0], np.float32))) == 1.0  # z = +0
    assert math.isnan(oracle.asum(np.array([1.0, np.nan], np.float32)))
    assert oracle.asum(np.array([-np.inf], np.float32)) == np.inf


def test_dot_is_not_asum_and_sign_sensitive():
    x = np.array([1.0, -2.0, 3.0], np.float32)
    y = np.array([-1.0, 1.0, 2.0], np.float32)
    assert oracle.dot(x, y) == 3.0          # -1 - 2 + 6
    assert oracle.dot(y, x) == 3.0
    assert oracle.dot(x, -y) == -3.0


def test_scal_exact():
    rng = np.random.default_rng(5)
    x = rng.uniform(-1e3, 1e3, 257).astype(np.float32)
    for a in (3.0, -0.1, 1.5e-7):
        got = oracle.scal(a, x)
        af = Fraction(float(np.float32(a)))
        for g, v in zip(got, x):
            assert Fraction(float(g)) == af * Fraction(float(v))


def test_gemv_identity_closed_form():
    # BASELINE north star: gemv with the identity matrix equals alpha*x + beta*y.
    # On the 2^-23 grid, 1.5x + 0.5y is exact in fp64 and in fp32.
    n = 300
    g = np.random.default_rng(9)
    x = (g.integers(-2 ** 23, 2 ** 23, n) * 2.0 ** -23).astype(np.float32)
    y = (g.integers(-2 ** 23, 2 ** 23, n) * 2.0 ** -23).astype(np.float32)
    out = oracle.gemv(np.eye(n, dtype=np.float32), x, y, 1.5, 0.5)
    exact = 1.5 * x.astype(np.float64) + 0.5 * y.astype(np.float64)
    assert np.array_equal(out, exact)


@pytest.mark.parametrize("shape", [(1, 1), (5, 7), (7, 5), (13, 64)])
def test_gemv_brute_force_nonsymmetric(shape):
    # Non-square, non-symmetric A: catches a transposed operand or swapped alpha/beta.
    m, n = shape
    g = np.random.default_rng(m * 100 + n)
    A = g.uniform(-1, 1, (m, n)).astype(np.float32)
    x = g.uniform(-1, 1, n).astype(np.float32)
    y = g.uniform(-1, 1, m).astype(np.float32)
    alpha, beta = 2.0, -3.0
    out = oracle.gemv(A, x, y, alpha, beta)
    for i in range(m):
        d = sum(Fraction(float(A[i, j])) * Fraction(float(x[j])) for j in range(n))
        ex = Fraction(alpha) * d + Fraction(beta) * Fraction(float(y[i]))
        terms = abs(Fraction(alpha)) * sum(abs(Fraction(float(A[i, j])) * Fraction(float(x[j])))
                                            for j in range(n)) + abs(Fraction(beta) * Fraction(float(y[i])))
        assert abs(Fraction(float(out[i])) - ex) <= Fraction(4 * U64) * terms


def test_gemv_row_major_with_padding():
    # lda > n: only the first n entries of each row are read (reading R8).
    m, n, lda = 4, 3, 5
    buf = np.full((m, lda), np.nan, np.float32)
    buf[:, :n] = np.arange(m * n, dtype=np.float32).reshape(m, n)
    out = oracle.gemv(buf[:, :n], [1.0, 0.0, -1.0], np.zeros(m), 1.0, 0.0)
    assert out.tolist() == [-2.0, -2.0, -2.0, -2.0]


def test_stream_equals_one_shot():
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, 10007).astype(np.float32)
    y = rng.uniform(-1, 1, 10007).astype(np.float32)
    s = oracle.Stream()
    for a in range(0, x.size, 1000):
        s.dot(x[a:a + 1000], y[a:a + 1000])
    assert s.value() == oracle.dot(x, y)
    s = oracle.Stream()
    for a in range(0, x.size, 333):
        s.asum(x[a:a + 333])
    assert s.value() == oracle.asum(x)


def test_dot_length_mismatch():
    with pytest.raises(ValueError):
        oracle.dot([1.0, 2.0], [1.0])
