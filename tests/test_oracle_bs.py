"""Pins for the BlackScholes oracle (NEXT-3 row): textbook prices, put-call parity,
limits and monotonicity — none of which retypes the oracle's formula."""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "blackscholes.json")


def _cases():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("c", _cases(), ids=lambda c: f"S{c['S']}")
def test_textbook_prices(c):
    call, put = oracle.blackscholes([c["S"]], c["K"], c["r"], c["v"], c["T"])
    half = 0.5 * 10.0 ** -c["digits"]
    assert abs(call[0] - c["call"]) <= half
    assert abs(put[0] - c["put"]) <= half


def test_put_call_parity():
    # C - P = S - K e^{-rT}, an identity of the model independent of N(.)
    s = np.linspace(1.0, 300.0, 1001).astype(np.float32)
    for K, r, v, T in [(100.0, 0.05, 0.2, 1.0), (40.0, 0.0, 0.6, 0.25), (15.0, 0.1, 0.05, 5.0)]:
        call, put = oracle.blackscholes(s, K, r, v, T)
        rhs = s.astype(np.float64) - K * math.exp(-r * T)
        assert np.allclose(call - put, rhs, rtol=0, atol=1e-9 * (K + s.max()))


def test_limits_and_bounds():
    K, r, T = 100.0, 0.05, 1.0
    s = np.array([1e-3, 50.0, 100.0, 150.0, 1e4], np.float32)
    call, put = oracle.blackscholes(s, K, r, 1e-6, T)  # v -> 0: intrinsic value of the forward
    disc = K * math.exp(-r * T)
    assert np.allclose(call, np.maximum(s - disc, 0), atol=1e-6)
    assert np.allclose(put, np.maximum(disc - s, 0), atol=1e-6)
    call, put = oracle.blackscholes(s, K, r, 0.3, T)
    assert np.all(call >= np.maximum(s - disc, 0) - 1e-12) and np.all(call <= s)
    assert np.all(put >= np.maximum(disc - s, 0) - 1e-12) and np.all(put <= disc + 1e-12)
    assert call[0] < 1e-12 and abs(put[0] - (disc - 1e-3)) < 1e-6        # s -> 0
    assert np.all(np.diff(call) > 0) and np.all(np.diff(put) < 0)       # monotone in s
