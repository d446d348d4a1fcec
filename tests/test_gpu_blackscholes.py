"""NEXT-3 row: BlackScholes (Fig. 9) on the GPU vs the fp64 oracle.

Bar (reading R22): per option |g - o| <= 5e-7 * (s + K) — fp32
arithmetic on prices bounded by s (call) and K (put); relative error is meaningless for
deep out-of-the-money prices near 0.  Put-call parity holds on the GPU results to the
same bound; any alignment gives the same bits."""
import numpy as np
import pytest
import torch

import lift_inputs as gen
import oracle

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
K, R, V, T = 100.0, 0.05, 0.2, 1.0   # reading R22: fixed per call


@pytest.fixture(scope="module")
def lift():
    import paper_1502_02389_b200 as m
    return m


def prices(n, seed=0):
    return gen.host(n, seed, gen.TID_X, lo=10.0, hi=200.0)


@pytest.mark.parametrize("n", [1, 7, 8, 9, 255, 1000, 100_003, 4 * 1024 * 1024])
def test_blackscholes_vs_oracle(lift, n):
    s = prices(n, n)
    c, p = lift.blackscholes(torch.from_numpy(s).to(DEV), K, R, V, T)
    oc, op = oracle.blackscholes(s, K, R, V, T)
    scale = s.astype(np.float64) + K
    ec = np.abs(c.cpu().numpy() - oc) / scale
    ep = np.abs(p.cpu().numpy() - op) / scale
    assert ec.max() <= 5e-7 and ep.max() <= 5e-7, (ec.max(), ep.max())
    par = c.cpu().numpy().astype(np.float64) - p.cpu().numpy() - (s - K * np.exp(-R * T))
    assert np.abs(par / scale).max() <= 1e-6


@pytest.mark.parametrize("params", [(40.0, 0.0, 0.6, 0.25), (15.0, 0.1, 0.05, 5.0),
                                    (100.0, -0.01, 1.5, 0.01)])
def test_blackscholes_other_params(lift, params):
    k, r, v, t = params
    s = gen.host(50_000, 3, gen.TID_X, lo=0.2 * k, hi=3.0 * k)
    c, p = lift.blackscholes(torch.from_numpy(s).to(DEV), k, r, v, t)
    oc, op = oracle.blackscholes(s, k, r, v, t)
    scale = s.astype(np.float64) + k
    assert (np.abs(c.cpu().numpy() - oc) / scale).max() <= 5e-7
    assert (np.abs(p.cpu().numpy() - op) / scale).max() <= 5e-7


def test_blackscholes_textbook(lift):
    s = torch.tensor([42.0, 100.0], device=DEV)
    c, p = lift.blackscholes(s[:1], 40.0, 0.1, 0.2, 0.5)
    assert abs(c.item() - 4.76) <= 0.005 and abs(p.item() - 0.81) <= 0.005
    c, p = lift.blackscholes(s[1:], 100.0, 0.05, 0.2, 1.0)
    assert abs(c.item() - 10.4506) <= 5e-4 and abs(p.item() - 5.5735) <= 5e-4


def test_blackscholes_alignment_and_empty(lift):
    n = 5003
    s = prices(n, 9)
    ref_c, ref_p = (t.cpu().numpy() for t in lift.blackscholes(torch.from_numpy(s).to(DEV), K, R, V, T))
    for off in (1, 3, 5):
        buf = torch.zeros(n + 16, device=DEV)
        sv = buf[off:off + n]
        sv.copy_(torch.from_numpy(s))
        cb = torch.zeros(n + 16, device=DEV)[(off * 3) % 8:(off * 3) % 8 + n]
        pb = torch.zeros(n + 16, device=DEV)[2:2 + n]
        lift.blackscholes(sv, K, R, V, T, call=cb, put=pb)
        assert np.array_equal(cb.cpu().numpy().view(np.uint32), ref_c.view(np.uint32))
        assert np.array_equal(pb.cpu().numpy().view(np.uint32), ref_p.view(np.uint32))
    e = torch.empty(0, device=DEV)
    c, p = lift.blackscholes(e, K, R, V, T)
    assert c.numel() == 0 and p.numel() == 0


def test_blackscholes_extreme_moneyness(lift):
    """Deep in/out of the money and s = 0 (d = -inf): finite, within the bar, and the
    limits call -> max(s - K e^{-rT}, 0), put -> max(K e^{-rT} - s, 0) hold."""
    s = np.array([0.0, 1e-30, 1e-3, 1.0, 1e4, 1e6, 3e7], dtype=np.float32)
    c, p = (t.cpu().numpy() for t in lift.blackscholes(torch.from_numpy(s).to(DEV), K, R, V, T))
    assert np.all(np.isfinite(c)) and np.all(np.isfinite(p))
    oc, op = oracle.blackscholes(s, K, R, V, T)
    scale = s.astype(np.float64) + K
    assert (np.abs(c - oc) / scale).max() <= 5e-7 and (np.abs(p - op) / scale).max() <= 5e-7
    assert c[0] == 0.0 and abs(p[0] - K * np.exp(-R * T)) <= 1e-4
