"""NEXT-2 row: the fused scal+asum (rule 5f across ops).

Bar: y bit-exact RN(alpha*x); result bit-identical to lift_asum(lift_scal(x)) (same
canonical fold over the same values) at every size and alignment; within 1e-5 of the
fp64 oracle's asum(y); exact on integer-valued inputs."""
import numpy as np
import pytest
import torch

import lift_inputs as gen
import oracle

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def lift():
    import paper_1502_02389_b200 as m
    return m


def bits(t):
    return t.detach().cpu().numpy().view(np.uint32).copy()


def at_offset(a, off):
    buf = torch.empty(a.size + off + 8, dtype=torch.float32, device=DEV)
    v = buf[off:off + a.size]
    v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return v


@pytest.mark.parametrize("n", [1, 7, 9, 8191, 8192, 8193, 100_003, (1 << 21) + 5, 1 << 24])
@pytest.mark.parametrize("alpha", [3.0, -0.37])
def test_fused_equals_composition(lift, n, alpha):
    x = gen.host(n, 5, gen.TID_X)
    xd = torch.from_numpy(x).to(DEV)
    y, r = lift.scal_asum(alpha, xd)
    y2 = lift.scal(alpha, xd)
    r2 = lift.asum(y2)
    assert np.array_equal(bits(y), bits(y2))
    assert np.array_equal(bits(r), bits(r2))
    yo = oracle.scal(alpha, x).astype(np.float32)
    assert np.array_equal(bits(y), yo.view(np.uint32))
    ao = oracle.asum(yo)
    assert abs(r.item() - ao) <= 1e-5 * ao


@pytest.mark.parametrize("ox,oy", [(1, 1), (0, 3), (5, 2)])
def test_fused_alignments(lift, ox, oy):
    n = 3 * 8192 + 77
    x = gen.host(n, 6, gen.TID_X, dist=gen.DIST_INT17)
    xd = at_offset(x, ox)
    yb = torch.empty(n + 16, dtype=torch.float32, device=DEV)[oy:oy + n]
    y, r = lift.scal_asum(2.0, xd, out=yb)
    assert np.array_equal(bits(y), (2.0 * x).astype(np.float32).view(np.uint32))
    assert r.item() == np.float32(oracle.asum(2.0 * x))  # integer-valued: exact


def test_fused_overflow_refold_and_empty(lift):
    x = np.full(40_000, 1e38, np.float32)
    y, r = lift.scal_asum(1.0, torch.from_numpy(x).to(DEV))
    assert r.item() == np.inf and np.array_equal(bits(y), x.view(np.uint32))
    x[5] = -3e38
    y, r = lift.scal_asum(0.5, torch.from_numpy(x).to(DEV))
    assert r.item() == lift.asum(y).item()
    e = torch.empty(0, device=DEV)
    y, r = lift.scal_asum(2.0, e)
    assert y.numel() == 0 and bits(r)[0] == 0


def test_fused_rejects_in_place(lift):
    x = torch.ones(100, device=DEV)
    with pytest.raises(lift.LiftError):
        lift.scal_asum(2.0, x, out=x)
