"""Randomised parity sweep (seeded): sizes, ragged tails, pointer alignments, lda
padding, on integer-valued inputs where every result is unique — so the CUDA path must
match the oracle BIT FOR BIT (asum, dot, their fp64 partials, scal, gemv, fused
scal+asum).  Complements the hand-picked cases in test_gpu_parity.py."""
import numpy as np
import pytest
import torch

import lift_inputs as gen
import oracle

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
RNG = np.random.default_rng(20261017)
CASES = [(int(np.exp(RNG.uniform(0, np.log(1 << 22)))), int(RNG.integers(0, 8)),
          int(RNG.integers(0, 8)), int(RNG.integers(1 << 30))) for _ in range(40)]
GEMV = [(int(RNG.integers(1, 300)), int(np.exp(RNG.uniform(0, np.log(40000)))),
         int(RNG.integers(0, 9)), int(RNG.integers(0, 4)), int(RNG.integers(1 << 30)))
        for _ in range(24)]


@pytest.fixture(scope="module")
def lift():
    import paper_1502_02389_b200 as m
    return m


def at_offset(a, off):
    buf = torch.empty(a.size + off + 8, dtype=torch.float32, device=DEV)
    v = buf[off:off + a.size]
    v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return v


def bits(t):
    return t.detach().cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("n,ox,oy,seed", CASES)
def test_fuzz_vectors(lift, n, ox, oy, seed):
    x = gen.host(n, seed, gen.TID_X, dist=gen.DIST_INT17)
    y = gen.host(n, seed, gen.TID_Y, dist=gen.DIST_INT17)
    xd, yd = at_offset(x, ox), at_offset(y, oy)
    assert lift.asum(xd).item() == np.float32(oracle.asum(x))
    assert lift.dot(xd, yd).item() == np.float32(oracle.dot(x, y))
    assert lift.asum_partial(xd).item() == oracle.asum(x)
    assert lift.dot_partial(xd, yd).item() == oracle.dot(x, y)
    out = torch.empty(n + 8, dtype=torch.float32, device=DEV)[oy:oy + n]
    lift.scal(-3.0, xd, out=out)
    assert np.array_equal(bits(out), oracle.scal(-3.0, x).astype(np.float32).view(np.uint32))
    ys, r = lift.scal_asum(0.5, xd, out=out)
    half = oracle.scal(0.5, x).astype(np.float32)
    assert np.array_equal(bits(ys), half.view(np.uint32))
    assert r.item() == np.float32(oracle.asum(half))


@pytest.mark.parametrize("m,n,pad,off,seed", GEMV)
def test_fuzz_gemv(lift, m, n, pad, off, seed):
    A = gen.host(m * n, seed, gen.TID_A, dist=gen.DIST_INT17).reshape(m, n)
    x = gen.host(n, seed, gen.TID_X, dist=gen.DIST_INT17)
    y = gen.host(m, seed, gen.TID_Y, dist=gen.DIST_INT17)
    buf = torch.zeros(m * (n + pad) + off + 8, dtype=torch.float32, device=DEV)
    Ad = buf[off:off + m * (n + pad)].view(m, n + pad)[:, :n]
    Ad.copy_(torch.from_numpy(A))
    got = lift.gemv(Ad, at_offset(x, off), at_offset(y, (off + 1) % 8), 1.5, 0.5)
    ref = oracle.gemv(A, x, y, 1.5, 0.5).astype(np.float32)  # exact: small integers
    assert np.array_equal(bits(got), ref.view(np.uint32))
