"""Maximum sizes: element counts past 2^32, where any 32-bit index arithmetic would wrap.

Reductions are checked through their fp64 partials against exact closed forms (constant
magnitudes with a sign pattern, plus marker values at indices 2^32 + 1 and n - 1), so a
single skipped or double-counted element shows; scal is checked bitwise around 2^32 and at
the end; gemv with more than 2^32 matrix elements (both row kernels) is checked on sampled
rows against the oracle and, for long rows, bitwise against lift_dot."""
import numpy as np
import pytest
import torch

import lift_inputs as gen
import oracle

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
N = (1 << 32) + 37


def _free_gib():
    free, _ = torch.cuda.mem_get_info()
    return free / 2**30


@pytest.fixture(scope="module")
def lift():
    import paper_1502_02389_b200 as m
    return m


def test_reductions_past_2_32(lift):
    if _free_gib() < 40:
        pytest.skip("needs ~34 GiB of device memory")
    x = torch.full((N,), 0.25, dtype=torch.float32, device=DEV)
    x[::3] = -0.25                       # sign pattern; |x| stays 0.25
    x[(1 << 32) + 1] = 1024.0            # markers past 2^32 and at the very end
    x[N - 1] = -2048.0
    n_neg = (N + 2) // 3                 # indices 0, 3, 6, ... (none of the markers)
    big = 0.25 * (N - 2) + 1024.0 + 2048.0
    assert lift.asum_partial(x).item() == big
    y = torch.ones(N, dtype=torch.float32, device=DEV)
    want_sum = 0.25 * (N - 2 - n_neg) - 0.25 * n_neg + 1024.0 - 2048.0
    assert lift.dot_partial(x, y).item() == want_sum
    assert lift.dot_partial(y, x).item() == want_sum
    assert lift.asum(x).item() == np.float32(big)
    del y
    # scal: y = 3 x, bitwise around 2^32 and at the end
    out = torch.full((N,), float("nan"), dtype=torch.float32, device=DEV)
    lift.scal(3.0, x, out=out)
    for a, b in [(0, 64), ((1 << 32) - 40, (1 << 32) + 40), (N - 64, N)]:
        assert torch.equal(out[a:b], 3.0 * x[a:b]), (a, b)
    assert not torch.isnan(out).any()


@pytest.mark.parametrize("m,n", [((1 << 19) + 3, 8192), (65537, 65541)])
def test_gemv_past_2_32_elements(lift, m, n):
    if _free_gib() < 24:
        pytest.skip("needs ~17 GiB of device memory")
    assert m * n > (1 << 32)
    A = gen.fill_device(torch.empty(m * n, device=DEV), 3, gen.TID_A, 0, 0, -1.0, 1.0).view(m, n)
    x = gen.fill_device(torch.empty(n, device=DEV), 3, gen.TID_X, 0, 0, -1.0, 1.0)
    y = gen.fill_device(torch.empty(m, device=DEV), 3, gen.TID_Y, 0, 0, -1.0, 1.0)
    got = lift.gemv(A, x, y, 1.5, 0.5).cpu().numpy()
    assert not np.isnan(got).any()
    xh = gen.host(n, 3, gen.TID_X, 0, lo=-1.0, hi=1.0)
    yh = gen.host(m, 3, gen.TID_Y, 0, lo=-1.0, hi=1.0)
    for r in [0, 1, m // 2, ((1 << 32) // n), m - 2, m - 1]:
        Ar = gen.host(n, 3, gen.TID_A, r * n, lo=-1.0, hi=1.0).reshape(1, n)
        ref = oracle.gemv(Ar, xh, yh[r:r + 1], 1.5, 0.5)[0]
        scale = 1.5 * float((np.abs(Ar.astype(np.float64)) @ np.abs(xh.astype(np.float64)))[0]) \
            + 0.5 * abs(float(yh[r]))
        assert abs(float(got[r]) - ref) <= 1e-6 * scale, r
        if n >= 65536:  # long rows: gemv row == lift_dot bitwise (alpha 1, beta 0)
            g1 = lift.gemv(A[r:r + 1], x, y[r:r + 1], 1.0, 0.0)
            assert torch.equal(g1, lift.dot(A[r], x)), r
