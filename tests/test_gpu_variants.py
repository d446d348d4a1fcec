"""NEXT-4 runtime strategy variants (lift_set_variant): every value of every knob computes the
SAME canonical order, so results must be bit-identical to the default (and hence to the
oracle-checked default path).  Shapes cover the vector bodies, scalar heads/tails, the
reduction's partial chunks and the gemv paths the knobs switch between."""
import numpy as np
import pytest
import torch

import lift_inputs as gen
import oracle

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.fixture
def lift():
    import paper_1502_02389_b200 as m
    yield m
    for k in m.VARIANTS:
        m.set_variant(k, 0)


def bits(t):
    return t.detach().cpu().numpy().view(np.uint32).copy()


def fill(n, seed, tid, lo=-1.0, hi=1.0, off=0):
    buf = torch.empty(n + off, dtype=torch.float32, device=DEV)
    v = buf[off:]
    return gen.fill_device(v, seed, tid, 0, gen.DIST_UNIFORM, lo, hi)


def run_all(lift, off):
    out = []
    for n in (1, 9, 8191, 8192 * 3 + 5, 1 << 20, (1 << 23) + 13):  # the last: > one resident wave
        x = fill(n, 1, gen.TID_X, off=off)
        y = fill(n, 1, gen.TID_Y, off=off)
        out += [bits(lift.scal(3.0, x)), bits(lift.asum(x)), bits(lift.dot(x, y))]
    for m, n in ((300, 2048), (257, 4096), (64, 8192), (50, 12288), (33, 16384), (16, 24576),
                 (7, 1000), (8200, 2048)):  # the last: more row blocks than resident CTAs
        A = fill(m * n, 2, gen.TID_A, 0.0, 3.0).view(m, n)
        gx = fill(n, 2, gen.TID_X, 0.0, 1.0)
        gy = fill(m, 2, gen.TID_Y, 0.0, 2.0)
        out.append(bits(lift.gemv(A, gx, gy, 1.5, 0.5)))
    return out


@pytest.mark.parametrize("knob,values", [("load_width", (1, 4, 8)), ("gemv_x", (1, 2, 3, 4, 5)),
                                         ("prefetch", (1, 2)), ("order", (1, 2)),
                                         ("stagger", (1, 2, 8))])
@pytest.mark.parametrize("off", [0, 4])
def test_variants_bit_identical(lift, knob, values, off):
    ref = run_all(lift, off)
    for v in values:
        lift.set_variant(knob, v)
        assert lift.get_variant(knob) == v
        got = run_all(lift, off)
        for i, (a, b) in enumerate(zip(ref, got)):
            assert np.array_equal(a, b), (knob, v, i)
        lift.set_variant(knob, 0)


@pytest.mark.parametrize("var", [2, 3, 4, 5])
def test_staged_x_gemv_matches_oracle(lift, var):
    """The gemv x-strategy kernels (LIFT_VAR_GEMV_X = 2: x in shared memory + register ring;
    3: + TMA ring; 4: two rows per thread) against the oracle directly, with a partial last
    row block and signed inputs."""
    lift.set_variant("gemv_x", var)
    for m, n in ((1001, 8192), (65, 4096), (3, 16384), (37, 2048), (9, 12288)):
        A = gen.host(m * n, 7, gen.TID_A).reshape(m, n)
        x = gen.host(n, 7, gen.TID_X)
        y = gen.host(m, 7, gen.TID_Y)
        got = lift.gemv(torch.from_numpy(A).to(DEV), torch.from_numpy(x).to(DEV),
                        torch.from_numpy(y).to(DEV), -1.25, 0.75).cpu().numpy().astype(np.float64)
        ref = oracle.gemv(A, x, y, -1.25, 0.75)
        assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref)), (m, n)


def test_stagger_full_size_bit_identical(lift):
    """The first-wave stagger (on by default for the reductions and the x-in-shared-memory
    gemv) at BASELINE's full sizes and in its launch configuration: asum 2^28, dot 2^26, the
    fused scal+asum 2^28 and gemv 8192^2 give the same bits with the stagger off, on (default)
    and wide (16 ns per 32 KiB), and scal (stagger only when forced) the same bytes."""
    n, nd, m = 1 << 28, 1 << 26, 8192
    x = fill(n, 5, gen.TID_X)
    y = fill(nd, 5, gen.TID_Y)
    A = fill(m * m, 5, gen.TID_A, 0.0, 3.0).view(m, m)
    gx = fill(m, 5, gen.TID_X, 0.0, 1.0)
    gy = fill(m, 5, gen.TID_Y, 0.0, 2.0)

    def run():
        _, r = lift.scal_asum(2.0, x[:nd])
        return [bits(lift.asum(x)), bits(lift.dot(x[:nd], y)), bits(r),
                bits(lift.gemv(A, gx, gy, 1.5, 0.5)),
                bits(lift.scal(3.0, x[:nd]))]

    ref = run()
    for v in (1, 16):
        lift.set_variant("stagger", v)
        got = run()
        for i, (a, b) in enumerate(zip(ref, got)):
            assert np.array_equal(a, b), (v, i)
    lift.set_variant("stagger", 0)
