"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Bars (BASELINE.json north_star):
  * scal: bit-exact RN(alpha*x_i) at every size, alignment and aliasing;
  * asum/dot: relative error |g-o| <= 1e-5 |o| (plain relative, also for
    signed inputs); bit-exact on integer-valued inputs, where the sum is unique;
    bit-identical run to run and across grid sizes;
  * gemv: per element relative error |g-o| <= 1e-6 |o| (plain relative, also for signed
    inputs); identity matrix bit-exact.
"""
import numpy as np
import pytest
import torch

import lift_inputs as gen
import oracle

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
from paper_1502_02389_b200._lib import lib as _abi  # noqa: E402

RED_C = int(_abi.lift_reduce_chunk_elems())        # canonical chunk (csrc/canon.h)
GROUP = RED_C * int(_abi.lift_reduce_group_chunks())  # canonical group


@pytest.fixture(scope="module")
def lift():
    import paper_1502_02389_b200 as m
    m.set_grid_limit(0)
    yield m
    m.set_grid_limit(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def at_offset(a, off):
    """Device copy of `a` whose data pointer is `off` floats past a 512-B boundary."""
    buf = torch.empty(a.size + off + 8, dtype=torch.float32, device=DEV)
    v = buf[off:off + a.size]
    v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return v


def bits(t):
    return t.detach().cpu().numpy().view(np.uint32).copy()


# ------------------------------------------------------------------ generator twin
@pytest.mark.parametrize("dist,lo,hi", [(0, -1.0, 1.0), (0, 0.0, 3.0), (1, 0.0, 0.0)])
def test_device_generator_matches_host(dist, lo, hi):
    for seed, tid, i0, n in [(0, 1, 0, 1 << 20), (3, 3, (1 << 31) + 5, 100_003)]:
        t = torch.empty(n, dtype=torch.float32, device=DEV)
        gen.fill_device(t, seed, tid, i0, dist, lo, hi)
        h = gen.host(n, seed, tid, i0, dist, lo, hi)
        assert np.array_equal(bits(t), h.view(np.uint32))


# ------------------------------------------------------------------------- scal
SIZES_SMALL = [0, 1, 2, 3, 7, 8, 9, 15, 16, 17, 31, 255, 256, 257, 1023, 1024, 1100]


@pytest.mark.parametrize("n", SIZES_SMALL + [8191, 8192, 8193, 100_003, 1 << 20])
def test_scal_bit_exact(lift, n):
    x = gen.host(n, 11, gen.TID_X, lo=-1e3, hi=1e3)
    for alpha in (3.0, -0.7):
        ref = oracle.scal(alpha, x).astype(np.float32)
        got = lift.scal(alpha, dev(x)).cpu().numpy()
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("ox,oy", [(0, 0), (1, 1), (3, 3), (7, 7), (1, 0), (0, 3), (2, 6), (5, 1)])
def test_scal_alignments(lift, ox, oy):
    n = 5003
    x = gen.host(n, 12, gen.TID_X)
    ref = oracle.scal(3.0, x).astype(np.float32)
    xd = at_offset(x, ox)
    y = torch.empty(n + oy + 8, dtype=torch.float32, device=DEV)[oy:oy + n]
    lift.scal(3.0, xd, out=y)
    assert np.array_equal(bits(y), ref.view(np.uint32))


def test_scal_in_place(lift):
    x = gen.host(77_777, 13, gen.TID_X)
    ref = oracle.scal(-2.5, x).astype(np.float32)
    for off in (0, 3):
        xd = at_offset(x, off)
        lift.scal(-2.5, xd, out=xd)
        assert np.array_equal(bits(xd), ref.view(np.uint32))


def test_scal_special_values(lift):
    x = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, 3e38, -1.0], np.float32)
    got = lift.scal(3.0, dev(x)).cpu().numpy()
    ref = oracle.scal(3.0, x).astype(np.float32)
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    m = ~np.isnan(ref)
    assert np.array_equal(got[m].view(np.uint32), ref[m].view(np.uint32))  # no FTZ (1e-45*3)


# ------------------------------------------------------------------- asum / dot
RED_SIZES = [1, 2, 7, 8, 9, 255, 256, 257, 4096, RED_C - 1, RED_C, RED_C + 1,
             3 * RED_C + 17, 100_003, GROUP - 5, GROUP + 7, (1 << 22) + 3]


@pytest.mark.parametrize("n", RED_SIZES)
def test_asum_dot_tolerance(lift, n):
    x = gen.host(n, 21, gen.TID_X)
    y = gen.host(n, 21, gen.TID_Y, lo=0.0, hi=2.0)
    a = float(lift.asum(dev(x)).item())
    ao = oracle.asum(x)
    assert abs(a - ao) <= 1e-5 * ao
    xp = gen.host(n, 21, gen.TID_X, lo=0.0, hi=1.0)
    d = float(lift.dot(dev(xp), dev(y)).item())
    do = oracle.dot(xp, y)
    assert abs(d - do) <= 1e-5 * abs(do)
    ds = float(lift.dot(dev(x), dev(y)).item())  # signed: plain relative too (A20)
    dso = oracle.dot(x, y)
    assert abs(ds - dso) <= 1e-5 * abs(dso), (ds, dso)


@pytest.mark.parametrize("n", [1, 9, 1000, RED_C + 1, 5 * RED_C + 3, GROUP + 1, 1 << 20])
@pytest.mark.parametrize("off", [0, 1, 4])
def test_integer_inputs_bit_exact(lift, n, off):
    """Integer-valued inputs make every partial sum exact, so the result is unique:
    this pins indexing, the tail, alignment handling and the cross-CTA fold."""
    x = gen.host(n, 31, gen.TID_X, dist=gen.DIST_INT17)
    y = gen.host(n, 31, gen.TID_Y, dist=gen.DIST_INT17)
    xd, yd = at_offset(x, off), at_offset(y, (off * 3) % 8)
    assert lift.asum(xd).item() == np.float32(oracle.asum(x))
    assert lift.dot(xd, yd).item() == np.float32(oracle.dot(x, y))
    assert lift.asum_partial(xd).item() == oracle.asum(x)
    assert lift.dot_partial(xd, yd).item() == oracle.dot(x, y)


def test_empty_reductions(lift):
    e = torch.empty(0, dtype=torch.float32, device=DEV)
    r = torch.full((1,), 7.0, device=DEV)
    lift.asum(e, out=r)
    assert bits(r)[0] == 0  # +0.0f
    r.fill_(7.0)
    lift.dot(e, e, out=r)
    assert bits(r)[0] == 0
    assert lift.asum_partial(e).item() == 0.0


def test_determinism_runs_and_grids(lift):
    n = 3 * GROUP + 12345
    xd = dev(gen.host(n, 41, gen.TID_X))
    yd = dev(gen.host(n, 41, gen.TID_Y))
    base_a, base_d = bits(lift.asum(xd)), bits(lift.dot(xd, yd))
    base_pa = lift.asum_partial(xd).item()
    for _ in range(10):
        assert np.array_equal(bits(lift.asum(xd)), base_a)
        assert np.array_equal(bits(lift.dot(xd, yd)), base_d)
    try:
        for g in (1, 2, 3, 7, 148, 1000):
            lift.set_grid_limit(g)
            assert np.array_equal(bits(lift.asum(xd)), base_a), g
            assert np.array_equal(bits(lift.dot(xd, yd)), base_d), g
            assert lift.asum_partial(xd).item() == base_pa
    finally:
        lift.set_grid_limit(0)


def test_alignment_does_not_change_bits(lift):
    n = 2 * RED_C + 99
    x = gen.host(n, 43, gen.TID_X)
    y = gen.host(n, 43, gen.TID_Y)
    ref_a = bits(lift.asum(at_offset(x, 0)))
    ref_d = bits(lift.dot(at_offset(x, 0), at_offset(y, 0)))
    for ox, oy in [(4, 4), (1, 1), (2, 5), (7, 0)]:
        assert np.array_equal(bits(lift.asum(at_offset(x, ox))), ref_a)
        assert np.array_equal(bits(lift.dot(at_offset(x, ox), at_offset(y, oy))), ref_d)


def test_invariants(lift):
    n = 200_001
    x = gen.host(n, 51, gen.TID_X)
    y = gen.host(n, 51, gen.TID_Y)
    xd, yd = dev(x), dev(y)
    assert np.array_equal(bits(lift.dot(xd, yd)), bits(lift.dot(yd, xd)))      # commutative
    assert np.array_equal(bits(lift.asum(xd)), bits(lift.asum(-xd)))           # abs even
    a = lift.asum(xd).item()
    assert lift.asum(xd * 4.0).item() == 4.0 * a                                # 2^k scaling
    xp = dev(np.abs(x))
    assert np.array_equal(bits(lift.dot(xp, torch.ones_like(xp))), bits(lift.asum(xp)))


@pytest.mark.parametrize("n,k", [(1 << 20, 3), (1 << 22, 10), (12345, 0)])
def test_asum_plus_minus_c_closed_form_gpu(lift, n, k):
    rng = np.random.default_rng(n + k)
    c = 2.0 ** -k
    x = np.where(rng.random(n) < 0.5, -c, c).astype(np.float32)
    assert lift.asum(dev(x)).item() == np.float32(n * c)


def test_workspace_ticket_reset(lift):
    n = GROUP * 2 + 5
    xd = dev(gen.host(n, 61, gen.TID_X))
    ws = lift.Workspace(n, xd.device)
    out = torch.empty(100, dtype=torch.float32, device=DEV)
    for i in range(100):
        lift.asum(xd, out=out[i:i + 1], ws=ws)
    o = out.cpu().numpy()
    assert np.all(o == o[0])
    wf = ws.nbytes // 16 * 16
    r = ((wf // 512 + 2) * 4 + 15) // 16 * 16  # tickets live in the last r bytes
    assert torch.count_nonzero(ws.buf[wf - r:wf]).item() == 0


def test_workspace_shared_across_sizes(lift):
    """One workspace serves calls of different n in any order (tickets never clobbered)."""
    ws = lift.Workspace(1 << 26, torch.device(DEV))
    sizes = [1 << 26, 1 << 24, 3 * RED_C + 5, 1 << 22, 1 << 26, 100, GROUP * 5 + 1]
    xs = {n: gen.host(n, 62, gen.TID_X, lo=0.0, hi=1.0) for n in set(sizes)}
    for n in sizes:
        g = lift.asum(dev(xs[n]), ws=ws).item()
        o = oracle.asum(xs[n])
        assert abs(g - o) <= 1e-5 * o, n


def test_special_values_propagate(lift):
    x = np.ones(70_000, np.float32)
    x[12345] = np.nan
    assert np.isnan(lift.asum(dev(x)).item())
    x[12345] = -np.inf
    assert lift.asum(dev(x)).item() == np.inf
    big = np.full(1 << 20, 3e38, np.float32)  # fp64 partials: no overflow until the final RN
    assert lift.asum(dev(big)).item() == np.inf
    assert lift.asum_partial(dev(big)).item() == pytest.approx(3e38 * (1 << 20), rel=1e-6)


def test_combine(lift):
    p = torch.tensor([1.0, 2.0 ** -30, -1.0, 3.0, 0.5], dtype=torch.float64, device=DEV)
    # pairwise over 8 leaves: ((1 + 2^-30) + (-1 + 3)) + (0.5 + 0) ...
    assert lift.combine(p).item() == np.float32(3.5 + 2.0 ** -30)
    one = torch.tensor([2.5], dtype=torch.float64, device=DEV)
    assert lift.combine(one).item() == 2.5


def test_sharded_partials_compose_bit_exactly(lift):
    """Shards of a power-of-two number of groups combine to the unsharded bits."""
    G = GROUP
    n = 8 * G
    x = gen.host(n, 71, gen.TID_X)
    y = gen.host(n, 71, gen.TID_Y)
    full_a = bits(lift.asum(dev(x)))
    full_d = bits(lift.dot(dev(x), dev(y)))
    for p in (2, 4, 8):
        s = n // p
        pa = torch.cat([lift.asum_partial(dev(x[r * s:(r + 1) * s])) for r in range(p)])
        pd = torch.cat([lift.dot_partial(dev(x[r * s:(r + 1) * s]), dev(y[r * s:(r + 1) * s]))
                        for r in range(p)])
        assert np.array_equal(bits(lift.combine(pa)), full_a)
        assert np.array_equal(bits(lift.combine(pd)), full_d)


# ------------------------------------------------------------------------- gemv
def gemv_inputs(m, n, seed, signed=False):
    lo = -1.0 if signed else 0.0
    A = gen.host(m * n, seed, gen.TID_A, lo=lo, hi=3.0 if not signed else 1.0).reshape(m, n)
    x = gen.host(n, seed, gen.TID_X, lo=lo, hi=1.0)
    y = gen.host(m, seed, gen.TID_Y, lo=lo, hi=2.0 if not signed else 1.0)
    return A, x, y


def check_gemv(got, A, x, y, alpha, beta):
    """Plain relative error per element; the condition-scaled error
    |g-o| / sum|terms| is reported as a diagnostic only."""
    ref = oracle.gemv(A, x, y, alpha, beta)
    scale = abs(alpha) * (np.abs(A.astype(np.float64)) @ np.abs(x.astype(np.float64))) \
        + abs(beta) * np.abs(y.astype(np.float64))
    err = np.abs(got.astype(np.float64) - ref)
    assert np.all(err <= 1e-6 * np.abs(ref)), (
        float(np.max(err / np.maximum(np.abs(ref), 1e-300))),
        float(np.max(err / np.maximum(scale, 1e-300))))
    return ref


@pytest.mark.parametrize("m,n", [(1, 1), (5, 7), (8, 256), (17, 255), (301, 1027), (64, 4096),
                                 (1000, 8192), (33, 16384), (20, 16385), (9, 40000), (3, 0)])
def test_gemv_tolerance(lift, m, n):
    A, x, y = gemv_inputs(m, n, m * 7 + n)
    got = lift.gemv(dev(A), dev(x), dev(y), 1.5, 0.5).cpu().numpy()
    ref = oracle.gemv(A, x, y, 1.5, 0.5)
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref))


@pytest.mark.parametrize("m,n", [(37, 1029), (8, 20000), (1000, 8192), (64, 70000)])
def test_gemv_signed_plain_relative(lift, m, n):
    A, x, y = gemv_inputs(m, n, 5, signed=True)
    got = lift.gemv(dev(A), dev(x), dev(y), -2.0, 0.75).cpu().numpy()
    check_gemv(got, A, x, y, -2.0, 0.75)


def test_gemv_identity_bit_exact(lift):
    n = 4096 + 37
    x = gen.host(n, 81, gen.TID_X)
    y = gen.host(n, 81, gen.TID_Y)
    eye = np.eye(n, dtype=np.float32)
    got = lift.gemv(dev(eye), dev(x), dev(y), 1.5, 0.5).cpu().numpy()
    exact = (1.5 * x.astype(np.float64) + 0.5 * y.astype(np.float64)).astype(np.float32)
    assert np.array_equal(got.view(np.uint32), exact.view(np.uint32))


@pytest.mark.parametrize("pad", [0, 1, 3, 4, 8])
def test_gemv_lda_and_alignment(lift, pad):
    m, n = 70, 3000
    A, x, y = gemv_inputs(m, n, 90 + pad)
    buf = torch.zeros(m, n + pad, dtype=torch.float32, device=DEV)
    buf[:, :n] = dev(A)
    Av = buf[:, :n]
    ref_bits = bits(lift.gemv(dev(A), dev(x), dev(y), 1.5, 0.5))
    got = lift.gemv(Av, dev(x), dev(y), 1.5, 0.5)
    assert np.array_equal(bits(got), ref_bits)  # load width never changes bits
    off = torch.zeros(m * n + 3, dtype=torch.float32, device=DEV)[1:1 + m * n].view(m, n)
    off.copy_(dev(A))
    assert np.array_equal(bits(lift.gemv(off, dev(x), dev(y), 1.5, 0.5)), ref_bits)


def test_gemv_in_place_and_zero_coeffs(lift):
    m, n = 129, 513
    A, x, y = gemv_inputs(m, n, 95)
    yd = dev(y)
    ref = oracle.gemv(A, x, y, 1.5, 0.5)
    lift.gemv(dev(A), dev(x), yd, 1.5, 0.5, out=yd)
    assert np.all(np.abs(yd.cpu().numpy() - ref) <= 1e-6 * np.abs(ref))
    # beta = 0 still reads y (literal semantics, reading R11): NaN in y propagates
    y2 = y.copy()
    y2[3] = np.nan
    got = lift.gemv(dev(A), dev(x), dev(y2), 1.0, 0.0).cpu().numpy()
    assert np.isnan(got[3]) and not np.isnan(got[4])
    got = lift.gemv(dev(A), dev(x), dev(y), 0.0, 1.0).cpu().numpy()
    assert np.array_equal(got, y)


def test_gemv_rows_independent_of_m(lift):
    """A row's bits do not depend on m or on which rows share a launch (sharding)."""
    m, n = 512, 2048 + 5
    A, x, y = gemv_inputs(m, n, 97)
    full = bits(lift.gemv(dev(A), dev(x), dev(y), 1.5, 0.5))
    for a, b in [(0, 1), (100, 356), (511, 512), (256, 512)]:
        part = bits(lift.gemv(dev(A[a:b]), dev(x), dev(y[a:b]), 1.5, 0.5))
        assert np.array_equal(part, full[a:b])
    try:
        lift.set_grid_limit(3)
        assert np.array_equal(bits(lift.gemv(dev(A), dev(x), dev(y), 1.5, 0.5)), full)
    finally:
        lift.set_grid_limit(0)


# ------------------------------------------------- full BASELINE sizes (device inputs)
def dev_gen(n, seed, tid, lo=-1.0, hi=1.0, dist=0):
    t = torch.empty(n, dtype=torch.float32, device=DEV)
    return gen.fill_device(t, seed, tid, 0, dist, lo, hi)


def test_full_scal_2p28_every_element(lift):
    """All 2^28 outputs compared bitwise with the oracle (in 2^24-element blocks)."""
    n = 1 << 28
    x = dev_gen(n, 0, gen.TID_X)
    y = lift.scal(3.0, x)
    xh, yh = x.cpu().numpy(), y.cpu().numpy()
    del x, y
    B = 1 << 24
    for i in range(0, n, B):
        ref = oracle.scal(3.0, xh[i:i + B]).astype(np.float32)
        assert np.array_equal(yh[i:i + B].view(np.uint32), ref.view(np.uint32)), i


def test_full_asum_2p28(lift):
    n = 1 << 28
    x = dev_gen(n, 0, gen.TID_X)
    g = lift.asum(x).item()
    o = oracle.asum(gen.host(n, 0, gen.TID_X))
    assert abs(g - o) <= 1e-5 * o


@pytest.mark.parametrize("n", [1 << 24, 1 << 26])
def test_full_dot(lift, n):
    x = dev_gen(n, 0, gen.TID_X, 0.0, 1.0)
    y = dev_gen(n, 0, gen.TID_Y, 0.0, 2.0)
    g = lift.dot(x, y).item()
    o = oracle.dot(gen.host(n, 0, gen.TID_X, lo=0.0, hi=1.0),
                   gen.host(n, 0, gen.TID_Y, lo=0.0, hi=2.0))
    assert abs(g - o) <= 1e-5 * o


def test_full_gemv_8192(lift):
    m = n = 8192
    A = dev_gen(m * n, 0, gen.TID_A, 0.0, 3.0).view(m, n)
    x = dev_gen(n, 0, gen.TID_X, 0.0, 1.0)
    y = dev_gen(m, 0, gen.TID_Y, 0.0, 2.0)
    got = lift.gemv(A, x, y, 1.5, 0.5).cpu().numpy()
    ref = oracle.gemv(gen.host(m * n, 0, gen.TID_A, lo=0.0, hi=3.0).reshape(m, n),
                      gen.host(n, 0, gen.TID_X, lo=0.0, hi=1.0),
                      gen.host(m, 0, gen.TID_Y, lo=0.0, hi=2.0), 1.5, 0.5)
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref))


@pytest.mark.parametrize("m,n", [(4096, 4096), (8192, 16384)])
def test_full_gemv_paper_sizes(lift, m, n):
    """The paper's own gemv inputs (reading R12): 4096^2 and 8192 x 16384 (the
    x-through-L1 path), every element against the oracle at plain relative 1e-6."""
    A = dev_gen(m * n, 1, gen.TID_A, 0.0, 3.0).view(m, n)
    x = dev_gen(n, 1, gen.TID_X, 0.0, 1.0)
    y = dev_gen(m, 1, gen.TID_Y, 0.0, 2.0)
    got = lift.gemv(A, x, y, 1.5, 0.5).cpu().numpy()
    ref = oracle.gemv(gen.host(m * n, 1, gen.TID_A, lo=0.0, hi=3.0).reshape(m, n),
                      gen.host(n, 1, gen.TID_X, lo=0.0, hi=1.0),
                      gen.host(m, 1, gen.TID_Y, lo=0.0, hi=2.0), 1.5, 0.5)
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref))


def test_full_dot_2p31(lift):
    """C5 at full size on one GPU (16 GiB of inputs); the oracle streams the same
    seeded values from the host generator block by block."""
    n = 1 << 31
    x = dev_gen(n, 0, gen.TID_X, 0.0, 1.0)
    y = dev_gen(n, 0, gen.TID_Y, 0.0, 2.0)
    g = lift.dot(x, y).item()
    del x, y
    torch.cuda.empty_cache()
    s = oracle.Stream()
    blk = 1 << 25
    xb = np.empty(blk, np.float32)
    yb = np.empty(blk, np.float32)
    for a in range(0, n, blk):
        gen.fill_host(xb, 0, gen.TID_X, a, gen.DIST_UNIFORM, 0.0, 1.0)
        gen.fill_host(yb, 0, gen.TID_Y, a, gen.DIST_UNIFORM, 0.0, 2.0)
        s.dot(xb, yb)
    o = s.value()
    assert abs(g - o) <= 1e-5 * o


# ------------------------------ canonical order: bits depend on n only (rounded sums)
def rough(n, seed, lo_exp=-20, hi_exp=20):
    """Full-mantissa values over a wide exponent range: fp64 sums of their products
    round, so any change of summation order shows up in the bits (the 2^-24-grid
    generator inputs sum exactly and cannot detect it)."""
    r = np.random.default_rng(seed)
    v = r.standard_normal(n) * np.exp2(r.integers(lo_exp, hi_exp, n))
    return v.astype(np.float32)


@pytest.mark.parametrize("m,n", [(300, 8192), (70, 3001), (130, 16384 + 9), (9, 5)])
def test_gemv_order_depends_on_n_only(lift, m, n):
    A = rough(m * n, 1).reshape(m, n)
    x, y = rough(n, 2), rough(m, 3)
    ref = bits(lift.gemv(dev(A), dev(x), dev(y), 1.5, 0.5))
    check_gemv(lift.gemv(dev(A), dev(x), dev(y), 1.5, 0.5).cpu().numpy(), A, x, y, 1.5, 0.5)
    # load width / alignment: A offset by 1 and 4 floats, padded lda, x offset
    for off, pad in [(1, 0), (4, 0), (0, 3), (0, 8)]:
        buf = torch.zeros(m * (n + pad) + off + 8, dtype=torch.float32, device=DEV)
        Av = buf[off:off + m * (n + pad)].view(m, n + pad)[:, :n]
        Av.copy_(dev(A))
        xb = torch.zeros(n + 8, dtype=torch.float32, device=DEV)
        xv = xb[off:off + n]
        xv.copy_(dev(x))
        assert np.array_equal(bits(lift.gemv(Av, xv, dev(y), 1.5, 0.5)), ref), (off, pad)
    # row subsets (sharding) and a capped grid
    for a, b in [(0, 1), (m // 3, m // 3 + 7), (m - 1, m)]:
        assert np.array_equal(bits(lift.gemv(dev(A[a:b]), dev(x), dev(y[a:b]), 1.5, 0.5)), ref[a:b])
    try:
        lift.set_grid_limit(2)
        assert np.array_equal(bits(lift.gemv(dev(A), dev(x), dev(y), 1.5, 0.5)), ref)
    finally:
        lift.set_grid_limit(0)


@pytest.mark.parametrize("n", [3001, (1 << 21) + 7])
def test_reduce_order_depends_on_n_only(lift, n):
    x, y = rough(n, 4), rough(n, 5)
    ra, rd = bits(lift.asum(dev(x))), bits(lift.dot(dev(x), dev(y)))
    for off in (1, 4):
        xb = torch.zeros(n + 8, dtype=torch.float32, device=DEV)
        yb = torch.zeros(n + 8, dtype=torch.float32, device=DEV)
        xv, yv = xb[off:off + n], yb[off:off + n]
        xv.copy_(dev(x))
        yv.copy_(dev(y))
        assert np.array_equal(bits(lift.asum(xv)), ra)
        assert np.array_equal(bits(lift.dot(xv, yv)), rd)
    try:
        lift.set_grid_limit(3)
        assert np.array_equal(bits(lift.asum(dev(x))), ra)
        assert np.array_equal(bits(lift.dot(dev(x), dev(y))), rd)
    finally:
        lift.set_grid_limit(0)


# ------------------------------------------- gemv long rows (n >= 65536): the dot order
@pytest.mark.parametrize("m,n", [(1, 1 << 16), (3, (1 << 20) + 5), (7, 200003), (40, 70000)])
def test_gemv_long_rows_equal_dot_bits(lift, m, n):
    A = rough(m * n, 11).reshape(m, n)
    x = rough(n, 12)
    y = rough(m, 13)
    Ad, xd = dev(A), dev(x)
    g = bits(lift.gemv(Ad, xd, dev(y), 1.0, 0.0))          # fp32(1 * d + 0 * y) = fp32(d)
    d = np.concatenate([bits(lift.dot(Ad[i], xd)) for i in range(m)])
    assert np.array_equal(g, d)
    check_gemv(lift.gemv(Ad, xd, dev(y), -1.5, 0.25).cpu().numpy(), A, x, y, -1.5, 0.25)
    # split path (workspace) == one CTA per row
    assert np.array_equal(bits(lift.gemv(Ad, xd, dev(y), -1.5, 0.25)),
                          bits(lift.gemv(Ad, xd, dev(y), -1.5, 0.25, split=False)))


def test_gemv_long_rows_many_rows_and_ws_reuse(lift):
    """Many long rows take the one-CTA-per-row kernel, a few take the split kernel: the
    same rows give the same bits; the split workspace is reused across shapes."""
    n = 65536 + 77
    m = 700
    A = dev(rough(m * n, 21).reshape(m, n))
    x, y = dev(rough(n, 22)), dev(rough(m, 23))
    full = bits(lift.gemv(A, x, y, 1.5, 0.5))
    for a, b in [(0, 3), (5, 6), (600, 700), (1, 300)]:
        assert np.array_equal(bits(lift.gemv(A[a:b], x, y[a:b], 1.5, 0.5)), full[a:b]), (a, b)
    for _ in range(3):
        assert np.array_equal(bits(lift.gemv(A[:2], x, y[:2], 1.5, 0.5)), full[:2])
        xs = dev(rough(1 << 20, 24))
        As = dev(rough(2 << 20, 25).reshape(2, 1 << 20))
        s1 = bits(lift.gemv(As, xs, y[:2], 1.0, 0.0))
        assert np.array_equal(s1, np.concatenate([bits(lift.dot(As[i], xs)) for i in range(2)]))


@pytest.mark.parametrize("n", [5, 24, 300, 3001, 8192 + 3, 70001])
def test_gemv_special_values_stay_in_their_row(lift, n):
    """NaN / Inf placed at the first column, the last column (the masked last batch or the
    partial last vector) and mid-row reach exactly their own row, for every threads-per-row
    class and the long-row path; Inf x 0 gives NaN as in the oracle."""
    m = 9
    A, x, y = gemv_inputs(m, n, 123)
    A = A.copy()
    x = x.copy()
    A[1, 0] = np.nan
    A[3, n - 1] = np.inf
    A[5, n // 2] = -np.inf
    A[7, n - 1] = np.inf
    x[n - 1] = 0.0 if n > 1 else x[n - 1]   # row 7: Inf * 0 = NaN; row 3 too
    got = lift.gemv(dev(A), dev(x), dev(y), 1.5, 0.5).cpu().numpy()
    ref = oracle.gemv(A, x, y, 1.5, 0.5).astype(np.float32)
    for i in range(m):
        if np.isnan(ref[i]):
            assert np.isnan(got[i]), i
        elif np.isinf(ref[i]):
            assert got[i] == ref[i], i
        else:
            assert np.isfinite(got[i]) and abs(got[i] - ref[i]) <= 1e-6 * abs(ref[i]), i
    assert np.isnan(got[1]) and np.isinf(got[5]) and got[5] < 0


def test_gemv_ws_too_small_or_null_falls_back_with_same_bits(lift):
    """lift_gemv_ws contract: a NULL or too-small workspace selects one CTA per row."""
    from paper_1502_02389_b200._lib import lib
    m, n = 3, 70001
    A = dev(rough(m * n, 31).reshape(m, n))
    x, y = dev(rough(n, 32)), dev(rough(m, 33))
    want = bits(lift.gemv(A, x, y, 1.5, 0.5))
    stream = torch.cuda.current_stream().cuda_stream
    small = torch.zeros(64, dtype=torch.uint8, device=DEV)
    for wp, wb in [(None, 0), (small.data_ptr(), small.numel())]:
        out = torch.full((m,), float("nan"), device=DEV)
        assert lib.lift_gemv_ws(m, n, 1.5, A.data_ptr(), n, x.data_ptr(), 0.5, y.data_ptr(),
                                out.data_ptr(), wp, wb, stream) == 0
        torch.cuda.synchronize()
        assert np.array_equal(bits(out), want)


def test_workspace_reset_restores_the_contract(lift):
    """A dirty ticket (the contract broken) is repaired by Workspace.reset(): the next
    call is correct again (bit-identical to a fresh workspace)."""
    n = 3 * GROUP + 5
    x = dev_gen(n, 4, gen.TID_X)
    ws = lift.Workspace(n, torch.device(DEV))
    good = lift.asum(x, ws=ws).item()
    wf = ws.nbytes & ~15
    region = ((wf // 512 + 2) * 4 + 15) & ~15
    t0 = wf - region
    assert ws.check()  # lift_workspace_check: every ticket zero after complete calls
    ws.buf[t0:t0 + 4].view(torch.int32).fill_(5)
    assert not ws.check()  # the broken contract is detected on the host
    lift.asum(x, ws=ws)
    ws.reset()
    assert ws.check()
    assert lift.asum(x, ws=ws).item() == good
    for k in (1, region // 4 - 1):  # any ticket of the region, not only the first
        ws.buf[t0 + 4 * k:t0 + 4 * k + 4].view(torch.int32).fill_(1)
        assert not ws.check()
        ws.reset()


# ---------------- accuracy beyond the bar: one fp32 rounding of an fp64-exact fold
def _ulp32(o):
    """The spacing of fp32 values at |o| (np.spacing of the fp32 rounding of o)."""
    return np.abs(np.spacing(np.abs(np.asarray(o, dtype=np.float64)).astype(np.float32))).astype(np.float64)


@pytest.mark.parametrize("op,n,lo", [("asum", 1 << 24, -1.0), ("dot", 1 << 26, -1.0),
                                     ("dot", 1 << 24, 0.0), ("asum", (1 << 22) + 77, -1.0)])
def test_reductions_within_one_fp32_ulp(lift, op, n, lo):
    """The kernels fold in fp64 (exact products for dot) and round once (reading R13), so
    their result is within one fp32 ulp of the fp64 oracle — far inside BASELINE's 1e-5 —
    signed inputs included."""
    xh = gen.host(n, 11, gen.TID_X, lo=lo, hi=1.0)
    if op == "asum":
        g, o = lift.asum(dev(xh)).item(), oracle.asum(xh)
    else:
        yh = gen.host(n, 11, gen.TID_Y, lo=lo, hi=2.0)
        g, o = lift.dot(dev(xh), dev(yh)).item(), oracle.dot(xh, yh)
    assert abs(g - o) <= _ulp32(o), (g, o)


@pytest.mark.parametrize("m,n,alpha,beta,lo", [(4096, 4096, 1.5, 0.5, 0.0), (1000, 8192, -1.25, 0.75, -1.0)])
def test_gemv_within_one_fp32_ulp(lift, m, n, alpha, beta, lo):
    """Every gemv element within one fp32 ulp of the oracle (exact products, fp64 row
    folds, the epilogue in fp64 rounded once: reading R10/R13)."""
    A = gen.host(m * n, 12, gen.TID_A, lo=lo, hi=3.0).reshape(m, n)
    x = gen.host(n, 12, gen.TID_X, lo=lo, hi=1.0)
    y = gen.host(m, 12, gen.TID_Y, lo=lo, hi=2.0)
    got = lift.gemv(dev(A), dev(x), dev(y), alpha, beta).cpu().numpy().astype(np.float64)
    ref = oracle.gemv(A, x, y, alpha, beta)
    assert np.all(np.abs(got - ref) <= _ulp32(ref))
