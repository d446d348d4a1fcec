"""Programmatic dependent launch: every lift kernel is launched with programmatic stream
serialization and may start while the previous kernel on the stream still runs; its
first statement, griddepcontrol.wait, must hold it until that kernel's writes are
visible.  These chains make each launch consume the previous launch's output, back to
back on one stream with no host synchronisation in between, and compare with the same
chain computed with a synchronisation after every call.

Negative control (run once by hand): a build whose pdl_wait() is empty but still
launches with the attribute fails test_consumer_reads_what_the_producer_writes_last."""
import numpy as np
import pytest
import torch

import lift_inputs as gen

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def lift():
    import paper_1502_02389_b200 as m
    return m


def bits(t):
    return t.cpu().numpy().view(np.uint32)


def test_lift_to_lift_chain(lift):
    """scal writes y, asum/dot read y, gemv reads y as its x, the next scal reads gemv's
    output region... each step depends on the previous kernel's stores."""
    n = (1 << 22) + 77
    x = gen.fill_device(torch.empty(n, device=DEV), 1, gen.TID_X, 0, 0, -1.0, 1.0)
    m, k = 512, 8192
    A = gen.fill_device(torch.empty(m * k, device=DEV), 1, gen.TID_A, 0, 0, 0.0, 3.0).view(m, k)

    def chain(sync):
        y = torch.empty(n, device=DEV)
        r1 = torch.empty(1, device=DEV)
        r2 = torch.empty(1, device=DEV)
        g = torch.empty(m, device=DEV)
        outs = []
        cur = x
        for it in range(6):
            lift.scal(1.0 + 0.25 * it, cur, out=y)            # y <- a * cur
            sync and torch.cuda.synchronize()
            lift.asum(y, out=r1)                               # reads y
            sync and torch.cuda.synchronize()
            lift.dot(y, x, out=r2)                             # reads y
            sync and torch.cuda.synchronize()
            lift.gemv(A, y[:k], y[k:k + m], 1.5, 0.5, out=g)   # x and y of gemv from scal's y
            sync and torch.cuda.synchronize()
            outs += [r1.clone(), r2.clone(), g.clone()]
            cur = y.clone()
            sync and torch.cuda.synchronize()
        torch.cuda.synchronize()
        return [bits(o) for o in outs]

    ref = chain(True)
    for _ in range(3):
        got = chain(False)
        for a, b in zip(ref, got):
            assert np.array_equal(a, b)


def test_torch_to_lift_and_back(lift):
    """A torch kernel (launched without the attribute) writes the input, lift reads it at
    once; lift writes, a torch kernel reads at once."""
    n = 3 << 20
    x = torch.empty(n, device=DEV)
    r = torch.empty(64, device=DEV)
    y = torch.empty(n, device=DEV)
    for i in range(64):
        x.fill_(float(i % 7) - 3.0)        # torch writes
        lift.asum(x, out=r[i:i + 1])        # lift reads immediately
        lift.scal(2.0, x, out=y)            # lift writes
        r[i:i + 1] += y[:1] * 0.0           # torch reads y right after
    torch.cuda.synchronize()
    want = np.array([abs(float(i % 7) - 3.0) * n for i in range(64)], np.float32)
    assert np.array_equal(r.cpu().numpy(), want)
    assert torch.all(y == 2.0 * (float(63 % 7) - 3.0))


def test_consumer_reads_what_the_producer_writes_last(lift):
    """The race window of an early start: a reduction's result is written by its LAST
    CTA, and the tail of scal's output by its last CTAs; the next launch reads exactly
    those first (a 1-element scal of the result; gemv with x = the tail of y)."""
    n = 1 << 24
    k, m = 8192, 64
    A = gen.fill_device(torch.empty(m * k, device=DEV), 2, gen.TID_A, 0, 0, 0.0, 3.0).view(m, k)
    xs = [gen.fill_device(torch.empty(n, device=DEV), s, gen.TID_X, 0, 0, -1.0, 1.0)
          for s in range(4)]
    reps = 40
    r = torch.full((reps,), float("nan"), device=DEV)
    s = torch.full((reps,), float("nan"), device=DEV)
    y = torch.empty(n, device=DEV)
    g = torch.full((reps, m), float("nan"), device=DEV)
    for i in range(reps):
        xi = xs[i % 4]
        lift.asum(xi, out=r[i:i + 1])                      # result stored by the last CTA
        lift.scal(2.0, r[i:i + 1], out=s[i:i + 1])          # reads it at once
        lift.scal(1.0 + i, xi, out=y)                       # tail of y written last
        lift.gemv(A, y[n - k:], y[n - k - m:n - k], 1.0, 1.0, out=g[i])  # reads the tail first
    torch.cuda.synchronize()
    want_r = [lift.asum(xs[i % 4]).item() for i in range(reps)]
    assert np.array_equal(r.cpu().numpy(), np.array(want_r, np.float32))
    assert np.array_equal(s.cpu().numpy(), 2.0 * np.array(want_r, np.float32))
    for i in range(reps):
        yi = lift.scal(1.0 + i, xs[i % 4])
        want = lift.gemv(A, yi[n - k:], yi[n - k - m:n - k], 1.0, 1.0)
        assert np.array_equal(bits(g[i]), bits(want)), i
