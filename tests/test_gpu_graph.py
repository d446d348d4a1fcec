"""The path captured in a CUDA graph and replayed: every call enqueues one kernel with no
host synchronisation or allocation, and the reduction / gemv-split workspaces are left
with zeroed tickets, so a captured step replays correctly any number of times."""
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


def test_graph_replay_of_a_step(lift):
    n = (3 << 21) + 11
    m, k = 300, 8192
    x = gen.fill_device(torch.empty(n, device=DEV), 5, gen.TID_X, 0, 0, -1.0, 1.0)
    y = gen.fill_device(torch.empty(n, device=DEV), 5, gen.TID_Y, 0, 0, -1.0, 1.0)
    A = gen.fill_device(torch.empty(m * k, device=DEV), 5, gen.TID_A, 0, 0, 0.0, 3.0).view(m, k)
    Al = gen.fill_device(torch.empty(2 * (1 << 17), device=DEV), 5, gen.TID_A, 0, 0, -1.0, 1.0).view(2, -1)
    xl = gen.fill_device(torch.empty(1 << 17, device=DEV), 6, gen.TID_X, 0, 0, -1.0, 1.0)
    ys = torch.empty(n, device=DEV)
    ra, rd, rf = (torch.empty(1, device=DEV) for _ in range(3))
    g_out = torch.empty(m, device=DEV)
    gl_out = torch.empty(2, device=DEV)
    ws = lift.Workspace(n, torch.device(DEV))

    def step():
        lift.scal(3.0, x, out=ys)
        lift.asum(ys, out=ra, ws=ws)
        lift.dot(x, y, out=rd, ws=ws)
        lift.scal_asum(0.5, x, out=ys, result=rf, ws=ws)
        lift.gemv(A, x[:k], y[:m], 1.5, 0.5, out=g_out)
        lift.gemv(Al, xl, y[:2], 1.0, 0.0, out=gl_out)   # long rows: split path + workspace

    s = torch.cuda.Stream(device=DEV)
    with torch.cuda.stream(s):
        step()
        torch.cuda.synchronize()
        ref = [bits(t) for t in (ra, rd, rf, g_out, gl_out)]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        for _ in range(5):
            for t in (ra, rd, rf, g_out, gl_out):
                t.fill_(float("nan"))
            g.replay()
            torch.cuda.synchronize()
            got = [bits(t) for t in (ra, rd, rf, g_out, gl_out)]
            for a, b in zip(ref, got):
                assert np.array_equal(a, b)
