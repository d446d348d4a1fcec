"""gemv under repetition: many launches into NaN-filled outputs at shapes with thousands
of row blocks per launch must write every row, with the same bits every time.

(History: an earlier gemv design stole row blocks with Cluster Launch Control; without a
proxy fence between reading the CLC response and the next try_cancel, 25 of 400
launches at 8192 x 8192 left one warp's rows unwritten.  Tolerance tests on recycled
output buffers had passed; this test is what caught it, and it stays for any
scheduling change.)"""
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


@pytest.mark.parametrize("m,n,runs", [(8192, 4096, 300), (8192, 8192, 200), (1024, 8192, 200),
                                      (4096, 8192, 200), (8192, 16384, 60)])
def test_gemv_repeated_launches_write_every_row_identically(lift, m, n, runs):
    A = gen.fill_device(torch.empty(m * n, device=DEV), 0, gen.TID_A, 0, 0, 0.0, 3.0).view(m, n)
    x = gen.fill_device(torch.empty(n, device=DEV), 0, gen.TID_X, 0, 0, 0.0, 1.0)
    y = gen.fill_device(torch.empty(m, device=DEV), 0, gen.TID_Y, 0, 0, 0.0, 2.0)
    outs = torch.full((runs, m), float("nan"), device=DEV)
    for i in range(runs):
        lift.gemv(A, x, y, 1.5, 0.5, out=outs[i])
    torch.cuda.synchronize()
    o = outs.cpu().numpy().view(np.uint32)
    assert not np.isnan(outs.cpu().numpy()).any(), "some launch left rows unwritten"
    bad = np.nonzero((o != o[0]).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} of {runs} launches differ from the first"
