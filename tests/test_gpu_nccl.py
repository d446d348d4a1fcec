"""The X1 'nccl' path through a real NCCL process group.  One GPU allows one NCCL rank, so
the group has world size 1 — the all-gathers still run as NCCL collectives on the device
(dist.py no longer short-cuts p = 1 when a group exists), followed by lift_combine; the
results must equal the unsharded calls bit for bit and the oracle within tolerance."""
import os
import socket

import numpy as np
import pytest
import torch

import lift_inputs as gen
import oracle

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_world1_sharded_path():
    import torch.distributed as dist

    import paper_1502_02389_b200 as lift
    from paper_1502_02389_b200 import dist as ldist
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        assert dist.get_backend() == "nccl"
        n = 3 * lift.GROUP_ELEMS + 77
        xh, yh = gen.host(n, 2, gen.TID_X), gen.host(n, 2, gen.TID_Y)
        x, y = torch.from_numpy(xh).to(dev), torch.from_numpy(yh).to(dev)
        ra, rd = ldist.sharded_asum(x), ldist.sharded_dot(x, y)
        assert ra.item() == lift.asum(x).item() and rd.item() == lift.dot(x, y).item()
        assert abs(ra.item() - oracle.asum(xh)) <= 1e-5 * oracle.asum(xh)
        assert abs(rd.item() - oracle.dot(xh, yh)) <= 1e-5 * abs(oracle.dot(xh, yh))
        m, k = 300, 8192
        A = gen.fill_device(torch.empty(m * k, device=dev), 2, gen.TID_A, 0).view(m, k)
        gx = gen.fill_device(torch.empty(k, device=dev), 2, gen.TID_X, 0)
        gy = gen.fill_device(torch.empty(m, device=dev), 2, gen.TID_Y, 0)
        yf = ldist.sharded_gemv(A, gx, gy, 1.5, 0.5, m)
        assert torch.equal(yf.view(torch.int32), lift.gemv(A, gx, gy, 1.5, 0.5).view(torch.int32))
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()
