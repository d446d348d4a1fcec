"""X1 on the GPU: the sharded path (dist.py) with real lift kernels, two processes.

Only one GPU is available, and NCCL refuses two ranks on one device, so both ranks run
on cuda:0 with the gloo backend (which gathers CUDA tensors through the host).  Every
kernel is the real one (lift_*_partial, lift_combine, lift_gemv); only the transport
differs from the NCCL runs.  Bars: each rank gets the SAME bits, and those bits equal
the unsharded call (shards are a power-of-two number of canonical groups); gemv row
slices gather to the unsharded y_out bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import lift_inputs as gen
    import paper_1502_02389_b200 as lift
    from paper_1502_02389_b200 import dist as ldist
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dev = torch.device("cuda:0")
        n = 8 * lift.GROUP_ELEMS  # 8 canonical groups -> 4 per rank
        a, b = ldist.shard_range(n, rank, world)
        x = gen.fill_device(torch.empty(b - a, device=dev), 3, gen.TID_X, a)
        y = gen.fill_device(torch.empty(b - a, device=dev), 3, gen.TID_Y, a)
        ra = ldist.sharded_asum(x)
        rd = ldist.sharded_dot(x, y)
        m, k = 1000, 777
        r0, r1 = ldist.row_range(m, rank, world)
        A = gen.fill_device(torch.empty((r1 - r0) * k, device=dev), 3, gen.TID_A, r0 * k).view(-1, k)
        gx = gen.fill_device(torch.empty(k, device=dev), 3, gen.TID_X, 0)
        gy = gen.fill_device(torch.empty(r1 - r0, device=dev), 3, gen.TID_Y, r0)
        yfull = ldist.sharded_gemv(A, gx, gy, 1.5, 0.5, m)
        q.put((rank, ra.cpu().numpy().view(np.uint32).tolist(),
               rd.cpu().numpy().view(np.uint32).tolist(),
               yfull.cpu().numpy().view(np.uint32).tolist()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface errors to the parent
        q.put((rank, "error", repr(e), None))


def test_sharded_path_two_processes_one_gpu():
    import lift_inputs as gen
    import paper_1502_02389_b200 as lift
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert res[r][1] != "error", res[r][2]
    assert res[0][1:] == res[1][1:]  # every rank holds the same bits
    dev = torch.device("cuda:0")
    n = 8 * lift.GROUP_ELEMS
    x = gen.fill_device(torch.empty(n, device=dev), 3, gen.TID_X, 0)
    y = gen.fill_device(torch.empty(n, device=dev), 3, gen.TID_Y, 0)
    assert res[0][1] == lift.asum(x).cpu().numpy().view(np.uint32).tolist()
    assert res[0][2] == lift.dot(x, y).cpu().numpy().view(np.uint32).tolist()
    m, k = 1000, 777
    A = gen.fill_device(torch.empty(m * k, device=dev), 3, gen.TID_A, 0).view(m, k)
    gx = gen.fill_device(torch.empty(k, device=dev), 3, gen.TID_X, 0)
    gy = gen.fill_device(torch.empty(m, device=dev), 3, gen.TID_Y, 0)
    full = lift.gemv(A, gx, gy, 1.5, 0.5)
    assert res[0][3] == full.cpu().numpy().view(np.uint32).tolist()
