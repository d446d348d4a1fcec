"""Multi-process (world_size 2, gloo, CPU) checks of the sharding layer's host logic:
shard arithmetic, rank-ordered gathers of partials and of gemv row slices.  The same
code runs with NCCL on GPUs (bench.py, N > 1); the combine there is lift_combine."""
import os
import socket
import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1502_02389_b200.dist import (GROUP_ELEMS, gather_partials, gather_rows, row_range,
                                        shard_range)


@pytest.mark.parametrize("n", [0, 1, 5, 1000, GROUP_ELEMS - 1, GROUP_ELEMS * 2,
                               GROUP_ELEMS * 8 + 3, 1 << 31])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_range_tiles_exactly(n, world):
    prev = 0
    for r in range(world):
        a, b = shard_range(n, r, world)
        assert a == prev and b >= a
        prev = b
    assert prev == n
    if n >= GROUP_ELEMS * world:
        for r in range(world):
            assert shard_range(n, r, world)[0] % GROUP_ELEMS == 0


def test_power_of_two_shards_hold_power_of_two_groups():
    # the bit-exact composition condition (reading R5)
    n = 1 << 31
    for world in (1, 2, 4, 8):
        a, b = shard_range(n, 0, world)
        groups = (b - a) // GROUP_ELEMS
        assert groups & (groups - 1) == 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pairwise(vals):
    """Pairwise fold zero-padded to a power of two (the combine's documented order)."""
    v = list(vals)
    p2 = 1
    while p2 < len(v):
        p2 *= 2
    v += [0.0] * (p2 - len(v))
    while len(v) > 1:
        v = [v[i] + v[i + 1] for i in range(0, len(v), 2)]
    return v[0]


def _worker(rank, world, port, q):
    import oracle
    import lift_inputs as gen
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n = 300_001
        a, b = shard_range(n, rank, world)
        xs = gen.host(b - a, 5, gen.TID_X, i0=a)
        ys = gen.host(b - a, 5, gen.TID_Y, i0=a)
        # asum / dot: one fp64 partial per rank, gathered in rank order
        pa = gather_partials(torch.tensor([oracle.asum(xs)], dtype=torch.float64))
        pd = gather_partials(torch.tensor([oracle.dot(xs, ys)], dtype=torch.float64))
        # gemv: uneven row split gathered back into the full y
        m = 7
        r0, r1 = row_range(m, rank, world)
        ysl = torch.arange(r0, r1, dtype=torch.float32) * 10
        full = gather_rows(ysl, m)
        q.put((rank, pa.tolist(), pd.tolist(), full.tolist(), (a, b)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface errors to the parent
        q.put((rank, "error", repr(e), None, None))


def test_gloo_world2_gathers_in_rank_order():
    import oracle
    import lift_inputs as gen
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert res[r][1] != "error", res[r][2]
    n = 300_001
    x = gen.host(n, 5, gen.TID_X)
    y = gen.host(n, 5, gen.TID_Y)
    # every rank holds the same rank-ordered partials
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]
    for r in range(world):
        a, b = res[r][4]
        assert res[0][1][r] == oracle.asum(x[a:b])
    # the pairwise combine of shard partials agrees with the unsharded definition
    assert abs(_pairwise(res[0][1]) - oracle.asum(x)) <= 1e-12 * oracle.asum(x)
    assert abs(_pairwise(res[0][2]) - oracle.dot(x, y)) <= 1e-12 * oracle.dot(np.abs(x), np.abs(y))
    # gemv row gather reproduces the full y in order
    assert res[0][3] == res[1][3] == [10.0 * i for i in range(7)]
