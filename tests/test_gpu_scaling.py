"""BASELINE configs[3] (C4: gemv 8192 x 8192 row-sharded) and configs[4] (C5: dot sharded
with a scalar combine) as 2-, 3- and 4-rank STRONG-scaling runs, checked against the ORACLE.

Only one GPU is available: both ranks run on cuda:0 as two processes with the gloo backend
(NCCL refuses two ranks on one device), so the 'nccl' X1 path's all-gathers travel through
gloo here; the kernels (lift_gemv, lift_*_partial, lift_combine) and the fused peer exchange
(lift_gemv_allgather, lift_dot_allreduce over CUDA IPC) are the real ones.

Bars (BASELINE north_star): every y element within 1e-6 relative of the fp64 oracle, the dot
within 1e-5; both X1 paths give the same bits on every rank, equal to the unsharded call
(row order / power-of-two canonical groups, R5); repeated calls with the same m
(both y banks) stay correct."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import lift_inputs as gen
import oracle

pytestmark = pytest.mark.gpu

M = N = 8192                 # C4
N5 = 1 << 28                 # C5-proportioned: 128 canonical groups, 64 per rank (2^31 at p=16)
ALPHA, BETA = 1.5, 0.5


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_1502_02389_b200 as lift
    from paper_1502_02389_b200 import dist as ldist
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        ex = ldist.PeerExchange(device=dev)
        res = {}
        # C4: rank r owns rows row_range(8192, r, 2); x replicated
        r0, r1 = ldist.row_range(M, rank, world)
        A = gen.fill_device(torch.empty((r1 - r0) * N, device=dev), 0, gen.TID_A, r0 * N,
                            gen.DIST_UNIFORM, 0.0, 3.0).view(r1 - r0, N)
        x = gen.fill_device(torch.empty(N, device=dev), 0, gen.TID_X, 0, gen.DIST_UNIFORM, 0.0, 1.0)
        y = gen.fill_device(torch.empty(r1 - r0, device=dev), 0, gen.TID_Y, r0,
                            gen.DIST_UNIFORM, 0.0, 2.0)
        yf = [ex.gemv(A, x, y, ALPHA, BETA, M, r0).clone() for _ in range(3)]  # both banks
        yn = ldist.sharded_gemv(A, x, y, ALPHA, BETA, M)
        res["c4_fused"] = [t.cpu().numpy().view(np.uint32) for t in yf]
        res["c4_nccl"] = yn.cpu().numpy().view(np.uint32)
        del A
        # C5-proportioned dot: shard_range on canonical groups
        a0, a1 = ldist.shard_range(N5, rank, world)
        xs = gen.fill_device(torch.empty(a1 - a0, device=dev), 0, gen.TID_X, a0,
                             gen.DIST_UNIFORM, 0.0, 1.0)
        ys = gen.fill_device(torch.empty(a1 - a0, device=dev), 0, gen.TID_Y, a0,
                             gen.DIST_UNIFORM, 0.0, 2.0)
        res["c5_fused"] = [ex.dot(xs, ys).cpu().numpy().view(np.uint32) for _ in range(3)]
        res["c5_nccl"] = ldist.sharded_dot(xs, ys).cpu().numpy().view(np.uint32)
        res["c5_range"] = (a0, a1)
        ex.check()
        ex.close()
        q.put((rank, res))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface errors to the parent
        import traceback
        q.put((rank, "error: " + repr(e) + traceback.format_exc()))


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r[1]
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    return res


@pytest.fixture(scope="module")
def two_rank_results():
    return _run(2)


def test_c4_two_ranks_match_oracle_and_unsharded(two_rank_results):
    import paper_1502_02389_b200 as lift
    res = two_rank_results
    # same bits on both ranks, both X1 paths, every repeated call
    for r in range(2):
        for yb in res[r]["c4_fused"]:
            assert np.array_equal(yb, res[0]["c4_nccl"])
        assert np.array_equal(res[r]["c4_nccl"], res[0]["c4_nccl"])
    got = res[0]["c4_nccl"].view(np.float32).astype(np.float64)
    A = gen.host(M * N, 0, gen.TID_A, lo=0.0, hi=3.0).reshape(M, N)
    x = gen.host(N, 0, gen.TID_X, lo=0.0, hi=1.0)
    y = gen.host(M, 0, gen.TID_Y, lo=0.0, hi=2.0)
    ref = oracle.gemv(A, x, y, ALPHA, BETA)
    assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref))
    dev = torch.device("cuda:0")
    full = lift.gemv(torch.from_numpy(A).to(dev), torch.from_numpy(x).to(dev),
                     torch.from_numpy(y).to(dev), ALPHA, BETA)
    assert np.array_equal(full.cpu().numpy().view(np.uint32), res[0]["c4_nccl"])


def test_c5_two_ranks_match_oracle_and_unsharded(two_rank_results):
    import paper_1502_02389_b200 as lift
    res = two_rank_results
    assert res[0]["c5_range"][1] == res[1]["c5_range"][0]
    for r in range(2):
        for d in res[r]["c5_fused"]:
            assert np.array_equal(d, res[0]["c5_nccl"])
        assert np.array_equal(res[r]["c5_nccl"], res[0]["c5_nccl"])
    got = float(res[0]["c5_nccl"].view(np.float32)[0])
    xh = gen.host(N5, 0, gen.TID_X, lo=0.0, hi=1.0)
    yh = gen.host(N5, 0, gen.TID_Y, lo=0.0, hi=2.0)
    ref = oracle.dot(xh, yh)
    assert abs(got - ref) <= 1e-5 * abs(ref)
    dev = torch.device("cuda:0")
    full = lift.dot(torch.from_numpy(xh).to(dev), torch.from_numpy(yh).to(dev))
    assert np.array_equal(full.cpu().numpy().view(np.uint32), res[0]["c5_nccl"])


@pytest.mark.parametrize("world", [3, 4])
def test_c4_c5_more_ranks(world):
    """Three (uneven split) and four ranks on the one GPU: gemv rows are independent, so the
    gathered y equals the unsharded call bit for bit at any split; the dot's combine is the
    pairwise tree over p partials — bit-identical to the unsharded call when every rank owns
    a power-of-two number of canonical groups (p = 4: 32 each), within 1e-5 of the oracle
    otherwise (p = 3: 43 + 43 + 42 groups)."""
    import paper_1502_02389_b200 as lift
    res = _run(world)
    for r in range(world):
        for yb in res[r]["c4_fused"]:
            assert np.array_equal(yb, res[0]["c4_nccl"])
        assert np.array_equal(res[r]["c4_nccl"], res[0]["c4_nccl"])
        for d in res[r]["c5_fused"]:
            assert np.array_equal(d, res[0]["c5_nccl"])
    dev = torch.device("cuda:0")
    A = gen.host(M * N, 0, gen.TID_A, lo=0.0, hi=3.0).reshape(M, N)
    x = gen.host(N, 0, gen.TID_X, lo=0.0, hi=1.0)
    y = gen.host(M, 0, gen.TID_Y, lo=0.0, hi=2.0)
    full = lift.gemv(torch.from_numpy(A).to(dev), torch.from_numpy(x).to(dev),
                     torch.from_numpy(y).to(dev), ALPHA, BETA)
    assert np.array_equal(full.cpu().numpy().view(np.uint32), res[0]["c4_nccl"])
    xh = gen.host(N5, 0, gen.TID_X, lo=0.0, hi=1.0)
    yh = gen.host(N5, 0, gen.TID_Y, lo=0.0, hi=2.0)
    got = float(res[0]["c5_nccl"].view(np.float32)[0])
    ref = oracle.dot(xh, yh)
    assert abs(got - ref) <= 1e-5 * abs(ref)
    if world == 4:
        fulld = lift.dot(torch.from_numpy(xh).to(dev), torch.from_numpy(yh).to(dev))
        assert np.array_equal(fulld.cpu().numpy().view(np.uint32), res[0]["c5_nccl"])
