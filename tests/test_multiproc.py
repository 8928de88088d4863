"""Multi-GPU host logic on CPU: world_size-2 process groups over gloo.

Points of a batch shard across ranks with no data-path collective
(SURVEY.md 8(e)); each rank's share, the max-over-ranks timing reduction and
the all-gather of finished value/gradient series are checked against a
single-process run. The per-point arithmetic here is the CPU oracle -- the
GPU engine is covered by the -m gpu tests; this file tests the plumbing."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2101_10881_b200 import dist as D


def test_point_range_partitions_exactly():
    for total in (0, 1, 5, 8, 1024, 1023):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                b, e = D.point_range(total, r, world)
                assert 0 <= b <= e <= total
                seen += list(range(b, e))
            assert seen == list(range(total))
            sizes = [D.point_range(total, r, world)[1] - D.point_range(total, r, world)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _points(total):
    import pyoracle as po

    base = po.gen_benchmark("p1", 4, 2, seed=7)
    out = []
    for b in range(total):
        zb = po.gen_benchmark("p1", 4, 2, seed=1000 + b)
        st = base.stat.copy()
        st[:, :, 1 + base.N:] = zb.stat[:, :, 1 + base.N:]
        out.append(po.Problem(base.n, base.d, base.m, False, base.nvars, base.idx, None, st))
    return out


def _worker(rank, world, port, total, outdir):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import pyoracle as po
    from paper_2101_10881_b200 import dist as DD

    dist = DD.init("gloo")
    b, e = DD.point_range(total, rank, world)
    probs = _points(total)[b:e]
    local = np.stack([po.evaluate(p, "port").reshape(2, 17, 5) for p in probs], axis=1)  # [Q][pts][n+1][d+1]
    allv = DD.gather_points(local, total)
    slowest = DD.max_over_ranks(float(rank + 1))
    count = DD.sum_over_ranks(float(e - b))
    if rank == 0:
        np.save(os.path.join(outdir, "gathered.npy"), allv)
        np.save(os.path.join(outdir, "scalars.npy"), np.array([slowest, count]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_points_gloo_world2():
    total = 5
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(2, _free_port(), total, tmp), nprocs=2, join=True)
        got = np.load(os.path.join(tmp, "gathered.npy"))
        slowest, count = np.load(os.path.join(tmp, "scalars.npy"))
    import pyoracle as po

    want = np.stack([po.evaluate(p, "port").reshape(2, 17, 5) for p in _points(total)], axis=1)
    assert got.shape == want.shape
    assert (got.view(np.uint64) == want.view(np.uint64)).all()  # bit-identical to one process
    assert slowest == 2.0 and count == total


class _FakePlan:
    """stands in for a sharded DevicePlan in connect_peers (host logic only)"""

    def __init__(self, rank, world, fail_rank):
        self.rank, self.nranks, self.fail_rank = rank, world, fail_rank
        self.opened = {}

    def ipc_handle(self):
        from paper_2101_10881_b200._lib import PseError

        if self.rank == self.fail_rank:
            raise PseError(-2, "no IPC on this device")
        return bytes([self.rank + 1]) * 64

    def open_peer(self, r, h):
        self.opened[r] = h


def _peer_worker(rank, world, port, fail_rank, outdir):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2101_10881_b200 import dist as DD

    dist = DD.init("gloo")
    plan = _FakePlan(rank, world, fail_rank)
    ok = DD.connect_peers(plan)
    np.save(os.path.join(outdir, f"r{rank}.npy"),
            np.array([int(ok)] + [plan.opened.get(r, b"\0")[0] for r in range(world)]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("fail_rank", [-1, 1])
def test_connect_peers_exchanges_handles_and_agrees_on_fallback(fail_rank):
    """every rank maps every other rank's handle; if any rank cannot export
    one, all ranks agree to fall back to the collective exchange"""
    world = 3
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_peer_worker, args=(world, _free_port(), fail_rank, tmp), nprocs=world, join=True)
        res = [np.load(os.path.join(tmp, f"r{r}.npy")) for r in range(world)]
    for r, v in enumerate(res):
        assert v[0] == (fail_rank < 0)
        if fail_rank < 0:
            assert [int(x) for x in v[1:]] == [0 if q == r else q + 1 for q in range(world)]


def _reps_worker(rank, world, port, outdir):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    from paper_2101_10881_b200 import dist as DD

    dist = DD.init("gloo")
    # ranks measure different evaluation times; a sharded evaluation has
    # collectives, so every rank must repeat it the same number of times
    reps = bench.repeat_count([0.2, 5.0][rank % 2])
    np.save(os.path.join(outdir, f"reps{rank}.npy"), np.array([reps]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_bench_repeat_count_agrees_across_ranks():
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_reps_worker, args=(2, _free_port(), tmp), nprocs=2, join=True)
        reps = [int(np.load(os.path.join(tmp, f"reps{r}.npy"))[0]) for r in range(2)]
    assert reps == [125, 125]
