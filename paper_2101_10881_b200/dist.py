"""Multi-GPU plumbing: one process per GPU, torch.distributed for the
barrier / timing reductions only.

The evaluation of independent points shards with no
data-path collective: each rank owns a contiguous range of points, keeps the
graph and coefficient slabs replicated, and produces bit-identical results to
a single GPU. Partial value/gradient series are never summed with NCCL's
native sum (it would add limbs as plain doubles); when one consumer needs all
points, ``gather_points`` moves the finished series with an all-gather.
"""
from __future__ import annotations

import os
from typing import Tuple


def env_rank() -> Tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def point_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [begin, end) share of `total` points for `rank`; sizes differ
    by at most one, lower ranks take the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(total, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def init(backend: str):
    import torch.distributed as dist

    if dist.is_available() and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend)
    return dist


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def connect_peers(plan) -> bool:
    """Map every other rank's arena into this plan (CUDA IPC handles
    exchanged over the process group once): NVLink peer memory between the
    GPUs of a node, plain device memory when ranks share a GPU. Returns
    False (and the collective exchange is used) when IPC is unavailable."""
    import torch.distributed as dist

    from ._lib import PseError

    world = plan.nranks
    try:
        mine = plan.ipc_handle()
    except PseError:
        mine = b""
    handles = [None] * world
    dist.all_gather_object(handles, mine)
    ok = all(h for h in handles)
    if ok:
        try:
            for r, h in enumerate(handles):
                if r != plan.rank:
                    plan.open_peer(r, h)
        except PseError:
            ok = False
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    return all(flags)


def evaluate_sharded(plan, batch: int = 1, detail: bool = True, p2p: bool = False):
    """One evaluation of a polynomial sharded over the process group: this
    rank's conv share, the exchange of the addition-stage term slots (a pure
    copy of limbs), then the exact addition tree on every rank. The exchange
    is either the peer gather (p2p, after connect_peers: every rank reads the
    slots it lacks straight from the peers' arenas, between two barriers) or
    an all-gather of packed blocks (NCCL over NVLink on GPUs, gloo through
    host memory when several ranks share a device).

    Returns (conv_report, finish_report). The finish report's times come from
    the kernels' %globaltimer stamps on this rank's device: conv_ms (the conv
    stage), exchange_ms (conv end -> first addition-stage kernel: the barriers
    and the gather), add_ms, and wall_ms (conv start -> last addition layer)."""
    import torch
    import torch.distributed as dist

    world = plan.nranks
    dev = torch.device(f"cuda:{plan.device}")
    rep = plan.execute(batch)  # returns once the conv stage has finished
    if p2p and world > 1:
        dist.barrier()  # every rank's term slots are final
        plan.gather_peers(batch)
        dist.barrier()  # every rank has read ours before our addition tree rewrites them
        return rep, plan.finish(batch)
    words = [plan.exchange_words(r, batch) for r in range(world)]
    width = max(1, max(words))
    mine = torch.zeros(width, dtype=torch.float64, device=dev)
    # the zero-fill runs on torch's stream, pack on the plan's non-blocking
    # stream: order them (otherwise the fill may land after the packed slots)
    torch.cuda.current_stream(dev).synchronize()
    plan.pack(mine.data_ptr(), batch)
    on_gpu = dist.is_initialized() and dist.get_backend() == "nccl"
    if world == 1 or not dist.is_initialized():
        blocks = [mine]
    elif on_gpu:
        blocks = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(blocks, mine)
        torch.cuda.synchronize(dev)
    else:
        host = mine.cpu()
        outs = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(outs, host)
        blocks = [o.to(dev) for o in outs]
        torch.cuda.synchronize(dev)
    for r in range(world):
        if r != plan.rank:
            plan.unpack(r, blocks[r].data_ptr(), batch)
    return rep, plan.finish(batch)


def gather_points(local, total: int, device=None):
    """All-gather per-rank blocks of finished series along axis 1 (points).
    local: numpy [Q][points_local][...]; returns numpy [Q][total][...].
    A pure data movement: no arithmetic is applied to the limbs."""
    import numpy as np
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    rows = [point_range(total, r, world) for r in range(world)]
    width = max(e - b for b, e in rows)
    shape = (local.shape[0], width) + tuple(local.shape[2:])
    buf = np.zeros(shape, np.float64)
    buf[:, : local.shape[1]] = local
    t = torch.from_numpy(buf).to(device) if device is not None else torch.from_numpy(buf)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    parts = [o.cpu().numpy()[:, : e - b] for o, (b, e) in zip(outs, rows)]
    return np.concatenate(parts, axis=1)
