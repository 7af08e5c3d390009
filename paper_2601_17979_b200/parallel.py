"""Multi-GPU batch splitting: problems are independent, so a batch
is partitioned into contiguous shards, one per rank (one process per GPU); no
collective is on the data path.  An optional gather brings the factors to one
rank (torch.distributed: NCCL over NVLink on the GPU box, gloo in the CPU tests).

The reference has no parallelism at all (src/batch.py:113-142 steps every
problem sequentially); the contract kept here is "batch == standalone": a
problem's factors do not depend on which rank solved it.
"""

from __future__ import annotations

import numpy as np


def shard(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous near-equal slice [start, stop) of `batch` problems for `rank`."""
    if world < 1 or not (0 <= rank < world) or batch < 0:
        raise ValueError(f"bad shard request batch={batch} rank={rank} world={world}")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    stop = start + base + (1 if rank < extra else 0)
    return start, stop


def gather_to_root(local: np.ndarray, batch: int, group=None, root: int = 0):
    """Gather per-rank shards (leading axis = problems) into the full batch on `root`.

    Uses torch.distributed.gather_object-free tensor collectives so it runs on
    gloo (CPU) and NCCL (GPU) alike; returns the assembled array on `root`, None
    elsewhere.  Shards may have unequal lengths (see `shard`).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(np.ascontiguousarray(local)).to(device)
    # pad every shard to the largest one so all_gather sees equal shapes
    sizes = [shard(batch, r, world)[1] - shard(batch, r, world)[0] for r in range(world)]
    width = max(sizes)
    pad = torch.zeros((width,) + tuple(t.shape[1:]), dtype=t.dtype, device=device)
    pad[: t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    if rank != root:
        return None
    parts = [bufs[r][: sizes[r]].cpu().numpy() for r in range(world)]
    return np.concatenate(parts, axis=0)


def max_over_ranks(value: float, group=None) -> float:
    """Job time = max over ranks (bench.py timing rule)."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
