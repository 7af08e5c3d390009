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
    if isinstance(local, torch.Tensor):  # device tensors go straight into the collective
        t = local.contiguous().to(device)
    else:
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


# ---------------------------------------------------------------------------
# Product entry points for one batch split over G devices (north star: "the batch is
# partitioned across the 8 GPUs of one box by plain batch splitting, with no NCCL needed beyond an
# optional gather").  Problem i of the global batch is solved by the device that owns shard(B, r, G)
# containing i; a problem's factors do not depend on the device (same kernel, same bits).
# ---------------------------------------------------------------------------
def slice_of(batch: int, rank: int | None = None, world: int | None = None) -> tuple[int, int]:
    """[start, stop) of this process's slice; rank/world default to torch.distributed's (1 process: all)."""
    if rank is None or world is None:
        try:
            import torch.distributed as dist

            if dist.is_available() and dist.is_initialized():
                rank, world = dist.get_rank(), dist.get_world_size()
        except Exception:  # pragma: no cover
            pass
    if rank is None or world is None:
        rank, world = 0, 1
    return shard(batch, rank, world)


def solve_rank_slice(a_global, m: int, n: int, opts, rank: int | None = None, world: int | None = None,
                     route=None, out=None, solve=None):
    """One rank's part of a global batch: solve problems [start, stop) of ``a_global`` (B, n, m).

    ``a_global`` holds the whole batch (every rank builds or loads the same one; the slice is a
    contiguous view, no copy).  Launches on the current device and stream; returns
    (start, stop, result).  ``solve`` is the per-slice solver (default: the device solver
    ``solver.solve_tensor``); the CPU tests pass the oracle here, the product never does.
    """
    from . import _lib

    B = int(a_global.shape[0])
    start, stop = slice_of(B, rank, world)
    local = a_global[start:stop]
    if solve is None:
        from .solver import solve_tensor

        res = solve_tensor(local, m, n, opts, _lib.DISPATCH if route is None else route, out=out)
    else:
        res = solve(local, m, n, opts)
    return start, stop, res


def gather_slices(parts, batch: int, group=None, root: int = 0):
    """Optional gather: every rank passes its slice's arrays/tensors (a tuple, leading axis = problems);
    root receives the assembled global arrays (numpy), others None.  Collective: every rank calls it."""
    out = []
    for p in parts:
        if p is None:
            out.append(None)
            continue
        out.append(gather_to_root(p if hasattr(p, "detach") else np.asarray(p), batch, group=group, root=root))
    return tuple(out) if out and out[0] is not None else None


def solve_multi_device(a_host, m: int, n: int, opts, devices, route=None, gather: bool = True):
    """One process, G devices: split the (B, n, m) host batch into contiguous shards, copy each to its
    device on that device's stream, launch every device's solve before waiting on any, and (optionally)
    gather U / sigma / V / info back to host arrays in global order.

    Returns dict(u, s, v, info (host numpy, global order, if gather), parts [(start, stop, device,
    DeviceResult)], wall_s (common start -> last device done), device_ms [per-device solve time]).
    """
    import time

    import torch

    from . import _lib
    from .solver import solve_tensor

    devs = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
    G = len(devs)
    if G < 1:
        raise ValueError("solve_multi_device needs at least one device")
    B = int(a_host.shape[0])
    src = a_host if a_host.device.type == "cpu" else a_host.cpu()
    if not src.is_pinned():
        src = src.pin_memory()
    for d in devs:
        torch.cuda.synchronize(d)
    parts, evs = [], []
    t0 = time.perf_counter()
    for g, d in enumerate(devs):  # enqueue every device before waiting on any (common start)
        start, stop = shard(B, g, G)
        with torch.cuda.device(d):
            st = torch.cuda.current_stream(d)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            loc = src[start:stop].to(d, non_blocking=True)
            e0.record(st)
            res = solve_tensor(loc, m, n, opts, _lib.DISPATCH if route is None else route) if stop > start else None
            e1.record(st)
        parts.append((start, stop, d, res))
        evs.append((e0, e1))
    for d in devs:
        torch.cuda.synchronize(d)
    wall = time.perf_counter() - t0
    out = {"parts": parts, "wall_s": wall, "device_ms": [a.elapsed_time(b) for a, b in evs]}
    if gather:
        k = min(m, n)
        cat = lambda xs: np.concatenate(xs, axis=0) if xs else None  # noqa: E731
        live = [p for p in parts if p[3] is not None]
        out["u"] = cat([p[3].u.cpu().numpy() for p in live])
        out["s"] = cat([p[3].s.cpu().numpy() for p in live])
        out["v"] = cat([p[3].v.cpu().numpy() for p in live]) if live and live[0][3].v is not None else None
        out["info"] = cat([p[3].info.cpu().numpy() for p in live])
        assert out["u"] is None or out["u"].shape[0] == B and out["u"].shape[1] == k
    return out
