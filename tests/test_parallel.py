"""Multi-process (world_size 2, gloo, CPU) tests of the batch-splitting path.

The GPU solve cannot run here, so each rank solves its shard with the CPU
restatement (oracle/, test infrastructure) and the shards are gathered with the
same helper the GPU path uses; the result must equal the single-process solve
of the whole batch bit for bit (batch == standalone, F8).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2601_17979_b200.parallel import shard


def test_shard_partitions_exactly():
    for batch in (0, 1, 7, 10, 10000, 10001):
        for world in (1, 2, 3, 4, 8):
            covered = []
            for r in range(world):
                a, b = shard(batch, r, world)
                assert 0 <= a <= b <= batch
                covered.extend(range(a, b))
            assert covered == list(range(batch))
            sizes = [shard(batch, r, world)[1] - shard(batch, r, world)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, batch, out_dir):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2601_17979_b200.parallel import gather_to_root, max_over_ranks

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(1234)
    A = rng.random((batch, 12, 10))  # every rank builds the same global batch
    a, b = shard(batch, rank, world)
    U, S, V, infos = O.solve_batch(A[a:b], None, None, nthreads=1)
    sweeps = np.array([i["outer_sweeps"] for i in infos], dtype=np.int64)
    S_all = gather_to_root(S, batch)
    U_all = gather_to_root(U, batch)
    sw_all = gather_to_root(sweeps, batch)
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        np.savez(os.path.join(out_dir, "gathered.npz"), S=S_all, U=U_all, sw=sw_all, t=t)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("batch", [9, 16])
def test_two_rank_split_and_gather_equals_single_process(tmp_path, batch):
    from oracle import oracle as O

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), batch, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "gathered.npz")
    rng = np.random.default_rng(1234)
    A = rng.random((batch, 12, 10))
    U, S, V, infos = O.solve_batch(A, None, None, nthreads=1)
    assert np.array_equal(got["S"], S)
    assert np.array_equal(got["U"], U)
    assert np.array_equal(got["sw"], [i["outer_sweeps"] for i in infos])
    assert float(got["t"]) == 2.0  # max over ranks


def _worker_entry(rank, world, port, batch, out_dir):
    """Same split through the product entry points (parallel.solve_rank_slice / gather_slices); the
    per-slice solver is injected (the CPU restatement here, the device solver on the GPU box)."""
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2601_17979_b200 import JacobiOptions
    from paper_2601_17979_b200.parallel import gather_slices, slice_of, solve_rank_slice

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(99)
    A = rng.random((batch, 20, 12))                       # user view: B matrices 20 x 12
    a_global = torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2)))  # (B, n, m) column-major layout

    def oracle_slice(local, m, n, opts):
        U, S, V, infos = O.solve_batch(np.swapaxes(local.numpy(), 1, 2), opts, None, nthreads=1)
        return U, S, V, np.array([i["outer_sweeps"] for i in infos], dtype=np.int64)

    start, stop, (U, S, V, sw) = solve_rank_slice(a_global, 20, 12, JacobiOptions(), solve=oracle_slice)
    assert (start, stop) == slice_of(batch)  # defaults come from the initialised process group
    got = gather_slices((U, S, V, sw), batch)
    if rank == 0:
        np.savez(os.path.join(out_dir, "entry.npz"), U=got[0], S=got[1], V=got[2], sw=got[3])
    else:
        assert got is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("batch", [7, 10])
def test_two_rank_product_entry_points(tmp_path, batch):
    from oracle import oracle as O

    mp.spawn(_worker_entry, args=(2, _free_port(), batch, str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "entry.npz")
    A = np.random.default_rng(99).random((batch, 20, 12))
    U, S, V, infos = O.solve_batch(A, None, None, nthreads=1)
    assert np.array_equal(got["S"], S) and np.array_equal(got["U"], U) and np.array_equal(got["V"], V)
    assert np.array_equal(got["sw"], [i["outer_sweeps"] for i in infos])


def test_slice_of_defaults_to_whole_batch_without_a_group():
    from paper_2601_17979_b200.parallel import slice_of

    assert slice_of(10000) == (0, 10000)
    assert slice_of(10000, 7, 8) == (8750, 10000)
