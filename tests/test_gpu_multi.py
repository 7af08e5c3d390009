"""GPU tests of the batch split: one global batch cut into contiguous slices, each slice
solved by its own launch (here on cuda:0 -- the round's GPU boxes have one device; on a multi-GPU box the
same entry points take one device per slice).  Batch == standalone: a problem's factors do not depend on
the slice it lands in, so the gathered result is bitwise the one-launch result."""

import numpy as np
import pytest

import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.parallel import shard, solve_multi_device, solve_rank_slice

pytestmark = pytest.mark.gpu


def _one_launch(a, m, n, opts):
    import torch

    r = bs.solve_tensor(a, m, n, opts)
    torch.cuda.synchronize()
    return r


@pytest.mark.parametrize("world", [2, 3, 8])
def test_rank_slices_concatenate_to_one_launch(world):
    import torch

    m = n = 32
    a = gen_batch_device("arith", m, n, 1000, np.float64, kappa=1e10, seed=3)
    opts = bs.JacobiOptions()
    full = _one_launch(a, m, n, opts)
    us, ss, vs = [], [], []
    for r in range(world):
        start, stop, res = solve_rank_slice(a, m, n, opts, r, world)
        assert (start, stop) == shard(1000, r, world)
        us.append(res.u)
        ss.append(res.s)
        vs.append(res.v)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(ss), full.s)
    assert torch.equal(torch.cat(us), full.u)
    assert torch.equal(torch.cat(vs), full.v)


@pytest.mark.parametrize("cfg", [("arith", 32, 32, np.float64, 1e10), ("random", 16, 16, np.float32, 1.0),
                                 ("geo", 64, 64, np.float64, 1e12)])
def test_solve_multi_device_gathers_in_global_order(cfg):
    import torch

    fam, m, n, dt, kappa = cfg
    B = 301
    a = gen_batch_device(fam, m, n, B, dt, kappa=kappa, seed=5)
    opts = bs.JacobiOptions()
    full = _one_launch(a, m, n, opts)
    out = solve_multi_device(a.cpu(), m, n, opts, devices=[0, 0, 0])
    assert [p[:2] for p in out["parts"]] == [shard(B, g, 3) for g in range(3)]
    assert np.array_equal(out["s"], full.s.cpu().numpy())
    assert np.array_equal(out["u"], full.u.cpu().numpy())
    assert np.array_equal(out["v"], full.v.cpu().numpy())
    from paper_2601_17979_b200.solver import INFO_DTYPE

    gi = np.frombuffer(out["info"].tobytes(), dtype=INFO_DTYPE)
    fi = np.frombuffer(full.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    for f in ("converged", "outer_sweeps", "rotations", "last_rotations", "path", "status"):
        assert np.array_equal(gi[f], fi[f]), f  # the kernel id may differ with the slice size, the bits not
    assert out["wall_s"] > 0 and len(out["device_ms"]) == 3


def test_concurrent_batch_svd_threads_match_standalone():
    """Two host threads calling batch_svd at once (the reference's batch_svd is pure numpy and safe to
    call concurrently): per-thread pinned staging, so each gets exactly its standalone results."""
    import threading

    from common import random_matrix

    sets = [[random_matrix(32, 32, np.float64, seed=6000 + 100 * t + b) for b in range(300)] for t in range(2)]
    solo = [bs.batch_svd(ms) for ms in sets]
    out = [None, None]
    errs = []

    def work(t):
        try:
            for _ in range(3):
                out[t] = bs.batch_svd(sets[t])
        except Exception as exc:  # pragma: no cover
            errs.append(exc)

    th = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs
    for t in range(2):
        for r, s in zip(out[t], solo[t]):
            assert np.array_equal(r.sigma, s.sigma) and np.array_equal(r.u, s.u) and np.array_equal(r.v, s.v)
