"""Outer-sweep differences GPU - reference restatement on BASELINE configs (development aid)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch, collections
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200 import _lib
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import INFO_DTYPE
from oracle import oracle as O
for fam, m, n, B, dt, kappa, rank, kern in [("geo", 64, 64, 2000, np.float64, 1e12, None, 0), ("geo", 64, 64, 2000, np.float64, 1e12, None, 2),
        ("geo", 64, 64, 2000, np.float64, 1e12, None, 8), ("rankdef", 64, 64, 2000, np.float64, 1e6, 48, 0),
        ("geo", 64, 64, 1000, np.float64, 1e8, None, 0), ("random", 128, 128, 500, np.float64, 1.0, None, 0)]:
    a = gen_batch_device(fam, m, n, B, dt, kappa=kappa, seed=0, rank=rank)
    r = bs.solve_tensor(a, m, n, bs.JacobiOptions(), kernel=kern); torch.cuda.synchronize()
    info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    A = np.swapaxes(a.cpu().numpy(), 1, 2)
    idx = np.arange(0, B, 4)
    _, S_ref, _, infos = O.solve_batch(A[idx], None, None, nthreads=0)
    d = info["outer_sweeps"][idx] - np.array([i["outer_sweeps"] for i in infos])
    print(fam, kappa, m, n, "kernel", int(info["kernel"][0]), "delta hist", sorted(collections.Counter(d.tolist()).items()),
          "gpu mean", info["outer_sweeps"].mean(), "ref mean", np.mean([i["outer_sweeps"] for i in infos]), flush=True)
