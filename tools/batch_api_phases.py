"""Phase timing of the list API host path on C1-10k shapes (development aid): pack, pipelined device
solve with copies, record building, batch telemetry."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_17979_b200 as bs
from paper_2601_17979_b200 import _lib, batch, solver

rng = np.random.default_rng(0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
mats = [np.asfortranarray(rng.random((32, 32))) for _ in range(B)]
opts = bs.JacobiOptions()
T = {}
orig_pack = _lib.load().bsvd_pack_host
orig_buf = solver.solve_host_buffers


def timed(name, fn):
    def w(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        return r
    return w


solver.solve_host_buffers = timed("device (H2D+solve+D2H)", orig_buf)
solver.solve_host = timed("solve_host", solver.solve_host)
batch._solve_problems = timed("_solve_problems", batch._solve_problems)
res = None
for it in range(12):
    T.clear()
    t0 = time.perf_counter()
    res = bs.batch_svd(mats, opts)
    t1 = time.perf_counter()
    tot = t1 - t0
    if it >= 2:
        print(f"B={B} batch_svd {tot * 1e3:.1f} ms ({B / tot:,.0f} mat/s) | " +
              " | ".join(f"{k} {v * 1e3:.1f}" for k, v in T.items()), flush=True)
r = res[7]
print("record", r.info.path, r.info.outer_sweeps, r.sigma[:2], type(r).__name__)
