"""Phase timing of the list API host path for C1-10k shapes (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_17979_b200 as bs
from paper_2601_17979_b200 import batch, solver

rng = np.random.default_rng(0)
B = 10000
mats = [np.asfortranarray(rng.random((32, 32))) for _ in range(B)]
opts = bs.JacobiOptions()
for it in range(4):
    t0 = time.perf_counter()
    U, S, V, info, kern = solver.solve_host(mats, opts)
    t1 = time.perf_counter()
    res, err, tele = batch._solve_problems(mats, opts, None, True)
    t2 = time.perf_counter()
    r = bs.batch_svd(mats, opts)
    t3 = time.perf_counter()
    print(f"solve_host {1e3 * (t1 - t0):.1f} ms | _solve_problems {1e3 * (t2 - t1):.1f} ms | batch_svd {1e3 * (t3 - t2):.1f} ms")
# inside solve_host
torch.cuda.synchronize()
hv = np.empty((B, 32, 32))
t0 = time.perf_counter(); solver._parallel_slices(B, lambda lo, hi: np.stack([a.T for a in mats[lo:hi]], out=hv[lo:hi])); t1 = time.perf_counter()
print(f"pack {1e3 * (t1 - t0):.1f} ms")
x = np.empty((B, 32, 32)); y = np.ones((B, 32, 32))
t0 = time.perf_counter(); solver._parallel_slices(B, lambda lo, hi: x.__setitem__(slice(lo, hi), y[lo:hi])); t1 = time.perf_counter()
print(f"copy-out 82 MB into fresh pages {1e3 * (t1 - t0):.1f} ms")
