"""Wall time of the reference-facing list API (batch_svd) on C1-10k-shaped inputs (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_17979_b200 as bs

rng = np.random.default_rng(0)
for B in (1000, 10000):
    mats = [np.asfortranarray(rng.random((32, 32))) for _ in range(B)]
    bs.batch_svd(mats[:10])
    torch.cuda.synchronize()
    for it in range(3):
        t0 = time.perf_counter()
        res = bs.batch_svd(mats, bs.JacobiOptions())
        t1 = time.perf_counter()
        print(f"batch_svd B={B}: {(t1 - t0) * 1e3:.1f} ms  ({B / (t1 - t0):,.0f} mat/s)", flush=True)
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    bs.batch_svd(mats, bs.JacobiOptions())
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
