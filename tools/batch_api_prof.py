"""cProfile of the list API on C1-10k (development aid)."""
import os, sys, time, cProfile, pstats, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
rng = np.random.default_rng(0)
mats = [np.asfortranarray(rng.random((32, 32))) for _ in range(10000)]
res = None
for _ in range(4):
    res = bs.batch_svd(mats)
ts = []
for _ in range(10):
    t0 = time.perf_counter(); res = bs.batch_svd(mats); ts.append(time.perf_counter() - t0)
print("median ms", sorted(ts)[5] * 1e3, "min", min(ts) * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    res = bs.batch_svd(mats)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
