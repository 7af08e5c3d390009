import sys, time, cProfile, pstats; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2601_17979_b200 as bs
rng = np.random.default_rng(0)
mats = [np.asfortranarray(rng.random((16, 16)).astype(np.float32)) for _ in range(10000)]
o = bs.JacobiOptions()
for _ in range(3): bs.batch_svd(mats, o)
pr = cProfile.Profile(); pr.enable()
for _ in range(10): bs.batch_svd(mats, o)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
