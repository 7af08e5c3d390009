import sys, time; sys.path.insert(0, "/root/repo")
import numpy as np, torch, gc
import paper_2601_17979_b200 as bs
rng = np.random.default_rng(0)
for (m, dt, wantv) in ((16, np.float32, True), (16, np.float32, False), (32, np.float64, True)):
    mats = [np.asfortranarray(rng.random((m, m)).astype(dt)) for _ in range(10000)]
    o = bs.JacobiOptions(compute_right_vectors=wantv)
    for _ in range(3): bs.batch_svd(mats, o)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); r = bs.batch_svd(mats, o); ts.append(time.perf_counter() - t0)
    print(m, dt.__name__, wantv, "median ms", round(sorted(ts)[5] * 1e3, 2), "M/s", round(10000 / sorted(ts)[5] / 1e6, 2), flush=True)
