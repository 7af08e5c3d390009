"""batch_svd (list API, gather-mode pipeline) time vs the pipeline's chunk divisor (development aid):
python tools/list_api_chunk_probe.py M DTYPE DIV[,DIV...]"""
import sys, time; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200 import solver
m, dt = int(sys.argv[1]), np.dtype(sys.argv[2])
divs = [int(x) for x in sys.argv[3].split(",")]
rng = np.random.default_rng(0)
mats = [np.asfortranarray(rng.random((m, m)).astype(dt)) for _ in range(10000)]
o = bs.JacobiOptions()
for rep in range(2):
    for div in divs:
        solver.default_chunk = lambda batch, *a, div=div: -(-batch // div)
        for _ in range(3): bs.batch_svd(mats, o)
        ts = []
        for _ in range(10):
            t0 = time.perf_counter(); r = bs.batch_svd(mats, o); ts.append(time.perf_counter() - t0)
        print(m, dt.name, "div", div, "median ms", round(sorted(ts)[5] * 1e3, 2), flush=True)
