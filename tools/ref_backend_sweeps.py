"""Sweep-count spread of the REFERENCE itself between its numba and numpy backends on C3a-shaped inputs
(geo kappa=1e12, 64x64, blocked) -- runs the reference from /root/reference in this container only:
  NUMBA_CACHE_DIR=/tmp/nc OPENBLAS_NUM_THREADS=1 python tools/ref_backend_sweeps.py"""
import sys, collections, numpy as np
sys.path.insert(0, "/root/reference/pkg/src")
import bsvd
from bsvd import backend
from bsvd.matgen import SpectrumSpec, gen_matrix
res = {}
mats = [gen_matrix(64, SpectrumSpec("geo", 64, kappa=1e12, seed=s)) for s in range(120)]
for name in ("numba", "numpy"):
    backend.select(name)
    res[name] = [bsvd.svd_dispatch(a).info.outer_sweeps for a in mats]
d = np.array(res["numba"]) - np.array(res["numpy"])
print("geo 1e12 64x64: reference numba - numpy backend sweep deltas", sorted(collections.Counter(d.tolist()).items()),
      "means", np.mean(res["numba"]), np.mean(res["numpy"]))
