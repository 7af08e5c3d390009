"""Stage timestamps inside batch._solve_problems for C2 (development aid)."""
import sys, time; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200 import _lib, batch, solver
rng = np.random.default_rng(0)
mats = [np.asfortranarray(rng.random((16, 16)).astype(np.float32)) for _ in range(10000)]
o = bs.JacobiOptions()
H = _lib.hostptrs()
stamps = []
orig_sh, orig_fill, orig_ho = solver.solve_host, H.bsvd_py_fill_lazy, solver._host_outputs
def sh(*a, **k):
    stamps.append(("solve_host in", time.perf_counter()))
    f = orig_sh(*a, **k)
    stamps.append(("solve_host out", time.perf_counter()))
    def fin():
        stamps.append(("finish in", time.perf_counter()))
        r = f()
        stamps.append(("finish out", time.perf_counter()))
        return r
    return fin
def fill(*a):
    stamps.append(("fill in", time.perf_counter()))
    r = orig_fill(*a)
    stamps.append(("fill out", time.perf_counter()))
    return r
def ho(*a):
    stamps.append(("host_outputs in", time.perf_counter()))
    r = orig_ho(*a)
    stamps.append(("host_outputs out", time.perf_counter()))
    return r
solver.solve_host, solver._host_outputs = sh, ho
H.bsvd_py_fill_lazy = fill
for it in range(8):
    stamps.clear()
    t0 = time.perf_counter(); r = batch._solve_problems(mats, o, None, True); t1 = time.perf_counter()
    if it >= 5:
        print(" | ".join(f"{n} {(t - t0) * 1e3:.3f}" for n, t in stamps), f"| end {(t1 - t0) * 1e3:.3f}")
