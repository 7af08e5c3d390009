"""batch_svd C2 component times (development aid): record fill alone, the pipeline call alone, the whole call."""
import sys, time; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200 import _lib, batch
from paper_2601_17979_b200.solver import solve_host
m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
dt = np.dtype(sys.argv[2] if len(sys.argv) > 2 else "float32")
rng = np.random.default_rng(0)
mats = [np.asfortranarray(rng.random((m, m)).astype(dt)) for _ in range(10000)]
o = bs.JacobiOptions()
H = _lib.hostptrs()
def med(fn, n=15):
    for _ in range(3): fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return round(sorted(ts)[n // 2] * 1e3, 3)
res = [None] * 10000
print("fill_lazy ms", med(lambda: H.bsvd_py_fill_lazy(res, 0, 10000, batch._LazyResult, batch._Group())))
ptrs = _lib.gather_fortran(mats)[0]
print("gather ms", med(lambda: _lib.gather_fortran(mats)))
print("solve_host ms", med(lambda: solve_host(mats, o, ptrs=ptrs)))
def enq():
    f = solve_host(mats, o, ptrs=ptrs, defer=True)
    t1 = time.perf_counter(); f(); return t1
ts = []
for _ in range(15):
    t0 = time.perf_counter(); f = solve_host(mats, o, ptrs=ptrs, defer=True); t1 = time.perf_counter(); f(); t2 = time.perf_counter()
    ts.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3))
ts.sort()
print("solve_host enqueue / drain ms", [round(x, 3) for x in ts[7]])
print("batch_svd ms", med(lambda: bs.batch_svd(mats, o)))
print("_solve_problems ms", med(lambda: batch._solve_problems(mats, o, None, True)))
import gc
def sp_nogc():
    gc.disable()
    try:
        return batch._solve_problems(mats, o, None, True)
    finally:
        gc.enable()
print("_solve_problems + gc toggle ms", med(sp_nogc))
print("gc.collect(0) after a call ms", med(lambda: (batch.batch_svd(mats, o), gc.collect(0))))
def spin(ms):
    t = time.perf_counter() + ms / 1e3
    while time.perf_counter() < t:
        pass
for busy in (0.0, 0.2, 0.44, 0.8):
    ts = []
    for _ in range(15):
        t0 = time.perf_counter(); f = solve_host(mats, o, ptrs=ptrs, defer=True); t1 = time.perf_counter()
        spin(busy); t2 = time.perf_counter(); f(); t3 = time.perf_counter()
        ts.append(((t1 - t0) * 1e3, (t3 - t2) * 1e3, (t3 - t0) * 1e3))
    ts.sort(key=lambda x: x[2])
    print(f"spin {busy} ms: enqueue / finish-after-spin / total ms", [round(x, 3) for x in ts[7]])
