"""Host-side overhead of one solve_tensor call (no synchronisation), development aid."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device

a = gen_batch_device("arith", 32, 32, 1000, np.float64, kappa=1e10, seed=0)
opts = bs.JacobiOptions()
out = None
for i in range(5):
    r = bs.solve_tensor(a, 32, 32, opts)
torch.cuda.synchronize()
ts = []
for i in range(50):
    t0 = time.perf_counter()
    r = bs.solve_tensor(a, 32, 32, opts)
    ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
print(f"solve_tensor host time per call: median {1e6 * np.median(ts):.1f} us, min {1e6 * min(ts):.1f} us")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for i in range(20):
    r = bs.solve_tensor(a, 32, 32, opts)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)

# the C-ABI call alone (arguments precomputed)
import ctypes
from paper_2601_17979_b200 import _lib
from paper_2601_17979_b200.solver import make_opts, _workspace
L = _lib.load()
o = make_opts(opts)
B, m, n, k = 1000, 32, 32, 32
u = torch.empty((B, k, m), dtype=torch.float64, device="cuda"); s = torch.empty((B, k), dtype=torch.float64, device="cuda")
v = torch.empty((B, k, n), dtype=torch.float64, device="cuda"); info = torch.empty((B * 48,), dtype=torch.uint8, device="cuda")
wsb = L.bsvd_workspace_bytes(1, m, n, B, ctypes.byref(o)); ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
args = (1, m, n, B, a.data_ptr(), m, m * n, u.data_ptr(), m, k * m, s.data_ptr(), k, v.data_ptr(), n, k * n,
        ctypes.byref(o), info.data_ptr(), ws.data_ptr(), wsb, st)
ts = []
for i in range(50):
    t0 = time.perf_counter(); L.bsvd_gesvj_batched(*args); ts.append(time.perf_counter() - t0); torch.cuda.synchronize()
print(f"bsvd_gesvj_batched ctypes call: median {1e6 * np.median(ts):.1f} us")
ts = []
for i in range(50):
    t0 = time.perf_counter(); L.bsvd_workspace_bytes(1, m, n, B, ctypes.byref(o)); ts.append(time.perf_counter() - t0)
print(f"bsvd_workspace_bytes: median {1e6 * np.median(ts):.1f} us")
