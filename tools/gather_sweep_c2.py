import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.solver import solve_host_buffers
B, m = 10000, 16
rng = np.random.default_rng(0)
mats = [np.asfortranarray(rng.random((m, m)).astype(np.float32)) for _ in range(B)]
ptrs = np.fromiter((a.__array_interface__["data"][0] for a in mats), dtype=np.uintp, count=B)
host = torch.empty((B, m, m), dtype=torch.float32, pin_memory=True)
u_h = torch.empty((B, m, m), dtype=torch.float32, pin_memory=True)
s_h = torch.empty((B, m), dtype=torch.float32, pin_memory=True)
v_h = torch.empty((B, m, m), dtype=torch.float32, pin_memory=True)
i_h = torch.empty((B * 48,), dtype=torch.uint8, pin_memory=True)
opts = bs.JacobiOptions()
for pt in (1, 2, 4, 8):
    ts, te = [], []
    for it in range(8):
        t0 = time.perf_counter()
        solve_host_buffers(host, u_h, s_h, v_h, i_h, m, m, opts, a_ptrs=ptrs, pack_threads=pt)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if it > 1:
            ts.append((t2 - t0) * 1e3); te.append((t1 - t0) * 1e3)
    print(f"pack_threads={pt}: total {np.median(ts):.3f} ms, call returns after {np.median(te):.3f} ms", flush=True)
