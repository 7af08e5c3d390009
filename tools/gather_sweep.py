"""Gather-mode host pipeline (list API path) sweep: pack threads x chunk, C1-10k (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.solver import solve_host_buffers, _pinned
B = 10000
rng = np.random.default_rng(0)
mats = [np.asfortranarray(rng.random((32, 32))) for _ in range(B)]
ptrs = np.fromiter((a.__array_interface__["data"][0] for a in mats), dtype=np.uintp, count=B)
host = torch.empty((B, 32, 32), dtype=torch.float64, pin_memory=True)
u_h = torch.empty((B, 32, 32), dtype=torch.float64, pin_memory=True)
s_h = torch.empty((B, 32), dtype=torch.float64, pin_memory=True)
v_h = torch.empty((B, 32, 32), dtype=torch.float64, pin_memory=True)
i_h = torch.empty((B * 48,), dtype=torch.uint8, pin_memory=True)
opts = bs.JacobiOptions()
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
for pt in (0, 2, 4, 8):
    for div in (16, 32):
        ts = []
        for it in range(5):
            t0 = time.perf_counter()
            solve_host_buffers(host, u_h, s_h, v_h, i_h, 32, 32, opts, chunk=-(-B // div),
                               a_ptrs=(ptrs if pt else None), pack_threads=max(pt, 1))
            torch.cuda.synchronize()
            if it:
                ts.append((time.perf_counter() - t0) * 1e3)
        print(f"pack_threads={pt:2d} (0 = pre-packed) chunk=B/{div}: {min(ts):.2f} ms  median {np.median(ts):.2f}", flush=True)

# event vs wall timing of the pre-packed call, random vs arith inputs
from paper_2601_17979_b200.matgen import gen_batch_device
for name, src in (("random", None), ("arith", gen_batch_device("arith", 32, 32, B, np.float64, kappa=1e10, seed=0))):
    if src is not None:
        host.copy_(src)
    st = torch.cuda.current_stream()
    for it in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        solve_host_buffers(host, u_h, s_h, v_h, i_h, 32, 32, opts, chunk=-(-B // 16))
        e1.record(st)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if it:
            print(f"{name}: events {e0.elapsed_time(e1):.2f} ms, host enqueue {(t1 - t0) * 1e3:.2f} ms, wall {(t2 - t0) * 1e3:.2f} ms", flush=True)
