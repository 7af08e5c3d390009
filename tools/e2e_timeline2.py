"""Host-buffer pipeline with a ramped chunk schedule (small first chunks start the D2H engine earlier):
total time of C1-10k for several schedules (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device

m = n = 32; B = 10000
a = gen_batch_device("arith", m, n, B, np.float64, kappa=1e10, seed=0)
a_h = torch.empty(a.shape, dtype=a.dtype, pin_memory=True); a_h.copy_(a)
u_h = torch.empty((B, 32, 32), dtype=torch.float64, pin_memory=True)
v_h = torch.empty((B, 32, 32), dtype=torch.float64, pin_memory=True)
s_h = torch.empty((B, 32), dtype=torch.float64, pin_memory=True)
opts = bs.JacobiOptions()
dev = torch.device("cuda", 0)

def sched(first, ramp, size):
    out, tot, cur = [], 0, first
    while tot < B:
        c = min(cur, B - tot); out.append(c); tot += c
        cur = min(size, int(cur * ramp))
    return out

for NS in (4, 8):
    streams = [torch.cuda.Stream(dev) for _ in range(NS)]
    bufs = [torch.empty((1250, 32, 32), dtype=torch.float64, device=dev) for _ in range(NS)]
    for first, ramp, size in ((625, 1, 625), (156, 2, 625), (80, 2, 625), (156, 2, 834), (156, 1.5, 625), (300, 2, 625), (80, 2, 500)):
        S = sched(first, ramp, size)
        best = 1e9
        for rep in range(4):
            base = torch.cuda.Event(enable_timing=True); base.record(torch.cuda.current_stream())
            lo = 0
            for c, cs in enumerate(S):
                st = streams[c % NS]
                st.wait_event(base)
                hi = lo + cs
                with torch.cuda.stream(st):
                    ad = bufs[c % NS][:cs]
                    ad.copy_(a_h[lo:hi], non_blocking=True)
                    r = bs.solve_tensor(ad, m, n, opts)
                    u_h[lo:hi].copy_(r.u, non_blocking=True)
                    v_h[lo:hi].copy_(r.v, non_blocking=True)
                    s_h[lo:hi].copy_(r.s, non_blocking=True)
                lo = hi
            end = torch.cuda.Event(enable_timing=True)
            for st in streams:
                torch.cuda.current_stream().wait_stream(st)
            end.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            if rep:
                best = min(best, base.elapsed_time(end))
        print(f"streams {NS} first {first} ramp {ramp} max {size} ({len(S)} chunks): {best:.3f} ms", flush=True)
