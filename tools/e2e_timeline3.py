"""Host-buffer pipeline with dedicated copy streams: every H2D on one stream, every D2H on another,
solves on S compute streams, events between them (so no H2D queues behind a D2H in a copy-engine
channel).  Total time of C1-10k per chunk count (development aid)."""
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
a_d = torch.empty_like(a)
h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
for NC, NS in ((16, 4), (16, 8), (8, 4), (32, 8), (20, 5)):
    comp = [torch.cuda.Stream(dev) for _ in range(NS)]
    chunk = -(-B // NC)
    best = 1e9
    for rep in range(4):
        base = torch.cuda.Event(enable_timing=True); base.record(torch.cuda.current_stream())
        h2d.wait_event(base); d2h.wait_event(base)
        for st in comp:
            st.wait_event(base)
        keep = []
        for c in range(NC):
            lo, hi = c * chunk, min(B, (c + 1) * chunk)
            if lo >= hi:
                break
            with torch.cuda.stream(h2d):
                a_d[lo:hi].copy_(a_h[lo:hi], non_blocking=True)
                e_in = torch.cuda.Event(); e_in.record(h2d)
            st = comp[c % NS]
            st.wait_event(e_in)
            with torch.cuda.stream(st):
                r = bs.solve_tensor(a_d[lo:hi], m, n, opts)
                e_sol = torch.cuda.Event(); e_sol.record(st)
            keep.append(r)
            d2h.wait_event(e_sol)
            with torch.cuda.stream(d2h):
                u_h[lo:hi].copy_(r.u, non_blocking=True)
                v_h[lo:hi].copy_(r.v, non_blocking=True)
                s_h[lo:hi].copy_(r.s, non_blocking=True)
        end = torch.cuda.Event(enable_timing=True)
        torch.cuda.current_stream().wait_stream(d2h)
        end.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        if rep:
            best = min(best, base.elapsed_time(end))
    print(f"chunks {NC} compute streams {NS}: {best:.3f} ms  ({B / best * 1e3:,.0f} mat/s)", flush=True)
