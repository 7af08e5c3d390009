"""Timeline of the C1-10k host-buffer pipeline (H2D / solve / D2H per chunk over S streams), rebuilt with
torch copies + solve_tensor and CUDA events, to see where the copy engines idle (development aid)."""
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
for NS, DIV in ((4, 16), (8, 16), (8, 32), (6, 24)):
    streams = [torch.cuda.Stream(dev) for _ in range(NS)]
    chunk = -(-B // DIV)
    bufs = [(torch.empty((chunk, 32, 32), dtype=torch.float64, device=dev),) for _ in range(NS)]
    for rep in range(3):
        base = torch.cuda.Event(enable_timing=True); base.record(torch.cuda.current_stream())
        marks = []
        for c in range(DIV):
            st = streams[c % NS]
            st.wait_event(base)
            lo, hi = c * chunk, min(B, (c + 1) * chunk)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            with torch.cuda.stream(st):
                ev[0].record(st)
                ad = bufs[c % NS][0][: hi - lo]
                ad.copy_(a_h[lo:hi], non_blocking=True)
                ev[1].record(st)
                r = bs.solve_tensor(ad, m, n, opts)
                ev[2].record(st)
                u_h[lo:hi].copy_(r.u, non_blocking=True)
                v_h[lo:hi].copy_(r.v, non_blocking=True)
                s_h[lo:hi].copy_(r.s, non_blocking=True)
                ev[3].record(st)
            marks.append(ev)
        end = torch.cuda.Event(enable_timing=True)
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
        end.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
    tot = base.elapsed_time(end)
    print(f"streams {NS} chunks {DIV} (x{chunk}): total {tot:.3f} ms", flush=True)
    for c, ev in enumerate(marks[: min(DIV, 12)]):
        t = [base.elapsed_time(e) for e in ev]
        print(f"  chunk {c:2d}: h2d {t[0]:6.3f}-{t[1]:6.3f}  solve -{t[2]:6.3f}  d2h -{t[3]:6.3f}")
