"""C2 kernels: timing and bitwise comparison of the 16x16 FP32 variants (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
kerns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "34,46").split(",")]
for fam, kappa in (("random", 1.0), ("geo", 1e4), ("arith", 1e5), ("rankdef", 1e3)):
    for B in (10000, 1000, 7):
        a = gen_batch_device(fam, 16, 16, B, np.float32, kappa=kappa, seed=3)
        for wantv in (True, False):
            opts = bs.JacobiOptions(compute_right_vectors=wantv)
            res = {}
            for k in kerns:
                r = bs.solve_tensor(a, 16, 16, opts, kernel=k); torch.cuda.synchronize()
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ts = []
                for _ in range(5):
                    ev0.record(); r = bs.solve_tensor(a, 16, 16, opts, kernel=k); ev1.record(); torch.cuda.synchronize()
                    ts.append(ev0.elapsed_time(ev1))
                res[k] = (r, min(ts))
            r0 = res[kerns[0]][0]
            same = all(torch.equal(r0.u, res[k][0].u) and torch.equal(r0.s, res[k][0].s) and
                       (not wantv or torch.equal(r0.v, res[k][0].v)) and torch.equal(r0.info, res[k][0].info) for k in kerns)
            if fam == "random" or not same:
                print(f"{fam:8s} B={B:6d} v={int(wantv)} " + " ".join(f"k{k} {res[k][1]*1e3:7.1f}us" for k in kerns) +
                      f"  bitwise={same}", flush=True)
