"""C2 (16x16 FP32): bitwise comparison of kernels 24 (gen. 2) and 34 (quarter-warp) and their
device times over batch sizes (development aid: picks the batch-size switch in make_plan)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device

def timed(a, opts, k, reps=7):
    bs.solve_tensor(a, 16, 16, opts, kernel=k); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); bs.solve_tensor(a, 16, 16, opts, kernel=k); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts) * 1e3

KS = [int(k) for k in (sys.argv[1] if len(sys.argv) > 1 else "24,34").split(",")]
for fam in ("random", "geo", "arith", "rankdef", "logrand"):
    a = gen_batch_device(fam, 16, 16, 4000, np.float32, kappa=1e5, seed=11)
    opts = bs.JacobiOptions()
    r0 = bs.solve_tensor(a, 16, 16, opts, kernel=24)
    for k in KS:
        r1 = bs.solve_tensor(a, 16, 16, opts, kernel=k)
        torch.cuda.synchronize()
        same = all(torch.equal(x, y) for x, y in ((r0.u, r1.u), (r0.s, r1.s), (r0.v, r1.v)))
        print(f"bitwise {fam:8s} k{k}: {'identical' if same else 'DIFFERENT'}", flush=True)
KS = [int(k) for k in (sys.argv[1] if len(sys.argv) > 1 else "24,34").split(",")]
BS = [int(b) for b in (sys.argv[2] if len(sys.argv) > 2 else "300,600,1000,1500,2000,2500,3000,4000,5000,7500,10000,20000").split(",")]
for B in BS:
    a = gen_batch_device("random", 16, 16, B, np.float32, seed=5)
    for wantv in (True, False):
        opts = bs.JacobiOptions(compute_right_vectors=wantv)
        ts = "  ".join(f"k{k} {timed(a, opts, k):7.1f} us" for k in KS)
        print(f"B={B:6d} v={int(wantv)}  {ts}", flush=True)
