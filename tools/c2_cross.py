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

for fam in ("random", "geo", "arith", "rankdef", "logrand"):
    a = gen_batch_device(fam, 16, 16, 4000, np.float32, kappa=1e5, seed=11)
    opts = bs.JacobiOptions()
    r0 = bs.solve_tensor(a, 16, 16, opts, kernel=24); r1 = bs.solve_tensor(a, 16, 16, opts, kernel=34)
    torch.cuda.synchronize()
    same = all(torch.equal(x, y) for x, y in ((r0.u, r1.u), (r0.s, r1.s), (r0.v, r1.v)))
    print(f"bitwise {fam:8s}: {'identical' if same else 'DIFFERENT'}", flush=True)
for B in (300, 600, 1000, 1500, 2000, 2500, 3000, 4000, 5000, 7500, 10000, 20000):
    a = gen_batch_device("random", 16, 16, B, np.float32, seed=5)
    for wantv in (True, False):
        opts = bs.JacobiOptions(compute_right_vectors=wantv)
        t24, t34, t35 = timed(a, opts, 24), timed(a, opts, 34), timed(a, opts, 35)
        print(f"B={B:6d} v={int(wantv)}  k24 {t24:7.1f} us  k34 {t34:7.1f} us  k35 {t35:7.1f} us", flush=True)
