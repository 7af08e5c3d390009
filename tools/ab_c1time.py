"""A/B device timing of two builds of the package (development aid): copy each build's package directory
(with its _lib/*.so) under DIR_A/ and DIR_B/, then `python tools/ab_c1time.py DIR_A` and `... DIR_B` on the
same box (C1 shapes, L2 flushed before every solve, CUDA events, 20 steps)."""
import os, sys
here = os.path.dirname(os.path.abspath(sys.argv[1]))
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import paper_2601_17979_b200 as bs
print("using", bs.__file__)
from paper_2601_17979_b200.matgen import gen_batch_device
dev = torch.device("cuda", 0)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for B in (500, 1000, 1184, 1250, 10000):
    a = gen_batch_device("arith", 32, 32, B, np.float64, kappa=1e10, seed=0)
    o = bs.JacobiOptions()
    for _ in range(3):
        flush.fill_(1.0); bs.solve_tensor(a, 32, 32, o)
    torch.cuda.synchronize()
    evs = []
    for _ in range(20):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); bs.solve_tensor(a, 32, 32, o); e1.record(); evs.append((e0, e1))
    torch.cuda.synchronize()
    ts = [e0.elapsed_time(e1) for e0, e1 in evs]
    print(f"B={B}: mean {np.mean(ts):.4f} ms  min {min(ts):.4f}", flush=True)
