"""Per-iteration latency of the 32x32 kernels vs batch size (development aid): device time / total sweep
iterations of the slowest problem."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import INFO_DTYPE
kernels = [int(x) for x in sys.argv[1].split(",")]
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 16, 148, 592, 1250, 2500, 5000, 10000]
a_all = gen_batch_device("arith", 32, 32, max(sizes), np.float64, kappa=1e10, seed=0)
opts = bs.JacobiOptions()
for B in sizes:
    a = a_all[:B].contiguous()
    line = f"B={B:6d}"
    for k in kernels:
        r = bs.solve_tensor(a, 32, 32, opts, kernel=k); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); bs.solve_tensor(a, 32, 32, opts, kernel=k); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
        its = int(info["outer_sweeps"].max()) * 31
        t = min(ts)
        line += f" | k{k}: {t*1e3:7.1f} us {t*1e-3*1.92e9/its:6.0f} cyc/it"
    print(line, flush=True)
