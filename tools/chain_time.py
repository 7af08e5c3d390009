"""Latency of one W iteration for a single warp per SM (development aid):
solve 2 x 148 problems with one warp per SM, values only and full, and
report device time per iteration in SM cycles."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import INFO_DTYPE
kern = int(sys.argv[1]) if len(sys.argv) > 1 else 16
per_warp = int(sys.argv[2]) if len(sys.argv) > 2 else 2
clk = torch.cuda.get_device_properties(0).clock_rate * 1e3 if hasattr(torch.cuda.get_device_properties(0), "clock_rate") else 1.965e9
for wantv in (False, True):
    B = per_warp * 148
    a = gen_batch_device("arith", 32, 32, B, np.float64, kappa=1e10, seed=0)
    opts = bs.JacobiOptions(compute_right_vectors=wantv)
    r = bs.solve_tensor(a, 32, 32, opts, kernel=kern); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = bs.solve_tensor(a, 32, 32, opts, kernel=kern); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    sw = info["outer_sweeps"].max()
    t = min(ts) * 1e-3
    print(f"kernel {kern} want_v={wantv}: {min(ts):.3f} ms, max sweeps {sw}, {t * 1.965e9 / (sw * 31):.0f} cycles/iteration (at 1.965 GHz, incl. launch+finalize)")
