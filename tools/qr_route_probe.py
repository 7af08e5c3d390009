"""QR-route timing probe for C4 (qr vs plain), with a torch.profiler kernel table (development aid)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import solve_tensor
a = gen_batch_device("random", 256, 32, 5000, np.complex128, kappa=1, seed=0)
for q in (True, False):
    opts = bs.JacobiOptions(use_qr_preprocess=q)
    r = solve_tensor(a, 256, 32, opts); torch.cuda.synchronize()
    for _ in range(3):
        t0=time.perf_counter(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); r = solve_tensor(a, 256, 32, opts); e1.record(); torch.cuda.synchronize()
        print("qr" if q else "plain", f"events {e0.elapsed_time(e1):.2f} ms wall {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    r = solve_tensor(a, 256, 32, bs.JacobiOptions(use_qr_preprocess=True)); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
