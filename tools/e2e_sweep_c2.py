"""Host-buffer pipeline sweep (streams x chunk) for C2 (10k x 16x16 FP32, full / values) (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import solve_host_buffers
B, m = 10000, 16
a = gen_batch_device("random", m, m, B, np.float32, kappa=1, seed=0)
dev = torch.device("cuda", 0)
for wantv in (True, False):
    a_h = torch.empty(a.shape, dtype=a.dtype, pin_memory=True); a_h.copy_(a)
    u_h = torch.empty((B, m, m), dtype=torch.float32, pin_memory=True)
    s_h = torch.empty((B, m), dtype=torch.float32, pin_memory=True)
    v_h = torch.empty((B, m, m), dtype=torch.float32, pin_memory=True) if wantv else None
    i_h = torch.empty((B * 48,), dtype=torch.uint8, pin_memory=True)
    opts = bs.JacobiOptions(compute_right_vectors=wantv)
    for nst in (2, 4, 8):
        for div in (1, 2, 4, 8, 16):
            streams = [torch.cuda.current_stream()] + [torch.cuda.Stream(dev) for _ in range(nst - 1)]
            ts = []
            for it in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                solve_host_buffers(a_h, u_h, s_h, v_h, i_h, m, m, opts, 0, chunk=-(-B // div), streams=streams)
                e1.record()
                torch.cuda.synchronize()
                if it:
                    ts.append(e0.elapsed_time(e1))
            print(f"v={wantv} streams={nst} chunk=B/{div}: {min(ts):.3f} ms  {B / min(ts) / 1e3:.1f} M/s", flush=True)
