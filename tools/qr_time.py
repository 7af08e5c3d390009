"""Time the qr+ route on the C4 shape (development aid; run under ncu for per-kernel shares)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
m, n, B = 256, 32, 5000
a = gen_batch_device("random", m, n, B, np.complex128, seed=0)
opts = bs.JacobiOptions(use_qr_preprocess=True)
for _ in range(2):
    r = bs.solve_tensor(a, m, n, opts)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); r = bs.solve_tensor(a, m, n, opts); e1.record(); torch.cuda.synchronize()
print(f"qr route C4: {e0.elapsed_time(e1):.2f} ms")
