"""Single-precision shapes that run on the general kernels vs their double-precision register kernels
(development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import INFO_DTYPE
for dt, m, n, B in ((np.float32, 32, 32, 10000), (np.float64, 32, 32, 10000), (np.complex64, 256, 32, 5000),
                    (np.complex128, 256, 32, 5000), (np.complex64, 32, 32, 5000), (np.complex128, 32, 32, 5000),
                    (np.float32, 24, 24, 10000)):
    a = gen_batch_device("random", m, n, B, dt, seed=1)
    for _ in range(3):
        r = bs.solve_tensor(a, m, n, bs.JacobiOptions()); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = bs.solve_tensor(a, m, n, bs.JacobiOptions()); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts)
    info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    print(f"{np.dtype(dt).name:10s} {m}x{n} B={B:5d} kernel={int(info['kernel'][0]):2d} {t:8.2f} ms "
          f"{B / t * 1e3:12,.0f} mat/s sweeps {info['outer_sweeps'].mean():.2f}", flush=True)
