"""Timing of the shapes that run on the general blocked kernel (complex / FP32 with n > 32), vs the FP64
register kernel on the same shape (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import INFO_DTYPE
for dt in (np.float64, np.float32, np.complex128, np.complex64):
    for n, B in ((64, 2000), (128, 500)):
        a = gen_batch_device("random", n, n, B, dt, seed=1)
        r = bs.solve_tensor(a, n, n, bs.JacobiOptions()); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = bs.solve_tensor(a, n, n, bs.JacobiOptions()); e1.record(); torch.cuda.synchronize()
        info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
        print(f"{np.dtype(dt).name:10s} n={n:3d} B={B:5d} kernel={int(info['kernel'][0]):2d} {e0.elapsed_time(e1):8.2f} ms "
              f"{B / e0.elapsed_time(e1) * 1e3:10,.0f} mat/s sweeps {info['outer_sweeps'].mean():.2f}", flush=True)
# accuracy of the promoted FP32 path vs the oracle (sigma parity in u_32, sweeps)
from oracle import oracle as O
u32 = 2.0 ** -24
for n, B in ((64, 200), (128, 40), (48, 40)):
    a = gen_batch_device("random", n, n, B, np.float32, seed=2)
    r = bs.solve_tensor(a, n, n, bs.JacobiOptions()); torch.cuda.synchronize()
    info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    ah = a.cpu().numpy(); S = r.s.cpu().numpy()
    ds, dsw = 0.0, []
    for i in range(0, B, max(1, B // 10)):
        _, s_ref, _, inf = O.solve(np.ascontiguousarray(ah[i].T).copy(order="F"), None, None)
        ds = max(ds, float(np.max(np.abs(S[i].astype(np.float64) - s_ref))) / (u32 * s_ref[0]))
        dsw.append(int(info["outer_sweeps"][i]) - inf["outer_sweeps"])
    print(f"f32 n={n}: kernel {int(info['kernel'][0])} max|ds| {ds:.2f} u32 s1 (bound n = {n}), sweeps diff {min(dsw)}..{max(dsw)}")
