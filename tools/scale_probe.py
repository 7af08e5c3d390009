"""Beyond the reference's exponent range (development aid): uniform scalings 1e+-150 (FP64) / 1e+-15
(FP32) and 1e+-100 / 1e+-8 graded columns and rows through every default kernel; sigma vs a float64
LAPACK SVD, finiteness of the factors.  (The reference's own guard product overflows here.)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.solver import INFO_DTYPE
from common import random_matrix, unit_roundoff, e2

CASES = [(np.float64, 32, 32, 0, False), (np.float64, 32, 32, 12, False), (np.float32, 16, 16, 0, False),
         (np.float32, 16, 16, 34, False), (np.float64, 64, 64, 0, False), (np.complex128, 256, 32, 0, False),
         (np.complex128, 40, 24, 0, False), (np.float32, 48, 48, 0, False), (np.float64, 96, 20, 0, True),
         (np.complex128, 256, 32, 0, True), (np.float64, 128, 128, 0, False), (np.complex128, 64, 32, 0, False)]
for dt, m, n, kernel, qr in CASES:
    single = unit_roundoff(dt) > 1e-10
    e, g = (15, 8) if single else (150, 100)
    base = [random_matrix(m, n, dt, seed=9100 + i) for i in range(4)]
    A = [base[0] * 10.0 ** -e, base[1] * 10.0 ** e, base[3] * np.geomspace(10.0 ** -g, 10.0 ** g, n)[None, :],
         base[0] * np.geomspace(10.0 ** g, 10.0 ** -g, m)[:, None]]
    A = np.stack([x.astype(dt) for x in A])
    a = torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2))).cuda()
    r = bs.solve_tensor(a, m, n, bs.JacobiOptions(use_qr_preprocess=qr), kernel=kernel)
    torch.cuda.synchronize()
    info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    U, S = np.swapaxes(r.u.cpu().numpy(), 1, 2), r.s.cpu().numpy()
    out = []
    for b in range(A.shape[0]):
        st = np.linalg.svd(A[b].astype(np.complex128 if np.iscomplexobj(A[b]) else np.float64), compute_uv=False)
        fin = np.isfinite(U[b]).all() and np.isfinite(S[b]).all()
        err = np.max(np.abs(S[b] - st)) / st[0] / unit_roundoff(dt) if fin else float("nan")
        out.append(f"[{'ok ' if fin else 'NaN'} conv={int(info['converged'][b])} sw={int(info['outer_sweeps'][b]):2d} dS={err:9.1f}u e2={e2(U[b]) / unit_roundoff(dt) if fin else float('nan'):9.1f}u]")
    print(f"{np.dtype(dt).name:10s} {m:3d}x{n:<3d} k={int(info['kernel'][0]):2d} qr={int(qr)} " + " ".join(out), flush=True)
