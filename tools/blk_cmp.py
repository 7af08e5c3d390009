"""Blocked FP64 variants (30 default, 49 scaled rotations): timing + accuracy vs the oracle (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import INFO_DTYPE
from oracle import oracle as O
kerns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "30,49").split(",")]
u = 2.0 ** -53
cases = [("geo", 64, 1e12, 10000, None), ("rankdef", 64, 1e6, 10000, 48), ("random", 128, 1, 2000, None),
         ("random", 64, 1, 2000, None), ("geo", 128, 1e12, 500, None), ("random", 96, 1, 500, None)]
for fam, n, kappa, B, rank in cases:
    a = gen_batch_device(fam, n, n, B, np.float64, kappa=kappa, seed=5, rank=rank)
    ah = a.cpu().numpy()
    samp = list(range(0, B, max(1, B // 8)))[:8]
    ref = [O.solve(np.ascontiguousarray(ah[i].T).copy(order="F"), None, None) for i in samp]
    line = f"{fam:7s} n={n:3d} B={B:5d}"
    for k in kerns:
        opts = bs.JacobiOptions()
        r = bs.solve_tensor(a, n, n, opts, kernel=k); torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(2):
            ev0.record(); r = bs.solve_tensor(a, n, n, opts, kernel=k); ev1.record(); torch.cuda.synchronize()
            ts.append(ev0.elapsed_time(ev1))
        info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
        S = r.s.cpu().numpy(); U = np.swapaxes(r.u.cpu().numpy(), 1, 2); V = np.swapaxes(r.v.cpu().numpy(), 1, 2)
        ds = max(float(np.max(np.abs(S[i] - ref[j][1]))) / (u * ref[j][1][0]) for j, i in enumerate(samp))
        dsw = [int(info["outer_sweeps"][i]) - ref[j][3]["outer_sweeps"] for j, i in enumerate(samp)]
        e1 = max(np.linalg.norm(ah[i].T - (U[i] * S[i]) @ V[i].T, 1) / np.linalg.norm(ah[i].T, 1) / (n * u) for i in samp)
        e2 = max(np.abs(U[i].T @ U[i] - np.eye(n)).max() / (n * u) for i in samp)
        e3 = max(np.abs(V[i].T @ V[i] - np.eye(n)).max() / (n * u) for i in samp)
        line += (f" | k{k} {min(ts):.2f} ms sw {info['outer_sweeps'].mean():.2f} dsw {min(dsw)}..{max(dsw)}"
                 f" ds {ds:.1f}u e {e1:.2f}/{e2:.2f}/{e3:.2f}")
    print(line, flush=True)
