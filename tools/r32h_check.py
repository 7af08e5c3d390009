"""reg32h (47/48) vs the default (42): timing + accuracy vs the oracle on a sample (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import INFO_DTYPE
from oracle import oracle as O
kerns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "42,47,48").split(",")]
u = 2.0 ** -53
for fam, kappa, B in (("arith", 1e10, 10000), ("arith", 1e10, 1250), ("random", 1, 10000), ("geo", 1e12, 2000),
                      ("rankdef", 1e6, 2000), ("arith", 1e10, 7)):
    a = gen_batch_device(fam, 32, 32, B, np.float64, kappa=kappa, seed=5)
    ah = a.cpu().numpy()
    samp = list(range(0, B, max(1, B // 24)))[:24]
    ref = [O.solve(np.ascontiguousarray(ah[i].T).copy(order="F"), None, None) for i in samp]
    line = f"{fam:7s} B={B:5d}"
    for k in kerns:
        opts = bs.JacobiOptions()
        try:
            r = bs.solve_tensor(a, 32, 32, opts, kernel=k); torch.cuda.synchronize()
        except Exception as e:
            line += f" | k{k} ERR {e}"; continue
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(3):
            ev0.record(); r = bs.solve_tensor(a, 32, 32, opts, kernel=k); ev1.record(); torch.cuda.synchronize()
            ts.append(ev0.elapsed_time(ev1))
        info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
        S = r.s.cpu().numpy(); U = np.swapaxes(r.u.cpu().numpy(), 1, 2); V = np.swapaxes(r.v.cpu().numpy(), 1, 2)
        ds = max(float(np.max(np.abs(S[i] - ref[j][1]))) / (u * ref[j][1][0]) for j, i in enumerate(samp))
        dsw = max(abs(int(info["outer_sweeps"][i]) - ref[j][3]["outer_sweeps"]) for j, i in enumerate(samp))
        e1 = max(np.linalg.norm(ah[i].T - (U[i] * S[i]) @ V[i].T) / np.linalg.norm(ah[i]) / u for i in samp)
        e2 = max(np.linalg.norm(U[i].T @ U[i] - np.eye(32)) / u for i in samp)
        e3 = max(np.linalg.norm(V[i].T @ V[i] - np.eye(32)) / u for i in samp)
        line += (f" | k{k} {min(ts):.3f} ms conv {info['converged'].mean():.3f} sw {info['outer_sweeps'].mean():.2f}"
                 f" ds {ds:.1f}u dsw {dsw} e {e1:.1f}/{e2:.1f}/{e3:.1f}")
    print(line, flush=True)
