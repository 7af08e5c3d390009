"""Accuracy comparison of kernel variants against the CPU restatement (development aid)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import INFO_DTYPE
from oracle import oracle as O
from common import e1, e2, e3
kernels = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [3]
u = 2.0 ** -53
for fam, kappa in (("arith", 1e10), ("random", 1), ("geo", 1e10)):
    B = 512
    a = gen_batch_device(fam, 32, 32, B, np.float64, kappa=kappa, seed=7)
    A = np.swapaxes(a.cpu().numpy(), 1, 2)
    _, S_ref, _, infos = O.solve_batch(A, None, None, nthreads=0)
    sw_ref = np.array([i["outer_sweeps"] for i in infos])
    for kern in kernels:
        r = bs.solve_tensor(a, 32, 32, bs.JacobiOptions(), kernel=kern)
        torch.cuda.synchronize()
        info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
        U = np.swapaxes(r.u.cpu().numpy(), 1, 2); S = r.s.cpu().numpy(); V = np.swapaxes(r.v.cpu().numpy(), 1, 2)
        E1 = np.array([e1(A[b], U[b], S[b], V[b]) for b in range(B)]) / u
        E2 = np.array([e2(U[b]) for b in range(B)]) / u
        E3 = np.array([e3(V[b]) for b in range(B)]) / u
        ds = np.max(np.abs(S - S_ref), axis=1) / S_ref[:, 0] / u
        dsw = info["outer_sweeps"] - sw_ref
        print(f"{fam:6s} k={kern}: e1 max {E1.max():5.2f} mean {E1.mean():5.2f} | e2 max {E2.max():5.2f} mean {E2.mean():5.2f} | "
              f"e3 max {E3.max():5.2f} mean {E3.mean():5.2f} | dsigma/u/s1 max {ds.max():5.2f} mean {ds.mean():5.2f} | "
              f"dsweeps {dsw.min()}..{dsw.max()} conv {info['converged'].mean():.3f}", flush=True)
