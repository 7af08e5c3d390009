"""Scaled-rotation (FG) accuracy probe: sigma and V corrected by V's column norms on the host (development aid)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from oracle import oracle as O
from common import e1, e2, e3
kern = int(sys.argv[1]) if len(sys.argv) > 1 else 42
u = 2.0 ** -53
for fam, kappa in (("arith", 1e10), ("random", 1), ("geo", 1e10)):
    B = 512
    a = gen_batch_device(fam, 32, 32, B, np.float64, kappa=kappa, seed=7)
    A = np.swapaxes(a.cpu().numpy(), 1, 2)
    _, S_ref, _, infos = O.solve_batch(A, None, None, nthreads=0)
    r = bs.solve_tensor(a, 32, 32, bs.JacobiOptions(), kernel=kern); torch.cuda.synchronize()
    U = np.swapaxes(r.u.cpu().numpy(), 1, 2); S = r.s.cpu().numpy(); V = np.swapaxes(r.v.cpu().numpy(), 1, 2)
    vn = np.linalg.norm(V, axis=1)  # (B, k) column norms
    for tag, Sx, Vx in (("raw", S, V), ("vnorm", S / vn, V / vn[:, None, :])):
        E1 = max(e1(A[b], U[b], Sx[b], Vx[b]) for b in range(B)) / u
        E3 = max(e3(Vx[b]) for b in range(B)) / u
        ds = np.max(np.abs(np.sort(Sx, axis=1)[:, ::-1] - S_ref), axis=1) / S_ref[:, 0] / u
        print(f"{fam:6s} {tag:5s}: e1 {E1:5.2f} e3 {E3:5.2f} dsigma/u/s1 max {ds.max():6.2f} mean {ds.mean():5.2f} "
              f"| vnorm dev max {np.abs(vn - 1).max() / u:6.2f}u", flush=True)
