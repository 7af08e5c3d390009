"""Accuracy of the blocked FP64 kernels vs LAPACK for inner_sweeps 0 (budget 100) and 1 on the reference's
c03 inputs (random n x n, seeds 9000 n + s) and c09's mass conservation (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
u = 2.0 ** -53
for n in (64, 128):
    A = np.stack([np.random.default_rng(9000 * n + s).random((n, n)) for s in range(50)])
    ref = np.stack([np.linalg.svd(a, compute_uv=False) for a in A])
    fro2 = np.sum(A ** 2, axis=(1, 2))
    a_t = torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2))).cuda()
    for kern in (30, 8):
        for inner in (0, 1):
            o = bs.JacobiOptions(inner_sweeps=inner)
            try:
                r = bs.solve_tensor(a_t, n, n, o, kernel=kern)
                torch.cuda.synchronize()
            except Exception as e:
                print(n, kern, inner, "unsupported", e); continue
            S = r.s.cpu().numpy()
            e_s = np.max(np.abs(S - ref), axis=1) / (u * ref[:, 0])
            e_m = np.abs(np.sum(S ** 2, axis=1) - fro2) / (u * fro2)
            print(f"n={n} kernel={kern} inner_sweeps={inner}: max |dsigma| {e_s.max():.1f} u s1 (median {np.median(e_s):.1f}), "
                  f"mass {e_m.max():.1f} u (median {np.median(e_m):.1f})", flush=True)
