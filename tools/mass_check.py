"""Frobenius-mass conservation |sum sigma^2 - ||A||_F^2| / (u ||A||_F^2) (the reference's acceptance c09 bar
is 30u) and max |sigma - sigma_LAPACK| / (u sigma_1) over random batches of every kernel family (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.solver import INFO_DTYPE
cases = [(32, 32, np.float64, 400), (16, 16, np.float32, 400), (64, 64, np.float64, 100), (128, 128, np.float64, 50),
         (96, 96, np.float64, 50), (256, 32, np.complex128, 100), (64, 64, np.complex128, 50), (128, 128, np.complex128, 30),
         (48, 48, np.float32, 50), (128, 128, np.float32, 30), (32, 32, np.complex64, 100)]
for m, n, dt, B in cases:
    rng = np.random.default_rng(m * 7 + n)
    A = rng.random((B, m, n))
    if np.dtype(dt).kind == "c":
        A = A + 1j * rng.random((B, m, n))
    A = A.astype(dt)
    a_t = torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2))).cuda()
    r = bs.solve_tensor(a_t, m, n, bs.JacobiOptions())
    torch.cuda.synchronize()
    S = r.s.cpu().numpy().astype(np.float64)
    kern = sorted(set(np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)["kernel"].tolist()))
    u = bs.unit_roundoff(dt)
    A64 = A.astype(np.complex128) if np.dtype(dt).kind == "c" else A.astype(np.float64)
    fro2 = np.sum(np.abs(A64) ** 2, axis=(1, 2))
    mass = np.abs(np.sum(S ** 2, axis=1) - fro2) / (u * fro2)
    ref = np.stack([np.linalg.svd(x, compute_uv=False) for x in A64])
    es = np.max(np.abs(S - ref), axis=1) / (u * ref[:, 0])
    print(f"{m}x{n} {np.dtype(dt).name} kernel {kern}: mass max {mass.max():.1f}u (median {np.median(mass):.1f}), "
          f"sigma max {es.max():.1f}u s1", flush=True)
