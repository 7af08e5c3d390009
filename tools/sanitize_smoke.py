"""One small batch through every kernel family, for compute-sanitizer runs (development aid):
    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_17979_b200 as bs

rng = np.random.default_rng(1)


def run(dt, m, n, route=0, kernel=0, B=3, tail=0, **kw):
    A = rng.random((B, n, m))
    if np.dtype(dt).kind == "c":
        A = A + 1j * rng.random((B, n, m))
    a = torch.from_numpy(A.astype(dt)).cuda()
    r = bs.solve_tensor(a, m, n, bs.JacobiOptions(**kw), route=route, kernel=kernel, tail=tail)
    torch.cuda.synchronize()
    print(dt.__name__, m, n, route, kernel, "ok", float(r.s[0, 0]), flush=True)


run(np.float64, 32, 32)                       # r32b scaled rotations, V in lockstep (52) + fused finalise
run(np.float64, 32, 32, kernel=42, B=5)       # r32b scaled rotations, two problems per warp (42)
run(np.float64, 32, 32, B=40, tail=13)        # r32b head (42) + tail (52) in one launch (k_reg32b_split)
run(np.float64, 32, 32, compute_right_vectors=False)  # r32b values only (12)
run(np.float32, 16, 16)                       # reg16b
run(np.float32, 16, 16, kernel=34, B=9)       # reg16c (quarter-warp)
run(np.float32, 16, 16, kernel=34, B=5, compute_right_vectors=False)
run(np.float64, 64, 64)                       # blocked_reg
run(np.float64, 128, 128, B=2)                # blocked_reg NWG 2
run(np.complex128, 256, 32, B=2)              # creg32 SP
run(np.complex128, 64, 32)                    # creg32 register V
run(np.complex128, 256, 32, B=2, use_qr_preprocess=True)  # qr_col + creg32 + applyq_col
run(np.float64, 96, 20, use_qr_preprocess=True)
run(np.complex64, 40, 24)                     # general unblocked
run(np.complex128, 64, 64, B=2)               # complex register blocked (k_cregb)
run(np.complex64, 48, 48, B=2)                # complex64 promoted to k_cregb
run(np.complex128, 128, 128, B=1)             # k_cregb delta mode (n > 64)
run(np.float64, 64, 64, B=2, inner_sweeps=0)  # blocked_reg delta mode (inner budget 100)
run(np.float32, 64, 64, B=2)                  # FP32 blocked promoted to the FP64 register blocked kernel
run(np.float32, 32, 32, B=3)                  # FP32 32x32 promoted to the FP64 32x32 kernel
run(np.complex64, 256, 32, B=2)               # complex64 promoted to creg32
run(np.complex128, 256, 32, B=2, kernel=45)   # creg32 with the TMA (bulk-copy) loader
run(np.float32, 48, 48)                       # general blocked
q, r = bs.householder_qr(rng.random((40, 12)))
f = bs.finalize(rng.random((20, 7)), rng.random((7, 7)))
g = rng.random((10, 10)); g = g + g.T
d = np.diag(g).copy(); m = np.zeros((10, 10))
w = np.triu(g, 1); w = np.asfortranarray(w + w.T)
bs.eig_sweeps(w, d, m, tol=1e-14, max_sweeps=5, delta=True)
ev = bs.jacobi_hermitian_eig(g)
print("all ok")
