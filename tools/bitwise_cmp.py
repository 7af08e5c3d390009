"""Bitwise comparison of 32x32 FP64 kernel variants against gen. 2 (kernel 12) on mixed inputs
(development aid: which variants may share a batch-size switch without breaking batch == standalone)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs

ks = [int(k) for k in (sys.argv[1] if len(sys.argv) > 1 else "20,21,22,23,26").split(",")]
rng = np.random.default_rng(5)
A = rng.standard_normal((300, 32, 32))
A[5] = np.diag(np.geomspace(1.0, 1e-12, 32)) @ A[5]
A[9][:, 4] = 0.0
A[17] = 1.0
A[23] *= 1e-200
A[24] *= 1e+200
A[25][:, 3] *= 1e-170  # one column 1e170 below the rest
A[26][:, 7:9] *= 1e-300
for fam_i in range(30, 60):
    A[fam_i] = A[fam_i] @ np.diag(np.geomspace(1, 1e-8, 32))
a = torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2))).cuda()
for want_v in (True, False):
    opts = bs.JacobiOptions(compute_right_vectors=want_v)
    r0 = bs.solve_tensor(a, 32, 32, opts, kernel=12)
    torch.cuda.synchronize()
    for k in ks:
        r = bs.solve_tensor(a, 32, 32, opts, kernel=k)
        torch.cuda.synchronize()
        same_s = torch.equal(r.s, r0.s); same_u = torch.equal(r.u, r0.u)
        same_v = (not want_v) or torch.equal(r.v, r0.v)
        nd = int(((r.s != r0.s).any(1) | (r.u != r0.u).flatten(1).any(1)).sum())
        print(f"v={int(want_v)} k={k}: s {same_s} u {same_u} v {same_v} problems differing {nd}", flush=True)
if "--detail" in sys.argv:
    from paper_2601_17979_b200.solver import INFO_DTYPE
    r0 = bs.solve_tensor(a, 32, 32, bs.JacobiOptions(), kernel=12)
    r1 = bs.solve_tensor(a, 32, 32, bs.JacobiOptions(), kernel=26)
    torch.cuda.synchronize()
    d = ((r1.s != r0.s).any(1) | (r1.u != r0.u).flatten(1).any(1)).nonzero().flatten().tolist()
    i0 = np.frombuffer(r0.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    i1 = np.frombuffer(r1.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    for b in d:
        print(b, i0[b], i1[b], "max|ds|", float((r1.s[b] - r0.s[b]).abs().max()), "s1", float(r0.s[b, 0]),
              "u-diff cols", (r1.u[b] != r0.u[b]).any(1).nonzero().flatten().tolist()[:10])
