import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from common import e1, e2, e3
from test_gpu_parity import _exactly_rank_deficient
from paper_2601_17979_b200.solver import INFO_DTYPE
A = _exactly_rank_deficient(32, np.float64)
a = torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2))).cuda()
for k in (12, 42):
    r = bs.solve_tensor(a, 32, 32, bs.JacobiOptions(), kernel=k); torch.cuda.synchronize()
    U, S, V = np.swapaxes(r.u.cpu().numpy(), 1, 2), r.s.cpu().numpy(), np.swapaxes(r.v.cpu().numpy(), 1, 2)
    info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    for b in range(A.shape[0]):
        print(k, b, f"e1 {e1(A[b],U[b],S[b],V[b]):.2e} e2 {e2(U[b]):.2e} e3 {e3(V[b]):.2e}", info["outer_sweeps"][b], info["converged"][b], S[b][:3], S[b][-3:])
        if e2(U[b]) > 1e-10:
            G = U[b].T @ U[b]; bad = np.where(np.abs(np.diag(G) - 1) > 1e-8)[0]
            print("  bad cols", bad, np.diag(G)[bad][:5], "norms", np.linalg.norm(U[b], axis=0)[:5])
