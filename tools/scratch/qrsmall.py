import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.solver import solve_tensor
for (m, n, dt) in [(96, 32, np.float64), (96, 32, np.complex128), (256, 32, np.complex128)]:
    rng = np.random.default_rng(0)
    A = rng.random((4, n, m)).astype(dt)
    a = torch.from_numpy(A).cuda()
    t0 = time.time()
    r = solve_tensor(a, m, n, bs.JacobiOptions(use_qr_preprocess=True))
    torch.cuda.synchronize()
    print(m, n, dt.__name__, "ok", time.time() - t0, r.s[0, :3].tolist(), flush=True)
