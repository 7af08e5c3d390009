import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.solver import INFO_DTYPE
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
kern = int(sys.argv[2]) if len(sys.argv) > 2 else 3
maxs = int(sys.argv[3]) if len(sys.argv) > 3 else 30
rng = np.random.default_rng(0)
A = rng.random((B, 32, 32))
a = torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2))).cuda()
r = bs.solve_tensor(a, 32, 32, bs.JacobiOptions(max_nsweeps=maxs), kernel=kern)
print("launched", flush=True)
torch.cuda.synchronize()
info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
print(info[:4])
s = r.s.cpu().numpy()
ref = np.linalg.svd(A, compute_uv=False)
print("max sigma err", np.abs(s - ref).max())
