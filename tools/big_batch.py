import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch, paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import INFO_DTYPE
for B in (100000, 200000):
    a = gen_batch_device("arith", 32, 32, B, np.float64, kappa=1e10, seed=3)
    o = bs.JacobiOptions()
    r = bs.solve_tensor(a, 32, 32, o); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); r = bs.solve_tensor(a, 32, 32, o); e1.record(); torch.cuda.synchronize()
    info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    idx = [0, B // 3, B - 1]
    ah = a[idx].cpu().numpy()
    err = max(np.max(np.abs(r.s[i].cpu().numpy() - np.linalg.svd(ah[j].T, compute_uv=False))) / np.linalg.svd(ah[j].T, compute_uv=False)[0] for j, i in enumerate(idx))
    print(f"B={B}: {e0.elapsed_time(e1):.2f} ms, {B / e0.elapsed_time(e1) * 1e3 / 1e6:.2f} M mat/s, converged {info['converged'].mean():.4f}, kernels {sorted(set(info['kernel'].tolist()))}, max rel sigma err {err / 2**-53:.1f} u", flush=True)
