import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_2601_17979_b200 as bs
A = np.outer(np.arange(1, 33), np.arange(1, 33)).astype(np.float64)[None]
a = torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2))).cuda()
for ms in (1, 2, 3, 5, 10, 20, 30):
    line = f"max_sweeps {ms:2d}"
    for k in (12, 42):
        r = bs.solve_tensor(a, 32, 32, bs.JacobiOptions(max_nsweeps=ms), kernel=k); torch.cuda.synchronize()
        S = r.s.cpu().numpy()[0]
        line += f" | k{k}: s2 {S[1]:.2e} s16 {S[15]:.2e} s32 {S[31]:.2e} fro(noise) {np.sqrt((S[1:]**2).sum()):.2e}"
    print(line)
