"""Save / compare the blocked FP64 register kernel's outputs across a refactor (development aid):
python tools/blk_bits.py save|cmp FILE.npz   (values compared with array_equal: +0 == -0)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
mode, path = sys.argv[1], sys.argv[2]
out = {}
for (fam, m, n, B, kappa, rank) in (("geo", 64, 64, 64, 1e12, None), ("rankdef", 64, 64, 64, 1e6, 48),
                                     ("random", 128, 128, 32, 1, None), ("random", 96, 96, 32, 1, None),
                                     ("geo", 128, 64, 32, 1e8, None), ("random", 200, 128, 16, 1, None),
                                     ("arith", 48, 48, 32, 1e4, None)):
    a = gen_batch_device(fam, m, n, B, np.float64, kappa=kappa, seed=m + n, rank=rank)
    for wantv in (True, False):
        r = bs.solve_tensor(a, m, n, bs.JacobiOptions(compute_right_vectors=wantv))
        torch.cuda.synchronize()
        key = f"{fam}_{m}_{n}_{int(wantv)}"
        out[key + "_u"] = r.u.cpu().numpy(); out[key + "_s"] = r.s.cpu().numpy()
        if wantv:
            out[key + "_v"] = r.v.cpu().numpy()
        out[key + "_i"] = r.info.cpu().numpy()
        out[key + "_k"] = np.array([r.kernel])
if mode == "save":
    np.savez_compressed(path, **out)
    print("saved", len(out))
else:
    ref = np.load(path)
    bad = [k for k in out if not np.array_equal(out[k], ref[k])]
    print("identical" if not bad else f"DIFFER: {bad}")
