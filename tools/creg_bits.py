"""Save / compare the complex register kernel's outputs (bitwise regression check across a refactor):
python tools/creg_bits.py save|cmp FILE"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hashlib, json
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
mode, path = sys.argv[1], sys.argv[2]
out = {}
for (m, B, route, fam) in ((256, 300, 0, "random"), (64, 300, 0, "geo"), (32, 300, 2, "random"), (100, 200, 0, "rankdef"),
                           (33, 100, 0, "random"), (256, 100, 2, "arith")):
    a = gen_batch_device(fam, m, 32, B, np.complex128, kappa=1e8, seed=m, rank=20 if fam == "rankdef" else None)
    for wantv in (True, False):
        r = bs.solve_tensor(a, m, 32, bs.JacobiOptions(compute_right_vectors=wantv), route=route)
        torch.cuda.synchronize()
        key = f"{m}_{B}_{route}_{fam}_{int(wantv)}"
        out[key + "_u"] = r.u.cpu().numpy(); out[key + "_s"] = r.s.cpu().numpy()
        if wantv:
            out[key + "_v"] = r.v.cpu().numpy()
        out[key + "_i"] = r.info.cpu().numpy()
dig = {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() for k, v in out.items()}
if mode == "save":
    json.dump(dig, open(path, "w"), indent=0)
    print("saved", len(dig))
else:
    ref = json.load(open(path))
    bad = [k for k in dig if dig[k] != ref.get(k)]
    print("bitwise identical" if not bad else f"DIFFER: {bad}")
