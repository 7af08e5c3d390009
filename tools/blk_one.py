"""One blocked FP64 solve (for ncu): python tools/blk_one.py c3|c5"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
cfg = sys.argv[1]
if cfg == "c3":
    a = gen_batch_device("geo", 64, 64, 10000, np.float64, kappa=1e12, seed=0); m = n = 64
else:
    a = gen_batch_device("random", 128, 128, 2000, np.float64, seed=0); m = n = 128
for _ in range(2):
    r = bs.solve_tensor(a, m, n, bs.JacobiOptions())
torch.cuda.synchronize()
