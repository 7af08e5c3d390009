"""One 32x32 FP64 solve with a forced kernel (for ncu): python tools/r32_one.py KERNEL BATCH"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
k, B = int(sys.argv[1]), int(sys.argv[2])
a = gen_batch_device("arith", 32, 32, B, np.float64, kappa=1e10, seed=5)
for _ in range(2):
    r = bs.solve_tensor(a, 32, 32, bs.JacobiOptions(), kernel=k)
torch.cuda.synchronize()
