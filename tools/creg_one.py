"""One complex solve with the default kernel (for ncu): python tools/creg_one.py M N BATCH"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
m, n, B = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a = gen_batch_device("random", m, n, B, np.complex128, kappa=1, seed=5)
for _ in range(2):
    r = bs.solve_tensor(a, m, n, bs.JacobiOptions())
torch.cuda.synchronize()
