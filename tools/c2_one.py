"""One C2 solve (10,000 x 16x16 FP32, full or values) for ncu: python tools/c2_one.py full|vals"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
a = gen_batch_device("random", 16, 16, 10000, np.float32, kappa=1, seed=0)
o = bs.JacobiOptions(compute_right_vectors=(sys.argv[1] == "full"))
for _ in range(2):
    r = bs.solve_tensor(a, 16, 16, o)
torch.cuda.synchronize()
