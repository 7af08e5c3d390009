import sys, time; sys.path.insert(0, "/root/repo")
import numpy as np, torch, paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
dev = torch.device("cuda", 0)
a = gen_batch_device("random", 16, 16, 10000, np.float32, kappa=1, seed=0)
o = bs.JacobiOptions()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for pre in ("none", "sleep2M", "flush x40", "solve x40"):
    time.sleep(0.3)
    for _ in range(3): bs.solve_tensor(a, 16, 16, o)
    torch.cuda.synchronize()
    if pre == "sleep2M": torch.cuda._sleep(2_000_000)
    if pre == "flush x40":
        for _ in range(40): flush.fill_(1.0)
    if pre == "solve x40":
        for _ in range(40): bs.solve_tensor(a, 16, 16, o)
    evs = []
    for _ in range(8):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); bs.solve_tensor(a, 16, 16, o); e1.record(); evs.append((e0, e1))
    torch.cuda.synchronize()
    print(pre, " ".join(f"{e0.elapsed_time(e1)*1e3:.0f}" for e0, e1 in evs), flush=True)
