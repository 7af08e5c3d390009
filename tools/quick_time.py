"""Quick device timing of the solver on BASELINE shapes (development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import INFO_DTYPE

cfgs = [("C1-10k", "arith", 32, 32, 10000, np.float64, 1e10, True),
        ("C1-1k", "arith", 32, 32, 1000, np.float64, 1e10, True),
        ("C1-3k", "arith", 32, 32, 3000, np.float64, 1e10, True),
        ("C1-1.5k", "arith", 32, 32, 1500, np.float64, 1e10, True),
        ("C1-1250", "arith", 32, 32, 1250, np.float64, 1e10, True),
        ("C1-2k", "arith", 32, 32, 2000, np.float64, 1e10, True),
        ("C1-2.5k", "arith", 32, 32, 2500, np.float64, 1e10, True),
        ("C1-500", "arith", 32, 32, 500, np.float64, 1e10, True),
        ("C1-1100", "arith", 32, 32, 1100, np.float64, 1e10, True),
        ("C1-1184", "arith", 32, 32, 1184, np.float64, 1e10, True),
        ("C2-full", "random", 16, 16, 10000, np.float32, 1, True),
        ("C2-vals", "random", 16, 16, 10000, np.float32, 1, False),
        ("C4", "random", 256, 32, 5000, np.complex128, 1, True),
        ("C3", "geo", 64, 64, 2000, np.float64, 1e12, True),
        ("C5", "random", 128, 128, 500, np.float64, 1, True),
        ("C3-10k", "geo", 64, 64, 10000, np.float64, 1e12, True),
        ("C5-2k", "random", 128, 128, 2000, np.float64, 1, True)]
args = sys.argv[1:]
kernels = [0]
if "--kernels" in args:
    i = args.index("--kernels"); kernels = [int(x) for x in args[i+1].split(",")]; del args[i:i+2]
tail = 0
if "--tail" in args:
    i = args.index("--tail"); tail = int(args[i+1]); del args[i:i+2]
only = args
for name, fam, m, n, B, dt, kappa, wantv in cfgs:
    if only and name not in only: continue
    a = gen_batch_device(fam, m, n, B, dt, kappa=kappa, seed=0)
    opts = bs.JacobiOptions(compute_right_vectors=wantv)
    for kern in kernels:
      try:
          r = bs.solve_tensor(a, m, n, opts, kernel=kern, tail=tail); torch.cuda.synchronize()
      except RuntimeError as exc:
          print(f"{name:8s} kernel={kern}: {exc}"); continue
      ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
      ts = []
      for _ in range(3):
        ev0.record(); r = bs.solve_tensor(a, m, n, opts, kernel=kern, tail=tail); ev1.record(); torch.cuda.synchronize()
        ts.append(ev0.elapsed_time(ev1))
      info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
      t = min(ts)
      print(f"{name:8s} B={B} {m}x{n} {np.dtype(dt).name} kernel={int(info['kernel'][0])} {t:.2f} ms  {B/t*1e3:,.0f} mat/s  "
          f"sweeps={info['outer_sweeps'].mean():.2f} conv={info['converged'].mean():.3f} rot/mat={info['rotations'].mean():.0f}", flush=True)
