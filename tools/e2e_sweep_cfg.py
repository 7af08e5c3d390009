"""Host-buffer pipeline sweep over chunk counts for any bench config (development aid):
python tools/e2e_sweep_cfg.py CONFIG [divisors]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200 import _lib
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import solve_host_buffers, torch_dtype
cfg = bench.CONFIGS[sys.argv[1]]
divs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "8,16,32,64").split(",")]
dt = np.dtype(cfg["dtype"])
m, n, B = cfg["m"], cfg["n"], cfg["batch"]
k = min(m, n)
a = gen_batch_device(cfg["family"], m, n, B, dt, kappa=cfg["kappa"], seed=0, rank=cfg.get("rank"))
opts = bs.JacobiOptions(compute_right_vectors=cfg["want_v"], use_qr_preprocess=cfg.get("use_qr", False))
route = {None: _lib.DISPATCH, "blocked": _lib.FORCE_BLOCKED}[cfg["route"]]
tdt = torch_dtype(dt)
rdt = torch.float64 if dt in (np.float64, np.complex128) else torch.float32
a_h = torch.empty(a.shape, dtype=a.dtype, pin_memory=True); a_h.copy_(a)
u_h = torch.empty((B, k, m), dtype=tdt, pin_memory=True)
s_h = torch.empty((B, k), dtype=rdt, pin_memory=True)
v_h = torch.empty((B, k, n), dtype=tdt, pin_memory=True) if cfg["want_v"] else None
i_h = torch.empty((B * 48,), dtype=torch.uint8, pin_memory=True)
dev = torch.device("cuda", 0)
streams = [torch.cuda.current_stream()] + [torch.cuda.Stream(dev) for _ in range(3)]
for div in divs:
    ts = []
    for it in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        solve_host_buffers(a_h, u_h, s_h, v_h, i_h, m, n, opts, route, chunk=-(-B // div), streams=streams)
        e1.record()
        torch.cuda.synchronize()
        if it:
            ts.append(e0.elapsed_time(e1))
    print(f"{sys.argv[1]} chunk=B/{div}: {min(ts):.2f} ms  {B / min(ts) * 1e3:,.0f} mat/s", flush=True)
