"""Host pipeline fill probe (development aid): e2e time of a bench config through solve_host_buffers with the
current BSVD_RAMP setting, plus the raw pinned H2D / D2H / concurrent copy rates of the same byte counts.
python tools/ramp_probe.py CONFIG"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200 import _lib
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import solve_host_buffers, torch_dtype, default_chunk, _sm_count
cfg = bench.CONFIGS[sys.argv[1]]
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
NS = int(os.environ.get("NSTREAMS", "4"))
streams = [torch.cuda.current_stream()] + [torch.cuda.Stream(dev) for _ in range(NS - 1)]
es = dt.itemsize
per = m * n * es + m * k * es + (n * k * es if cfg["want_v"] else 0)
chunk = int(os.environ.get("CHUNK", "0")) or default_chunk(B, per, m * n, NS, _sm_count(dev))
ev = lambda: torch.cuda.Event(enable_timing=True)
def timed(fn, reps=6):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); e0, e1 = ev(), ev(); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]
t = timed(lambda: solve_host_buffers(a_h, u_h, s_h, v_h, i_h, m, n, opts, route, kernel=int(os.environ.get('KERNEL', '0')), chunk=chunk, streams=streams))
dout = torch.empty(u_h.numel() * es + (v_h.numel() * es if v_h is not None else 0), dtype=torch.uint8, device=dev)
hout = torch.empty(dout.numel(), dtype=torch.uint8, pin_memory=True)
din = torch.empty(a_h.numel() * es, dtype=torch.uint8, device=dev)
hin = a_h.view(-1).view(torch.uint8)
th = timed(lambda: din.copy_(hin, non_blocking=True))
td = timed(lambda: hout.copy_(dout, non_blocking=True))
s2 = streams[1]
def both():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        din.copy_(hin, non_blocking=True)
    hout.copy_(dout, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
tb = timed(both)
print(f"kernel={os.environ.get('KERNEL', '0')} ns={NS} ramp={os.environ.get('BSVD_RAMP', '1')} chunk={chunk} e2e {t:.3f} ms ({B / t * 1e3 / 1e6:.3f} M/s) | "
      f"H2D {hin.numel() / 1e6:.0f} MB {th:.3f} ms ({hin.numel() / th / 1e6:.1f} GB/s) D2H {hout.numel() / 1e6:.0f} MB "
      f"{td:.3f} ms ({hout.numel() / td / 1e6:.1f} GB/s) both {tb:.3f} ms", flush=True)
import time
hs = []
for _ in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    solve_host_buffers(a_h, u_h, s_h, v_h, i_h, m, n, opts, route, kernel=int(os.environ.get('KERNEL', '0')), chunk=chunk, streams=streams)
    hs.append((time.perf_counter() - t0) * 1e3)
    torch.cuda.synchronize()
print("host enqueue ms", [round(x, 3) for x in hs], flush=True)
# chunk-kernel latency alone
from paper_2601_17979_b200.solver import solve_tensor
ad = a[:chunk].contiguous()
print("kernel on one chunk ms", round(timed(lambda: solve_tensor(ad, m, n, opts, route)), 3),
      "full batch ms", round(timed(lambda: solve_tensor(a, m, n, opts, route)), 3), flush=True)
