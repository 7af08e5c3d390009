"""Host-buffer pipeline sweep (streams x chunk; argv: streams, divisors, batch) for C1-10k through bsvd_gesvj_batched_host, plus raw PCIe
copies (development aid).  Measured on B200: 4 streams x B/16 best (4.02 ms vs 4.26 ms at 3 x B/8);
raw D2H of the 167 MB of factors alone takes 2.93 ms, H2D of the 82 MB input 1.49 ms."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
from paper_2601_17979_b200.solver import solve_host_buffers

m = n = 32
B = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
a = gen_batch_device("arith", m, n, B, np.float64, kappa=1e10, seed=0)
a_h = torch.empty(a.shape, dtype=a.dtype, pin_memory=True)
a_h.copy_(a)
u_h = torch.empty((B, 32, 32), dtype=torch.float64, pin_memory=True)
s_h = torch.empty((B, 32), dtype=torch.float64, pin_memory=True)
v_h = torch.empty((B, 32, 32), dtype=torch.float64, pin_memory=True)
i_h = torch.empty((B * 48,), dtype=torch.uint8, pin_memory=True)
opts = bs.JacobiOptions()
dev = torch.device("cuda", 0)
NST = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,3,4,6").split(",")]
DIV = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,8,16,32").split(",")]
for nst in NST:
    for div in DIV:
        streams = [torch.cuda.current_stream()] + [torch.cuda.Stream(dev) for _ in range(nst - 1)]
        chunk = -(-B // div)
        ts = []
        for it in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            solve_host_buffers(a_h, u_h, s_h, v_h, i_h, m, n, opts, 0, chunk=chunk, streams=streams)
            e1.record()
            torch.cuda.synchronize()
            if it:
                ts.append(e0.elapsed_time(e1))
        t = min(ts)
        print(f"streams={nst} chunk=B/{div}: {t:.2f} ms  {B / t * 1e3 / 1e6:.2f} M mat/s", flush=True)
if B != 10000:
    sys.exit(0)
x = torch.empty(167_000_000 // 8, dtype=torch.float64, device=dev)
xh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    xh.copy_(x, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
print(f"D2H 167 MB: {e0.elapsed_time(e1):.2f} ms")
y = torch.empty(82_000_000 // 8, dtype=torch.float64, device=dev)
yh = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    y.copy_(yh, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
print(f"H2D 82 MB: {e0.elapsed_time(e1):.2f} ms")
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        xh.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        y.copy_(yh, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
print(f"D2H 167 MB + H2D 82 MB concurrently: {e0.elapsed_time(e1):.2f} ms")
