import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch, paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device
dev = torch.device("cuda", 0)
for (fam, m, n, B, dt, wantv) in (("random", 16, 16, 10000, np.float32, True), ("random", 16, 16, 10000, np.float32, False),
                                  ("arith", 32, 32, 10000, np.float64, True), ("arith", 32, 32, 1000, np.float64, True)):
    a = gen_batch_device(fam, m, n, B, dt, kappa=1e10 if m == 32 else 1, seed=0)
    o = bs.JacobiOptions(compute_right_vectors=wantv)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(3): bs.solve_tensor(a, m, n, o)
    torch.cuda.synchronize()
    res = {}
    for mode in ("idle", "behind_flush", "behind_long"):
        ts = []
        for _ in range(10):
            if mode == "behind_flush":
                flush.fill_(1.0)
            elif mode == "behind_long":
                torch.cuda._sleep(2_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); bs.solve_tensor(a, m, n, o); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res[mode] = np.median(ts)
    print(f"{m}x{n} B={B} v={wantv}: " + ", ".join(f"{k} {v:.1f} us" for k, v in res.items()), flush=True)

# the bench loop: flush, e0, solve_rank_slice, e1 -- no synchronisation between steps
from paper_2601_17979_b200.parallel import solve_rank_slice
import time
for (fam, m, n, B, dt, wantv) in (("random", 16, 16, 10000, np.float32, True), ("random", 16, 16, 10000, np.float32, False)):
    a = gen_batch_device(fam, m, n, B, dt, kappa=1, seed=0)
    o = bs.JacobiOptions(compute_right_vectors=wantv)
    out = None
    for _ in range(3):
        res = solve_rank_slice(a, m, n, o, 0, 1)[2]
    out = (res.u, res.s, res.v, res.info)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    evs = []
    th = []
    st = torch.cuda.current_stream()
    for _ in range(10):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        h0 = time.perf_counter()
        res = solve_rank_slice(a, m, n, o, 0, 1, out=out)[2]
        th.append((time.perf_counter() - h0) * 1e6)
        e1.record(st)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ts = [e0.elapsed_time(e1) * 1e3 for e0, e1 in evs]
    print(f"bench-loop {m}x{n} v={wantv}: device per step {ts}  host per step median {np.median(th):.1f} us", flush=True)
