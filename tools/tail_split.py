"""C1-10k split into a two-problems-per-warp head (kernel 42) and a one-problem-per-warp tail (kernel 52)
launched concurrently on two streams (development aid): does the tail wave finish sooner as 52?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_17979_b200 as bs
from paper_2601_17979_b200.matgen import gen_batch_device

B = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
a = gen_batch_device("arith", 32, 32, B, np.float64, kappa=1e10, seed=0)
opts = bs.JacobiOptions()
main = torch.cuda.current_stream()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(X, order):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        ev0.record(main)
        s1.wait_stream(main); s2.wait_stream(main)
        parts = [(s1, a[:B - X], 42), (s2, a[B - X:], 52)]
        if order:
            parts = parts[::-1]
        for st, aa, k in parts:
            if aa.shape[0] == 0:
                continue
            with torch.cuda.stream(st):
                bs.solve_tensor(aa, 32, 32, opts, kernel=k)
        main.wait_stream(s1); main.wait_stream(s2)
        ev1.record(main)
        torch.cuda.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    return min(ts), float(np.median(ts))


for X in [0, 296, 592, 888, 1184, 1480, 1776, 2368]:
    for order in (0, 1):
        if X == 0 and order:
            continue
        t, med = run(X, order)
        print(f"B={B} tail={X:5d} {'52 first' if order else '42 first'}: min {t:.3f} ms median {med:.3f} ms", flush=True)
