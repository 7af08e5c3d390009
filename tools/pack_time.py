"""Host packing cost of the list API (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2601_17979_b200 import _lib, solver
B = 10000
rng = np.random.default_rng(0)
mats = [np.asfortranarray(rng.random((32, 32))) for _ in range(B)]
host = solver._pinned("a", (B, 32, 32), torch.float64)
dt = np.dtype(np.float64)
for it in range(3):
    t0 = time.perf_counter(); ok = all(a.flags.f_contiguous and a.dtype == dt for a in mats); t1 = time.perf_counter()
    ptrs = np.fromiter((a.__array_interface__["data"][0] for a in mats), dtype=np.uintp, count=B); t2 = time.perf_counter()
    ptrs2 = np.fromiter((a.ctypes.data for a in mats), dtype=np.uintp, count=B); t3 = time.perf_counter()
    _lib.load().bsvd_pack_host(ptrs.ctypes.data, B, 8192, host.data_ptr(), 8); t4 = time.perf_counter()
    _lib.load().bsvd_pack_host(ptrs.ctypes.data, B, 8192, host.data_ptr(), 16); t5 = time.perf_counter()
    print(f"check {1e3*(t1-t0):.2f} | ptrs(array_interface) {1e3*(t2-t1):.2f} | ptrs(ctypes) {1e3*(t3-t2):.2f} | pack8 {1e3*(t4-t3):.2f} | pack16 {1e3*(t5-t4):.2f} ms")
print(os.cpu_count())
