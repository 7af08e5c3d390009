"""Generate BSVD / BSVR fixtures by running the REFERENCE package itself (src/fileio.py).

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_fileio.py

Writes tests/golden/ref_*.bsvd / ref_*.bsvr (small files) that tests/test_fileio.py reads back.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import bsvd  # noqa: E402
from bsvd import fileio  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def rm(m, n, dt, seed):
    rng = np.random.default_rng(seed)
    a = rng.random((m, n))
    if np.dtype(dt).kind == "c":
        a = a + 1j * rng.random((m, n))
    return np.asarray(a, dtype=dt, order="F")


def main():
    for dt, nm in ((np.float32, "f32"), (np.float64, "f64"), (np.complex64, "c64"), (np.complex128, "c128")):
        mats = [rm(6, 4, dt, 1), rm(3, 5, dt, 2), rm(8, 8, dt, 3)]  # mixed shapes
        fileio.write_matrices(os.path.join(HERE, f"ref_mixed_{nm}.bsvd"), mats)
        uni = [rm(5, 3, dt, 10 + b) for b in range(4)]
        fileio.write_matrices(os.path.join(HERE, f"ref_uniform_{nm}.bsvd"), uni)
        res = [bsvd.svd_dispatch(a) for a in uni]
        res[2] = None  # a failed slot
        fileio.write_results(os.path.join(HERE, f"ref_uniform_{nm}.bsvr"), uni, res)
    fileio.write_matrices(os.path.join(HERE, "ref_empty.bsvd"), [])
    print("fixtures written")


if __name__ == "__main__":
    main()
