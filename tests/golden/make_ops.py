"""Golden vectors for the standalone finalize and householder_qr operators, made by running the
REFERENCE package itself (bsvd.finalize, src/svd.py:278-303; bsvd.householder_qr, src/core.py:118-168).

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_ops.py

writes tests/golden/ops.npz; the GPU box has no /root/reference, the tests only read the file.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import bsvd  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ALL = (np.float32, np.float64, np.complex64, np.complex128)


def rand(m, n, dt, seed):
    rng = np.random.default_rng(seed)
    a = rng.random((m, n))
    if np.dtype(dt).kind == "c":
        a = a + 1j * rng.random((m, n))
    return np.asarray(a, dtype=dt, order="F")


def main():
    out = {}
    cases = []
    for di, dt in enumerate(ALL):
        name = np.dtype(dt).name
        # finalize: an orthogonalised working copy (solve with V, then W = U diag(s)), plus edge columns
        for tag, (m, n) in {"sq": (12, 12), "tall": (20, 7)}.items():
            a = rand(m, n, dt, 100 + di)
            r = bsvd.svd_unblocked(a)
            w = np.asfortranarray((r.u * r.sigma).astype(dt))
            perm = np.random.default_rng(7 + di).permutation(n)
            w = np.asfortranarray(w[:, perm])           # unsorted columns
            v = np.asfortranarray(r.v[:, perm].astype(dt))
            w[:, 2] = 0                                   # a hole: orthogonal completion
            w[:, 4] = w[:, 3]                             # an exact tie (stable order)
            v[:, 4] = v[:, 3]
            f = bsvd.finalize(w, v)
            key = f"fin_{name}_{tag}"
            out[key + "_w"], out[key + "_v"] = w, v
            out[key + "_u"], out[key + "_s"], out[key + "_vo"] = f.u, f.sigma, f.v
            f0 = bsvd.finalize(w)
            out[key + "_u0"], out[key + "_s0"] = f0.u, f0.sigma
            cases.append(key)
        # householder_qr: random, a zero column, a rank-deficient tall matrix, wide-enough square
        for tag, (m, n) in {"tall": (30, 9), "sq": (10, 10), "skinny": (64, 32)}.items():
            a = rand(m, n, dt, 200 + di + m)
            if tag == "tall":
                a[:, 3] = 0
            if tag == "sq":
                a[:, 7] = a[:, 1]
            q, rr = bsvd.householder_qr(a)
            key = f"hqr_{name}_{tag}"
            out[key + "_a"], out[key + "_q"], out[key + "_r"] = a, q, rr
            cases.append(key)
    out["cases"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **out)
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
