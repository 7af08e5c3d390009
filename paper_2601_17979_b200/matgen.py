"""Synthetic benchmark inputs with prescribed spectra, generated on the device.

Restates the spectrum families of /root/reference/pkg/src/bsvd/matgen.py
(make_sigma :52-84; A = U diag(sigma) V^H with orthonormal factors from QR
of Gaussians, :96-122) for whole batches at once on the GPU, so the bench
can build 10k-problem inputs in milliseconds.  The factors come from torch's
batched QR instead of the reference's Householder loop, so matrices are not
bit-identical to ``gen_batch`` -- only the spectra are (which is what the
accuracy metrics e4 and the bench workload need).  Harness only; not on the
solve path.
"""

from __future__ import annotations

import numpy as np

FAMILIES = ("random", "arith", "cluster0", "cluster1", "logrand", "geo", "rankdef")


def make_sigma(family: str, n: int, kappa: float = 1.0, seed: int = 0, rank: int | None = None) -> np.ndarray:
    """Prescribed singular values, descending (src/matgen.py:52-84; rankdef = BASELINE C3b)."""
    i = np.arange(n, dtype=np.float64)
    if family == "arith":
        return 1.0 - (i / (n - 1)) * (1.0 - 1.0 / kappa)
    if family == "geo":
        return kappa ** (-i / (n - 1))
    if family == "cluster0":
        s = np.full(n, 1.0 / kappa)
        s[0] = 1.0
        return s
    if family == "cluster1":
        s = np.ones(n)
        s[-1] = 1.0 / kappa
        return s
    if family == "logrand":
        rng = np.random.default_rng(seed)
        s = np.empty(n)
        s[0] = 1.0
        if n > 1:
            s[1:] = np.exp(rng.uniform(np.log(1.0 / kappa), 0.0, size=n - 1))
        s[::-1].sort()
        return s
    if family == "rankdef":
        r = rank if rank is not None else (3 * n) // 4
        j = np.arange(r, dtype=np.float64)
        return np.concatenate([kappa ** (-j / (r - 1)), np.zeros(n - r)])
    raise ValueError(f"family {family!r} has no prescribed spectrum")


def gen_batch_device(family: str, m: int, n: int, batch: int, dtype=np.float64, kappa: float = 1.0,
                     seed: int = 0, rank: int | None = None, device="cuda"):
    """(batch, n, m) C-contiguous device tensor: column-major m x n matrices."""
    import torch

    from .solver import torch_dtype

    dt = np.dtype(dtype)
    tdt = torch_dtype(dt)
    cplx = dt.kind == "c"
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) * 1000003 + 17)
    if family == "random":
        if cplx:
            re = torch.rand((batch, n, m), generator=g, device=device, dtype=torch.float64)
            im = torch.rand((batch, n, m), generator=g, device=device, dtype=torch.float64)
            return torch.complex(re, im).to(tdt).contiguous()
        return torch.rand((batch, n, m), generator=g, device=device, dtype=torch.float64).to(tdt).contiguous()
    sig = torch.as_tensor(make_sigma(family, n, kappa, seed, rank), device=device, dtype=torch.float64)
    wdt = torch.complex128 if cplx else torch.float64

    def orth(rows, cols):
        if cplx:
            z = torch.complex(torch.randn((batch, rows, cols), generator=g, device=device, dtype=torch.float64),
                              torch.randn((batch, rows, cols), generator=g, device=device, dtype=torch.float64))
        else:
            z = torch.randn((batch, rows, cols), generator=g, device=device, dtype=torch.float64)
        q, _ = torch.linalg.qr(z)
        return q

    u = orth(m, n)
    v = orth(n, n)
    a = (u * sig.to(wdt)) @ v.mH  # (batch, m, n)
    return a.transpose(1, 2).to(tdt).contiguous()
