"""Kernel-level operators on the device, shaped like the reference's API.

The reference routes its hot loops through ``Backend(onesided_sweeps,
eig_sweeps, fused_pair_update)`` (src/backend.py:30-35) plus
``compute_gram`` (src/svd.py:144).  These wrappers run the same operations
on the B200 through the batch-granular C-ABI entry points
(bsvd_onesided_sweeps_batched, bsvd_gram_batched,
bsvd_fused_pair_update_batched) for a single problem, with the reference's
argument checks and in-place semantics, so the reference's kernel-level
tests can be replayed against the GPU.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .core import DTYPE_CODE, DomainError, ShapeError, check_dtype


def _dev(x_np):
    from .solver import _torch

    torch = _torch()
    # column-major matrix -> C-contiguous transpose on the device
    return torch.from_numpy(np.ascontiguousarray(x_np.T)).cuda()


def _back(t, like_shape):
    return np.asfortranarray(t.cpu().numpy().T).reshape(like_shape, order="F")


def onesided_sweeps(a, v, pairs=None, starts=None, tol=None, max_sweeps=1):
    """In place on a (m x n) and v (vrows x n); returns (sweeps, rotations, converged).

    Mirrors src/_kernels_numba.py:85-138.  ``pairs``/``starts`` are accepted for
    signature parity; the device evaluates the same round-robin schedule in
    closed form.
    """
    from .solver import _torch

    torch = _torch()
    L = _lib.load()
    m, n = a.shape
    vrows = v.shape[0] if v is not None else 0
    at = _dev(a)
    vt = _dev(v) if vrows else None
    rot = torch.zeros(1, dtype=torch.int64, device="cuda")
    sw = torch.zeros(1, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    rc = L.bsvd_onesided_sweeps_batched(DTYPE_CODE[a.dtype], m, n, 1, at.data_ptr(), max(m, 1), m * n, vrows,
                                        vt.data_ptr() if vt is not None else None, max(vrows, 1), vrows * n,
                                        float(tol), int(max_sweeps), rot.data_ptr(), sw.data_ptr(), stream)
    _lib.check(rc, "bsvd_onesided_sweeps_batched")
    a[...] = _back(at, a.shape)
    if vrows:
        v[...] = _back(vt, v.shape)
    raw = int(sw.item())
    sweeps = raw & ((1 << 30) - 1)
    converged = bool(raw >> 30)
    rotations = int(rot.item())
    return sweeps, rotations, converged


def compute_gram(ai: np.ndarray, aj: np.ndarray) -> np.ndarray:
    """Hermitian Gram [Ai Aj]^H [Ai Aj] of two column blocks (src/svd.py:144-179)."""
    from .solver import _torch

    torch = _torch()
    a_i = np.asarray(ai)
    a_j = np.asarray(aj)
    check_dtype(a_i)
    check_dtype(a_j)
    if a_i.ndim != 2 or a_j.ndim != 2:
        raise ShapeError("block views must be 2-d")
    if a_i.shape[0] != a_j.shape[0]:
        raise ShapeError(f"row-count mismatch: {a_i.shape[0]} vs {a_j.shape[0]}")
    if a_i.dtype != a_j.dtype:
        raise DomainError(f"dtype mismatch: {a_i.dtype} vs {a_j.dtype}")
    wi, wj = a_i.shape[1], a_j.shape[1]
    if wi < 1 or wj < 1:
        raise ShapeError("block widths must be >= 1")
    m = a_i.shape[0]
    w = wi + wj
    blk = np.hstack([a_i, a_j])
    at = _dev(blk)
    gt = torch.empty((w, w), dtype=at.dtype, device="cuda")
    L = _lib.load()
    rc = L.bsvd_gram_batched(DTYPE_CODE[a_i.dtype], m, wi, wj, 1, at.data_ptr(), max(m, 1), m * w,
                             gt.data_ptr(), w, w * w, torch.cuda.current_stream().cuda_stream)
    _lib.check(rc, "bsvd_gram_batched")
    return np.asfortranarray(gt.cpu().numpy().T)


def fused_pair_update(bi: np.ndarray, bj: np.ndarray, j: np.ndarray, row_block: int = 64,
                      delta: bool = False) -> None:
    """[Bi Bj] <- [Bi Bj] @ J in place (or += with delta) (src/svd.py:182-210)."""
    from .solver import _torch

    torch = _torch()
    b_i = np.asarray(bi)
    b_j = np.asarray(bj)
    jm = np.asarray(j)
    if b_i.ndim != 2 or b_j.ndim != 2 or jm.ndim != 2:
        raise ShapeError("fused_pair_update expects 2-d arrays")
    if b_i.shape[0] != b_j.shape[0]:
        raise ShapeError(f"row-count mismatch: {b_i.shape[0]} vs {b_j.shape[0]}")
    wt = b_i.shape[1] + b_j.shape[1]
    if jm.shape != (wt, wt):
        raise ShapeError(f"J must be {wt}x{wt}, got {jm.shape}")
    if b_i.dtype != b_j.dtype:
        raise DomainError(f"dtype mismatch: {b_i.dtype} vs {b_j.dtype}")
    if row_block < 1:
        raise DomainError(f"row_block must be >= 1, got {row_block}")
    if jm.dtype != b_i.dtype:
        jm = jm.astype(b_i.dtype)
    m = b_i.shape[0]
    if m == 0:
        return
    blk = np.hstack([b_i, b_j])
    bt = _dev(blk)
    jt = _dev(np.asfortranarray(jm))
    L = _lib.load()
    rc = L.bsvd_fused_pair_update_batched(DTYPE_CODE[b_i.dtype], m, wt, 1, bt.data_ptr(), m, m * wt,
                                          jt.data_ptr(), wt, wt * wt, int(bool(delta)),
                                          torch.cuda.current_stream().cuda_stream)
    _lib.check(rc, "bsvd_fused_pair_update_batched")
    out = _back(bt, blk.shape)
    wi = b_i.shape[1]
    bi[...] = out[:, :wi]
    bj[...] = out[:, wi:]


def householder_qr(a) -> tuple[np.ndarray, np.ndarray]:
    """Reduced non-pivoted Householder QR on the device (src/core.py:118-168): (q m x n, r n x n upper
    triangular with a real non-negative diagonal), through bsvd_householder_qr_batched."""
    from .core import fmatrix
    from .solver import _torch, torch_dtype

    torch = _torch()
    a = fmatrix(a)
    m, n = a.shape
    if m < n:
        raise ShapeError(f"householder_qr needs m >= n, got {m}x{n}")
    dt = a.dtype
    tdt = torch_dtype(dt)
    L = _lib.load()
    if n == 0:
        return np.zeros((m, 0), dtype=dt, order="F"), np.zeros((0, 0), dtype=dt, order="F")
    at = _dev(a)
    qt = torch.empty((n, m), dtype=tdt, device="cuda")
    rt = torch.empty((n, n), dtype=tdt, device="cuda")
    wb = L.bsvd_householder_qr_workspace_bytes(DTYPE_CODE[dt], m, n, 1)
    ws = torch.empty(max(int(wb), 1), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    rc = L.bsvd_householder_qr_batched(DTYPE_CODE[dt], m, n, 1, at.data_ptr(), m, m * n, qt.data_ptr(), m, m * n,
                                       rt.data_ptr(), n, n * n, ws.data_ptr(), int(wb), stream)
    _lib.check(rc, "bsvd_householder_qr_batched")
    return _back(qt, (m, n)), _back(rt, (n, n))


def finalize_factors(w, v=None):
    """(u, sigma, v_permuted) of a converged working copy on the device (src/svd.py:243-275) through
    bsvd_finalize_batched; inputs are not modified."""
    from .core import real_dtype
    from .solver import _torch, torch_dtype

    torch = _torch()
    w = np.asarray(w)
    dt = check_dtype(w.dtype)
    if w.ndim != 2:
        raise ShapeError("finalize expects a 2-d working copy")
    m, n = w.shape
    if n > m:
        raise ShapeError(f"finalize expects m >= n, got {w.shape}")
    vrows = 0
    if v is not None:
        v = np.asarray(v)
        if v.ndim != 2 or v.shape[1] != n:
            raise ShapeError("V must be 2-d with the same column count as workA")
        if v.dtype != dt:
            raise DomainError(f"V dtype {v.dtype} differs from workA dtype {dt}")
        vrows = v.shape[0]
    rdt = real_dtype(dt)
    if n == 0:
        return (np.zeros((m, 0), dtype=dt, order="F"), np.zeros(0, dtype=rdt),
                None if v is None else np.zeros((vrows, 0), dtype=dt, order="F"))
    tdt = torch_dtype(dt)
    L = _lib.load()
    wt = _dev(w)
    vt = _dev(v) if v is not None and vrows else None
    ut = torch.empty((n, m), dtype=tdt, device="cuda")
    st_ = torch.empty((n,), dtype=torch_dtype(rdt), device="cuda")
    vo = torch.empty((n, vrows), dtype=tdt, device="cuda") if vt is not None else None
    stream = torch.cuda.current_stream().cuda_stream
    rc = L.bsvd_finalize_batched(DTYPE_CODE[dt], m, n, 1, wt.data_ptr(), m, m * n, vrows,
                                 vt.data_ptr() if vt is not None else None, max(vrows, 1), vrows * n, ut.data_ptr(),
                                 m, m * n, st_.data_ptr(), n, vo.data_ptr() if vo is not None else None,
                                 max(vrows, 1), vrows * n, stream)
    _lib.check(rc, "bsvd_finalize_batched")
    u = _back(ut, (m, n))
    s = st_.cpu().numpy().astype(rdt, copy=False)
    vv = None
    if v is not None:
        vv = _back(vo, (vrows, n)) if vo is not None else np.zeros((0, n), dtype=dt, order="F")
    return u, s, vv


def eig_sweeps(g, d, m, pairs=None, starts=None, tol=None, max_sweeps=1, delta=False):
    """In place on g (n x n Hermitian; off-diagonal rotated, pivots zeroed), d (n real pivots) and m
    (n x n accumulator; delta: P - I, start it at zero); returns (sweeps, rotations, converged).

    Mirrors src/_kernels_numba.py:17-82 through bsvd_eig_sweeps_batched.  ``pairs``/``starts`` are
    accepted for signature parity; the device evaluates the same round-robin schedule in closed form.
    """
    from .solver import INFO_DTYPE, _torch, torch_dtype

    torch = _torch()
    g = np.asarray(g)
    dt = check_dtype(g.dtype)
    n = g.shape[0]
    if g.ndim != 2 or g.shape[1] != n:
        raise ShapeError(f"expected a square matrix, got shape {g.shape}")
    if m.shape != (n, n):
        raise ShapeError(f"m must be {n} x {n}, got {m.shape}")
    if d.shape != (n,):
        raise ShapeError(f"d must have length {n}, got {d.shape}")
    L = _lib.load()
    gt = _dev(g)
    mt = _dev(np.asarray(m, dtype=dt))
    dtt = torch.from_numpy(np.ascontiguousarray(d)).cuda()
    info = torch.zeros((_lib.INFO_BYTES,), dtype=torch.uint8, device="cuda")
    wb = int(L.bsvd_heevj_workspace_bytes(DTYPE_CODE[dt], n, 1))
    ws = torch.empty(max(wb, 1), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    rc = L.bsvd_eig_sweeps_batched(DTYPE_CODE[dt], n, 1, gt.data_ptr(), max(n, 1), n * n, dtt.data_ptr(), n,
                                   mt.data_ptr(), max(n, 1), n * n, float(tol), int(max_sweeps), 1 if delta else 0,
                                   info.data_ptr(), ws.data_ptr() if wb else None, wb, stream)
    _lib.check(rc, "bsvd_eig_sweeps_batched")
    g[...] = _back(gt, g.shape)
    m[...] = _back(mt, m.shape)
    d[...] = dtt.cpu().numpy()
    if n == 0:
        return 1, 0, True
    inf = np.frombuffer(info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)[0]
    return int(inf["outer_sweeps"]), int(inf["rotations"]), bool(inf["converged"])
