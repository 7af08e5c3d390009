"""Scalar 2x2 rotation record (host side).

Mirrors /root/reference/pkg/src/bsvd/eig.py:23-80.  ``compute_rotation`` is
the reference's scalar formula (the kernels evaluate the same formula in
float64 per pair, csrc/common.cuh rot_params); it is kept here as the
known-answer companion of the device rotation core.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import DomainError


@dataclass(frozen=True)
class Rotation:
    """Plane rotation J = [[c, -phase*s], [conj(phase)*s, c]] (src/eig.py:23-49)."""

    c: float
    s: float
    phase: complex
    t: float
    i: int | None = None
    j: int | None = None

    def as_matrix(self, dtype=None) -> np.ndarray:
        j = np.array([[self.c, -self.phase * self.s], [np.conj(self.phase) * self.s, self.c]])
        if dtype is not None:
            j = j.astype(dtype)
        return j


def compute_rotation(a_ii, a_jj, a_ij) -> Rotation:
    """Rotation annihilating the off-diagonal of [[a_ii, a_ij], [conj(a_ij), a_jj]] (src/eig.py:52-80)."""
    if np.iscomplexobj(a_ii) and np.imag(a_ii) != 0:
        raise DomainError("diagonal entry a_ii must be real")
    if np.iscomplexobj(a_jj) and np.imag(a_jj) != 0:
        raise DomainError("diagonal entry a_jj must be real")
    dii = float(np.real(a_ii))
    djj = float(np.real(a_jj))
    g = complex(a_ij) if np.iscomplexobj(a_ij) else float(a_ij)
    absg = abs(g)
    if absg == 0.0:
        return Rotation(c=1.0, s=0.0, phase=1.0, t=0.0)
    if absg < 2.0 ** -966:
        gs = g * 2.0 ** 1022
        phase = gs / abs(gs)
    else:
        phase = g / absg
    tau = (dii - djj) / (2.0 * absg)
    sgn = 1.0 if tau >= 0.0 else -1.0
    t = sgn / (abs(tau) + np.sqrt(1.0 + tau * tau))
    c = 1.0 / np.sqrt(1.0 + t * t)
    return Rotation(c=float(c), s=float(t * c), phase=phase, t=float(t))


@dataclass(frozen=True)
class EigInfo:
    """Inner eigensolver telemetry (src/eig.py:83-87)."""

    sweeps_run: int
    rotations: int
    converged: bool


def _validate_hermitian(g, k: float, max_sweeps: int):
    from .core import ShapeError, check_dtype, unit_roundoff

    a = np.asarray(g)
    check_dtype(a)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ShapeError(f"expected a square matrix, got shape {a.shape}")
    n = a.shape[0]
    if k <= 0:
        raise DomainError(f"guard multiplier k must be positive, got {k}")
    if max_sweeps < 1:
        raise DomainError(f"max_sweeps must be at least 1, got {max_sweeps}")
    u = unit_roundoff(a.dtype)
    herm_tol = 4.0 * u * float(np.linalg.norm(a))
    asym = float(np.max(np.abs(a - a.conj().T))) if n else 0.0
    if asym > herm_tol:
        raise DomainError(f"matrix is not Hermitian: max asymmetry {asym:.3e} exceeds {herm_tol:.3e}")
    return a


def batch_hermitian_eig(mats, k: float = 30.0, max_sweeps: int = 30, eigvecs=None):
    """Equal-size Hermitian matrices -> [(d, m, EigInfo)] on the device (bsvd_heevj_batched).

    Each entry follows ``jacobi_hermitian_eig`` (src/eig.py:90-148): ``g ~= m @ diag(d) @ m^H``,
    d unsorted; ``eigvecs`` (optional list of F-ordered n-column matrices of the same dtype)
    accumulate the rotations in place instead of a fresh identity.
    """
    import ctypes

    from . import _lib
    from .core import DTYPE_CODE, ShapeError, real_dtype
    from .solver import _torch, _workspace, torch_dtype
    from .solver import INFO_DTYPE

    mats = [_validate_hermitian(g, k, max_sweeps) for g in mats]
    if not mats:
        return []
    n = mats[0].shape[0]
    dt = mats[0].dtype
    if any(g.shape != (n, n) or g.dtype != dt for g in mats):
        raise ShapeError("batch_hermitian_eig needs equal shapes and dtypes")
    B = len(mats)
    if eigvecs is not None:
        for m in eigvecs:
            if m.dtype != dt or m.ndim != 2 or m.shape[1] != n:
                raise ShapeError("eigvecs must be 2-d with n columns and matching dtype")
            if not m.flags.f_contiguous:
                raise ShapeError("eigvecs must be F-contiguous")
    if n < 2:  # src/eig.py:136-137
        out = []
        for b, g in enumerate(mats):
            d = np.ascontiguousarray(np.real(np.diag(g)), dtype=real_dtype(dt))
            m = eigvecs[b] if eigvecs is not None else np.eye(n, dtype=dt, order="F")
            out.append((d, m, EigInfo(sweeps_run=1, rotations=0, converged=True)))
        return out
    torch = _torch()
    L = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    tdt = torch_dtype(dt)
    g_h = torch.empty((B, n, n), dtype=tdt, pin_memory=True)
    gv = g_h.numpy()
    for b, g in enumerate(mats):
        gv[b] = g.T  # column-major per matrix
    m_h = torch.empty((B, n, n), dtype=tdt, pin_memory=True)
    # n x n accumulators are rotated in place on the device; any other row count (the reference accepts
    # any n-column matrix, src/eig.py:128-133) gets the device's rotation product Q: eigvecs <- eigvecs Q
    square = eigvecs is not None and all(m.shape[0] == n for m in eigvecs)
    if square:
        mv = m_h.numpy()
        for b, m in enumerate(eigvecs):
            mv[b] = m.T
    g_d = g_h.to(dev, non_blocking=True)
    m_d = m_h.to(dev, non_blocking=True)
    d_d = torch.empty((B, n), dtype=torch_dtype(real_dtype(dt)), device=dev)
    info_d = torch.empty((B * _lib.INFO_BYTES,), dtype=torch.uint8, device=dev)
    code = DTYPE_CODE[dt]
    ws_bytes = L.bsvd_heevj_workspace_bytes(code, n, B)
    ws = _workspace(ws_bytes, dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = L.bsvd_heevj_batched(code, n, B, g_d.data_ptr(), n, n * n, d_d.data_ptr(), n, m_d.data_ptr(), n, n * n,
                              1 if square else 0, float(k), int(max_sweeps), info_d.data_ptr(),
                              ws.data_ptr() if ws is not None else None, ws_bytes, stream)
    _lib.check(rc, f"bsvd_heevj_batched({dt.name}, n={n}, batch={B})")
    d_h = d_d.cpu().numpy()
    m_out = np.swapaxes(m_d.cpu().numpy(), 1, 2)
    info = np.frombuffer(info_d.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    out = []
    for b in range(B):
        if square:
            eigvecs[b][...] = m_out[b]
            m = eigvecs[b]
        elif eigvecs is not None:
            eigvecs[b][...] = eigvecs[b] @ m_out[b]
            m = eigvecs[b]
        else:
            m = np.asfortranarray(m_out[b])
        out.append((np.ascontiguousarray(d_h[b]), m, EigInfo(sweeps_run=int(info["outer_sweeps"][b]),
                                                              rotations=int(info["rotations"][b]),
                                                              converged=bool(info["converged"][b]))))
    return out


def jacobi_hermitian_eig(g, k: float = 30.0, max_sweeps: int = 30, eigvecs=None):
    """Diagonalize a Hermitian matrix by cyclic Jacobi rotations (src/eig.py:90-148), on the device.

    Returns ``(d, m, info)`` with ``g ~= m @ diag(d) @ m.conj().T``; a pair rotates only when
    its off-diagonal magnitude exceeds ``k * u * sqrt(|d_i| * |d_j|)`` and a quiet sweep (counted
    in ``sweeps_run``) ends the iteration.  ``eigvecs`` accumulates the rotations in place.
    """
    return batch_hermitian_eig([g], k, max_sweeps, [eigvecs] if eigvecs is not None else None)[0]
