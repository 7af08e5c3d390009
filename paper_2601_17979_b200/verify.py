"""Accuracy metrics e1-e4 and pass thresholds, evaluated on the device.

Mirrors /root/reference/pkg/src/bsvd/verify.py:39-190 (``threshold``,
``residual_e1``, ``orthogonality_e2_e3``, ``sigma_error_e4``,
``ErrorReport``, ``error_report``) with the metrics computed by the batched
kernel ``bsvd_verify_batched`` (csrc/verify.cu, float64 accumulation):

    e1 = |A - U diag(s) V^H|_1 / (n |A|_1)
    e2 = |I - U^H U|_1 / m,   e3 = |I - V^H V|_1 / n
    e4 = |s - s_ref|_F / min(m, n)

``verify_tensor`` checks a whole device-resident batch (the solve_tensor
layout) without leaving the GPU; the per-problem functions wrap it.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import DTYPE_CODE, DomainError, ShapeError, check_dtype, unit_roundoff

__all__ = ["ErrorReport", "threshold", "residual_e1", "orthogonality_e2_e3", "sigma_error_e4", "error_report",
           "verify_tensor"]


def threshold(dtype, k: float = 30.0) -> float:
    """Pass bound k*u for the given element type (src/verify.py:39-41)."""
    return float(k) * unit_roundoff(dtype)


def verify_tensor(a_t, m: int, n: int, res, sigma_ref=None):
    """(B, 4) float64 device tensor of (e1, e2, e3, e4) for a solve_tensor result.

    a_t (B, n, m), res.u (B, k, m), res.s (B, k), res.v (B, k, n) | None; sigma_ref an optional
    (B, k) float64 device tensor.  Launched on the current stream, no synchronisation.
    """
    from .solver import _torch, np_dtype_of

    torch = _torch()
    L = _lib.load()
    B = a_t.shape[0]
    k = min(m, n)
    dt = np_dtype_of(a_t.dtype)
    out = torch.empty((B, 4), dtype=torch.float64, device=a_t.device)
    if sigma_ref is not None:
        sigma_ref = sigma_ref.to(device=a_t.device, dtype=torch.float64).contiguous()
    stream = torch.cuda.current_stream(a_t.device).cuda_stream
    rc = L.bsvd_verify_batched(
        DTYPE_CODE[dt], m, n, B, a_t.data_ptr(), max(m, 1), m * n, res.u.data_ptr(), max(m, 1), k * m,
        res.s.data_ptr(), k, res.v.data_ptr() if res.v is not None else None, max(n, 1), k * n,
        sigma_ref.data_ptr() if sigma_ref is not None else None, k, out.data_ptr(), stream)
    _lib.check(rc, f"bsvd_verify_batched({dt.name}, {m}x{n}, batch={B})")
    return out


def _metrics(a, result, sigma_ref=None):
    """(e1, e2, e3, e4) of one host (matrix, SvdResult) pair through the device kernel."""
    from .solver import _torch, torch_dtype

    torch = _torch()
    a = np.asarray(a)
    check_dtype(a.dtype)
    m, n = a.shape
    k = min(m, n)
    dev = torch.device("cuda", torch.cuda.current_device())

    class _R:
        pass

    r = _R()
    tdt = torch_dtype(a.dtype)
    a_t = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev, tdt).reshape(1, n, m)
    r.u = torch.from_numpy(np.ascontiguousarray(np.asarray(result.u).T)).to(dev, tdt).reshape(1, k, m)
    r.s = torch.from_numpy(np.ascontiguousarray(result.sigma)).to(dev).reshape(1, k)
    r.v = (torch.from_numpy(np.ascontiguousarray(np.asarray(result.v).T)).to(dev, tdt).reshape(1, k, n)
           if result.v is not None else None)
    sr = None
    if sigma_ref is not None:
        sr_np = np.asarray(sigma_ref, dtype=np.float64)
        if sr_np.shape != (k,):
            raise ShapeError(f"length mismatch: {sr_np.shape} vs {(k,)}")
        sr = torch.from_numpy(sr_np).to(dev).reshape(1, k)
    out = verify_tensor(a_t, m, n, r, sr).cpu().numpy()[0]
    return tuple(float(x) for x in out)


def residual_e1(a, result) -> float:
    """|A - U diag(sigma) V^H|_1 / (n |A|_1) (src/verify.py:44-56)."""
    if result.v is None:
        raise DomainError("e1 needs right singular vectors; solve with compute_right_vectors=True")
    return _metrics(a, result)[0]


def orthogonality_e2_e3(result, a=None) -> tuple[float, float]:
    """(|I - U^H U|_1 / m, |I - V^H V|_1 / n) (src/verify.py:59-73)."""
    if result.v is None:
        raise DomainError("e3 needs right singular vectors; solve with compute_right_vectors=True")
    m, n = np.asarray(result.u).shape[0], np.asarray(result.v).shape[0]
    if a is None:
        a = np.zeros((m, n), dtype=np.asarray(result.u).dtype, order="F")
    e = _metrics(a, result)
    return e[1], e[2]


def sigma_error_e4(sigma, sigma_ref, m: int, n: int) -> float:
    """|sigma - sigma_ref|_F / min(m, n) (src/verify.py:76-84; host arithmetic on two vectors)."""
    s = np.asarray(sigma, dtype=np.float64)
    r = np.asarray(sigma_ref, dtype=np.float64)
    if s.shape != r.shape:
        raise ShapeError(f"length mismatch: {s.shape} vs {r.shape}")
    md = min(m, n)
    return 0.0 if md == 0 else float(np.linalg.norm(s - r)) / md


@dataclass(frozen=True)
class ErrorReport:
    """Metrics and verdicts for one solved problem (src/verify.py:120-143)."""

    e1: float
    e2: float
    e3: float
    e4: float | None
    threshold: float
    e3_threshold: float
    passes: tuple[bool, bool, bool, bool]
    family: str | None = None
    n: int = 0
    m: int = 0
    dtype: str = ""
    batch_index: int | None = None

    @property
    def all_pass(self) -> bool:
        return all(self.passes)


def error_report(a, result, sigma_ref=None, k: float = 30.0, e3_threshold: float | None = None,
                 family: str | None = None, batch_index: int | None = None) -> ErrorReport:
    """All four metrics for one (matrix, result) pair (src/verify.py:146-190), computed on the device."""
    a = np.asarray(a)
    m, n = a.shape
    thr = threshold(a.dtype, k)
    e3_thr = thr if e3_threshold is None else float(e3_threshold)
    if result.v is None:
        raise DomainError("e1 needs right singular vectors; solve with compute_right_vectors=True")
    e1, e2, e3, e4 = _metrics(a, result, sigma_ref)
    if sigma_ref is None:
        e4v, p4 = None, True
    else:
        e4v, p4 = e4, e4 < thr
    return ErrorReport(e1=e1, e2=e2, e3=e3, e4=e4v, threshold=thr, e3_threshold=e3_thr,
                       passes=(e1 < thr, e2 < thr, e3 < e3_thr, p4), family=family, n=n, m=m,
                       dtype=str(a.dtype), batch_index=batch_index)
