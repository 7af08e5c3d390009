"""ctypes front-end of the CPU restatement (oracle/bsvd_oracle.cpp).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline / --impl reference) as the checker and the CPU
baseline; the product package never imports it.

Each wrapper mirrors a reference function so tests read like the reference's
own: ``solve`` ~ ``svd_dispatch``/``svd_unblocked``/``svd_blocked``
(src/svd.py:550-582), ``onesided_sweeps`` / ``eig_sweeps`` /
``fused_pair_update`` ~ src/_kernels_numba.py, ``compute_gram`` ~
src/svd.py:144, ``schedule`` ~ src/ordering.py:58.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libbsvd_oracle.so")

DTYPE_CODE = {
    np.dtype(np.float32): 0,
    np.dtype(np.float64): 1,
    np.dtype(np.complex64): 2,
    np.dtype(np.complex128): 3,
}
REAL_OF = {
    np.dtype(np.float32): np.dtype(np.float32),
    np.dtype(np.float64): np.dtype(np.float64),
    np.dtype(np.complex64): np.dtype(np.float32),
    np.dtype(np.complex128): np.dtype(np.float64),
}
PATHS = {0: "empty", 1: "unblocked", 2: "blocked"}
FORCE = {None: 0, "unblocked": 1, "blocked": 2, "qr": 3}


class OrcOpts(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_double),
        ("max_nsweeps", ctypes.c_int),
        ("nb", ctypes.c_int),
        ("inner_sweeps", ctypes.c_int),
        ("want_v", ctypes.c_int),
        ("fused_updates", ctypes.c_int),
        ("row_block", ctypes.c_int),
        ("force", ctypes.c_int),
        ("use_qr", ctypes.c_int),
    ]


class OrcInfo(ctypes.Structure):
    _fields_ = [
        ("converged", ctypes.c_int32),
        ("outer_sweeps", ctypes.c_int32),
        ("inner_rotations", ctypes.c_int64),
        ("path", ctypes.c_int32),
        ("transposed", ctypes.c_int32),
        ("gram_calls", ctypes.c_int64),
        ("eig_calls", ctypes.c_int64),
        ("update_calls", ctypes.c_int64),
        ("status", ctypes.c_int32),
        ("qr", ctypes.c_int32),
    ]


_lib = None


def build() -> str:
    """Compile the restatement (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        vp, ci, cd = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        L.orc_solve.argtypes = [ci, ci, ci, vp, vp, vp, vp, ctypes.POINTER(OrcOpts), ctypes.POINTER(OrcInfo)]
        L.orc_solve.restype = ci
        L.orc_solve_batch.argtypes = [ci, ci, ci, ci, vp, vp, vp, vp, ctypes.POINTER(OrcOpts),
                                      ctypes.POINTER(OrcInfo), ci]
        L.orc_solve_batch.restype = ci
        L.orc_onesided_sweeps.argtypes = [ci, ci, ci, vp, ci, vp, cd, ci, ctypes.POINTER(ci), ctypes.POINTER(ci)]
        L.orc_onesided_sweeps.restype = ctypes.c_int64
        L.orc_eig_sweeps.argtypes = [ci, ci, vp, vp, ci, vp, cd, ci, ci, ctypes.POINTER(ci), ctypes.POINTER(ci)]
        L.orc_eig_sweeps.restype = ctypes.c_int64
        L.orc_compute_gram.argtypes = [ci, ci, ci, ci, vp, vp, vp]
        L.orc_compute_gram.restype = None
        L.orc_fused_pair_update.argtypes = [ci, ci, ci, ci, vp, vp, vp, ci, ci]
        L.orc_fused_pair_update.restype = None
        L.orc_schedule.argtypes = [ci, vp, vp, ctypes.POINTER(ci)]
        L.orc_schedule.restype = ci
        L.orc_max_threads.argtypes = []
        L.orc_max_threads.restype = ci
        _lib = L
    return _lib


def _opts(opts=None, force=None) -> OrcOpts:
    o = OrcOpts()
    o.k = float(getattr(opts, "k", 30.0))
    o.max_nsweeps = int(getattr(opts, "max_nsweeps", 30))
    o.nb = int(getattr(opts, "nb", 16))
    o.inner_sweeps = int(getattr(opts, "inner_sweeps", 1))
    o.want_v = int(bool(getattr(opts, "compute_right_vectors", True)))
    o.fused_updates = int(bool(getattr(opts, "fused_updates", True)))
    o.row_block = int(getattr(opts, "row_block", 64))
    o.force = FORCE[force]
    o.use_qr = int(bool(getattr(opts, "use_qr_preprocess", False)))
    return o


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def unit_roundoff(dtype) -> float:
    return 2.0 ** -24 if REAL_OF[np.dtype(dtype)] == np.dtype(np.float32) else 2.0 ** -53


def _info_dict(inf: OrcInfo) -> dict:
    path = PATHS[inf.path]
    if inf.qr and path != "empty":
        path = "qr+" + path
    if inf.transposed and path != "empty":
        path = "transpose+" + path
    return dict(
        converged=bool(inf.converged),
        outer_sweeps=int(inf.outer_sweeps),
        inner_rotations=int(inf.inner_rotations),
        path=path,
        gram_calls=int(inf.gram_calls),
        eig_calls=int(inf.eig_calls),
        update_calls=int(inf.update_calls),
        status=int(inf.status),
    )


def solve(a, opts=None, force=None):
    """One problem; returns (u, sigma, v_or_None, info_dict)."""
    a = np.asarray(a)
    dt = a.dtype
    if dt not in DTYPE_CODE:
        raise ValueError(f"unsupported dtype {dt}")
    m, n = a.shape
    k = min(m, n)
    af = np.asfortranarray(a)
    o = _opts(opts, force)
    u = np.zeros((m, k), dtype=dt, order="F")
    s = np.zeros(k, dtype=REAL_OF[dt])
    v = np.zeros((n, k), dtype=dt, order="F") if o.want_v else None
    inf = OrcInfo()
    rc = lib().orc_solve(DTYPE_CODE[dt], m, n, _ptr(af), _ptr(u), _ptr(s), _ptr(v),
                         ctypes.byref(o), ctypes.byref(inf))
    if rc != 0:
        raise ValueError(f"oracle solve failed rc={rc} shape={a.shape} force={force}")
    return u, s, v, _info_dict(inf)


def solve_batch(a3, opts=None, force=None, nthreads: int = 0):
    """Equal-shape batch a3[b] (m x n, any layout); returns (U, S, V, infos).

    U: (B, m, k) with each U[b] column-major contents, S: (B, k), V: (B, n, k).
    """
    a3 = np.asarray(a3)
    B, m, n = a3.shape
    dt = a3.dtype
    k = min(m, n)
    # column-major per problem: transpose last two axes into C order
    af = np.ascontiguousarray(np.swapaxes(a3, 1, 2))
    o = _opts(opts, force)
    u = np.zeros((B, k, m), dtype=dt)
    s = np.zeros((B, k), dtype=REAL_OF[dt])
    v = np.zeros((B, k, n), dtype=dt) if o.want_v else None
    infos = (OrcInfo * B)()
    rc = lib().orc_solve_batch(DTYPE_CODE[dt], m, n, B, _ptr(af), _ptr(u), _ptr(s), _ptr(v),
                               ctypes.byref(o), infos, int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle batch solve failed rc={rc}")
    U = np.swapaxes(u, 1, 2)
    V = np.swapaxes(v, 1, 2) if v is not None else None
    return U, s, V, [_info_dict(i) for i in infos]


def onesided_sweeps(a, v, tol, max_sweeps):
    """In-place, like src/_kernels_numba.py:85 (a, v F-order)."""
    assert a.flags.f_contiguous and v.flags.f_contiguous
    sw, cv = ctypes.c_int(), ctypes.c_int()
    rot = lib().orc_onesided_sweeps(DTYPE_CODE[a.dtype], a.shape[0], a.shape[1], _ptr(a),
                                    v.shape[0], _ptr(v), float(tol), int(max_sweeps),
                                    ctypes.byref(sw), ctypes.byref(cv))
    return sw.value, int(rot), bool(cv.value)


def eig_sweeps(g, d, mm, tol, max_sweeps, delta=False):
    """In-place, like src/_kernels_numba.py:17 (g, mm F-order; d real)."""
    assert g.flags.f_contiguous and mm.flags.f_contiguous
    sw, cv = ctypes.c_int(), ctypes.c_int()
    rot = lib().orc_eig_sweeps(DTYPE_CODE[g.dtype], g.shape[0], _ptr(g), _ptr(d), mm.shape[0],
                               _ptr(mm), float(tol), int(max_sweeps), int(bool(delta)),
                               ctypes.byref(sw), ctypes.byref(cv))
    return sw.value, int(rot), bool(cv.value)


def compute_gram(ai, aj):
    ai = np.asfortranarray(ai)
    aj = np.asfortranarray(aj)
    w = ai.shape[1] + aj.shape[1]
    g = np.zeros((w, w), dtype=ai.dtype, order="F")
    lib().orc_compute_gram(DTYPE_CODE[ai.dtype], ai.shape[0], ai.shape[1], aj.shape[1],
                           _ptr(ai), _ptr(aj), _ptr(g))
    return g


def fused_pair_update(bi, bj, j, row_block=64, delta=False):
    assert bi.flags.f_contiguous and bj.flags.f_contiguous
    j = np.asfortranarray(j, dtype=bi.dtype)
    lib().orc_fused_pair_update(DTYPE_CODE[bi.dtype], bi.shape[0], bi.shape[1], bj.shape[1],
                                _ptr(bi), _ptr(bj), _ptr(j), int(row_block), int(bool(delta)))


def schedule(ell):
    """(pairs (P,2) int64, starts (T+1,) int64) like src/ordering.py:58."""
    pairs = np.zeros(2 * ell * ell, dtype=np.int32)
    starts = np.zeros(ell + 2, dtype=np.int32)
    nit = ctypes.c_int()
    P = lib().orc_schedule(int(ell), _ptr(pairs), _ptr(starts), ctypes.byref(nit))
    if P < 0:
        raise ValueError(f"need at least 2 indices, got {ell}")
    return pairs[: 2 * P].reshape(P, 2).astype(np.int64), starts[: nit.value + 1].astype(np.int64)


def max_threads() -> int:
    return int(lib().orc_max_threads())
