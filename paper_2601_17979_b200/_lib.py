"""ctypes binding of the C-ABI library (include/bsvd_b200.h).

The product path goes through this module only.  There is no CPU fallback:
if the in-tree libbsvd_b200.so is missing, or no CUDA device is present, the
call raises.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libbsvd_b200.so")

BSVD_OK = 0
DISPATCH, FORCE_UNBLOCKED, FORCE_BLOCKED, FORCE_QR = 0, 1, 2, 3


class BsvdOpts(ctypes.Structure):
    _fields_ = [
        ("k", ctypes.c_double),
        ("max_sweeps", ctypes.c_int),
        ("nb", ctypes.c_int),
        ("inner_sweeps", ctypes.c_int),
        ("masking", ctypes.c_int),
        ("want_v", ctypes.c_int),
        ("route", ctypes.c_int),
        ("fused_updates", ctypes.c_int),
        ("row_block", ctypes.c_int),
        ("kernel", ctypes.c_int),
        ("use_qr", ctypes.c_int),
        ("reserved", ctypes.c_int * 2),
    ]


class BsvdInfo(ctypes.Structure):
    _fields_ = [
        ("converged", ctypes.c_int32),
        ("outer_sweeps", ctypes.c_int32),
        ("rotations", ctypes.c_int64),
        ("gram_calls", ctypes.c_int64),
        ("update_calls", ctypes.c_int64),
        ("last_rotations", ctypes.c_int32),
        ("path", ctypes.c_int32),
        ("status", ctypes.c_int32),
        ("kernel", ctypes.c_int32),
    ]


INFO_BYTES = ctypes.sizeof(BsvdInfo)

# exported symbols, one per declaration in include/bsvd_b200.h
EXPORTS = (
    "bsvd_gesvj_batched",
    "bsvd_gesvj_batched_host",
    "bsvd_workspace_bytes",
    "bsvd_host_workspace_bytes",
    "bsvd_select_kernel",
    "bsvd_select_kernel_batched",
    "bsvd_default_opts",
    "bsvd_strerror",
    "bsvd_abi_version",
    "bsvd_onesided_sweeps_batched",
    "bsvd_gram_batched",
    "bsvd_fused_pair_update_batched",
    "bsvd_bench_fma_peak",
    "bsvd_heevj_batched",
    "bsvd_heevj_workspace_bytes",
    "bsvd_verify_batched",
    "bsvd_finalize_batched",
    "bsvd_pack_host",
    "bsvd_gesvj_batched_host_gather",
    "bsvd_eig_sweeps_batched",
    "bsvd_householder_qr_workspace_bytes",
    "bsvd_householder_qr_batched",
)

_lib = None


def load():
    """Load libbsvd_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2601_17979_b200/csrc); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    vp, ci, i64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
    popts = ctypes.POINTER(BsvdOpts)
    L.bsvd_gesvj_batched.argtypes = [ci, ci, ci, ci, vp, i64, i64, vp, i64, i64, vp, i64, vp, i64, i64,
                                     popts, vp, vp, sz, vp]
    L.bsvd_gesvj_batched.restype = ci
    L.bsvd_gesvj_batched_host.argtypes = [ci, ci, ci, ci, vp, vp, vp, vp, popts, vp, ci, vp, sz,
                                          ctypes.POINTER(vp), ci]
    L.bsvd_gesvj_batched_host.restype = ci
    L.bsvd_gesvj_batched_host_gather.argtypes = [ci, ci, ci, ci, vp, vp, ci, vp, vp, vp, popts, vp, ci, vp, sz,
                                                 ctypes.POINTER(vp), ci]
    L.bsvd_gesvj_batched_host_gather.restype = ci
    L.bsvd_host_workspace_bytes.argtypes = [ci, ci, ci, ci, ci, popts]
    L.bsvd_host_workspace_bytes.restype = sz
    L.bsvd_workspace_bytes.argtypes = [ci, ci, ci, ci, popts]
    L.bsvd_workspace_bytes.restype = sz
    L.bsvd_select_kernel.argtypes = [ci, ci, ci, popts]
    L.bsvd_select_kernel.restype = ci
    L.bsvd_select_kernel_batched.argtypes = [ci, ci, ci, ci, popts]
    L.bsvd_select_kernel_batched.restype = ci
    L.bsvd_default_opts.argtypes = [popts]
    L.bsvd_default_opts.restype = None
    L.bsvd_strerror.argtypes = [ci]
    L.bsvd_strerror.restype = ctypes.c_char_p
    L.bsvd_abi_version.argtypes = []
    L.bsvd_abi_version.restype = ci
    L.bsvd_onesided_sweeps_batched.argtypes = [ci, ci, ci, ci, vp, i64, i64, ci, vp, i64, i64, ctypes.c_double,
                                               ci, vp, vp, vp]
    L.bsvd_onesided_sweeps_batched.restype = ci
    L.bsvd_gram_batched.argtypes = [ci, ci, ci, ci, ci, vp, i64, i64, vp, i64, i64, vp]
    L.bsvd_gram_batched.restype = ci
    L.bsvd_fused_pair_update_batched.argtypes = [ci, ci, ci, ci, vp, i64, i64, vp, i64, i64, ci, vp]
    L.bsvd_fused_pair_update_batched.restype = ci
    L.bsvd_heevj_batched.argtypes = [ci, ci, ci, vp, i64, i64, vp, i64, vp, i64, i64, ci, ctypes.c_double, ci, vp,
                                     vp, sz, vp]
    L.bsvd_heevj_batched.restype = ci
    L.bsvd_heevj_workspace_bytes.argtypes = [ci, ci, ci]
    L.bsvd_heevj_workspace_bytes.restype = sz
    L.bsvd_verify_batched.argtypes = [ci, ci, ci, ci, vp, i64, i64, vp, i64, i64, vp, i64, vp, i64, i64, vp, i64,
                                      vp, vp]
    L.bsvd_verify_batched.restype = ci
    L.bsvd_eig_sweeps_batched.argtypes = [ci, ci, ci, vp, i64, i64, vp, i64, vp, i64, i64, ctypes.c_double, ci, ci,
                                          vp, vp, ctypes.c_size_t, vp]
    L.bsvd_eig_sweeps_batched.restype = ci
    L.bsvd_pack_host.argtypes = [vp, ci, ctypes.c_size_t, vp, ci]
    L.bsvd_pack_host.restype = ci
    L.bsvd_finalize_batched.argtypes = [ci, ci, ci, ci, vp, i64, i64, ci, vp, i64, i64, vp, i64, i64, vp, i64, vp,
                                        i64, i64, vp]
    L.bsvd_finalize_batched.restype = ci
    L.bsvd_householder_qr_workspace_bytes.argtypes = [ci, ci, ci, ci]
    L.bsvd_householder_qr_workspace_bytes.restype = ctypes.c_size_t
    L.bsvd_householder_qr_batched.argtypes = [ci, ci, ci, ci, vp, i64, i64, vp, i64, i64, vp, i64, i64, vp,
                                              ctypes.c_size_t, vp]
    L.bsvd_householder_qr_batched.restype = ci
    L.bsvd_bench_fma_peak.argtypes = [ci, ci, ci, vp, vp]
    L.bsvd_bench_fma_peak.restype = ci
    _lib = L
    return L


_hostptrs = None
HOSTPTRS_PATH = os.path.join(HERE, "_lib", "libbsvd_hostptrs.so")


def gather_fortran(problems: list):
    """(ptrs uintp[B], (m, n), itemsize) when every item of the list exports an F-contiguous 2-D buffer of
    the same format and shape (one C pass, csrc/hostptrs.c), else None (the caller's per-item path)."""
    global _hostptrs
    if _hostptrs is None:
        if not os.path.exists(HOSTPTRS_PATH):
            return None
        H = ctypes.PyDLL(HOSTPTRS_PATH)  # CPython API inside: keeps the GIL
        H.bsvd_py_gather_fortran.argtypes = [ctypes.py_object, ctypes.c_ssize_t, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_char_p, ctypes.c_ssize_t]
        H.bsvd_py_gather_fortran.restype = ctypes.c_int
        H.bsvd_py_gather_ndarray.argtypes = [ctypes.py_object, ctypes.c_ssize_t, ctypes.py_object, ctypes.c_void_p,
                                             ctypes.c_void_p]
        H.bsvd_py_gather_ndarray.restype = ctypes.c_int
        H.bsvd_py_fill_lazy.argtypes = [ctypes.py_object, ctypes.c_ssize_t, ctypes.c_ssize_t, ctypes.py_object,
                                        ctypes.py_object]
        H.bsvd_py_fill_lazy.restype = ctypes.c_int
        H.bsvd_py_fill_pair_stats.argtypes = [ctypes.py_object, ctypes.c_ssize_t, ctypes.c_ssize_t,
                                              ctypes.c_void_p, ctypes.py_object]
        H.bsvd_py_fill_pair_stats.restype = ctypes.c_int
        _hostptrs = H
    import numpy as np

    n = len(problems)
    ptrs = np.empty(n, dtype=np.uintp)
    shape = np.zeros(2, dtype=np.intp)
    if _hostptrs.bsvd_py_gather_ndarray(problems, n, np.ndarray, ptrs.ctypes.data, shape.ctypes.data) == 0:
        return ptrs, (int(shape[0]), int(shape[1])), int(problems[0].dtype.itemsize)
    isz = np.zeros(1, dtype=np.intp)
    fmt = ctypes.create_string_buffer(32)
    rc = _hostptrs.bsvd_py_gather_fortran(problems, n, ptrs.ctypes.data, shape.ctypes.data, isz.ctypes.data, fmt, 32)
    if rc != 0:
        return None
    return ptrs, (int(shape[0]), int(shape[1])), int(isz[0])


def hostptrs():
    """The CPython helper library (csrc/hostptrs.c) or None when it was not built."""
    if _hostptrs is None and os.path.exists(HOSTPTRS_PATH):
        gather_fortran([])  # loads and declares it
    return _hostptrs


def check(rc: int, what: str = "bsvd call") -> None:
    if rc != BSVD_OK:
        msg = load().bsvd_strerror(rc).decode()
        raise RuntimeError(f"{what} failed: {msg} (code {rc})")
