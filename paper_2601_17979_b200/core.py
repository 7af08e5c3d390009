"""Dtype policy, errors and layout contract.

Mirrors /root/reference/pkg/src/bsvd/core.py:14-60: four element types
(float32, float64, complex64, complex128), u = 2^-24 / 2^-53, column-major
matrices, ShapeError / DomainError (both ValueError subclasses).
"""

from __future__ import annotations

import numpy as np


class ShapeError(ValueError):
    """Operand dimensions do not conform (src/core.py:14-15)."""


class DomainError(ValueError):
    """Input lies outside an operation's domain (src/core.py:18-19)."""


_REAL_OF = {
    np.dtype(np.float32): np.dtype(np.float32),
    np.dtype(np.float64): np.dtype(np.float64),
    np.dtype(np.complex64): np.dtype(np.float32),
    np.dtype(np.complex128): np.dtype(np.float64),
}
SUPPORTED_DTYPES = tuple(_REAL_OF)
# C-ABI dtype codes (include/bsvd_b200.h; equal to src/fileio.py:49-54)
DTYPE_CODE = {
    np.dtype(np.float32): 0,
    np.dtype(np.float64): 1,
    np.dtype(np.complex64): 2,
    np.dtype(np.complex128): 3,
}


def check_dtype(dtype) -> np.dtype:
    """src/core.py:32-37."""
    dt = dtype.dtype if isinstance(dtype, np.ndarray) else np.dtype(dtype)
    if dt not in _REAL_OF:
        raise DomainError(f"unsupported element type {dt}; "
                          f"expected one of {[str(d) for d in SUPPORTED_DTYPES]}")
    return dt


def real_dtype(dtype) -> np.dtype:
    return _REAL_OF[check_dtype(dtype)]


def is_complex(dtype) -> bool:
    return np.dtype(dtype).kind == "c"


def unit_roundoff(dtype) -> float:
    """u = 2**-24 for single-precision fields, 2**-53 for double (src/core.py:49-51)."""
    return 2.0 ** -24 if real_dtype(dtype) == np.dtype(np.float32) else 2.0 ** -53


def fmatrix(a, dtype=None) -> np.ndarray:
    """Copy `a` into a 2-d Fortran-ordered array of a supported dtype (src/core.py:54-60)."""
    arr = np.array(a, dtype=dtype, order="F")
    if arr.ndim != 2:
        raise ShapeError(f"expected a 2-d array, got ndim={arr.ndim}")
    check_dtype(arr.dtype)
    return arr
