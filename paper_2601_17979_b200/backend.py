"""The reference's kernel plugin interface (src/backend.py:30-35) with one implementation: the B200.

``Backend(name, eig_sweeps, onesided_sweeps, fused_pair_update)`` has the reference's fields and call
signatures; here every operator runs on the device through the batch-granular C-ABI (kernels.py).
There is deliberately no second backend and no dispatch: ``select``/``use`` accept only "b200" (or
"auto", which means the same thing) and reject the reference's CPU backends ("numba", "numpy") --
this package has no CPU fallback.
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass
from typing import Callable

from . import kernels

_VALID = ("auto", "b200")


@dataclass(frozen=True)
class Backend:
    name: str
    eig_sweeps: Callable
    onesided_sweeps: Callable
    fused_pair_update: Callable


_B200 = Backend(name="b200", eig_sweeps=kernels.eig_sweeps, onesided_sweeps=kernels.onesided_sweeps,
                fused_pair_update=kernels.fused_pair_update)


def _resolve(name: str) -> Backend:
    if str(name).lower() not in _VALID:
        raise ValueError(f"unknown backend {name!r}; this package runs only on the B200 (expected one of "
                         f"{', '.join(_VALID)}; the reference's numba/numpy CPU backends are not provided)")
    return _B200


def active() -> Backend:
    """The backend in effect (always the B200 one)."""
    return _B200


def select(name: str) -> Backend:
    """Validate ``name`` and return the backend (src/backend.py:98-103)."""
    return _resolve(name)


@contextlib.contextmanager
def use(name: str):
    """Scoped form of select (src/backend.py:106-115)."""
    yield _resolve(name)
