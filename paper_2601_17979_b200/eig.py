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
