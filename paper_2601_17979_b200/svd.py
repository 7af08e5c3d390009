"""Solver options, result records and the single-problem entry points.

Mirrors /root/reference/pkg/src/bsvd/svd.py: ``JacobiOptions`` (:58-91),
``WorkCounters`` (:93-124), ``SolveInfo`` (:126-133), ``SvdResult``
(:136-141) and ``svd_unblocked`` / ``svd_blocked`` / ``svd_dispatch``
(:559-582).  Every solve runs on the B200 through the batch path
(``batch.batch_svd``); a single problem is a batch of one.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import DomainError, ShapeError

# dispatch thresholds (src/svd.py:51-55)
SMALL_CUTOFF = 32
QR_RATIO = 3.0
INNER_BUDGET = 100


@dataclass(frozen=True)
class JacobiOptions:
    """Solver knobs shared by every entry point (src/svd.py:58-91)."""

    k: float = 30.0
    max_nsweeps: int = 30
    nb: int = 16
    inner_sweeps: int = 1
    masking: bool = False
    use_qr_preprocess: bool = False
    compute_right_vectors: bool = True
    fused_updates: bool = True
    row_block: int = 64

    def __post_init__(self):
        if self.k <= 0:
            raise DomainError(f"k must be positive, got {self.k}")
        if self.max_nsweeps < 1:
            raise DomainError(f"max_nsweeps must be >= 1, got {self.max_nsweeps}")
        if self.nb < 1:
            raise DomainError(f"nb must be >= 1, got {self.nb}")
        if self.inner_sweeps < 0:
            raise DomainError(f"inner_sweeps must be >= 0, got {self.inner_sweeps}")
        if self.row_block < 1:
            raise DomainError(f"row_block must be >= 1, got {self.row_block}")


@dataclass
class WorkCounters:
    """Work and stage-time accounting (src/svd.py:93-124).

    Call counts follow the reference's own bookkeeping.  Times, per problem: ``t_eig`` is the device
    stage -- the pipelined host-to-device copy, solve and device-to-host copy of the problem's group
    (wall time, synchronised) shared evenly by its problems; ``t_aux`` the host stage (validation,
    pointer gathering, result handling).  The B200 kernels fuse the Gram, eigensolve and update stages
    of the blocked path into one launch, so ``t_gram`` and ``t_vec`` stay 0 (their work is in t_eig).
    """

    gram_calls: int = 0
    eig_calls: int = 0
    update_calls: int = 0
    masked_pair_skips: int = 0
    t_aux: float = 0.0
    t_gram: float = 0.0
    t_eig: float = 0.0
    t_vec: float = 0.0

    def add(self, other: "WorkCounters") -> None:
        self.gram_calls += other.gram_calls
        self.eig_calls += other.eig_calls
        self.update_calls += other.update_calls
        self.masked_pair_skips += other.masked_pair_skips
        self.t_aux += other.t_aux
        self.t_gram += other.t_gram
        self.t_eig += other.t_eig
        self.t_vec += other.t_vec

    def total_seconds(self) -> float:
        return self.t_aux + self.t_gram + self.t_eig + self.t_vec


@dataclass(frozen=True)
class SolveInfo:
    converged: bool
    outer_sweeps: int
    inner_rotations: int
    masked_pair_skips: int
    path: str
    counters: WorkCounters | None = None


@dataclass(frozen=True)
class SvdResult:
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray | None
    info: SolveInfo


def _run_standalone(a, opts: JacobiOptions | None, force: str | None) -> SvdResult:
    from .batch import _solve_problems

    if opts is None:
        opts = JacobiOptions()
    results, errors, _ = _solve_problems([a], opts, force=force, masked_rounds=False)
    if 0 in errors:
        raise errors[0]
    return results[0]


def svd_unblocked(a, opts: JacobiOptions | None = None) -> SvdResult:
    """SVD by scalar column rotations; requires m >= n (src/svd.py:559-561)."""
    return _run_standalone(a, opts, force="unblocked")


def svd_blocked(a, opts: JacobiOptions | None = None) -> SvdResult:
    """SVD by block-column rotations with an inner eigensolver; m >= n (src/svd.py:564-566)."""
    return _run_standalone(a, opts, force="blocked")


def svd_qr_preprocessed(a, opts: JacobiOptions | None = None) -> SvdResult:
    """QR first, Jacobi SVD on the small R factor, then U = Q @ Uhat (src/svd.py:569-571); m >= n."""
    return _run_standalone(a, opts, force="qr")


def svd_dispatch(a, opts: JacobiOptions | None = None) -> SvdResult:
    """Shape-aware entry point (src/svd.py:574-582)."""
    return _run_standalone(a, opts, force=None)


def _check_2d(a) -> np.ndarray:
    from .core import check_dtype

    a = np.asarray(a)
    check_dtype(a)
    if a.ndim != 2:
        raise ShapeError(f"expected a 2-d matrix, got ndim={a.ndim}")
    return a


def finalize(work_a, v=None) -> SvdResult:
    """Turn a converged working copy into (U, sigma, V) on the device (src/svd.py:278-303):
    sigma_i = ||w_i|| (float64), U = W / sigma with orthogonal completion of columns below tiny/u,
    stable descending order, V permuted identically."""
    from .kernels import finalize_factors

    u, sigma, vv = finalize_factors(work_a, v)
    info = SolveInfo(converged=True, outer_sweeps=0, inner_rotations=0, masked_pair_skips=0, path="finalize")
    return SvdResult(u=u, sigma=sigma, v=vv, info=info)
