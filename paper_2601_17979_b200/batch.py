"""Batch driver: the drop-in for the reference's ``batch_svd``.

Mirrors /root/reference/pkg/src/bsvd/batch.py:24-157.  The reference steps
every problem one sweep per round from Python and masks converged problems
after each round (convergence_scan, :62-82).  Here each uniform
(dtype, m, n) group is ONE device launch: every problem runs its sweeps on
the device and stops after its own first quiet sweep (the per-problem early
exit of the masked batch), so results equal the reference's masked and
unmasked modes alike (a quiet sweep never writes, F7).  The batch telemetry
(rounds, masked pair skips, call counts) is reconstructed exactly from the
per-problem sweep counts the kernels report.

Per-problem failures keep the reference's semantics: a problem that fails
validation yields ``None`` and its exception is kept in ``state.errors``;
the batch never aborts (:105-111).
"""

from __future__ import annotations

import gc
import time
from dataclasses import dataclass, field
from math import ceil

import numpy as np

from . import _lib
from .core import DomainError, ShapeError, check_dtype, real_dtype
from .svd import QR_RATIO, SMALL_CUTOFF, JacobiOptions, SolveInfo, SvdResult, WorkCounters

__all__ = ["BatchState", "batch_svd", "convergence_scan"]

_ROUTE = {None: _lib.DISPATCH, "unblocked": _lib.FORCE_UNBLOCKED, "blocked": _lib.FORCE_BLOCKED,
          "qr": _lib.FORCE_QR}


@dataclass
class BatchState:
    """Observable batch telemetry (src/batch.py:24-59)."""

    active: np.ndarray
    outer_sweeps: np.ndarray
    pair_stats: list
    counters: WorkCounters = field(default_factory=WorkCounters)
    errors: dict = field(default_factory=dict)

    @classmethod
    def for_batch(cls, n_problems: int) -> "BatchState":
        return cls(
            active=np.ones(n_problems, dtype=bool),
            outer_sweeps=np.zeros(n_problems, dtype=np.int64),
            pair_stats=[None] * n_problems,
        )

    def _reset(self, n_problems: int) -> None:
        self.active = np.ones(n_problems, dtype=bool)
        self.outer_sweeps = np.zeros(n_problems, dtype=np.int64)
        self.pair_stats = [None] * n_problems
        self.counters = WorkCounters()
        self.errors = {}

    @property
    def n_problems(self) -> int:
        return len(self.pair_stats)


def convergence_scan(state: BatchState) -> bool:
    """Mask off problems whose latest sweep applied no rotation (src/batch.py:62-82)."""
    all_done = True
    for i in range(state.n_problems):
        if i in state.errors:
            continue
        if not state.active[i]:
            continue
        stats = state.pair_stats[i]
        if stats is None:
            all_done = False
            continue
        if all(rot == 0 for (_, _, rot) in stats):
            state.active[i] = False
        else:
            all_done = False
    return all_done


@dataclass
class _Prep:
    a: np.ndarray
    m: int
    n: int
    bn: int
    trans: bool
    blocked: bool
    trivial: bool
    pairs_per_sweep: int
    qr: bool = False


def _prepare(a, opts: JacobiOptions, force: str | None) -> _Prep:
    """Validation and routing of _ProblemRun.__init__ (src/svd.py:323-413)."""
    a = np.asarray(a)
    check_dtype(a)
    if a.ndim != 2:
        raise ShapeError(f"expected a 2-d matrix, got ndim={a.ndim}")
    m, n = a.shape
    if force is not None and m < n:
        raise ShapeError(f"{force} solver requires m >= n, got {m}x{n}; use svd_dispatch")
    trans = force is None and m < n
    bm, bn = (n, m) if trans else (m, n)
    trivial = bm == 0 or bn == 0
    # QR first (src/svd.py:364-371): forced, or dispatch with use_qr_preprocess and bm >= 3 bn
    qr = not trivial and (force == "qr" or (force is None and opts.use_qr_preprocess and bm >= QR_RATIO * bn))
    if force == "unblocked":
        blocked = False
    elif force == "blocked":
        blocked = True
    else:
        blocked = bn > SMALL_CUTOFF
    if trivial:
        pps = 0
    elif not blocked:
        pps = bn * (bn - 1) // 2 if bn >= 2 else 0
    else:
        ell = ceil(bn / opts.nb)
        pps = ell * (ell - 1) // 2 if ell >= 2 else 1
    return _Prep(a=a, m=m, n=n, bn=bn, trans=trans, blocked=blocked, trivial=trivial, pairs_per_sweep=pps, qr=qr)


def _clone_exc(exc: Exception) -> Exception:
    try:
        return type(exc)(*exc.args)
    except Exception:  # pragma: no cover - exotic exception signatures
        return exc


def _solve_problems(problems, opts: JacobiOptions, force: str | None, masked_rounds: bool):
    """Solve a list of problems on the device; returns (results, errors, telemetry).

    Validation depends only on (dtype, shape), so it runs once per distinct pair; each uniform group is
    one device launch; the per-problem records are built from column lists of the device telemetry.
    """
    from .solver import solve_host

    n_prob = len(problems)
    errors: dict = {}
    preps: list = [None] * n_prob
    arrays: list = [None] * n_prob
    proto: dict = {}
    groups: dict = {}
    trivial: list = []
    for idx, a in enumerate(problems):
        if type(a) is not np.ndarray:
            try:
                a = np.asarray(a)
            except Exception as exc:  # per-problem isolation (src/batch.py:105-111)
                errors[idx] = exc
                continue
        key = (a.dtype.str, a.shape)
        t = proto.get(key)
        if t is None:
            try:
                t = _prepare(a, opts, force)
            except Exception as exc:
                t = exc
            proto[key] = t
        if isinstance(t, Exception):
            errors[idx] = _clone_exc(t)
            continue
        arrays[idx] = a
        preps[idx] = t
        if t.trivial:
            trivial.append(idx)
        else:
            groups.setdefault(key, []).append(idx)

    solved: list = []  # (idxs, prep, U, S, V, columns, dt, kern)
    for key, idxs in groups.items():
        t0 = time.perf_counter()
        try:
            U, S, V, info, kern = solve_host([arrays[i] for i in idxs], opts, route=_ROUTE[force])
        except Exception as exc:
            for i in idxs:
                errors[i] = exc
            continue
        dt = (time.perf_counter() - t0) / len(idxs)
        cols = {f: info[f].tolist() for f in ("outer_sweeps", "converged", "rotations", "update_calls", "path",
                                             "last_rotations")}
        solved.append((idxs, preps[idxs[0]], U, S, V, cols, dt, kern))

    # rounds the reference's lockstep loop would run (src/batch.py:113-142)
    unconverged = any(not all(c["converged"]) for *_, c, _dt, _k in solved)
    mx = max([max(max(c["outer_sweeps"]), 1) for *_, c, _dt, _k in solved] + ([1] if trivial else []), default=0)
    rounds = opts.max_nsweeps if unconverged else mx

    results: list = [None] * n_prob
    tele: dict = {}
    want_v = opts.compute_right_vectors
    for idx in trivial:
        p = preps[idx]
        m, n = p.m, p.n
        k = min(m, n)
        dt = arrays[idx].dtype
        u = np.zeros((m, k), dtype=dt, order="F")
        sigma = np.zeros(k, dtype=real_dtype(dt))
        v = np.zeros((n, k), dtype=dt, order="F") if want_v else None
        info = SolveInfo(converged=True, outer_sweeps=0, inner_rotations=0, masked_pair_skips=0, path="empty",
                         counters=WorkCounters())
        results[idx] = SvdResult(u=u, sigma=sigma, v=v, info=info)
        tele[idx] = dict(outer_sweeps=0, converged=True, last=0, pair_stats=[])
    paths: dict = {}
    for idxs, p, U, S, V, cols, dtime, kern in solved:
        pps, blocked = p.pairs_per_sweep, p.blocked
        eig_unit = 0 if (not blocked and p.bn < 2) else 1
        masking = bool(masked_rounds and opts.masking)
        sw_l, cv_l, rot_l, up_l, path_l, last_l = (cols["outer_sweeps"], cols["converged"], cols["rotations"],
                                                   cols["update_calls"], cols["path"], cols["last_rotations"])
        for j, idx in enumerate(idxs):
            s_i = sw_l[j]
            conv = bool(cv_l[j])
            calls = s_i if masked_rounds is False or opts.masking else rounds
            masked = (rounds - max(s_i, 1)) * pps if (masking and conv) else 0
            if blocked:
                cnt = WorkCounters(gram_calls=calls * pps, eig_calls=calls * pps, update_calls=up_l[j],
                                   masked_pair_skips=masked, t_eig=dtime)
            else:
                cnt = WorkCounters(eig_calls=calls * eig_unit, masked_pair_skips=masked, t_eig=dtime)
            pv = path_l[j]
            path = paths.get(pv)
            if path is None:
                base = "blocked" if (pv & 0xFF) == 2 else "unblocked"
                path = ("transpose+" if pv & 0x100 else "") + ("qr+" if pv & 0x200 else "") + base
                paths[pv] = path
            info = SolveInfo(converged=conv, outer_sweeps=s_i, inner_rotations=rot_l[j], masked_pair_skips=masked,
                             path=path, counters=cnt)
            results[idx] = SvdResult(u=U[j], sigma=S[j], v=V[j] if (want_v and V is not None) else None, info=info)
            last = last_l[j]
            if not blocked:
                stats = [(last == 0, 1, last)]
            else:
                stats = [(True, 1, 0)] * pps if last == 0 else [(False, 1, last)] + [(True, 1, 0)] * (pps - 1)
            tele[idx] = dict(outer_sweeps=s_i, converged=conv, last=last, pair_stats=stats, kernel=kern)
    return results, errors, tele


def batch_svd(problems, opts: JacobiOptions | None = None, state: BatchState | None = None):
    """Solve every problem in the batch; results align with the input order (src/batch.py:85-157)."""
    if opts is None:
        opts = JacobiOptions()
    problems = list(problems)
    if not problems:
        raise DomainError("batch must contain at least one problem")
    st = state if state is not None else BatchState.for_batch(len(problems))
    st._reset(len(problems))
    # the records are tens of thousands of small objects: keep the cyclic collector out of the way
    gc_was = gc.isenabled()
    gc.disable()
    try:
        results, errors, tele = _solve_problems(problems, opts, force=None, masked_rounds=True)
    finally:
        if gc_was:
            gc.enable()
    st.errors = dict(errors)
    c = st.counters
    for idx, t in tele.items():
        st.outer_sweeps[idx] = t["outer_sweeps"]
        st.pair_stats[idx] = t["pair_stats"]
        st.active[idx] = not t["converged"]
        w = results[idx].info.counters
        c.gram_calls += w.gram_calls
        c.eig_calls += w.eig_calls
        c.update_calls += w.update_calls
        c.masked_pair_skips += w.masked_pair_skips
        c.t_aux += w.t_aux
        c.t_gram += w.t_gram
        c.t_eig += w.t_eig
        c.t_vec += w.t_vec
    return results
