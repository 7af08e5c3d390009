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


class _Group:
    """One device launch's outputs and the per-problem accounting rules its lazy records share."""

    __slots__ = ("U", "S", "V", "cols", "calls", "masked", "blocked", "pps", "eig_unit", "dtime", "atime", "paths")


_PATHS: dict = {}


def _set_ref(r, g, j):
    object.__setattr__(r, "_g", g)
    object.__setattr__(r, "_j", j)


def _path_string(pv: int) -> str:
    p = _PATHS.get(pv)
    if p is None:
        base = "blocked" if (pv & 0xFF) == 2 else "unblocked"
        p = _PATHS[pv] = ("transpose+" if pv & 0x100 else "") + ("qr+" if pv & 0x200 else "") + base
    return p


class _LazyResult(SvdResult):
    """An ``SvdResult`` whose fields (views into the group's factor arrays, the ``SolveInfo`` record)
    are built on first access.  A 10k-problem batch would otherwise spend longer building 60k Python
    objects than the device spends solving it; the record is otherwise the reference's frozen
    dataclass (same fields, equality, repr, immutability; copies and pickles are plain SvdResults)."""

    __slots__ = ("_g", "_j")  # set by the C helper straight into the slots (no per-record dict until first use)

    def __getattr__(self, name):
        if name not in ("u", "sigma", "v", "info"):
            raise AttributeError(name)
        try:
            g = object.__getattribute__(self, "_g")
        except AttributeError:
            raise AttributeError(name) from None
        if g is None:
            raise AttributeError(name)
        j = object.__getattribute__(self, "_j")
        d = self.__dict__
        c = g.cols
        if g.blocked:
            cnt = WorkCounters(gram_calls=int(g.calls[j]) * g.pps, eig_calls=int(g.calls[j]) * g.pps,
                               update_calls=int(c["update_calls"][j]), masked_pair_skips=int(g.masked[j]),
                               t_eig=g.dtime, t_aux=g.atime)
        else:
            cnt = WorkCounters(eig_calls=int(g.calls[j]) * g.eig_unit, masked_pair_skips=int(g.masked[j]),
                               t_eig=g.dtime, t_aux=g.atime)
        info = SolveInfo(converged=bool(c["converged"][j]), outer_sweeps=int(c["outer_sweeps"][j]),
                         inner_rotations=int(c["rotations"][j]), masked_pair_skips=int(g.masked[j]),
                         path=_path_string(int(c["path"][j])), counters=cnt)
        d.update(u=g.U[j], sigma=g.S[j], v=g.V[j] if g.V is not None else None, info=info)
        object.__setattr__(self, "_g", None)  # materialised: the fields now live in the instance dict
        return d[name]

    def __reduce__(self):
        return (SvdResult, (self.u, self.sigma, self.v, self.info))


def _solve_problems(problems, opts: JacobiOptions, force: str | None, masked_rounds: bool):
    """Solve a list of problems on the device; returns (results, errors, telemetry).

    Validation depends only on (dtype, shape), so it runs once per distinct pair; each uniform group is
    one device launch; records are lazy views of the group's arrays and the batch telemetry is computed
    with array operations on the kernels' per-problem counters.  Telemetry: (groups, trivial), groups a
    list of (problem indices, outer sweeps, converged, last-sweep rotations, _Group).
    """
    from .solver import solve_host

    n_prob = len(problems)
    errors: dict = {}
    preps: list = [None] * n_prob
    arrays: list = [None] * n_prob
    proto: dict = {}
    groups: dict = {}
    trivial: list = []
    uniform = None
    if n_prob > 64 and type(problems) is list and type(problems[0]) is np.ndarray:
        # one C pass: every problem an F-contiguous matrix of one dtype and shape (the common case)
        g = _lib.gather_fortran(problems)
        if g is not None and g[1] == problems[0].shape and g[2] == problems[0].dtype.itemsize:
            try:
                t = _prepare(problems[0], opts, force)
            except Exception:
                t = None  # per-problem path reports the error for every problem
            if t is not None and not t.trivial:
                uniform = (g[0], t)
    for idx, a in enumerate(problems if uniform is None else ()):
        if type(a) is not np.ndarray:
            try:
                a = np.asarray(a)
            except Exception as exc:  # per-problem isolation (src/batch.py:105-111)
                errors[idx] = exc
                continue
        key = (a.dtype, a.shape)
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

    from .solver import last_device_seconds

    solved: list = []  # (idxs, prep, U, S, V, info, (device, host) seconds per problem, group)
    results: list = [None] * n_prob
    if uniform is not None:
        ptrs, t = uniform
        groups = {None: range(n_prob)}
        preps = [t]
    H = _lib.hostptrs()
    for key, idxs in groups.items():
        t0 = time.perf_counter()
        g = _Group()
        try:
            if uniform is not None:
                finish = solve_host(problems, opts, route=_ROUTE[force], ptrs=ptrs, defer=True)
                if H is not None:  # the records (lazy views of g) are built while the device pipeline drains
                    H.bsvd_py_fill_lazy(results, 0, n_prob, _LazyResult, g)
                U, S, V, info, _kern = finish()
            else:
                U, S, V, info, _kern = solve_host([arrays[i] for i in idxs], opts, route=_ROUTE[force])
        except Exception as exc:
            for i in idxs:
                errors[i] = exc
                results[i] = None
            continue
        wall, dev = time.perf_counter() - t0, last_device_seconds()
        solved.append((idxs, preps[idxs[0]], U, S, V, info, (dev / len(idxs), max(0.0, wall - dev) / len(idxs)),
                       g if (uniform is not None and H is not None) else None))

    # rounds the reference's lockstep loop would run (src/batch.py:113-142)
    unconverged = any(not info["converged"].all() for *_, info, _dt, _g in solved)
    mx = max([max(int(info["outer_sweeps"].max()), 1) for *_, info, _dt, _g in solved] + ([1] if trivial else []),
             default=0)
    rounds = opts.max_nsweeps if unconverged else mx

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
    tele = []
    masking = bool(masked_rounds and opts.masking)
    new = object.__new__
    for idxs, p, U, S, V, info, dtime, pre in solved:
        g = pre if pre is not None else _Group()
        sw = info["outer_sweeps"].astype(np.int64)
        conv = info["converged"] != 0
        g.U, g.S, g.V = U, S, (V if want_v else None)
        g.cols = info
        g.calls = sw if (masked_rounds is False or opts.masking) else np.full_like(sw, rounds)
        g.masked = ((rounds - np.maximum(sw, 1)) * p.pairs_per_sweep) * (conv & masking)
        g.blocked, g.pps = p.blocked, p.pairs_per_sweep
        g.eig_unit = 0 if (not p.blocked and p.bn < 2) else 1
        g.dtime, g.atime = dtime
        if pre is not None:
            pass  # records already built (during the device pipeline)
        elif isinstance(idxs, range) and H is not None:  # one C pass (csrc/hostptrs.c): records with (_g, _j)
            H.bsvd_py_fill_lazy(results, idxs.start, len(idxs), _LazyResult, g)
        elif isinstance(idxs, range):
            recs = [new(_LazyResult) for _ in idxs]
            for j, r in enumerate(recs):
                _set_ref(r, g, j)
            results[idxs.start:idxs.stop] = recs
        else:
            for j, idx in enumerate(idxs):
                r = new(_LazyResult)
                _set_ref(r, g, j)
                results[idx] = r
        tele.append((idxs, sw, conv, info["last_rotations"], g))
    return results, errors, (tele, trivial)


def batch_svd(problems, opts: JacobiOptions | None = None, state: BatchState | None = None):
    """Solve every problem in the batch; results align with the input order (src/batch.py:85-157)."""
    if opts is None:
        opts = JacobiOptions()
    problems = list(problems)
    if not problems:
        raise DomainError("batch must contain at least one problem")
    if state is not None:
        state._reset(len(problems))
    # the records are tens of thousands of small objects: keep the cyclic collector out of the way
    gc_was = gc.isenabled()
    gc.disable()
    try:
        results, errors, tele = _solve_problems(problems, opts, force=None, masked_rounds=True)
    finally:
        if gc_was:
            gc.enable()
    if state is None:  # no caller-visible state: the per-problem batch telemetry would only be discarded
        return results
    st = state
    st.errors = dict(errors)
    c = st.counters
    groups, trivial = tele
    for idx in trivial:
        st.outer_sweeps[idx] = 0
        st.pair_stats[idx] = []
        st.active[idx] = False
    quiet1 = (True, 1, 0)
    for idxs, sw, conv, last, g in groups:
        ix = slice(idxs.start, idxs.stop) if isinstance(idxs, range) else np.asarray(idxs)
        st.outer_sweeps[ix] = sw
        st.active[ix] = ~conv
        pps = g.pps
        if not g.blocked:
            H = _lib.hostptrs() if isinstance(idxs, range) else None
            if H is not None:  # one C pass; one shared tuple for the common quiet last sweep
                lc = np.ascontiguousarray(last, dtype=np.int32)
                H.bsvd_py_fill_pair_stats(st.pair_stats, idxs.start, len(idxs), lc.ctypes.data, quiet1)
            elif isinstance(idxs, range):
                st.pair_stats[ix] = [[quiet1] if l == 0 else [(False, 1, l)] for l in last.tolist()]
            else:
                for i, l in zip(idxs, last.tolist()):
                    st.pair_stats[i] = [(l == 0, 1, l)]
        else:
            quiet = [(True, 1, 0)] * pps
            for i, l in zip(idxs, last.tolist()):
                st.pair_stats[i] = list(quiet) if l == 0 else [(False, 1, l)] + [(True, 1, 0)] * (pps - 1)
        n = len(idxs)
        calls = int(g.calls.sum())
        if g.blocked:
            c.gram_calls += calls * pps
            c.eig_calls += calls * pps
            c.update_calls += int(g.cols["update_calls"].sum())
        else:
            c.eig_calls += calls * g.eig_unit
        c.masked_pair_skips += int(g.masked.sum())
        c.t_eig += g.dtime * n
        c.t_aux += g.atime * n
    return results
