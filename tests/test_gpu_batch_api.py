"""The reference-facing list API on the fast host path (batch.py, solver.solve_host): lazily built records,
pooled pinned result buffers, the one-pass pointer gather + packing overlapped with the pipeline
(bsvd_gesvj_batched_host_gather), stage times.  Semantics from the reference's tests/test_batch.py and
tests/test_svd.py (records are frozen SvdResult dataclasses, inputs never mutated, batch == standalone)."""

import copy
import dataclasses
import pickle

import numpy as np
import pytest

import paper_2601_17979_b200 as bs

pytestmark = pytest.mark.gpu


def _mats(B, seed, m=32, n=32, dt=np.float64):
    rng = np.random.default_rng(seed)
    return [np.asfortranarray(rng.random((m, n)).astype(dt)) for _ in range(B)]


def test_lazy_records_are_svd_results():
    mats = _mats(200, 1)
    res = bs.batch_svd(mats)
    r = res[17]
    assert isinstance(r, bs.SvdResult) and isinstance(r.info, bs.SolveInfo)
    s = bs.svd_dispatch(mats[17])
    assert np.array_equal(r.sigma, s.sigma) and np.array_equal(r.u, s.u) and np.array_equal(r.v, s.v)
    assert r.info.path == s.info.path == "unblocked" and r.info.outer_sweeps == s.info.outer_sweeps
    with pytest.raises(dataclasses.FrozenInstanceError):
        r.u = None
    assert "SvdResult" in repr(r) or "LazyResult" in repr(r)
    for c in (copy.copy(r), copy.deepcopy(r), pickle.loads(pickle.dumps(r))):
        assert np.array_equal(c.sigma, r.sigma) and np.array_equal(c.u, r.u) and c.info == r.info
    r2 = dataclasses.replace(res[3], sigma=np.zeros(32))
    assert np.array_equal(r2.u, res[3].u) and not r2.sigma.any()
    assert r.info.counters.t_eig > 0 and r.info.counters.t_aux >= 0


def test_pooled_results_survive_later_calls():
    """Results are views into pooled pinned buffers; a buffer is reused only after every view of it is gone."""
    a, b = _mats(300, 2), _mats(300, 3)
    ra = bs.batch_svd(a)
    keep = [(x.sigma.copy(), x.u.copy(), x.v.copy()) for x in ra]
    for _ in range(6):  # more calls than pooled buffers per shape, while ra is alive
        rb = bs.batch_svd(b)
    for x, (s, u, v) in zip(ra, keep):
        assert np.array_equal(x.sigma, s) and np.array_equal(x.u, u) and np.array_equal(x.v, v)
    s0 = ra[5].sigma
    del ra, x
    rc = bs.batch_svd(a)  # may reuse ra's buffer now; s0 still holds it alive
    assert np.array_equal(s0, keep[5][0]) and np.array_equal(rc[5].sigma, keep[5][0])
    assert np.array_equal(rb[9].sigma, bs.svd_dispatch(b[9]).sigma)


def test_gather_path_equals_per_item_path():
    """The one-pass C gather (uniform F-ordered ndarrays) and the per-item Python path (a C-ordered
    member forces it) give identical bits; inputs are never mutated."""
    mats = _mats(150, 4)
    orig = [m.copy() for m in mats]
    r1 = bs.batch_svd(mats)
    mixed = list(mats)
    mixed[7] = np.ascontiguousarray(mats[7])  # same values, C order
    r2 = bs.batch_svd(mixed)
    for x, y in zip(r1, r2):
        assert np.array_equal(x.sigma, y.sigma) and np.array_equal(x.u, y.u) and np.array_equal(x.v, y.v)
    assert all(np.array_equal(m, o) for m, o in zip(mats, orig))


def test_gather_path_fault_isolation_and_state():
    mats = _mats(100, 5)
    mats[4] = np.arange(9).reshape(3, 3)  # integer: DomainError, None slot
    st = bs.BatchState.for_batch(len(mats))
    res = bs.batch_svd(mats, state=st)
    assert res[4] is None and isinstance(st.errors[4], bs.DomainError)
    assert all(r is not None for i, r in enumerate(res) if i != 4)
    assert st.outer_sweeps[0] == res[0].info.outer_sweeps and not st.active[0]
    assert st.counters.t_eig > 0 and st.counters.eig_calls > 0
    assert st.pair_stats[0] == [(True, 1, 0)]
