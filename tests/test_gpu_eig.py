"""GPU tests of the batched Hermitian Jacobi eigensolver (bsvd_heevj_batched; the reference's
jacobi_hermitian_eig, src/eig.py:90-148).  Mirrors tests/test_eig.py:88-160 of the reference and
checks parity with the reference's golden vectors and the CPU restatement."""

import numpy as np
import pytest

import paper_2601_17979_b200 as bs
from common import ALL_DTYPES, unit_roundoff
from test_oracle import _oracle_heev

pytestmark = pytest.mark.gpu


def random_hermitian(n, dtype=np.float64, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.random((n, n))
    if np.dtype(dtype).kind == "c":
        x = x + 1j * rng.random((n, n))
    return np.asfortranarray(((x + x.conj().T) / 2).astype(dtype))


def off_norm(a):
    return float(np.linalg.norm(a - np.diag(np.diag(a))))


def _check_eig(g, d, m, info, dt):
    n = g.shape[0]
    u = unit_roundoff(dt)
    gf = np.linalg.norm(g)
    assert info.converged
    assert np.linalg.norm(m @ np.diag(d).astype(dt) @ m.conj().T - g) < 50 * n * u * gf
    assert np.linalg.norm(m.conj().T @ m - np.eye(n)) < 50 * n * u
    assert np.allclose(np.sort(d), np.linalg.eigvalsh(g.astype(np.complex128 if np.iscomplexobj(g) else np.float64)),
                       atol=50 * n * u * gf)


@pytest.mark.parametrize("dt", ALL_DTYPES)
def test_diagonalizes(dt):
    g = random_hermitian(12, dt, seed=3)
    d, m, info = bs.jacobi_hermitian_eig(g)
    _check_eig(g, d, m, info, dt)


def test_golden_vs_reference(golden):
    for eid, e in golden.eig.items():
        g = golden.get(eid, "g")
        d, m, info = bs.jacobi_hermitian_eig(g)
        dt = g.dtype
        u = unit_roundoff(dt)
        d_ref = golden.get(eid, "d")
        # eigenvalue parity, normwise and as sets: the GPU runs the disjoint pairs of an iteration
        # concurrently, and near-equal eigenvalues may settle in each other's positions
        assert np.max(np.abs(np.sort(d) - np.sort(d_ref))) <= 2 * g.shape[0] * u * np.linalg.norm(g), eid
        assert abs(info.sweeps_run - e["sweeps_run"]) <= 1 and info.converged == e["converged"], eid
        _check_eig(g, d, m, info, dt)


@pytest.mark.parametrize("dt", ALL_DTYPES)
@pytest.mark.parametrize("n", [2, 5, 16, 31, 64, 96])
def test_batches_vs_oracle(dt, n):
    gs = [random_hermitian(n, dt, seed=200 + 7 * b + n) for b in range(5)]
    res = bs.batch_hermitian_eig(gs)
    u = unit_roundoff(dt)
    for g, (d, m, info) in zip(gs, res):
        d_o, m_o, sw, rot, cv = _oracle_heev(g)
        assert np.max(np.abs(np.sort(d) - np.sort(d_o))) <= 2 * n * u * np.linalg.norm(g)
        assert abs(info.sweeps_run - sw) <= 1 and info.converged == cv
        _check_eig(g, d, m, info, dt)


def test_known_two_by_two():
    d, m, info = bs.jacobi_hermitian_eig(np.asfortranarray([[9.0, 12.0], [12.0, 41.0]]))
    assert np.allclose(d, [5.0, 45.0]) and info.rotations == 1


def test_already_diagonal_quiet_first_sweep():
    d, m, info = bs.jacobi_hermitian_eig(np.asfortranarray(np.diag([4.0, 1.0, 2.0])))
    assert info == bs.EigInfo(sweeps_run=1, rotations=0, converged=True)
    assert np.array_equal(d, [4.0, 1.0, 2.0]) and np.array_equal(m, np.eye(3))


def test_trivial_and_guard_and_max_sweeps():
    d, m, info = bs.jacobi_hermitian_eig(np.asfortranarray([[7.0]]))
    assert d[0] == 7.0 and info.converged
    d, m, info = bs.jacobi_hermitian_eig(random_hermitian(8, seed=9), k=1e30)
    assert info.rotations == 0 and info.converged
    g = random_hermitian(16, seed=4)
    d1, m1, i1 = bs.jacobi_hermitian_eig(g, max_sweeps=1)
    assert i1.sweeps_run == 1 and not i1.converged
    assert off_norm(m1.conj().T @ g @ m1) < off_norm(g)
    dc, mc, ic = bs.jacobi_hermitian_eig(g)
    assert ic.converged and ic.sweeps_run > 1


def test_eigvecs_accumulate_in_place_and_validation():
    g = random_hermitian(6, seed=6)
    pre = np.asfortranarray(np.eye(6))
    d0, m0, _ = bs.jacobi_hermitian_eig(g)
    d1, m1, _ = bs.jacobi_hermitian_eig(g, eigvecs=pre)
    assert m1 is pre and np.array_equal(m0, m1) and np.array_equal(d0, d1)
    g4 = random_hermitian(4, seed=7)
    with pytest.raises(bs.ShapeError):
        bs.jacobi_hermitian_eig(g4, eigvecs=np.eye(4))  # C order
    with pytest.raises(bs.ShapeError):
        bs.jacobi_hermitian_eig(g4, eigvecs=np.asfortranarray(np.eye(3)))
    with pytest.raises(bs.DomainError):
        bs.jacobi_hermitian_eig(np.asfortranarray([[1.0, 2.0], [5.0, 1.0]]))


@pytest.mark.parametrize("rows", [3, 9])
def test_eigvecs_any_row_count(rows):
    """The reference accepts any F-contiguous n-column accumulator (src/eig.py:128-133) and rotates its
    columns in place: the result is eigvecs @ Q for the rotation product Q (the square run's m)."""
    g = random_hermitian(6, seed=8)
    rng = np.random.default_rng(rows)
    pre = np.asfortranarray(rng.random((rows, 6)))
    want = pre.copy()
    d0, q, _ = bs.jacobi_hermitian_eig(g)
    d1, m1, i1 = bs.jacobi_hermitian_eig(g, eigvecs=pre)
    assert m1 is pre and np.array_equal(d0, d1) and i1.converged
    np.testing.assert_allclose(m1, want @ q, rtol=0, atol=64 * 2.0 ** -53 * np.abs(want).sum())
    # and batched, rows differing per problem
    pres = [np.asfortranarray(rng.random((r, 6))) for r in (rows, 6, 2)]
    outs = bs.batch_hermitian_eig([g, g, g], eigvecs=[p.copy(order="F") for p in pres])
    for p, (d, m, _) in zip(pres, outs):
        np.testing.assert_allclose(m, p @ q, rtol=0, atol=64 * 2.0 ** -53 * np.abs(p).sum())


def test_single_sweep_reduces_off_norm():  # reference tests/test_eig.py:133-136
    g = random_hermitian(10, seed=5)
    d, m, info = bs.jacobi_hermitian_eig(g, max_sweeps=1)
    assert info.sweeps_run == 1 and off_norm(m.conj().T @ g @ m) < off_norm(g)


def test_rejections_and_input_not_mutated():  # reference tests/test_eig.py:156-178
    with pytest.raises(bs.DomainError):
        bs.jacobi_hermitian_eig(np.asfortranarray([[1.0, 2.0], [5.0, 1.0]]))
    with pytest.raises(bs.ShapeError):
        bs.jacobi_hermitian_eig(np.zeros((2, 3), order="F"))
    g = random_hermitian(4)
    for kw in ({"k": 0.0}, {"max_sweeps": 0}):
        with pytest.raises(bs.DomainError):
            bs.jacobi_hermitian_eig(g, **kw)
    g8 = random_hermitian(8, seed=8)
    keep = g8.copy()
    bs.jacobi_hermitian_eig(g8)
    assert np.array_equal(g8, keep)


from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=25, deadline=None)
@given(n=st.integers(2, 24), seed=st.integers(0, 2 ** 16))
def test_property_spectrum_matches_lapack(n, seed):  # reference tests/test_eig.py:180-187
    g = random_hermitian(n, np.float64, seed=seed)
    d, m, info = bs.jacobi_hermitian_eig(g)
    assert info.converged
    tol = 64 * n * 2.0 ** -53 * max(np.linalg.norm(g), 1.0)
    assert np.allclose(np.sort(d), np.linalg.eigvalsh(g), atol=tol)
