"""GPU parity of the standalone operators against the reference's own outputs (tests/golden/ops.npz,
made by tests/golden/make_ops.py from bsvd itself): finalize (src/svd.py:278-303) and householder_qr
(src/core.py:118-168), all four dtypes."""

import os

import numpy as np
import pytest

import paper_2601_17979_b200 as bs
from common import unit_roundoff

pytestmark = pytest.mark.gpu

OPS = np.load(os.path.join(os.path.dirname(__file__), "golden", "ops.npz"))
FIN = [str(c) for c in OPS["cases"] if str(c).startswith("fin_")]
HQR = [str(c) for c in OPS["cases"] if str(c).startswith("hqr_")]


@pytest.mark.parametrize("key", FIN)
def test_finalize_matches_reference(key):
    w, v = OPS[key + "_w"], OPS[key + "_v"]
    u_ref, s_ref, v_ref = OPS[key + "_u"], OPS[key + "_s"], OPS[key + "_vo"]
    w_keep, v_keep = w.copy(), v.copy()
    r = bs.finalize(w, v)
    assert np.array_equal(w, w_keep) and np.array_equal(v, v_keep)  # inputs never mutated
    uu = unit_roundoff(w.dtype)
    n = w.shape[1]
    assert r.sigma.dtype == s_ref.dtype and r.u.dtype == u_ref.dtype and r.info.path == "finalize"
    assert np.max(np.abs(r.sigma - s_ref)) <= 4 * n * uu * s_ref[0]
    assert np.array_equal(r.v, v_ref)  # same stable permutation: V columns are copied, not computed
    assert np.max(np.abs(r.u - u_ref)) <= 50 * uu
    r0 = bs.finalize(w)
    assert r0.v is None and np.array_equal(r0.sigma, r.sigma) and np.array_equal(r0.u, r.u)
    assert np.max(np.abs(r0.sigma - OPS[key + "_s0"])) <= 4 * n * uu * s_ref[0]


@pytest.mark.parametrize("key", HQR)
def test_householder_qr_matches_reference(key):
    a = OPS[key + "_a"]
    q_ref, r_ref = OPS[key + "_q"], OPS[key + "_r"]
    q, r = bs.householder_qr(a)
    m, n = a.shape
    uu = unit_roundoff(a.dtype)
    an = float(np.abs(a).sum(axis=0).max())
    assert q.shape == (m, n) and r.shape == (n, n) and q.dtype == a.dtype and r.dtype == a.dtype
    assert np.allclose(np.tril(r, -1), 0) and np.all(np.real(np.diag(r)) >= 0) and np.all(np.imag(np.diag(r)) == 0)
    assert np.abs(q @ r - a).sum(axis=0).max() <= 30 * n * uu * an
    assert np.abs(np.eye(n) - q.conj().T @ q).sum(axis=0).max() <= 30 * n * uu
    if key.endswith("_sq"):  # column 7 duplicates column 1: reflector 7 is rounding noise, so rows 7.. of R
        # and columns 7.. of Q are determined only up to a unitary in that subspace
        assert np.max(np.abs(r[:7] - r_ref[:7])) <= 30 * n * uu * an
        assert np.max(np.abs(q[:, :7] - q_ref[:, :7])) <= 30 * n * uu * max(1.0, an)
    else:
        assert np.max(np.abs(r - r_ref)) <= 30 * n * uu * an
        assert np.max(np.abs(q - q_ref)) <= 30 * n * uu * max(1.0, an)


def test_operator_shape_errors():
    with pytest.raises(bs.ShapeError):
        bs.householder_qr(np.zeros((3, 5)))
    with pytest.raises(bs.ShapeError):
        bs.finalize(np.zeros((3, 5)))
    with pytest.raises(bs.ShapeError):
        bs.finalize(np.zeros((5, 3)), np.zeros((3, 4)))


# ---- the reference's householder_qr scenarios (pkg/tests/test_core.py: TestHouseholderQR) ----
from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

from common import ALL_DTYPES, random_matrix  # noqa: E402


@pytest.mark.parametrize("dt", ALL_DTYPES)
@pytest.mark.parametrize("shape", [(6, 6), (10, 4), (600, 16)])
def test_householder_factorization_all_dtypes(dt, shape):  # test_core.py:116-132
    m, n = shape
    a = random_matrix(m, n, dt, seed=m + n)
    q, r = bs.householder_qr(a)
    u = unit_roundoff(dt)
    one = lambda x: float(np.abs(x).sum(axis=0).max())  # noqa: E731
    assert q.shape == (m, n) and r.shape == (n, n)
    assert np.allclose(q @ r, a, atol=50 * u * one(a))
    assert one(np.eye(n) - q.conj().T @ q) < 50 * n * u
    assert np.allclose(np.tril(r, -1), 0.0)
    d = np.diag(r)
    assert np.all(np.real(d) >= 0)
    if np.iscomplexobj(a):
        assert np.max(np.abs(np.imag(d))) < 10 * u * one(a)


@settings(max_examples=40, deadline=None)
@given(m=st.integers(1, 30), n=st.integers(1, 30), seed=st.integers(0, 2 ** 16))
def test_householder_property_reconstruction(m, n, seed):  # test_core.py:137-149
    if m < n:
        m, n = n, m
    a = random_matrix(m, n, np.float64, seed=seed)
    q, r = bs.householder_qr(a)
    u = 2.0 ** -53
    assert np.linalg.norm(a - q @ r) <= 100 * m * u * max(np.linalg.norm(a), 1e-300)
    assert np.linalg.norm(np.eye(n) - q.T @ q) <= 100 * m * u
