"""The reference's own svd-level test scenarios (pkg/tests/test_svd.py: TestUnblocked, TestBlocked,
TestDispatchAndQR) replayed on the GPU path: same inputs and assertions where the reference states exact
outcomes, and the oracle (the CPU restatement of the reference algorithm) as the sigma reference where
it states tolerances (c n u sigma_1)."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2601_17979_b200 as bs
from common import Opts, check_factors, check_sigma_parity, random_matrix, unit_roundoff
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ALL = [np.float32, np.float64, np.complex64, np.complex128]


def _fact(a, r, k=30.0):
    check_factors(a, r.u, r.sigma, r.v, k=k)


def test_triangular_two_by_two():  # test_svd.py:162-168
    a = np.asfortranarray([[3.0, 4.0], [0.0, 5.0]])
    r = bs.svd_unblocked(a)
    assert np.allclose(r.sigma, [np.sqrt(45.0), np.sqrt(5.0)], rtol=1e-14)
    _fact(a, r)
    assert r.info.converged and r.info.path == "unblocked"


def test_identity_converges_in_one_sweep():  # test_svd.py:170-175
    r = bs.svd_unblocked(np.asfortranarray(np.eye(4)))
    assert r.info.outer_sweeps == 1 and r.info.inner_rotations == 0
    assert np.array_equal(r.sigma, np.ones(4))


@pytest.mark.parametrize("dt", ALL)
def test_unblocked_random_all_dtypes(dt):  # test_svd.py:177-183
    a = random_matrix(20, 12, dt, seed=21)
    r = bs.svd_unblocked(a)
    _fact(a, r)
    _, s_ref, _, _ = O.solve(a, None, "unblocked")
    check_sigma_parity(r.sigma, s_ref, 12, unit_roundoff(dt))


def test_no_right_vectors_and_input_not_mutated():  # test_svd.py:185-196
    a = random_matrix(10, 6, seed=23)
    keep = a.copy()
    r = bs.svd_unblocked(a, bs.JacobiOptions(compute_right_vectors=False))
    assert r.v is None and np.array_equal(a, keep)
    _fact(a, r)


@pytest.mark.parametrize("dt", ALL)
def test_blocked_matches_unblocked(dt):  # test_svd.py:199-207
    a = random_matrix(48, 48, dt, seed=31)
    u = unit_roundoff(dt)
    rb = bs.svd_blocked(a, bs.JacobiOptions(nb=8))
    ru = bs.svd_unblocked(a)
    _fact(a, rb)
    assert np.max(np.abs(rb.sigma.astype(np.float64) - ru.sigma)) <= 60 * u * float(ru.sigma[0])


def test_nb_larger_than_n_degenerates_to_single_block():  # test_svd.py:209-213
    r = bs.svd_blocked(np.asfortranarray(np.diag([2.0, 1.0])), bs.JacobiOptions(nb=16))
    assert np.array_equal(r.sigma, [2.0, 1.0]) and r.info.converged


@pytest.mark.parametrize("n,nb", [(24, 8), (20, 8), (48, 16), (40, 16)])
def test_odd_and_uneven_block_counts(n, nb):  # test_svd.py:215-223 (3 blocks with a phantom; 8, 8, 4)
    a = random_matrix(n, n, seed=32 + n)
    r = bs.svd_blocked(a, bs.JacobiOptions(nb=nb))
    _fact(a, r)
    _, s_ref, _, info = O.solve(a, Opts(nb=nb), "blocked")
    check_sigma_parity(r.sigma, s_ref, n, 2.0 ** -53)
    assert abs(r.info.outer_sweeps - info["outer_sweeps"]) <= 1


def test_fused_and_twostage_agree_and_inner_budget_zero():  # test_svd.py:225-240
    a = random_matrix(40, 40, seed=34)
    u = 2.0 ** -53
    r1 = bs.svd_blocked(a, bs.JacobiOptions(nb=8, fused_updates=True))
    r2 = bs.svd_blocked(a, bs.JacobiOptions(nb=8, fused_updates=False))
    assert np.max(np.abs(r1.sigma - r2.sigma)) <= 30 * u * float(r2.sigma[0])
    b = random_matrix(32, 32, seed=35)
    r0 = bs.svd_blocked(b, bs.JacobiOptions(nb=8, inner_sweeps=0))
    rr = bs.svd_blocked(b, bs.JacobiOptions(nb=8, inner_sweeps=1))
    _fact(b, r0)
    _fact(b, rr)
    assert np.max(np.abs(r0.sigma - rr.sigma)) <= 30 * u * float(r0.sigma[0])


def test_blocked_counters_populated():  # test_svd.py:242-250
    r = bs.svd_blocked(random_matrix(40, 40, seed=36), bs.JacobiOptions(nb=8))
    c = r.info.counters
    assert c is not None and c.gram_calls > 0 and c.eig_calls > 0 and c.update_calls > 0
    assert c.gram_calls == c.eig_calls and r.info.outer_sweeps >= 1


def test_path_selection():  # test_svd.py:253-260
    assert bs.svd_dispatch(random_matrix(16, 16)).info.path == "unblocked"
    assert bs.svd_dispatch(random_matrix(64, 64)).info.path == "blocked"
    opts = bs.JacobiOptions(use_qr_preprocess=True)
    assert bs.svd_dispatch(random_matrix(600, 16), opts).info.path == "qr+unblocked"
    assert bs.svd_dispatch(random_matrix(300, 90), opts).info.path == "qr+blocked"
    assert bs.svd_dispatch(random_matrix(80, 40), opts).info.path == "blocked"


def test_wide_inputs_transposed():  # test_svd.py:262-274
    a = random_matrix(2, 5, seed=41)
    r = bs.svd_dispatch(a)
    assert r.info.path.startswith("transpose+") and r.u.shape == (2, 2) and r.v.shape == (5, 2)
    _fact(a, r)
    b = random_matrix(3, 7, seed=42)
    r2 = bs.svd_dispatch(b, bs.JacobiOptions(compute_right_vectors=False))
    assert r2.v is None and r2.u.shape == (3, 3)
    _fact(b, r2)


def test_qr_path_matches_direct_and_single_column():  # test_svd.py:276-288
    a = random_matrix(200, 12, seed=43)
    rq = bs.svd_qr_preprocessed(a)
    rd = bs.svd_unblocked(a)
    assert np.max(np.abs(rq.sigma - rd.sigma)) <= 30 * 2.0 ** -53 * float(rd.sigma[0])
    _fact(a, rq)
    r1 = bs.svd_qr_preprocessed(np.asfortranarray([[3.0], [4.0]]))
    assert r1.sigma[0] == pytest.approx(5.0) and np.allclose(np.abs(r1.u[:, 0]), [0.6, 0.8])


def test_empty_tiny_and_rejected_inputs():  # test_svd.py:290-309
    r = bs.svd_dispatch(np.zeros((0, 0), order="F"))
    assert r.sigma.shape == (0,) and r.info.path == "empty"
    assert bs.svd_dispatch(np.asfortranarray([[2.0]])).sigma[0] == 2.0
    with pytest.raises(bs.DomainError):
        bs.svd_dispatch(np.zeros((3, 3), dtype=np.int64, order="F"))
    a = random_matrix(2, 5)
    for f in (bs.svd_unblocked, bs.svd_blocked, bs.svd_qr_preprocessed):
        with pytest.raises(bs.ShapeError):
            f(a)


@settings(max_examples=25, deadline=None)
@given(m=st.integers(1, 40), n=st.integers(1, 40), seed=st.integers(0, 2 ** 16))
def test_property_dispatch_factorizes(m, n, seed):  # test_svd.py:311-325
    a = random_matrix(m, n, np.float64, seed=seed)
    r = bs.svd_dispatch(a)
    check_factors(a, r.u, r.sigma, r.v, k=80.0)
    ref = np.linalg.svd(a, compute_uv=False)
    mn = min(m, n)
    tol = 80 * max(m, n) * 2.0 ** -53 * max(float(ref[0]) if mn else 1.0, 1.0)
    assert np.allclose(r.sigma, ref[:mn], atol=tol)
