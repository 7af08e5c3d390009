"""GPU tests of the "qr+" route (householder_qr, src/core.py:118-168; src/svd.py:364-371, :529-530):
batched Householder QR on the device, Jacobi on R, U = Q diag(p) U_R.  Mirrors the reference's
tests/test_svd.py:250-262 (path selection) and tests/test_acceptance.py:284-293 (c07 QR equivalence)."""

import numpy as np
import pytest

import paper_2601_17979_b200 as bs
from common import ALL_DTYPES, Opts, check_factors, check_sigma_parity, random_matrix, unit_roundoff
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_qr_path_selection():
    opts = bs.JacobiOptions(use_qr_preprocess=True)
    assert bs.svd_dispatch(random_matrix(600, 16), opts).info.path == "qr+unblocked"
    assert bs.svd_dispatch(random_matrix(300, 90), opts).info.path == "qr+blocked"
    assert bs.svd_dispatch(random_matrix(80, 40), opts).info.path == "blocked"  # under the 3x ratio
    assert bs.svd_dispatch(random_matrix(600, 16)).info.path == "unblocked"  # option off
    assert bs.svd_qr_preprocessed(random_matrix(40, 30)).info.path == "qr+unblocked"  # forced: any ratio
    with pytest.raises(bs.ShapeError):
        bs.svd_qr_preprocessed(random_matrix(3, 5))


def test_c07_qr_path_equivalence():
    # tests/test_acceptance.py:284-293: the QR route agrees with the unblocked solver within 30 u sigma_1
    u = 2.0 ** -53
    for s in range(6):
        rng = np.random.default_rng(7000 + s)
        a = np.asfortranarray(rng.random((512, 16)))
        rq = bs.svd_qr_preprocessed(a)
        rd = bs.svd_unblocked(a)
        check_factors(a, rq.u, rq.sigma, rq.v)
        assert float(np.max(np.abs(rq.sigma - rd.sigma))) <= 30.0 * u * float(rd.sigma[0])
        _, s_ref, _, _ = O.solve(a, None, "unblocked")
        check_sigma_parity(rq.sigma, s_ref, min(a.shape), u)


@pytest.mark.parametrize("dt", ALL_DTYPES)
@pytest.mark.parametrize("shape,want_v", [((96, 20), True), ((256, 32), True), ((120, 36), False), ((20, 70), True)])
def test_qr_route_all_dtypes(dt, shape, want_v):
    m, n = shape
    opts = bs.JacobiOptions(use_qr_preprocess=True, compute_right_vectors=want_v)
    mats = [random_matrix(m, n, dt, seed=4100 + b + m) for b in range(3)]
    st = bs.BatchState.for_batch(len(mats))
    res = bs.batch_svd(mats, opts, st)
    uu = unit_roundoff(dt)
    k = min(m, n)
    for a, r in zip(mats, res):
        assert r is not None
        bm, bn = max(m, n), min(m, n)
        mode = "unblocked" if bn <= 32 else "blocked"
        assert r.info.path == ("transpose+" if m < n else "") + "qr+" + mode
        assert r.info.converged and r.u.shape == (m, k) and r.sigma.shape == (k,)
        _, s_ref, _, _ = O.solve(a, None, None)  # dispatch without QR: same singular values
        check_sigma_parity(r.sigma, s_ref, min(bm, bn), uu)
        if want_v:
            assert r.v.shape == (n, k)
            check_factors(a, r.u, r.sigma, r.v)
        else:
            assert r.v is None
            # U orthonormal and U^H A = diag(sigma) V^H has row norms sigma
            assert np.linalg.norm(r.u.conj().T @ r.u - np.eye(k)) < 50 * bm * uu
            assert np.allclose(np.linalg.norm(r.u.conj().T @ a, axis=1), r.sigma, rtol=0,
                               atol=100 * bm * uu * float(r.sigma[0]))


def test_qr_rank_deficient_and_zero_columns():
    a = random_matrix(200, 12, seed=77)
    a[:, 3] = 0.0
    a[:, 7] = a[:, 2]
    r = bs.svd_qr_preprocessed(a)
    check_factors(a, r.u, r.sigma, r.v)
    assert r.sigma[-1] < 1e-13 * r.sigma[0] and r.sigma[-2] < 1e-13 * r.sigma[0]
