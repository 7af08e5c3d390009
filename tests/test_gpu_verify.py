"""GPU tests of the on-device accuracy metrics (bsvd_verify_batched; the reference's verify.py:44-190)
against the host restatement in tests/common.py on the same factors, plus a full-size C1 batch."""

import numpy as np
import pytest

import paper_2601_17979_b200 as bs
from common import ALL_DTYPES, e1, e2, e3, random_matrix, unit_roundoff

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dt", ALL_DTYPES)
@pytest.mark.parametrize("shape", [(8, 8), (20, 12), (12, 20), (64, 64), (96, 20)])
def test_device_metrics_match_host(dt, shape):
    m, n = shape
    a = random_matrix(m, n, dt, seed=300 + m + n)
    r = bs.svd_dispatch(a)
    rep = bs.error_report(a, r, sigma_ref=np.asarray(r.sigma, dtype=np.float64) * (1 + 1e-3))
    u = unit_roundoff(dt)
    # host metrics in the working precision vs device metrics in float64: agree to a few u
    assert abs(rep.e1 - e1(a, r.u, r.sigma, r.v)) <= 4 * u
    assert abs(rep.e2 - e2(r.u)) <= 4 * u
    assert abs(rep.e3 - e3(r.v)) <= 4 * u
    assert rep.e4 == pytest.approx(np.linalg.norm(r.sigma.astype(np.float64) * 1e-3) / min(m, n), rel=1e-6)
    assert rep.passes[:3] == (True, True, True) and not rep.passes[3]
    assert rep.threshold == 30 * u


def test_detects_corrupted_factors():
    a = random_matrix(16, 16, seed=4)
    r = bs.svd_dispatch(a)
    u_bad = r.u.copy()
    u_bad[:, 0] *= 1.0 + 1e-10
    bad = bs.SvdResult(u=u_bad, sigma=r.sigma, v=r.v, info=r.info)
    rep = bs.error_report(a, bad)
    assert not rep.passes[0] and not rep.passes[1] and rep.passes[2]


def test_full_batch_on_device():
    import torch

    from paper_2601_17979_b200.matgen import gen_batch_device

    a = gen_batch_device("arith", 32, 32, 10000, np.float64, kappa=1e10, seed=3)
    res = bs.solve_tensor(a, 32, 32, bs.JacobiOptions())
    met = bs.verify_tensor(a, 32, 32, res).cpu().numpy()
    u = 2.0 ** -53
    assert np.isnan(met[:, 3]).all()
    assert met[:, :3].max() < 30 * u, met[:, :3].max(axis=0) / u


# ---- the reference's metric scenarios (pkg/tests/test_verify.py: TestThreshold, TestMetrics) ----
from common import random_matrix  # noqa: E402


def test_threshold_values():  # test_verify.py:26-31
    assert bs.threshold(np.float32) == pytest.approx(30 * 2.0 ** -24)
    assert bs.threshold(np.float64) == pytest.approx(30 * 2.0 ** -53)
    assert bs.threshold(np.complex64) == bs.threshold(np.float32)
    assert bs.threshold(np.complex128, k=100.0) == pytest.approx(100 * 2.0 ** -53)


def test_exact_factorization_scores_zero():  # test_verify.py:34-39
    a = np.asfortranarray(np.diag([3.0, 2.0]))
    r = bs.svd_dispatch(a)
    assert bs.residual_e1(a, r) == 0.0
    e2, e3 = bs.orthogonality_e2_e3(r)
    assert e2 == 0.0 and e3 == 0.0


def test_e1_detects_wrong_factors_and_requires_v():  # test_verify.py:41-51
    a = random_matrix(8, 8, seed=60)
    r = bs.svd_dispatch(a)
    wrong = bs.SvdResult(u=r.u, sigma=r.sigma * 2.0, v=r.v, info=r.info)
    assert bs.residual_e1(a, wrong) > 0.01
    b = random_matrix(8, 8, seed=61)
    with pytest.raises(bs.DomainError):
        bs.residual_e1(b, bs.svd_dispatch(b, bs.JacobiOptions(compute_right_vectors=False)))


def test_e4_normalizes_by_min_dim():  # test_verify.py:53-57
    assert bs.sigma_error_e4(np.array([3.0, 0.0]), np.array([0.0, 0.0]), 4, 2) == pytest.approx(1.5)
    with pytest.raises(bs.ShapeError):
        bs.sigma_error_e4(np.ones(3), np.ones(2), 3, 3)


@pytest.mark.parametrize("dt", [np.float32, np.float64, np.complex64, np.complex128])
def test_report_passes_on_good_solves(dt):  # test_verify.py:59-66 (arith spectrum, kappa 1e2)
    from paper_2601_17979_b200.matgen import gen_batch_device

    a = gen_batch_device("arith", 24, 24, 1, dt, kappa=1e2, seed=62)[0].cpu().numpy().T.copy(order="F")
    r = bs.svd_dispatch(a)
    sref = bs.make_sigma("arith", 24, 1e2)
    rep = bs.error_report(a, r, sigma_ref=sref)
    assert rep.all_pass and rep.threshold == pytest.approx(bs.threshold(dt)) and len(rep.passes) == 4


def test_report_thresholds_and_missing_reference():  # test_verify.py:68-87
    a = random_matrix(8, 8, seed=63)
    r = bs.svd_dispatch(a)
    assert bs.error_report(a, r, e3_threshold=100 * 2.0 ** -53).e3_threshold == pytest.approx(100 * 2.0 ** -53)
    rep = bs.error_report(a, r)
    assert rep.e4 is None and rep.all_pass
    bad = bs.error_report(a, r, sigma_ref=np.linspace(5, 1, 8))
    assert not bad.passes[3] and not bad.all_pass
