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
