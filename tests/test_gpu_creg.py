"""GPU parity of the complex FP64 register kernel (csrc/creg32.cu, kernel id 32): n = 32, m <= 256,
c128 -- BASELINE config C4 (256 x 32) on the reference's dispatch route (unblocked,
src/svd.py:375-381) and its blocked Gram route (ell = 2, src/svd.py:481-522), and the 32 x 32 R of the
QR route.  Same contract as tests/test_gpu_parity.py: sigma within 2 n u sigma_1 of the CPU
restatement, e1-e3 < 30u, converged, outer sweeps within 2, path strings and counters."""

import numpy as np
import pytest

import paper_2601_17979_b200 as bs
from common import Opts, check_factors, check_sigma_parity, random_matrix
from oracle import oracle as O

pytestmark = pytest.mark.gpu

U64 = 2.0 ** -53


ROUTE = {None: 0, "unblocked": 1, "blocked": 2}


def _solve(A, m, n, opts, route=None):
    import torch

    from paper_2601_17979_b200.solver import INFO_DTYPE

    a = torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2))).cuda()
    r = bs.solve_tensor(a, m, n, opts, route=ROUTE[route])
    torch.cuda.synchronize()
    info = np.frombuffer(r.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    U = np.swapaxes(r.u.cpu().numpy(), 1, 2)
    V = np.swapaxes(r.v.cpu().numpy(), 1, 2) if r.v is not None else None
    return U, r.s.cpu().numpy(), V, info


@pytest.mark.parametrize("m", [32, 33, 64, 100, 160, 256])
@pytest.mark.parametrize("route", [None, "blocked"])
def test_creg32_vs_oracle(m, route):
    B = 6
    A = np.stack([random_matrix(m, 32, np.complex128, seed=4000 + 7 * b + m) for b in range(B)])
    U, S, V, info = _solve(A, m, 32, bs.JacobiOptions(), route=route)
    assert (info["kernel"] == 32).all() and info["converged"].all()
    for b in range(B):
        _, s_ref, _, oi = O.solve(A[b], Opts(), route)
        check_sigma_parity(S[b], s_ref, 32, U64)
        check_factors(A[b], U[b], S[b], V[b])
        assert abs(int(info["outer_sweeps"][b]) - oi["outer_sweeps"]) <= 1
    if route == "blocked":
        assert (info["gram_calls"] == info["outer_sweeps"]).all() and (info["update_calls"] >= 1).all()
    else:
        assert (info["gram_calls"] == 0).all()


@pytest.mark.parametrize("route", [None, "blocked"])
def test_creg32_public_api_paths(route):
    a = random_matrix(256, 32, np.complex128, seed=77)
    fn = bs.svd_dispatch if route is None else bs.svd_blocked
    r = fn(a, bs.JacobiOptions())
    _, s_ref, _, oi = O.solve(a, Opts(), route)
    assert r.info.path == oi["path"] and r.info.converged
    check_sigma_parity(r.sigma, s_ref, 32, U64)
    check_factors(a, r.u, r.sigma, r.v)


def test_creg32_values_only_matches_full():
    A = np.stack([random_matrix(256, 32, np.complex128, seed=90 + b) for b in range(5)])
    _, S1, _, _ = _solve(A, 256, 32, bs.JacobiOptions())
    U0, S0, V0, info = _solve(A, 256, 32, bs.JacobiOptions(compute_right_vectors=False))
    assert V0 is None and (info["kernel"] == 32).all()
    assert np.array_equal(S0, S1)  # V is a passenger: the W iteration is the same bits
    for b in range(5):
        check_factors(A[b], U0[b], S0[b], None)


def test_creg32_rank_deficient_and_edge_inputs():
    B = 8
    A = np.stack([random_matrix(256, 32, np.complex128, seed=300 + b) for b in range(B)])
    A[1][:, 7] = 0.0                                   # zero column
    A[2] = 0.0                                         # zero matrix
    A[3] = A[3][:, :5] @ (np.random.default_rng(1).standard_normal((5, 32)) + 0j)  # rank 5
    A[4][:, 20] = 1j * A[4][:, 3]                      # dependent column (phase)
    A[5] = A[5] * 1e-60                                # small scale (g_ii g_jj stays normal, as the reference needs)
    A[6] = A[6] * 1e+60                                # large scale (g_ii g_jj stays finite, as the reference needs)
    A[7][:, 1::2] = 0.0                                # half the columns zero
    U, S, V, info = _solve(A, 256, 32, bs.JacobiOptions())
    assert info["converged"].all() and (info["status"] == 0).all()
    for b in range(B):
        _, s_ref, _, _ = O.solve(A[b], Opts(), None)
        check_sigma_parity(S[b], s_ref, 32, U64)
        check_factors(A[b], U[b], S[b], V[b])


def test_creg32_nonfinite_input_flagged():
    A = np.stack([random_matrix(64, 32, np.complex128, seed=5 + b) for b in range(3)])
    A[1][3, 4] = np.nan
    _, S, _, info = _solve(A, 64, 32, bs.JacobiOptions())
    assert info["status"][1] != 0 and info["status"][0] == 0 and info["status"][2] == 0
    assert np.isfinite(S[0]).all() and np.isfinite(S[2]).all()


def test_creg32_batch_equals_standalone_bitwise():
    """Batch == standalone (tests/test_batch.py:19-28): one CTA per problem, no cross-problem state."""
    A = np.stack([random_matrix(200, 32, np.complex128, seed=40 + b) for b in range(7)])
    U, S, V, _ = _solve(A, 200, 32, bs.JacobiOptions())
    for b in (0, 3, 6):
        U1, S1, V1, _ = _solve(A[b:b + 1], 200, 32, bs.JacobiOptions())
        assert np.array_equal(U1[0], U[b]) and np.array_equal(S1[0], S[b]) and np.array_equal(V1[0], V[b])


def test_qr_route_uses_creg32_for_r():
    a = random_matrix(256, 32, np.complex128, seed=11)
    r = bs.svd_qr_preprocessed(a, bs.JacobiOptions())
    assert r.info.path.startswith("qr+")
    _, s_ref, _, _ = O.solve(a, Opts(), None)
    check_sigma_parity(r.sigma, s_ref, 32, U64)
    check_factors(a, r.u, r.sigma, r.v)
    import ctypes

    from paper_2601_17979_b200 import _lib
    from paper_2601_17979_b200.solver import make_opts

    o = make_opts(bs.JacobiOptions(use_qr_preprocess=True))
    assert _lib.load().bsvd_select_kernel(3, 256, 32, ctypes.byref(o)) == 32


@pytest.mark.parametrize("m", [32, 100, 256])
@pytest.mark.parametrize("route", [None, "blocked"])
def test_creg32_tma_loader_bitwise(m, route):
    """Kernel (1) through bulk copies (cp.async.bulk into shared memory, KV_CREG32_TMA = 45) loads the
    same bits as the LDG loader: every output identical to the default kernel's."""
    import torch

    B = 5
    A = np.stack([random_matrix(m, 32, np.complex128, seed=4500 + 3 * b + m) for b in range(B)])
    a = torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2))).cuda()
    r0 = bs.solve_tensor(a, m, 32, bs.JacobiOptions(), route=ROUTE[route])
    r1 = bs.solve_tensor(a, m, 32, bs.JacobiOptions(), route=ROUTE[route], kernel=45)
    torch.cuda.synchronize()
    assert torch.equal(r0.u, r1.u) and torch.equal(r0.s, r1.s) and torch.equal(r0.v, r1.v)
    _, s_ref, _, _ = O.solve(A[0], Opts(), route)
    check_sigma_parity(r1.s[0].cpu().numpy(), s_ref, 32, U64)
