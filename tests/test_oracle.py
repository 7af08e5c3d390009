"""Pin the CPU restatement (oracle/) against the reference's golden vectors.

CPU-only.  The unblocked path and the kernel-level routines must match the
reference bit for bit; the blocked path differs only through the BLAS Gram
(src/svd.py:170-174 uses numpy/OpenBLAS), so it is held to the parity
tolerance and the reference's accuracy thresholds.
"""

import numpy as np
import pytest

from common import ALL_DTYPES, REAL_OF, Opts, check_factors, check_sigma_parity, unit_roundoff
from oracle import oracle as O


def _solve_case(golden, cid):
    c = golden.cases[cid]
    a = golden.get(cid, "a")
    opts = Opts(**c["opts"])
    u, s, v, info = O.solve(a, opts, c["force"])
    return c, a, u, s, v, info


def _unblocked_bitwise(c):
    # the unblocked path is bitwise except where finalize's zero-column completion
    # calls BLAS (np.vdot / np.linalg.norm, src/svd.py:224-240)
    # the qr+ route runs numpy/BLAS Householder QR first (src/core.py:118-168): tolerance only
    return (c["path"].endswith("unblocked") and "qr+" not in c["path"]
            and c["id"] not in ("ka_zerocol", "ka_zero4"))


def test_golden_cases_unblocked_bitwise(golden):
    n_bit = 0
    for cid, c in golden.cases.items():
        if not _unblocked_bitwise(c):
            continue
        c, a, u, s, v, info = _solve_case(golden, cid)
        assert info["path"] == c["path"], cid
        assert np.array_equal(u, golden.get(cid, "u")), cid
        assert np.array_equal(s, golden.get(cid, "s")), cid
        if c["has_v"]:
            assert np.array_equal(v, golden.get(cid, "v")), cid
        assert info["outer_sweeps"] == c["outer_sweeps"], cid
        assert info["inner_rotations"] == c["inner_rotations"], cid
        assert info["converged"] == c["converged"], cid
        n_bit += 1
    assert n_bit >= 40


def test_golden_cases_blocked_tolerance(golden):
    n = 0
    for cid, c in golden.cases.items():
        if _unblocked_bitwise(c):
            continue
        c, a, u, s, v, info = _solve_case(golden, cid)
        assert info["path"] == c["path"], cid
        assert info["converged"] == c["converged"], cid
        assert abs(info["outer_sweeps"] - c["outer_sweeps"]) <= 1, cid
        uu = unit_roundoff(a.dtype)
        s_ref = golden.get(cid, "s")
        check_sigma_parity(s, s_ref, min(a.shape), uu)
        if a.size:
            e3k = 100.0 if cid.startswith("c3_") else None
            check_factors(a, u, s, v if c["has_v"] else None, e3_k=e3k)
        n += 1
    assert n >= 20


@pytest.mark.parametrize("dt", ALL_DTYPES)
def test_kernel_onesided_bitwise(golden, dt):
    nm = np.dtype(dt).name
    kid = f"k_os_{nm}"
    a = np.asfortranarray(golden.get(kid, "a0").copy())
    v = np.asfortranarray(golden.get(kid, "v0").copy())
    sw, rot, cv = O.onesided_sweeps(a, v, golden.kernels[kid]["tol"], 1)
    assert rot == golden.kernels[kid]["rotations"]
    assert np.array_equal(a, golden.get(kid, "a1"))
    assert np.array_equal(v, golden.get(kid, "v1"))


@pytest.mark.parametrize("dt", ALL_DTYPES)
def test_kernel_eig_delta_bitwise(golden, dt):
    nm = np.dtype(dt).name
    kid = f"k_eig_{nm}"
    g = np.asfortranarray(golden.get(kid, "g0").copy())
    d = golden.get(kid, "d0").copy()
    mm = np.zeros(g.shape, dtype=g.dtype, order="F")
    sw, rot, cv = O.eig_sweeps(g, d, mm, golden.kernels[kid]["tol"], 1, delta=True)
    assert rot == golden.kernels[kid]["rotations"]
    assert np.array_equal(g, golden.get(kid, "g1"))
    assert np.array_equal(d, golden.get(kid, "d1"))
    assert np.array_equal(mm, golden.get(kid, "m1"))


@pytest.mark.parametrize("dt", ALL_DTYPES)
def test_kernel_fused_update_bitwise(golden, dt):
    nm = np.dtype(dt).name
    kid = f"k_fu_{nm}"
    bi = np.asfortranarray(golden.get(kid, "bi0").copy())
    bj = np.asfortranarray(golden.get(kid, "bj0").copy())
    O.fused_pair_update(bi, bj, golden.get(kid, "j"), 16, delta=True)
    assert np.array_equal(bi, golden.get(kid, "bi1"))
    assert np.array_equal(bj, golden.get(kid, "bj1"))


@pytest.mark.parametrize("ell", [2, 3, 4, 5, 7, 8, 9, 16, 31, 32])
def test_schedule_matches_reference(golden, ell):
    pairs, starts = O.schedule(ell)
    assert np.array_equal(pairs, golden.get(f"sched_{ell}", "pairs"))
    assert np.array_equal(starts, golden.get(f"sched_{ell}", "starts"))


def test_oracle_batch_equals_standalone(golden):
    # F8: batch == standalone (bitwise), here through the threaded batch entry
    rng = np.random.default_rng(3)
    a3 = rng.random((9, 12, 10))
    U, S, V, infos = O.solve_batch(a3, Opts(), nthreads=3)
    for b in range(9):
        u, s, v, info = O.solve(a3[b], Opts())
        assert np.array_equal(U[b], u) and np.array_equal(S[b], s) and np.array_equal(V[b], v)
        assert infos[b] == info


def _oracle_heev(g, k=30.0, max_sweeps=30):
    """jacobi_hermitian_eig (src/eig.py:90-148) through the oracle's eig_sweeps (non-delta)."""
    n = g.shape[0]
    d = np.ascontiguousarray(np.real(np.diag(g)), dtype=np.dtype(REAL_OF[np.dtype(g.dtype)]))
    w = np.triu(g, 1)
    w = np.asfortranarray(w + w.conj().T)
    m = np.asfortranarray(np.eye(n, dtype=g.dtype))
    sw, rot, cv = O.eig_sweeps(w, d, m, k * unit_roundoff(g.dtype), max_sweeps, delta=False)
    return d, m, sw, rot, cv


def test_golden_hermitian_eig(golden):
    # the eigensolver's arithmetic is the eig_sweeps kernel the oracle restates bitwise
    assert len(golden.eig) >= 9
    for eid, e in golden.eig.items():
        g = golden.get(eid, "g")
        d, m, sw, rot, cv = _oracle_heev(g)
        assert (sw, rot, cv) == (e["sweeps_run"], e["rotations"], e["converged"]), eid
        assert np.array_equal(d, golden.get(eid, "d")), eid
        assert np.array_equal(m, golden.get(eid, "m")), eid
