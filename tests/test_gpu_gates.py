"""The reference's release gates replayed on the GPU, and full-batch checks at BASELINE sizes.

* c01 -- the accuracy protocol over every spectrum family x dtype x n in {8, 16, 32, 64, 96}, 20 problems
  each, design4 options (/root/reference/pkg/tests/test_acceptance.py:63-93): e1, e2, e3 < 30u (e3 < 100u
  for double logrand / geo), e4 < 30u against the prescribed spectrum (make_sigma, src/matgen.py:52-84) or,
  for the random family, against the reference's verification oracle (oracle_svd, src/verify.py:90-123:
  the unblocked solver in double at k = 1, 100 sweeps -- here its CPU restatement, oracle/).
  The inputs follow gen_matrix's recipe (src/matgen.py:96-122: uniform [0,1) entries for random,
  A = U diag(sigma) V^H from QR of standard normals in double, cast last) with numpy's QR for the
  orthonormal factors, so they realise the same spectra but are not bit-identical to gen_batch.
* c02 -- the paper's section 6.1 8x8 nb = 2 worked example (:96-138) through the GPU operators.
* the delta-mode fused_pair_update against the reference's own kernel-level golden case.
* C3a / C3b / C4 / C5 at their BASELINE batch sizes: e1-e3 on every problem (device verify), e4 on every
  problem where a spectrum is prescribed, sigma against the CPU restatement on a >= 1 % sample.
"""

import numpy as np
import pytest

import paper_2601_17979_b200 as bs
from common import Opts, check_sigma_parity, unit_roundoff
from oracle import oracle as O

pytestmark = pytest.mark.gpu

FAMILIES = ("random", "arith", "cluster0", "cluster1", "logrand", "geo")
DTYPES = (np.float32, np.float64, np.complex64, np.complex128)


def _design4():
    return bs.JacobiOptions(inner_sweeps=1, fused_updates=True, masking=True)


def _gen(fam, n, count, dt, kappa, seed0=0):
    """count n x n problems of family fam (gen_matrix's recipe, numpy QR for the factors)."""
    cplx = np.dtype(dt).kind == "c"
    out, sig = [], []
    for i in range(count):
        seed = seed0 + i
        rng = np.random.default_rng([seed, 4242, n])
        if fam == "random":
            a = rng.random((n, n))
            if cplx:
                a = a + 1j * rng.random((n, n))
            out.append(np.asfortranarray(a.astype(dt)))
            sig.append(None)
            continue
        s = bs.make_sigma(fam, n, kappa, seed=seed)

        def orth():
            z = rng.standard_normal((n, n))
            if cplx:
                z = z + 1j * rng.standard_normal((n, n))
            q, r = np.linalg.qr(z)
            return q * (np.diag(r) / np.abs(np.diag(r)))  # Haar-distributed

        u, v = orth(), orth()
        out.append(np.asfortranarray(((u * s) @ v.conj().T).astype(dt)))
        sig.append(s)
    return out, sig


def _oracle_sigma(a):
    """oracle_svd (src/verify.py:90-123): unblocked, double precision, k = 1, 100 sweeps."""
    wide = np.complex128 if np.iscomplexobj(a) else np.float64
    _, s, _, _ = O.solve(np.asfortranarray(a, dtype=wide), Opts(k=1.0, max_nsweeps=100), "unblocked")
    return s


@pytest.mark.parametrize("dt", DTYPES)
@pytest.mark.parametrize("fam", FAMILIES)
def test_c01_accuracy_protocol(fam, dt):
    single = np.dtype(dt) in (np.dtype(np.float32), np.dtype(np.complex64))
    kappa = 1e5 if single else 1e10
    e3_lim = 100.0 * unit_roundoff(dt) if (not single and fam in ("logrand", "geo")) else None
    failures = []
    for n in (8, 16, 32, 64, 96):
        mats, sig = _gen(fam, n, 20, dt, kappa)
        res = bs.batch_svd(mats, _design4())
        for i, (a, r) in enumerate(zip(mats, res)):
            sref = _oracle_sigma(a) if fam == "random" else sig[i]
            rep = bs.error_report(a, r, sigma_ref=sref, e3_threshold=e3_lim)
            if not (rep.all_pass and r.info.converged):
                failures.append((n, i, rep.e1, rep.e2, rep.e3, rep.e4, r.info.converged))
    assert not failures, f"{len(failures)} out of bounds, first: {failures[0]}"


def test_c02_fixed_example_reproduction():
    """Paper section 6.1: the 8x8 nb = 2 example, values quoted to 4 decimals (hence 5e-3)."""
    a = np.asfortranarray(np.array([
        [0.1206, 0.7675, 0.3103, 0.3527, 0.7382, 0.7008, 0.6985, 0.6836],
        [0.6438, 0.8468, 0.4922, 0.1086, 0.8833, 0.9463, 0.4762, 0.0463],
        [0.0623, 0.1681, 0.0378, 0.8734, 0.3093, 0.4652, 0.1508, 0.0702],
        [0.4903, 0.4045, 0.6989, 0.9629, 0.4463, 0.3890, 0.5055, 0.4994],
        [0.3061, 0.3025, 0.1704, 0.5332, 0.0403, 0.4388, 0.8133, 0.2996],
        [0.8164, 0.7730, 0.4167, 0.4056, 0.9273, 0.3014, 0.1878, 0.6929],
        [0.9972, 0.3156, 0.1199, 0.8503, 0.7538, 0.8448, 0.3805, 0.0510],
        [0.4246, 0.8355, 0.2274, 0.1604, 0.5861, 0.0802, 0.5890, 0.6763],
    ]))
    ref_first = np.array([0.4876, 7.7671, 0.1913, 1.2676])
    ref_second = np.array([[0.3739, -0.0001, -0.0108, -0.1912], [-0.0001, 7.7672, 0.1312, 0.4160],
                           [-0.0108, 0.1312, 0.1880, 0.0000], [-0.1912, 0.4160, 0.0000, 1.3463]])
    w = a.copy(order="F")

    def pair_step(bi, bj):
        g = bs.compute_gram(w[:, 2 * bi:2 * bi + 2], w[:, 2 * bj:2 * bj + 2])   # GPU operator
        d, vecs, _ = bs.jacobi_hermitian_eig(g)                                  # GPU eigensolver
        blk = np.hstack([w[:, 2 * bi:2 * bi + 2], w[:, 2 * bj:2 * bj + 2]])
        bi_, bj_ = np.asfortranarray(blk[:, :2]), np.asfortranarray(blk[:, 2:])
        bs.fused_pair_update(bi_, bj_, vecs)                                     # GPU update, [Bi Bj] @ J
        w[:, 2 * bi:2 * bi + 2] = bi_
        w[:, 2 * bj:2 * bj + 2] = bj_
        return d

    assert np.max(np.abs(pair_step(0, 1) - ref_first)) < 5e-3
    pair_step(2, 3)
    pair_step(0, 3)
    pair_step(1, 2)
    assert np.max(np.abs(bs.compute_gram(w[:, 0:2], w[:, 2:4]) - ref_second)) < 5e-3
    res = bs.svd_blocked(a, bs.JacobiOptions(nb=2, inner_sweeps=0))
    assert bs.error_report(a, res).all_pass and res.info.converged


@pytest.mark.parametrize("nm", ["float32", "float64", "complex64", "complex128"])
def test_fused_pair_update_delta_golden(golden, nm):
    """Delta mode ([Bi Bj] += [Bi Bj] Delta, src/_kernels_numba.py:141-175) against the reference's own
    kernel-level output (tests/golden/make_golden.py k_fu_*): same inputs, within a few ulps."""
    kid = f"k_fu_{nm}"
    bi = np.asfortranarray(golden.get(kid, "bi0").copy())
    bj = np.asfortranarray(golden.get(kid, "bj0").copy())
    jm = golden.get(kid, "j")
    bs.fused_pair_update(bi, bj, jm, row_block=16, delta=True)
    u = unit_roundoff(bi.dtype)
    ref = np.hstack([golden.get(kid, "bi1"), golden.get(kid, "bj1")])
    scale = np.abs(np.hstack([golden.get(kid, "bi0"), golden.get(kid, "bj0")])).max() * (1 + np.abs(jm).sum(0).max())
    assert np.max(np.abs(np.hstack([bi, bj]) - ref)) <= 8 * 8 * u * scale


_FULL = [  # BASELINE configs at their batch sizes (id, family, m, n, batch, dtype, kappa, rank, route)
    ("c3a", "geo", 64, 64, 10000, np.float64, 1e12, None, None),
    ("c3b", "rankdef", 64, 64, 10000, np.float64, 1e6, 48, None),
    ("c4", "random", 256, 32, 5000, np.complex128, 1.0, None, None),
    ("c4-blocked", "random", 256, 32, 5000, np.complex128, 1.0, None, "blocked"),
    ("c5", "random", 128, 128, 2000, np.float64, 1.0, None, None),
]


@pytest.mark.parametrize("cid,fam,m,n,B,dt,kappa,rank,route", _FULL, ids=[c[0] for c in _FULL])
def test_full_batch_baseline_configs(cid, fam, m, n, B, dt, kappa, rank, route):
    import torch

    from paper_2601_17979_b200 import _lib
    from paper_2601_17979_b200.matgen import gen_batch_device
    from paper_2601_17979_b200.solver import INFO_DTYPE

    a = gen_batch_device(fam, m, n, B, dt, kappa=kappa, seed=0, rank=rank)
    rt = _lib.FORCE_BLOCKED if route == "blocked" else _lib.DISPATCH
    res = bs.solve_tensor(a, m, n, bs.JacobiOptions(), route=rt)
    sref = None
    if fam != "random":
        sref = torch.as_tensor(bs.make_sigma(fam, n, kappa, rank=rank)).expand(B, n).contiguous().cuda()
    met = bs.verify_tensor(a, m, n, res, sigma_ref=sref).cpu().numpy()
    torch.cuda.synchronize()
    info = np.frombuffer(res.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    assert info["converged"].all() and (info["status"] == 0).all()
    u = unit_roundoff(dt)
    e3_lim = 100.0 if fam == "geo" else 30.0  # src/cli.py:209
    assert met[:, 0].max() < 30 * u and met[:, 1].max() < 30 * u and met[:, 2].max() < e3_lim * u
    if sref is not None:
        assert met[:, 3].max() < 30 * u  # e4 on every problem against the prescribed spectrum
    S = res.s.cpu().numpy()
    assert np.all(np.diff(S, axis=1) <= 0)
    A = np.swapaxes(a.cpu().numpy(), 1, 2)
    sample = np.arange(0, B, 100 if B >= 5000 else 50)  # 1 % (2 % for C5)
    _, S_ref, _, infos = O.solve_batch(A[sample], None, "blocked" if route == "blocked" else None, nthreads=0)
    for j, b in enumerate(sample):
        check_sigma_parity(S[b], S_ref[j], min(m, n), u)
    d = info["outer_sweeps"][sample].astype(np.int64) - np.array([i["outer_sweeps"] for i in infos])
    if kappa >= 1e6:
        # squared condition >= 1e12 on the blocked path: the sweep count is chaotic in the rounding; the
        # reference's own numba and numpy backends differ by -2..+3 on these inputs
        # (profiles/r2_sweep_spread.md), so the contract is the spread and the mean
        assert np.abs(d).max() <= 3 and abs(d.mean()) <= 0.25, (np.abs(d).max(), d.mean())
    else:
        assert np.abs(d).max() <= 1


# ---- acceptance c03, c06, c09 (/root/reference/pkg/tests/test_acceptance.py:141-331) ----
def _design(name):  # src/cli.py:46-58 design presets (cumulative variants)
    import dataclasses

    base = bs.JacobiOptions()
    return {"baseline": dataclasses.replace(base, inner_sweeps=0, fused_updates=False, masking=False),
            "design2": dataclasses.replace(base, inner_sweeps=1, fused_updates=False, masking=False),
            "design3": dataclasses.replace(base, inner_sweeps=1, fused_updates=True, masking=False),
            "design4": dataclasses.replace(base, inner_sweeps=1, fused_updates=True, masking=True)}[name]


def test_c03_design_variant_equivalence():
    """sigma of every design variant within 30u of the baseline; design4 == design3 bitwise (batched: the
    50 seeds of each n in one call per design)."""
    u = 2.0 ** -53
    for n in (16, 64, 128):
        mats = [np.asfortranarray(np.random.default_rng(9000 * n + s).random((n, n))) for s in range(50)]
        base = bs.batch_svd(mats, _design("baseline"))
        res = {name: bs.batch_svd(mats, _design(name)) for name in ("design2", "design3", "design4")}
        for name, rs in res.items():
            for b, r in zip(base, rs):
                assert float(np.max(np.abs(r.sigma - b.sigma))) < 30 * u * float(b.sigma[0]), (name, n)
        for r3, r4 in zip(res["design3"], res["design4"]):
            assert np.array_equal(r3.sigma, r4.sigma) and np.array_equal(r3.u, r4.u) and np.array_equal(r3.v, r4.v)


def test_c06_masked_batch_work_saving():
    rng = np.random.default_rng(606)
    probs = [np.asfortranarray(np.diag(rng.uniform(0.5, 2.0, 64))) for _ in range(8)] + \
            [np.asfortranarray(rng.random((64, 64))) for _ in range(8)]
    st3, st4 = bs.BatchState.for_batch(len(probs)), bs.BatchState.for_batch(len(probs))
    r3 = bs.batch_svd(probs, _design("design3"), st3)
    r4 = bs.batch_svd(probs, _design("design4"), st4)
    assert not st3.errors and not st4.errors
    assert st4.counters.masked_pair_skips > 0 and st4.counters.eig_calls < st3.counters.eig_calls
    for a3, a4 in zip(r3, r4):
        assert np.array_equal(a3.sigma, a4.sigma) and np.array_equal(a3.u, a4.u) and np.array_equal(a3.v, a4.v)


def test_c09_frobenius_mass_conservation():
    """sum sigma^2 equals ||A||_F^2 within 30u, at most 30 outer sweeps (logrand spectra and random)."""
    from paper_2601_17979_b200.matgen import gen_batch_device

    rng = np.random.default_rng(909)
    for n in (16, 64):
        for dt in (np.float32, np.complex128):
            a = gen_batch_device("logrand", n, n, 3, dt, kappa=1e3, seed=1).cpu().numpy()
            mats = [np.asfortranarray(x.T) for x in a]
            for m_, r in zip(mats, bs.batch_svd(mats, _design("design4"))):
                u = unit_roundoff(dt)
                fro2 = float(np.sum(np.abs(m_.astype(np.complex128)) ** 2))
                ssq = float(np.sum(np.asarray(r.sigma, dtype=np.float64) ** 2))
                assert r.info.outer_sweeps <= 30 and abs(ssq - fro2) < 30 * u * fro2
        mats = [np.asfortranarray(rng.random((n, n))) for _ in range(5)]
        for m_, r in zip(mats, bs.batch_svd(mats, _design("baseline"))):
            fro2 = float(np.sum(m_ ** 2))
            assert abs(float(np.sum(r.sigma ** 2)) - fro2) < 30 * 2.0 ** -53 * fro2


@pytest.mark.parametrize("m,n,dt,B,inner", [(32, 32, np.float64, 200, 1), (16, 16, np.float32, 200, 1),
                                            (64, 64, np.float64, 30, 1), (64, 64, np.float64, 30, 0),
                                            (128, 128, np.float64, 12, 1), (128, 128, np.float64, 8, 0),
                                            (256, 32, np.complex128, 30, 1), (128, 128, np.complex128, 8, 1)])
def test_c09_mass_and_sigma_every_family(m, n, dt, B, inner):
    """The c09 bar (sum sigma^2 = ||A||_F^2 within 30u) and sigma within 30u s1 of LAPACK on random batches of
    every kernel family, the large blocked shapes and the inner-budget-100 design included (the blocked
    kernels' delta mode; tools/mass_check.py)."""
    import torch

    rng = np.random.default_rng(m * 31 + n + inner)
    A = rng.random((B, m, n))
    if np.dtype(dt).kind == "c":
        A = A + 1j * rng.random((B, m, n))
    A = A.astype(dt)
    r = bs.solve_tensor(torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2))).cuda(), m, n,
                        bs.JacobiOptions(inner_sweeps=inner))
    torch.cuda.synchronize()
    S = r.s.cpu().numpy().astype(np.float64)
    u = unit_roundoff(dt)
    A64 = A.astype(np.complex128) if np.dtype(dt).kind == "c" else A.astype(np.float64)
    fro2 = np.sum(np.abs(A64) ** 2, axis=(1, 2))
    assert np.max(np.abs(np.sum(S ** 2, axis=1) - fro2) / (u * fro2)) < 30
    ref = np.stack([np.linalg.svd(x, compute_uv=False) for x in A64])
    assert np.max(np.max(np.abs(S - ref), axis=1) / (u * ref[:, 0])) < 30
