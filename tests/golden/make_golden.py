"""Generate golden vectors by running the REFERENCE package itself.

Run here (the reference is importable read-only in this container):

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py

It imports bsvd from /root/reference/pkg/src and writes
tests/golden/golden.npz (arrays) + tests/golden/golden.json (case metadata).
The GPU box has no /root/reference; the tests only read these committed files.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
import bsvd  # noqa: E402
import bsvd.cli  # noqa: E402
from bsvd.matgen import _random_orthonormal  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ALL = (np.float32, np.float64, np.complex64, np.complex128)


def random_matrix(m, n, dtype=np.float64, seed=0):
    # tests/conftest.py:10-16 of the reference
    rng = np.random.default_rng(seed)
    a = rng.random((m, n))
    if np.dtype(dtype).kind == "c":
        a = a + 1j * rng.random((m, n))
    return np.asarray(a, dtype=dtype, order="F")


def rank_deficient(n, rank, kappa, seed, dtype=np.float64):
    # BASELINE.md C3b construction: geo spectrum on the first `rank` values, zeros after
    i = np.arange(rank, dtype=np.float64)
    sig = np.concatenate([kappa ** (-i / (rank - 1)), np.zeros(n - rank)])
    rng = np.random.default_rng([seed, 2])
    cplx = np.dtype(dtype).kind == "c"
    u = _random_orthonormal(rng, n, n, cplx)
    v = _random_orthonormal(rng, n, n, cplx)
    return np.asfortranarray(((u * sig) @ v.conj().T).astype(dtype))


arrays: dict[str, np.ndarray] = {}
cases: list[dict] = []


def add_solve(cid, a, force=None, **kw):
    opts = bsvd.JacobiOptions(**kw)
    fn = {None: bsvd.svd_dispatch, "unblocked": bsvd.svd_unblocked, "blocked": bsvd.svd_blocked,
          "qr": bsvd.svd_qr_preprocessed}[force]
    r = fn(a, opts)
    arrays[f"{cid}__a"] = np.asarray(a)
    arrays[f"{cid}__u"] = r.u
    arrays[f"{cid}__s"] = r.sigma
    if r.v is not None:
        arrays[f"{cid}__v"] = r.v
    cases.append(dict(
        id=cid, kind="solve", force=force, opts=kw, dtype=np.dtype(a.dtype).name,
        shape=list(a.shape), has_v=r.v is not None,
        converged=bool(r.info.converged), outer_sweeps=int(r.info.outer_sweeps),
        inner_rotations=int(r.info.inner_rotations), path=r.info.path,
        gram_calls=int(r.info.counters.gram_calls), update_calls=int(r.info.counters.update_calls),
    ))


def main():
    # --- dispatch over dtypes and shapes (unblocked ≤ 32 columns) ---
    for dt in ALL:
        nm = np.dtype(dt).name
        for (m, n) in [(8, 8), (20, 12), (16, 16), (32, 32), (2, 5), (33, 31)]:
            add_solve(f"disp_{nm}_{m}x{n}", random_matrix(m, n, dt, seed=1000 + 37 * m + n))
        add_solve(f"novec_{nm}_3x7", random_matrix(3, 7, dt, seed=42), compute_right_vectors=False)
        add_solve(f"novec_{nm}_16x16", random_matrix(16, 16, dt, seed=43), compute_right_vectors=False)
        add_solve(f"blk_{nm}_48x48_nb8", random_matrix(48, 48, dt, seed=31), force="blocked", nb=8)
        add_solve(f"disp_{nm}_64x64", random_matrix(64, 64, dt, seed=64))
    # --- known answers (reference tests) ---
    add_solve("ka_tri2", np.asfortranarray([[3.0, 4.0], [0.0, 5.0]]), force="unblocked")
    add_solve("ka_eye4", np.asfortranarray(np.eye(4)), force="unblocked")
    add_solve("ka_diag3", np.asfortranarray(np.diag([1.0, 10.0, 100.0])))
    zc = np.zeros((3, 2), order="F")
    zc[0, 0] = 2.0
    add_solve("ka_zerocol", zc)
    add_solve("ka_zero4", np.zeros((4, 4), order="F"))
    add_solve("ka_one", np.asfortranarray([[2.0]]))
    add_solve("ka_col", np.asfortranarray([[3.0], [4.0]]))
    add_solve("ka_empty", np.zeros((0, 0), order="F"))
    add_solve("ka_diag8", np.asfortranarray(np.diag(np.arange(1.0, 9.0))))
    add_solve("ka_diaglin48", np.asfortranarray(np.diag(np.linspace(1.0, 0.25, 48))), nb=8)
    add_solve("ka_rank5_8", rank_deficient(8, 5, 1e3, 7))
    # --- BASELINE config shapes (small counts) ---
    for s in range(3):
        a = bsvd.gen_matrix(32, bsvd.SpectrumSpec("arith", 32, 1e10, s), np.float64)
        add_solve(f"c1_arith_{s}", a, **bsvd.cli.design_options("design4").__dict__)
        a = bsvd.gen_matrix(32, bsvd.SpectrumSpec("random", 32, 1.0, s), np.float64)
        add_solve(f"c1_random_{s}", a)
        a = bsvd.gen_matrix(16, bsvd.SpectrumSpec("random", 16, 1.0, s), np.float32)
        add_solve(f"c2_full_{s}", a)
        add_solve(f"c2_vals_{s}", a, compute_right_vectors=False)
    for s in range(2):
        a = bsvd.gen_matrix(64, bsvd.SpectrumSpec("geo", 64, 1e12, s), np.float64)
        add_solve(f"c3_geo_{s}", a)
    add_solve("c3_rank48_0", rank_deficient(64, 48, 1e6, 0))
    a = bsvd.gen_matrix(256, bsvd.SpectrumSpec("random", 32, 1.0, 0), np.complex128)
    add_solve("c4_disp_0", a)
    add_solve("c4_blk_0", a, force="blocked")
    a = bsvd.gen_matrix(128, bsvd.SpectrumSpec("random", 128, 1.0, 0), np.float64)
    add_solve("c5_0", a)
    # --- blocked variants (reference tests/test_svd.py:199-249) ---
    add_solve("blk_odd_24", random_matrix(24, 24, seed=32), force="blocked", nb=8)
    add_solve("blk_ragged_20", random_matrix(20, 20, seed=33), force="blocked", nb=8)
    add_solve("blk_fused_40", random_matrix(40, 40, seed=34), force="blocked", nb=8, fused_updates=True)
    add_solve("blk_twostage_40", random_matrix(40, 40, seed=34), force="blocked", nb=8, fused_updates=False)
    add_solve("blk_inner0_32", random_matrix(32, 32, seed=35), force="blocked", nb=8, inner_sweeps=0)
    add_solve("blk_single_2", np.asfortranarray(np.diag([2.0, 1.0])), force="blocked", nb=16)
    add_solve("blk_single_12", random_matrix(12, 10, seed=36), force="blocked", nb=16)
    add_solve("blk_tall_80x40", random_matrix(80, 40, seed=37))
    add_solve("blk_wide_40x96", random_matrix(40, 96, seed=38))
    add_solve("unb_k1_20", random_matrix(20, 20, seed=39), force="unblocked", k=1.0, max_nsweeps=100)
    add_solve("unb_cap_32", random_matrix(32, 32, seed=40), force="unblocked", max_nsweeps=3)
    # --- QR-preprocessed route (src/core.py:118-168, src/svd.py:364-371; tests/test_svd.py:250-262) ---
    add_solve("qr_f64_600x16", random_matrix(600, 16, seed=50), use_qr_preprocess=True)
    add_solve("qr_f64_300x90", random_matrix(300, 90, seed=51), use_qr_preprocess=True)
    add_solve("qr_c128_256x32", random_matrix(256, 32, np.complex128, seed=52), use_qr_preprocess=True)
    add_solve("qr_f32_96x20", random_matrix(96, 20, np.float32, seed=53), force="qr")
    add_solve("qr_c64_20x70", random_matrix(20, 70, np.complex64, seed=54), use_qr_preprocess=True)
    add_solve("qr_f64_512x16_c07", random_matrix(512, 16, seed=7000), force="qr")
    add_solve("qr_f64_40x30_forced", random_matrix(40, 30, seed=55), force="qr", compute_right_vectors=False)

    # --- kernel-level vectors (bitwise restatement checks) ---
    kern = []
    for dt in ALL:
        nm = np.dtype(dt).name
        a = random_matrix(16, 8, dt, seed=5)
        v = np.asfortranarray(np.eye(8, dtype=dt))
        arrays[f"k_os_{nm}__a0"] = a.copy(order="F")
        arrays[f"k_os_{nm}__v0"] = v.copy(order="F")
        pairs, starts = bsvd.schedule_arrays(8)
        tol = 30.0 * bsvd.unit_roundoff(dt)
        sw, rot, cv = bsvd.backend.active().onesided_sweeps(a, v, pairs, starts, tol, 1)
        arrays[f"k_os_{nm}__a1"] = a
        arrays[f"k_os_{nm}__v1"] = v
        kern.append(dict(id=f"k_os_{nm}", kind="onesided", dtype=nm, tol=tol, rotations=int(rot)))

        g = bsvd.compute_gram(random_matrix(20, 6, dt, seed=6), random_matrix(20, 6, dt, seed=7))
        d = np.ascontiguousarray(np.real(np.diag(g)), dtype=bsvd.real_dtype(dt))
        off = np.triu(g, 1)
        off = np.asfortranarray(off + off.conj().T)
        mm = np.zeros((12, 12), dtype=dt, order="F")
        arrays[f"k_eig_{nm}__g0"] = off.copy(order="F")
        arrays[f"k_eig_{nm}__d0"] = d.copy()
        pairs, starts = bsvd.schedule_arrays(12)
        sw, rot, cv = bsvd.backend.active().eig_sweeps(off, d, mm, pairs, starts, tol, 1, True)
        arrays[f"k_eig_{nm}__g1"] = off
        arrays[f"k_eig_{nm}__d1"] = d
        arrays[f"k_eig_{nm}__m1"] = mm
        kern.append(dict(id=f"k_eig_{nm}", kind="eig_delta", dtype=nm, tol=tol, rotations=int(rot)))

        bi = random_matrix(70, 5, dt, seed=8)
        bj = random_matrix(70, 3, dt, seed=9)
        jm = random_matrix(8, 8, dt, seed=10)
        arrays[f"k_fu_{nm}__bi0"] = bi.copy(order="F")
        arrays[f"k_fu_{nm}__bj0"] = bj.copy(order="F")
        arrays[f"k_fu_{nm}__j"] = jm
        bsvd.backend.active().fused_pair_update(bi, bj, jm, 16, True)
        arrays[f"k_fu_{nm}__bi1"] = bi
        arrays[f"k_fu_{nm}__bj1"] = bj
        kern.append(dict(id=f"k_fu_{nm}", kind="fused_delta", dtype=nm))

    # --- standalone Hermitian eigensolver (src/eig.py:90-148; tests/test_eig.py:88-160) ---
    eig = []
    for dt in ALL:
        nm = np.dtype(dt).name
        for n_, seed in ((12, 3), (33, 11)):
            rng = np.random.default_rng(seed)
            x = rng.random((n_, n_))
            if np.dtype(dt).kind == "c":
                x = x + 1j * rng.random((n_, n_))
            g = np.asfortranarray(((x + x.conj().T) / 2).astype(dt))
            d, m, inf = bsvd.jacobi_hermitian_eig(g)
            eid = f"eig_{nm}_{n_}"
            arrays[f"{eid}__g"] = g
            arrays[f"{eid}__d"] = d
            arrays[f"{eid}__m"] = m
            eig.append(dict(id=eid, dtype=nm, n=n_, sweeps_run=int(inf.sweeps_run), rotations=int(inf.rotations),
                            converged=bool(inf.converged)))
    g = np.asfortranarray([[9.0, 12.0], [12.0, 41.0]])
    d, m, inf = bsvd.jacobi_hermitian_eig(g)
    arrays["eig_ka2__g"], arrays["eig_ka2__d"], arrays["eig_ka2__m"] = g, d, m
    eig.append(dict(id="eig_ka2", dtype="float64", n=2, sweeps_run=int(inf.sweeps_run), rotations=int(inf.rotations),
                    converged=bool(inf.converged)))

    for ell in (2, 3, 4, 5, 7, 8, 9, 16, 31, 32):
        pairs, starts = bsvd.schedule_arrays(ell)
        arrays[f"sched_{ell}__pairs"] = np.asarray(pairs)
        arrays[f"sched_{ell}__starts"] = np.asarray(starts)
    rot = bsvd.compute_rotation(9.0, 41.0, 12.0)
    meta = dict(
        cases=cases,
        kernels=kern,
        eig=eig,
        rotation_9_41_12=dict(c=rot.c, s=rot.s, t=rot.t),
        generator="tests/golden/make_golden.py",
        reference="bsvd " + bsvd.__version__ + " (numba backend) from /root/reference/pkg/src",
        numpy=np.__version__,
    )
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"{len(cases)} solve cases, {len(kern)} kernel cases, {len(arrays)} arrays")


if __name__ == "__main__":
    main()
