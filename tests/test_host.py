"""CPU-only tests of the host side: schedule closed form, options, the C-ABI
library (loads, exports every declared symbol), result metadata, and that the
product path refuses to run without a GPU (no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2601_17979_b200 as bs
from paper_2601_17979_b200 import _lib
from paper_2601_17979_b200.ordering import rr_pair

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("ell", [2, 3, 4, 5, 7, 8, 9, 16, 31, 32])
def test_schedule_closed_form_matches_reference(golden, ell):
    pairs, starts = bs.schedule_arrays(ell)
    assert np.array_equal(pairs, golden.get(f"sched_{ell}", "pairs"))
    assert np.array_equal(starts, golden.get(f"sched_{ell}", "starts"))
    assert not pairs.flags.writeable


@pytest.mark.parametrize("ell", range(2, 97))
def test_schedule_covers_all_pairs_disjointly(ell):
    # reference tests/test_ordering.py:48-68 and acceptance c08
    sched = bs.round_robin_schedule(ell)
    seen = set()
    for it in sched.iterations:
        idx = [x for p in it for x in p]
        assert len(idx) == len(set(idx))
        for i, j in it:
            assert 0 <= i < j < ell
            seen.add((i, j))
    assert len(seen) == ell * (ell - 1) // 2


def test_schedule_layouts_of_reference_tests():
    # tests/test_ordering.py:12-30
    assert bs.round_robin_schedule(2).iterations == (((0, 1),),)
    assert bs.round_robin_schedule(4).iterations == (((0, 1), (2, 3)), ((0, 3), (1, 2)), ((0, 2), (1, 3)))
    assert bs.round_robin_schedule(8).iterations[0] == ((0, 1), (2, 3), (4, 5), (6, 7))
    with pytest.raises(bs.DomainError):
        bs.round_robin_schedule(1)


def test_rr_pair_phantom():
    # odd ell: exactly one pair per iteration touches the phantom
    for ell in (3, 5, 9, 31):
        S = ell + 1
        for t in range(S - 1):
            flags = [rr_pair(t, k, S, ell)[2] for k in range(S // 2)]
            assert flags.count(False) == 1


def test_options_defaults_and_validation():
    o = bs.JacobiOptions()
    assert (o.k, o.max_nsweeps, o.nb, o.inner_sweeps, o.masking, o.use_qr_preprocess,
            o.compute_right_vectors, o.fused_updates, o.row_block) == (30.0, 30, 16, 1, False, False, True, True, 64)
    for kw in ({"k": 0.0}, {"k": -1.0}, {"max_nsweeps": 0}, {"nb": 0}, {"inner_sweeps": -1}, {"row_block": 0}):
        with pytest.raises(bs.DomainError):
            bs.JacobiOptions(**kw)


def test_compute_rotation_known_answer(golden):
    # tests/test_eig.py:23-32
    r = bs.compute_rotation(9.0, 41.0, 12.0)
    g = golden.meta["rotation_9_41_12"]
    assert r.c == g["c"] and r.s == g["s"] and r.t == g["t"]
    assert abs(r.c - 3 / np.sqrt(10)) < 1e-15 and abs(r.t + 1 / 3) < 1e-15


def test_library_loads_and_exports_header_symbols():
    L = _lib.load()
    with open(os.path.join(ROOT, "include", "bsvd_b200.h")) as fh:
        hdr = fh.read()
    declared = set(re.findall(r"^\s*(?:int|size_t|void|const char\*)\s+(bsvd_\w+)\s*\(", hdr, flags=re.M))
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    for sym in declared:
        assert hasattr(L, sym)
    assert L.bsvd_abi_version() == 1
    o = _lib.BsvdOpts()
    L.bsvd_default_opts(ctypes.byref(o))
    assert (o.k, o.max_sweeps, o.nb, o.inner_sweeps, o.want_v, o.row_block) == (30.0, 30, 16, 1, 1, 64)
    assert L.bsvd_strerror(-2).decode() == "workspace too small"


def test_library_argument_errors_without_device():
    # argument checks run on the host and fail before any device work
    L = _lib.load()
    o = _lib.BsvdOpts()
    L.bsvd_default_opts(ctypes.byref(o))
    rc = L.bsvd_gesvj_batched(7, 4, 4, 1, None, 4, 16, None, 4, 16, None, 4, None, 4, 16,
                              ctypes.byref(o), None, None, 0, None)
    assert rc == -1
    o.route = 1  # forced unblocked on a wide matrix -> ShapeError analogue
    rc = L.bsvd_gesvj_batched(1, 2, 5, 1, None, 2, 10, None, 2, 4, None, 2, None, 5, 10,
                              ctypes.byref(o), None, None, 0, None)
    assert rc == -1
    o.route = 0
    o.max_sweeps = 0
    assert L.bsvd_gesvj_batched(1, 4, 4, 1, None, 4, 16, None, 4, 16, None, 4, None, 4, 16,
                                ctypes.byref(o), None, None, 0, None) == -1


def test_kernel_selection_routes():
    L = _lib.load()
    o = _lib.BsvdOpts()
    L.bsvd_default_opts(ctypes.byref(o))
    assert L.bsvd_select_kernel(1, 64, 64, ctypes.byref(o)) == 30     # blocked FP64: register block pairs
    assert L.bsvd_select_kernel(3, 64, 64, ctypes.byref(o)) == 51     # blocked complex: complex register blocked
    assert L.bsvd_select_kernel(3, 40, 40, ctypes.byref(o)) == 2      # n % 16 != 0: general blocked kernel
    assert L.bsvd_select_kernel(0, 16, 16, ctypes.byref(o)) == 24     # 16x16 FP32 register kernel (2nd gen)
    assert L.bsvd_select_kernel(1, 32, 32, ctypes.byref(o)) == 42     # 32x32 FP64: 2nd gen, scaled rotations
    o.want_v = 0
    assert L.bsvd_select_kernel(1, 32, 32, ctypes.byref(o)) == 12     # values only: unscaled 2nd gen
    o.want_v = 1
    assert L.bsvd_select_kernel(3, 256, 32, ctypes.byref(o)) == 32    # c128 n = 32: complex register kernel
    assert L.bsvd_select_kernel(3, 300, 32, ctypes.byref(o)) == 1     # m > 256: general unblocked kernel
    assert L.bsvd_select_kernel(2, 256, 32, ctypes.byref(o)) == 32    # c64 n = 32: on the c128 register kernel
    assert L.bsvd_select_kernel(2, 256, 24, ctypes.byref(o)) == 1     # c64, other n: general unblocked kernel
    assert L.bsvd_select_kernel(0, 64, 64, ctypes.byref(o)) == 30     # FP32 blocked: on the FP64 register kernel
    assert L.bsvd_select_kernel(0, 32, 32, ctypes.byref(o)) == 42     # FP32 32x32: on the FP64 register kernel
    # by batch size (148 SMs assumed without a device): one problem per warp up to one resident wave (8 per SM)
    assert L.bsvd_select_kernel_batched(1, 32, 32, 1000, ctypes.byref(o)) == 52
    assert L.bsvd_select_kernel_batched(0, 32, 32, 1000, ctypes.byref(o)) == 52
    assert L.bsvd_select_kernel_batched(1, 32, 32, 10000, ctypes.byref(o)) == 42
    o.want_v = 0
    assert L.bsvd_select_kernel_batched(1, 32, 32, 1000, ctypes.byref(o)) == 12
    o.want_v = 1
    o.route = _lib.FORCE_BLOCKED
    assert L.bsvd_select_kernel(3, 256, 32, ctypes.byref(o)) == 32    # blocked route, ell = 2: same kernel
    o.nb = 8
    assert L.bsvd_select_kernel(3, 256, 32, ctypes.byref(o)) == 2     # ell = 4: general blocked kernel
    o.nb = 16
    o.route = _lib.DISPATCH
    assert L.bsvd_select_kernel(1, 0, 5, ctypes.byref(o)) == 0        # empty


def test_info_struct_layout():
    from paper_2601_17979_b200.solver import INFO_DTYPE

    assert INFO_DTYPE.itemsize == ctypes.sizeof(_lib.BsvdInfo) == 48


def test_batch_rejects_bad_problems_without_device():
    # per-problem isolation (src/batch.py:105-111) happens before any device work
    bad = np.zeros((4, 4), dtype=np.int8, order="F")
    st = bs.BatchState.for_batch(2)
    out = bs.batch_svd([bad, np.zeros((2, 2, 2))], bs.JacobiOptions(), st)
    assert out == [None, None]
    assert isinstance(st.errors[0], bs.DomainError)
    assert isinstance(st.errors[1], bs.ShapeError)
    with pytest.raises(bs.DomainError):
        bs.batch_svd([])


def test_empty_shapes_need_no_device():
    r = bs.svd_dispatch(np.zeros((0, 0), order="F"))
    assert r.sigma.shape == (0,) and r.info.path == "empty" and r.info.converged
    r = bs.svd_dispatch(np.zeros((0, 3), order="F"))
    assert r.u.shape == (0, 0) and r.v.shape == (3, 0)


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    a = np.eye(4)
    st = bs.BatchState.for_batch(1)
    out = bs.batch_svd([a], bs.JacobiOptions(), st)
    assert out == [None]
    assert isinstance(st.errors[0], RuntimeError)
    with pytest.raises(RuntimeError):
        bs.svd_dispatch(a)


def test_backend_interface_single_b200_backend():
    """src/backend.py:30-35 interface: one B200 backend, CPU backends rejected (no fallback)."""
    b = bs.active()
    assert b.name == "b200" and b is bs.select("auto") and b is bs.select("b200")
    assert b.onesided_sweeps is bs.onesided_sweeps and b.eig_sweeps is bs.eig_sweeps
    assert b.fused_pair_update is bs.fused_pair_update
    for bad in ("numba", "numpy", "cuda"):
        with pytest.raises(ValueError):
            bs.select(bad)
    with bs.use("b200") as bb:
        assert bb is b


def test_pack_host_helper_packs_column_major_batches():
    """bsvd_pack_host (host-only, no GPU): the list API's packing of F-ordered matrices."""
    L = _lib.load()
    rng = np.random.default_rng(3)
    mats = [np.asfortranarray(rng.random((5, 3))) for _ in range(37)]
    out = np.empty((37, 3, 5))
    ptrs = np.fromiter((a.__array_interface__["data"][0] for a in mats), dtype=np.uintp, count=len(mats))
    for nt in (1, 4):
        out[...] = 0
        assert L.bsvd_pack_host(ptrs.ctypes.data, len(mats), 15 * 8, out.ctypes.data, nt) == 0
        assert np.array_equal(out, np.stack([a.T for a in mats]))


def test_default_chunk_policy():
    from paper_2601_17979_b200.solver import default_chunk

    per32 = 3 * 32 * 32 * 8
    assert default_chunk(1000, per32, 32 * 32, 4, 148) == 250      # latency-bound: one chunk per stream
    assert default_chunk(1250, per32, 32 * 32, 4, 148) == 313
    assert default_chunk(10000, per32, 32 * 32, 4, 148) == 1250    # small problems: at most 8 chunks
    assert default_chunk(10000, 3 * 16 * 16 * 4, 16 * 16, 4, 148) == 2500    # ~8 MB chunks, at least 4
    assert default_chunk(2000, 3 * 128 * 128 * 8, 128 * 128, 4, 148) == 125  # large problems: 16 chunks
    assert default_chunk(3, per32, 32 * 32, 4, 148) == 1
    assert default_chunk(10000, per32, 32 * 32, 4, 148, gather=True) == 417         # packed ahead: B/24
    assert default_chunk(10000, 3 * 16 * 16 * 4, 16 * 16, 4, 148, gather=True) == 2500


def test_lazy_records_filled_by_c_helper():
    """bsvd_py_fill_lazy writes the records' (_g, _j) slots directly; a record materialises its fields on
    first use and otherwise behaves as the reference's frozen SvdResult (repr, copy, pickle, replace)."""
    import copy
    import dataclasses
    import pickle

    from paper_2601_17979_b200 import batch
    from paper_2601_17979_b200.solver import INFO_DTYPE

    H = _lib.hostptrs()
    if H is None:
        pytest.skip("CPython helper not built")
    g = batch._Group()
    g.U = np.arange(5 * 4, dtype=float).reshape(5, 2, 2)
    g.S = np.ones((5, 2))
    g.V = None
    g.cols = np.zeros(5, dtype=INFO_DTYPE)
    g.cols["converged"] = 1
    g.cols["outer_sweeps"] = 3
    g.calls = np.full(5, 3)
    g.masked = np.zeros(5, dtype=int)
    g.blocked, g.pps, g.eig_unit, g.dtime, g.atime = False, 1, 1, 1e-6, 1e-7
    recs = [None] * 6
    assert H.bsvd_py_fill_lazy(recs, 1, 5, batch._LazyResult, g) == 0
    assert recs[0] is None and all(isinstance(r, bs.SvdResult) for r in recs[1:])
    r = recs[4]
    assert np.array_equal(r.u, g.U[3]) and np.array_equal(r.sigma, g.S[3]) and r.v is None
    assert r.info.outer_sweeps == 3 and r.info.converged and "SvdResult" in repr(r) or "LazyResult" in repr(r)
    for c in (copy.copy(r), copy.deepcopy(r), pickle.loads(pickle.dumps(r))):
        assert type(c) is bs.SvdResult and np.array_equal(c.u, r.u) and c.info == r.info
    r2 = dataclasses.replace(recs[2], sigma=np.zeros(2))
    assert np.array_equal(r2.u, g.U[1]) and not r2.sigma.any()
    with pytest.raises(dataclasses.FrozenInstanceError):
        r.u = None
