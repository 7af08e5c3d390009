"""BSVD / BSVR containers (src/fileio.py of the reference): read the reference-written fixtures
(tests/golden/make_fileio.py), write byte-identical files, reject malformed streams, and the
uniform fast path into a pinned-layout host tensor.  CPU only."""

import os

import numpy as np
import pytest

from paper_2601_17979_b200 import fileio as F

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ("f32", "f64", "c64", "c128")


class _Info:
    def __init__(self, c):
        self.converged = c


class _Res:
    def __init__(self, rec):
        self.u, self.sigma, self.v, self.info = rec.u, rec.sigma, rec.v, _Info(rec.converged)


@pytest.mark.parametrize("nm", NAMES)
def test_matrix_round_trip_byte_identical(nm, tmp_path):
    for kind in ("mixed", "uniform"):
        src = os.path.join(G, f"ref_{kind}_{nm}.bsvd")
        mats = F.read_matrices(src)
        assert all(a.flags.f_contiguous for a in mats)
        out = tmp_path / "x.bsvd"
        F.write_matrices(out, mats)
        assert out.read_bytes() == open(src, "rb").read()


@pytest.mark.parametrize("nm", NAMES)
def test_result_round_trip_byte_identical(nm, tmp_path):
    mats = F.read_matrices(os.path.join(G, f"ref_uniform_{nm}.bsvd"))
    recs = F.read_results(os.path.join(G, f"ref_uniform_{nm}.bsvr"))
    assert [r.failed for r in recs] == [False, False, True, False]
    res = [None if r.failed else _Res(r) for r in recs]
    out = tmp_path / "x.bsvr"
    F.write_results(out, mats, res)
    assert out.read_bytes() == open(os.path.join(G, f"ref_uniform_{nm}.bsvr"), "rb").read()
    # the uniform C-ABI-layout writer produces the same bytes for the non-failed slots
    ok = [r for r in recs if not r.failed]
    m, n = ok[0].m, ok[0].n
    u = np.stack([np.ascontiguousarray(r.u.T) for r in ok])
    s = np.stack([r.sigma for r in ok])
    v = np.stack([np.ascontiguousarray(r.v.T) for r in ok])
    F.write_results_batch(tmp_path / "b.bsvr", m, n, u, s, v, [r.converged for r in ok])
    F.write_results(tmp_path / "c.bsvr", [mats[i] for i in (0, 1, 3)], [_Res(r) for r in ok])
    assert (tmp_path / "b.bsvr").read_bytes() == (tmp_path / "c.bsvr").read_bytes()


@pytest.mark.parametrize("nm", NAMES)
def test_uniform_fast_path(nm):
    mats = F.read_matrices(os.path.join(G, f"ref_uniform_{nm}.bsvd"))
    t, m, n = F.read_matrices_pinned(os.path.join(G, f"ref_uniform_{nm}.bsvd"), pin=False)
    assert (m, n) == mats[0].shape and t.shape == (len(mats), n, m)
    for b, a in enumerate(mats):  # t[b] is the column-major matrix, i.e. A^T row-major
        assert np.array_equal(t[b].numpy().T, a)
    with pytest.raises(F.DomainError):
        F.read_matrices_pinned(os.path.join(G, f"ref_mixed_{nm}.bsvd"), pin=False)


def test_empty_and_malformed(tmp_path):
    assert F.read_matrices(os.path.join(G, "ref_empty.bsvd")) == []
    good = open(os.path.join(G, "ref_uniform_f64.bsvd"), "rb").read()
    cases = {
        "magic": b"XSVD" + good[4:],
        "version": good[:4] + bytes([2]) + good[5:],
        "dtype": good[:5] + bytes([9]) + good[6:],
        "reserved": good[:6] + bytes([1]) + good[7:],
        "trailing": good + b"\0",
        "truncated": good[:-3],
        "short": good[:7],
    }
    for name, blob in cases.items():
        p = tmp_path / f"{name}.bsvd"
        p.write_bytes(blob)
        with pytest.raises(F.FormatError):
            F.read_matrices(p)
    with pytest.raises(F.FormatError):
        F.read_results(os.path.join(G, "ref_uniform_f64.bsvd"))  # wrong magic for a result file
    with pytest.raises(F.DomainError):
        F.write_matrices(tmp_path / "z.bsvd", [np.zeros((2, 2)), np.zeros((2, 2), np.float32)])
    with pytest.raises(F.DomainError):
        F.write_results(tmp_path / "z.bsvr", [np.zeros((2, 2))], [])
