"""BSVD/BSVR container I/O around the device solver (src/fileio.py:105-218): a
uniform BSVD file lands in a pinned (B, n, m) host tensor, goes through the host-buffer C-ABI entry
(bsvd_gesvj_batched_host), and the factors are written as a BSVR file byte-identical to the one
write_results produces from the list API's records."""

import numpy as np
import pytest

import paper_2601_17979_b200 as bs
from common import check_factors, random_matrix
from paper_2601_17979_b200 import fileio

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dt,m,n", [(np.float64, 32, 32), (np.float32, 16, 16), (np.complex128, 64, 32),
                                    (np.complex64, 12, 9)])
def test_bsvd_file_to_bsvr_file_through_host_pipeline(tmp_path, dt, m, n):
    import torch

    from paper_2601_17979_b200.solver import INFO_DTYPE, real_dtype, solve_host_buffers, torch_dtype

    B = 23
    mats = [random_matrix(m, n, dt, seed=5100 + b) for b in range(B)]
    src = tmp_path / "in.bsvd"
    fileio.write_matrices(src, mats)
    a_h, mm, nn = fileio.read_matrices_pinned(src)
    assert (mm, nn) == (m, n) and a_h.is_pinned() and tuple(a_h.shape) == (B, n, m)
    k = min(m, n)
    tdt = torch_dtype(np.dtype(dt))
    u_h = torch.empty((B, k, m), dtype=tdt).pin_memory()
    s_h = torch.empty((B, k), dtype=torch_dtype(real_dtype(np.dtype(dt)))).pin_memory()
    v_h = torch.empty((B, k, n), dtype=tdt).pin_memory()
    i_h = torch.empty((B * 48,), dtype=torch.uint8).pin_memory()
    solve_host_buffers(a_h, u_h, s_h, v_h, i_h, m, n, bs.JacobiOptions(), chunk=7)
    torch.cuda.synchronize()
    info = np.frombuffer(i_h.numpy().tobytes(), dtype=INFO_DTYPE)
    out_fast = tmp_path / "fast.bsvr"
    fileio.write_results_batch(out_fast, m, n, u_h.numpy(), s_h.numpy(), v_h.numpy(), info["converged"])
    # the same batch through the list API and the record writer
    res = bs.batch_svd(mats, bs.JacobiOptions())
    out_ref = tmp_path / "ref.bsvr"
    fileio.write_results(out_ref, mats, res)
    assert out_fast.read_bytes() == out_ref.read_bytes()
    back = fileio.read_results(out_fast)
    for a, rec in zip(mats, back):
        assert rec.converged and not rec.failed
        check_factors(a, rec.u, rec.sigma, rec.v)
