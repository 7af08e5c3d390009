"""bsvd_gesvj_batched through the C-ABI with padded leading dimensions and batch strides (lda > m,
ldu > m, ldv > n, gaps between problems), as a C caller with its own allocations would pass them
(include/bsvd_b200.h): results match the contiguous solve -- bitwise where the same kernel runs (the
single-precision problems promoted to the double-precision register kernels widen into a contiguous
copy), within the parity tolerance where a padded lda moves a problem to a general kernel -- and the
workspace query covers both plans."""

import ctypes

import numpy as np
import pytest

import paper_2601_17979_b200 as bs
from common import check_sigma_parity, random_matrix
from oracle import oracle as O
from paper_2601_17979_b200 import _lib
from paper_2601_17979_b200.core import DTYPE_CODE
from paper_2601_17979_b200.solver import INFO_DTYPE, make_opts, torch_dtype

pytestmark = pytest.mark.gpu

CASES = [
    (np.float64, 32, 32), (np.float32, 32, 32), (np.float32, 64, 64), (np.float32, 16, 16),
    (np.complex64, 256, 32), (np.complex64, 40, 32), (np.complex128, 256, 32), (np.float64, 64, 64),
    (np.float32, 48, 33), (np.float64, 128, 128), (np.complex128, 128, 128),
]


@pytest.mark.parametrize("dt,m,n", CASES)
def test_padded_strides_match_contiguous(dt, m, n):
    import torch

    L = _lib.load()
    B, pad, gap = 5, 3, 7
    k = min(m, n)
    dtn = np.dtype(dt)
    rdt = np.float32 if dtn in (np.float32, np.complex64) else np.float64
    A = np.stack([random_matrix(m, n, dt, seed=6100 + b + m) for b in range(B)])
    lda, ldu, ldv = m + pad, m + pad, n + pad
    sA, sU, sV, sS = lda * n + gap, ldu * k + gap, ldv * k + gap, k + gap
    tdt = torch_dtype(dtn)
    a_buf = torch.zeros(B * sA, dtype=tdt)
    for b in range(B):  # column-major problem b at offset b * sA with leading dimension lda
        view = a_buf[b * sA: b * sA + lda * n].view(n, lda)
        view[:, :m] = torch.from_numpy(np.ascontiguousarray(A[b].T))
    dev = torch.device("cuda", torch.cuda.current_device())
    a_d = a_buf.to(dev)
    u_d = torch.zeros(B * sU, dtype=tdt, device=dev)
    v_d = torch.zeros(B * sV, dtype=tdt, device=dev)
    s_d = torch.zeros(B * sS, dtype=torch_dtype(np.dtype(rdt)), device=dev)
    info_d = torch.zeros(B * _lib.INFO_BYTES, dtype=torch.uint8, device=dev)
    opts = bs.JacobiOptions()
    o = make_opts(opts, _lib.DISPATCH, 0)
    code = DTYPE_CODE[dtn]
    ws_bytes = L.bsvd_workspace_bytes(code, m, n, B, ctypes.byref(o))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    rc = L.bsvd_gesvj_batched(code, m, n, B, a_d.data_ptr(), lda, sA, u_d.data_ptr(), ldu, sU, s_d.data_ptr(), sS,
                              v_d.data_ptr(), ldv, sV, ctypes.byref(o), info_d.data_ptr(), ws.data_ptr(), ws_bytes,
                              torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(rc, "padded bsvd_gesvj_batched")
    torch.cuda.synchronize()
    info = np.frombuffer(info_d.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    # the contiguous solve of the same problems
    ref = bs.solve_tensor(torch.from_numpy(np.ascontiguousarray(np.swapaxes(A, 1, 2))).to(dev), m, n, opts)
    torch.cuda.synchronize()
    Sr, Ur, Vr = ref.s.cpu().numpy(), ref.u.cpu().numpy(), ref.v.cpu().numpy()
    info_r = np.frombuffer(ref.info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
    ub, vb, sb = u_d.cpu().numpy(), v_d.cpu().numpy(), s_d.cpu().numpy()
    same_kernel = (info["kernel"] == info_r["kernel"]).all()
    for b in range(B):
        S = sb[b * sS: b * sS + k]
        U = ub[b * sU: b * sU + ldu * k].reshape(k, ldu)[:, :m]
        V = vb[b * sV: b * sV + ldv * k].reshape(k, ldv)[:, :n]
        assert info["converged"][b]
        if same_kernel:
            assert np.array_equal(S, Sr[b]) and np.array_equal(U, Ur[b]) and np.array_equal(V, Vr[b])
        _, s_ref, _, _ = O.solve(A[b], None, None)
        check_sigma_parity(S, s_ref, k, bs.unit_roundoff(dt))
        # padding and gaps untouched
        if b + 1 < B:
            assert not ub[b * sU + ldu * k: (b + 1) * sU].any() and not sb[b * sS + k: (b + 1) * sS].any()
        assert not ub[b * sU: b * sU + ldu * k].reshape(k, ldu)[:, m:].any()
