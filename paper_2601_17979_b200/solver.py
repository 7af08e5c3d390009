"""Device-side batch solve through the C-ABI (the hot path).

``solve_tensor`` is the tensor fast path: a device-resident batch in, device
factors out, one ``bsvd_gesvj_batched`` launch on the current stream, no host
synchronisation.  ``solve_host`` is the host-buffer path used by the
reference-shaped API (``batch_svd``): pinned staging, H2D, the same launch,
D2H.  Layout contract (include/bsvd_b200.h): each matrix column-major, so a
batch is stored as a C-contiguous (B, n, m) tensor whose [b] slice is the
transpose view of A_b.
"""

from __future__ import annotations

import ctypes
import threading
import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import DTYPE_CODE, real_dtype

INFO_DTYPE = np.dtype([
    ("converged", "<i4"),
    ("outer_sweeps", "<i4"),
    ("rotations", "<i8"),
    ("gram_calls", "<i8"),
    ("update_calls", "<i8"),
    ("last_rotations", "<i4"),
    ("path", "<i4"),
    ("status", "<i4"),
    ("kernel", "<i4"),
])
assert INFO_DTYPE.itemsize == _lib.INFO_BYTES


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2601_17979_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")
    return torch


_TORCH_OF = {}


def torch_dtype(np_dtype):
    import torch

    if not _TORCH_OF:
        _TORCH_OF.update({
            np.dtype(np.float32): torch.float32,
            np.dtype(np.float64): torch.float64,
            np.dtype(np.complex64): torch.complex64,
            np.dtype(np.complex128): torch.complex128,
        })
    return _TORCH_OF[np.dtype(np_dtype)]


_NP_OF: dict = {}


def np_dtype_of(tdtype):
    if not _NP_OF:
        torch = _torch()
        _NP_OF.update({torch.float32: np.dtype(np.float32), torch.float64: np.dtype(np.float64),
                       torch.complex64: np.dtype(np.complex64), torch.complex128: np.dtype(np.complex128)})
    return _NP_OF[tdtype]


_OPTS_CACHE: dict = {}
_WSB_CACHE: dict = {}


def _cached_opts(opts, route: int, kernel: int, tail: int) -> _lib.BsvdOpts:
    """make_opts memoised on the (frozen, hashable) JacobiOptions: the C side only reads the struct."""
    key = (opts, int(route), int(kernel), int(tail))
    o = _OPTS_CACHE.get(key)
    if o is None:
        o = make_opts(opts, route, kernel, tail)
        _OPTS_CACHE[key] = o
    return o


def make_opts(opts, route: int = _lib.DISPATCH, kernel: int = 0, tail: int = 0) -> _lib.BsvdOpts:
    """JacobiOptions -> POD bsvd_opts (src/svd.py:70-78 field by field)."""
    o = _lib.BsvdOpts()
    o.k = float(opts.k)
    o.max_sweeps = int(opts.max_nsweeps)
    o.nb = int(opts.nb)
    o.inner_sweeps = int(opts.inner_sweeps)
    o.masking = int(bool(opts.masking))
    o.want_v = int(bool(opts.compute_right_vectors))
    o.route = int(route)
    o.fused_updates = int(bool(opts.fused_updates))
    o.row_block = int(opts.row_block)
    o.kernel = int(kernel)
    o.use_qr = int(bool(opts.use_qr_preprocess))
    o.reserved[0] = int(tail)  # experimental: 32x32 FP64 tail size (0 automatic, < 0 off)
    return o


_WS_CACHE: dict = {}


def _workspace(nbytes: int, device, stream_handle=None):
    torch = _torch()
    if nbytes == 0:
        return None
    if stream_handle is None:
        stream_handle = torch.cuda.current_stream(device).cuda_stream
    key = (str(device), stream_handle)
    buf = _WS_CACHE.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _WS_CACHE[key] = buf
    return buf


@dataclass
class DeviceResult:
    u: object      # (B, k, m) tensor: u[b] is U_b^T (column-major U_b)
    s: object      # (B, k) real tensor
    v: object      # (B, k, n) tensor or None
    info: object   # (B * INFO_BYTES,) uint8 tensor
    kernel: int


def solve_tensor(a_t, m: int, n: int, opts, route: int = _lib.DISPATCH, kernel: int = 0,
                 out=None, tail: int = 0) -> DeviceResult:
    """Batched SVD of a device tensor a_t (B, n, m) (column-major matrices).

    Launches on torch's current stream; returns device tensors without
    synchronising.  ``out`` may pass preallocated (u, s, v, info) tensors.
    """
    torch = _torch()
    L = _lib.load()
    B = a_t.shape[0]
    assert a_t.shape == (B, n, m) and a_t.is_contiguous() and a_t.is_cuda
    dt = np_dtype_of(a_t.dtype)
    code = DTYPE_CODE[dt]
    k = min(m, n)
    o = _cached_opts(opts, route, kernel, tail)
    dev = a_t.device
    if out is None:
        u = torch.empty((B, k, m), dtype=a_t.dtype, device=dev)
        s = torch.empty((B, k), dtype=torch_dtype(real_dtype(dt)), device=dev)
        v = torch.empty((B, k, n), dtype=a_t.dtype, device=dev) if o.want_v else None
        info = torch.empty((B * _lib.INFO_BYTES,), dtype=torch.uint8, device=dev)
    else:
        u, s, v, info = out
    wkey = (code, m, n, B, id(o))
    ws_bytes = _WSB_CACHE.get(wkey)
    if ws_bytes is None:
        ws_bytes = L.bsvd_workspace_bytes(code, m, n, B, ctypes.byref(o))
        _WSB_CACHE[wkey] = ws_bytes
    stream = torch.cuda.current_stream(dev).cuda_stream
    ws = _workspace(ws_bytes, dev, stream)
    rc = L.bsvd_gesvj_batched(
        code, m, n, B,
        a_t.data_ptr(), max(m, 1), m * n,
        u.data_ptr(), max(m, 1), k * m,
        s.data_ptr(), k,
        v.data_ptr() if v is not None else None, max(n, 1), k * n,
        ctypes.byref(o), info.data_ptr(),
        ws.data_ptr() if ws is not None else None, ws_bytes, stream)
    _lib.check(rc, f"bsvd_gesvj_batched({dt.name}, {m}x{n}, batch={B})")
    kern = L.bsvd_select_kernel_batched(code, m, n, B, ctypes.byref(o))  # the batch size can pick the kernel
    return DeviceResult(u=u, s=s, v=v, info=info, kernel=int(kern))


def solve_host_buffers(a_h, u_h, s_h, v_h, info_h, m: int, n: int, opts, route: int = _lib.DISPATCH,
                       kernel: int = 0, chunk: int = 0, streams=None, a_ptrs=None, pack_threads: int = 4):
    """Pipelined host-buffer solve through bsvd_gesvj_batched_host.

    With ``a_ptrs`` (uintp array of the B problems' column-major data) the batch is packed into a_h by
    ``pack_threads`` host threads chunk by chunk while earlier chunks are in flight
    (bsvd_gesvj_batched_host_gather); otherwise a_h already holds the packed batch.

    a_h (B, n, m), u_h (B, k, m), s_h (B, k), v_h (B, k, n) | None, info_h
    (B * INFO_BYTES,) are CPU tensors (pinned for full PCIe bandwidth).  The
    batch is cut into ``chunk``-problem pieces whose H2D, solve and D2H
    overlap across ``streams`` (torch streams; default: the current stream
    plus three side streams; chunk default: ``default_chunk``).  Asynchronous on streams[0]: synchronise it
    before reading the outputs.
    """
    torch = _torch()
    L = _lib.load()
    B = a_h.shape[0]
    dt = np_dtype_of(a_h.dtype)
    code = DTYPE_CODE[dt]
    o = make_opts(opts, route, kernel)
    dev = torch.device("cuda", torch.cuda.current_device())
    if streams is None:
        streams = [torch.cuda.current_stream(dev)] + _side_streams(dev, 3)
    if chunk <= 0:
        k = min(m, n)
        es = np.dtype(dt).itemsize
        per = m * n * es + m * k * es + (n * k * es if opts.compute_right_vectors else 0)  # bytes in + out
        chunk = default_chunk(B, per, m * n, len(streams), _sm_count(dev), gather=a_ptrs is not None)
    ws_bytes = L.bsvd_host_workspace_bytes(code, m, n, chunk, len(streams), ctypes.byref(o))
    ws = _workspace(ws_bytes, dev)
    arr = (ctypes.c_void_p * len(streams))(*[st.cuda_stream for st in streams])
    if a_ptrs is None:
        rc = L.bsvd_gesvj_batched_host(
            code, m, n, B, a_h.data_ptr(), u_h.data_ptr(), s_h.data_ptr(),
            v_h.data_ptr() if v_h is not None else None, ctypes.byref(o),
            info_h.data_ptr() if info_h is not None else None, chunk,
            ws.data_ptr() if ws is not None else None, ws_bytes, arr, len(streams))
    else:  # gather mode: the problems are packed into a_h chunk by chunk, overlapping the pipeline
        rc = L.bsvd_gesvj_batched_host_gather(
            code, m, n, B, a_ptrs.ctypes.data, a_h.data_ptr(), pack_threads, u_h.data_ptr(), s_h.data_ptr(),
            v_h.data_ptr() if v_h is not None else None, ctypes.byref(o),
            info_h.data_ptr() if info_h is not None else None, chunk,
            ws.data_ptr() if ws is not None else None, ws_bytes, arr, len(streams))
    _lib.check(rc, f"bsvd_gesvj_batched_host({dt.name}, {m}x{n}, batch={B})")
    # the kernel of a chunk: with more than two waves of kernel 52 in flight the pipeline turns it off
    # (csrc/api.cu pipeline_throughput)
    o_sel = make_opts(opts, route, kernel, -1) if len(streams) * min(chunk, B) > 16 * _sm_count(dev) else o
    return int(L.bsvd_select_kernel_batched(code, m, n, min(B, chunk), ctypes.byref(o_sel)))


def default_chunk(batch: int, bytes_per_problem: int, elems: int = 0, nstreams: int = 4, sms: int = 148,
                  gather: bool = False) -> int:
    """Host-pipeline chunk: about 8 MB of copies per chunk, between 4 and 16 chunks -- at most 8 for
    problems of m n <= 1,024 (measured on B200, tools/e2e_sweep.py, tools/e2e_sweep_c2.py,
    tools/ramp_probe.py: C1-10k best at B/8 with the pipeline's kernel 42, 3.86 vs 3.96 ms at B/16; C2 full
    at B/4, 0.635 vs 0.679 ms at B/8; C4 at B/16).  Small problems (m n <= 1,024, a problem per warp or
    half-warp) in batches of at most 16 per SM take one chunk per stream: their solve is a single-problem
    latency whatever the chunk size, so more chunks than streams queue a second latency behind the first
    (C1 1,000 problems: 0.65 ms at B/4 vs 0.75 ms at B/6).  ``gather``: the batch is packed on host threads
    ahead of the pipeline, and the first H2D waits for its whole chunk, so small problems go down to B/24
    (batch_svd C1-10k, tools/list_api_chunk_probe.py: 5.39 ms at B/24, 5.42-5.67 at B/16, 5.98-6.33 at B/8;
    C2 unchanged at its ~8 MB chunks, 1.47-1.61 ms at B/4, 1.60 at B/16)."""
    small = 0 < elems <= 1024
    if small and batch <= 16 * sms:
        return max(1, -(-batch // max(1, nstreams)))
    lo, hi = -(-batch // (24 if small and gather else 8 if small else 16)), -(-batch // 4)
    want = -(-(8 << 20) // max(1, bytes_per_problem))
    return max(1, min(max(want, lo), hi))


def _sm_count(dev) -> int:
    torch = _torch()
    return int(torch.cuda.get_device_properties(dev).multi_processor_count)


_SIDE: dict = {}


def _side_streams(dev, count):
    torch = _torch()
    key = str(dev)
    lst = _SIDE.setdefault(key, [])
    while len(lst) < count:
        lst.append(torch.cuda.Stream(dev))
    return lst[:count]


_TLS = threading.local()  # per-thread pinned staging: concurrent batch_svd calls never share buffers
_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        import concurrent.futures
        import os

        _POOL = concurrent.futures.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1))
    return _POOL


def _parallel_slices(total: int, fn, min_per: int = 256) -> None:
    """fn(lo, hi) over [0, total) in parallel host threads (numpy copies release the GIL)."""
    nt = max(1, min(8, total // min_per))
    if nt == 1:
        fn(0, total)
        return
    step = -(-total // nt)
    futs = [_pool().submit(fn, lo, min(total, lo + step)) for lo in range(0, total, step)]
    for f in futs:
        f.result()


def _pinned(key, shape, tdt):
    """Pinned staging reused across calls of the same host thread (pinned allocation is slow; results are
    copied out before the call returns), so two threads calling batch_svd at once never share it."""
    torch = _torch()
    pinned = getattr(_TLS, "pinned", None)
    if pinned is None:
        pinned = _TLS.pinned = {}
    buf = pinned.get(key)
    n = int(np.prod(shape))
    if buf is None or buf.numel() < n or buf.dtype != tdt:
        buf = torch.empty(max(n, 1), dtype=tdt, pin_memory=True)
        pinned[key] = buf
    return buf[:n].view(shape)


class _PinnedOwner:
    """Owner of one pooled pinned result buffer, exposed to numpy through __array_interface__: every
    array or view handed to the caller keeps it alive, so the pool can tell (by a weak reference) when
    the caller has dropped all of them and the buffer may be written again."""

    def __init__(self, t):
        self.tensor = t
        self.__array_interface__ = t.numpy().__array_interface__


_RESULTS: dict = {}  # (tag, shape, dtype) -> [[tensor, weakref to the live _PinnedOwner | None], ...]
_RESULTS_LOCK = threading.Lock()
_RESULTS_PER_KEY = 4  # at most this many pinned result sets per shape; beyond it, fresh pageable arrays


def _result_array(tag, shape, tdt, dt):
    """A pinned array for results that go to the caller without a copy, or None when every pooled buffer
    of this shape is still referenced by earlier results (the caller then copies into fresh memory)."""
    torch = _torch()
    key = (tag, tuple(shape), tdt)
    with _RESULTS_LOCK:
        lst = _RESULTS.setdefault(key, [])
        ent = next((e for e in lst if e[1] is None or e[1]() is None), None)
        if ent is None:
            if len(lst) >= _RESULTS_PER_KEY:
                return None
            ent = [torch.empty(tuple(shape), dtype=tdt, pin_memory=True), None]
            lst.append(ent)
        owner = _PinnedOwner(ent[0])
        ent[1] = weakref.ref(owner)
    arr = np.asarray(owner)
    assert arr.dtype == dt
    return arr


def last_device_seconds() -> float:
    """Wall time of this thread's latest solve_host device pipeline (H2D, kernels, D2H; synchronised)."""
    return getattr(_TLS, "device_seconds", 0.0)


def solve_host(mats: list, opts, route: int = _lib.DISPATCH, kernel: int = 0, device=None, ptrs=None,
               defer: bool = False):
    """Equal shape/dtype numpy matrices -> (U (B,m,k), S (B,k), V (B,n,k)|None, info records).

    Host-buffer path: the column-major batch is packed (one C-level copy; ``ptrs`` may pass the
    problems' data pointers when the caller already checked them) into pinned staging that is
    reused across calls of the thread, and the pipelined bsvd_gesvj_batched_host overlaps H2D / solve /
    D2H in chunks.  The factors land directly in pooled pinned result buffers that are handed to the
    caller (no copy-out; a buffer is reused only once every array viewing it has been dropped); when the
    pool is exhausted the factors are copied into fresh arrays.  Returned U[b] / V[b] are F-ordered views.
    ``defer``: return a callable instead, which waits for the device and returns the same tuple, so the
    caller can do host work (building records) while the pipeline drains.
    """
    torch = _torch()
    B = len(mats)
    m, n = mats[0].shape
    dt = np.dtype(mats[0].dtype)
    k = min(m, n)
    device = device or torch.device("cuda", torch.cuda.current_device())
    tdt = torch_dtype(dt)
    rdt = real_dtype(dt)
    host = _pinned("a", (B, n, m), tdt)
    hv = host.numpy()
    if ptrs is None and all(a.flags.f_contiguous and a.dtype == dt for a in mats):
        ptrs = np.fromiter((a.__array_interface__["data"][0] for a in mats), dtype=np.uintp, count=B)
    if ptrs is not None:  # raw column-major copies in C, overlapped with the pipeline (gather mode)
        pass
    else:
        _parallel_slices(B, lambda lo, hi: np.stack([a.T for a in mats[lo:hi]], out=hv[lo:hi]))
    want_v = bool(opts.compute_right_vectors)
    Uo = _result_array("u", (B, k, m), tdt, dt)
    Vo = _result_array("v", (B, k, n), tdt, dt) if want_v else None
    So = _result_array("s", (B, k), torch_dtype(rdt), rdt)
    direct = Uo is not None and So is not None and (Vo is not None or not want_v)
    if direct:
        u_h = torch.from_numpy(Uo)
        s_h = torch.from_numpy(So)
        v_h = torch.from_numpy(Vo) if want_v else None
    else:
        u_h = _pinned("u", (B, k, m), tdt)
        s_h = _pinned("s", (B, k), torch_dtype(rdt))
        v_h = _pinned("v", (B, k, n), tdt) if want_v else None
    info_h = _pinned("i", (B * _lib.INFO_BYTES,), torch.uint8)
    t_dev0 = time.perf_counter()
    with torch.cuda.device(device):
        kern = solve_host_buffers(host, u_h, s_h, v_h, info_h, m, n, opts, route, kernel, a_ptrs=ptrs)
        stream = torch.cuda.current_stream(device)

    def finish():
        stream.synchronize()
        _TLS.device_seconds = time.perf_counter() - t_dev0  # the pipelined H2D / solve / D2H, for WorkCounters
        return _host_outputs(direct, Uo, So, Vo, u_h, s_h, v_h, info_h, B, k, m, n, dt, kern)

    return finish if defer else finish()


def _host_outputs(direct, Uo, So, Vo, u_h, s_h, v_h, info_h, B, k, m, n, dt, kern):
    if direct:
        Uc, S, Vc = Uo, So, Vo
    else:  # copy the factors out of the reusable staging (threaded: ~250 MB for C1-10k)
        Uc = np.empty((B, k, m), dtype=dt)
        Vc = np.empty((B, k, n), dtype=dt) if v_h is not None else None
        un, vn = u_h.numpy(), (v_h.numpy() if v_h is not None else None)

        def _out(lo, hi):
            Uc[lo:hi] = un[lo:hi]
            if Vc is not None:
                Vc[lo:hi] = vn[lo:hi]

        _parallel_slices(B, _out)
        S = s_h.numpy().copy()
    U = np.swapaxes(Uc, 1, 2)
    V = np.swapaxes(Vc, 1, 2) if Vc is not None else None
    info = np.frombuffer(info_h.numpy().tobytes(), dtype=INFO_DTYPE)
    return U, S, V, info, kern
