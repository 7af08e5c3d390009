"""Time the REFERENCE's own CPU path (numba backend, batch_svd with design4) on this host's cores, beside the
oracle/ C++ port -- SURVEY 8(d)'s CPU protocol (development tool; the reference package is the unmodified
/root/reference/pkg installed into baseline/_ref, which travels to the GPU box with the snapshot):

    python -m pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of /root/reference/pkg>
    python tools/ref_numba_time.py [config ...]     (on the GPU box: gpurun -- python tools/ref_numba_time.py)

N forked worker processes (N = usable cores), OPENBLAS_NUM_THREADS=1, numba cache warmed first; each worker builds
its strided share (i::N) of the inputs (reference gen_batch, seeds 0..B-1) before a barrier; wall = max(end) -
min(start).  Also one core on a prefix.  Prints one JSON line per config.
"""

from __future__ import annotations

import json
import multiprocessing as mp
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bsvd")
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

CONFIGS = {  # id: (family, m, n, kappa, dtype, batch, want_v, one-core prefix, multi-core sample)
    "c1-10k": ("arith", 32, 32, 1e10, "float64", 10000, True, 1000, 10000),
    "c2-full": ("random", 16, 16, 1.0, "float32", 10000, True, 2000, 10000),
    "c3-geo": ("geo", 64, 64, 1e12, "float64", 10000, True, 16, 400),
    "c4": ("random", 256, 32, 1.0, "complex128", 5000, True, 8, 200),
    "c5": ("random", 128, 128, 1.0, "float64", 2000, True, 4, 100),
}


def _problems(cfg, idx):
    import numpy as np
    from bsvd.matgen import SpectrumSpec, gen_matrix

    fam, m, n, kappa, dt = cfg[:5]
    return [gen_matrix(m, SpectrumSpec(fam, n, kappa=kappa, seed=int(i)), dtype=np.dtype(dt)) for i in idx]


def _worker(cfg, idx, barrier, q):
    from bsvd import JacobiOptions, batch_svd
    from bsvd.cli import design_options

    probs = _problems(cfg, idx)
    opts = design_options("design4", JacobiOptions(compute_right_vectors=cfg[6]))
    barrier.wait()
    t0 = time.perf_counter()
    batch_svd(probs, opts)
    q.put((t0, time.perf_counter(), len(probs)))


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    import numba
    import numpy as np
    from bsvd import JacobiOptions, backend, batch_svd
    from bsvd.cli import design_options

    assert backend.active().name == "numba", backend.active().name
    cores = len(os.sched_getaffinity(0))
    ids = sys.argv[1:] or list(CONFIGS)
    # warm the numba cache (compile once in the parent; forked children inherit it)
    batch_svd(_problems(CONFIGS["c1-10k"], range(2)), design_options("design4"))
    batch_svd(_problems(CONFIGS["c4"], range(1)), design_options("design4"))
    for cid in ids:
        cfg = CONFIGS[cid]
        pre = cfg[7]
        probs = _problems(cfg, range(pre))
        opts = design_options("design4", JacobiOptions(compute_right_vectors=cfg[6]))
        t0 = time.perf_counter()
        batch_svd(probs, opts)
        one = pre / (time.perf_counter() - t0)
        count = cfg[8]
        ctx = mp.get_context("fork")
        barrier, q = ctx.Barrier(cores), ctx.Queue()
        procs = [ctx.Process(target=_worker, args=(cfg, np.arange(w, count, cores), barrier, q)) for w in range(cores)]
        for p in procs:
            p.start()
        res = [q.get() for _ in procs]
        for p in procs:
            p.join()
        wall = max(r[1] for r in res) - min(r[0] for r in res)
        # the oracle/ C++ port (bench.py's reference arm) on the same problems, same cores
        sys.path.insert(0, ROOT)
        from oracle import oracle as O

        A = np.stack(_problems(cfg, range(count)))
        t0 = time.perf_counter()
        O.solve_batch(A, None, None, nthreads=cores)
        port = count / (time.perf_counter() - t0)
        print(json.dumps({"config": cid, "impl": "reference numba batch_svd design4", "cores": cores,
                          "matrices_per_s": count / wall, "sample": f"{count} of {cfg[5]} (reference gen_batch seeds)",
                          "one_core_matrices_per_s": one, "one_core_sample": pre,
                          "port_matrices_per_s": port, "port_over_numba": port / (count / wall),
                          "cpu": _cpu_model(), "numpy": np.__version__, "numba": numba.__version__,
                          "python": platform.python_version()}), flush=True)


if __name__ == "__main__":
    main()
