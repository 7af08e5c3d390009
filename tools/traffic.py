"""Per-config DRAM traffic of the dominant solver kernel (development aid; run under ncu).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \\
        -k regex:'^k_' --csv --log-file traffic.csv python tools/traffic.py
    python tools/traffic.py --parse traffic.csv > profiles/ncu_traffic.json

One solve per bench config (same generator, seed and options as bench.py, rank 0), L2 cold (ncu flushes).
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ORDER = ["c1-10k", "c1", "c1r", "c2-full", "c2-vals", "c3-geo", "c3-rank", "c4", "c4-blocked", "c4-qr", "c5"]


def run():
    import numpy as np
    import torch

    import bench
    import paper_2601_17979_b200 as bs
    from paper_2601_17979_b200 import _lib
    from paper_2601_17979_b200.matgen import gen_batch_device
    from paper_2601_17979_b200.solver import solve_tensor

    for cid in ORDER:
        cfg = bench.CONFIGS[cid]
        dt = np.dtype(cfg["dtype"])
        a = gen_batch_device(cfg["family"], cfg["m"], cfg["n"], cfg["batch"], dt, kappa=cfg["kappa"], seed=0,
                             rank=cfg.get("rank"))
        opts = bs.JacobiOptions(compute_right_vectors=cfg["want_v"], use_qr_preprocess=cfg.get("use_qr", False))
        route = {None: _lib.DISPATCH, "blocked": _lib.FORCE_BLOCKED}[cfg["route"]]
        torch.cuda.nvtx.range_push(cid)
        solve_tensor(a, cfg["m"], cfg["n"], opts, route)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        print(cid, "done", file=sys.stderr, flush=True)


def parse(path):
    txt = open(path).read().splitlines()
    i = [k for k, l in enumerate(txt) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[i:]))))
    launches = {}
    for r in rows:
        key = int(r["ID"])
        d = launches.setdefault(key, {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    # launches come in bench-config order; a config's launches end with its finalisation / path kernel
    seq = [launches[k] for k in sorted(launches)]
    out = {"_source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none (tools/traffic.py): dram bytes per launch of each config's dominant "
                      "(longest) kernel, cold L2"}
    groups, cur = [], []
    for l in seq:
        cur.append(l)
        if "finalize" in l["name"] or "qr_path" in l["name"]:
            groups.append(cur)
            cur = []
    merged = []
    for g in groups:  # the QR route finalises R's factors before applying Q: keep those together
        if merged and ("applyq" in g[0]["name"] or "qr_path" in g[0]["name"]):
            merged[-1].extend(g)
        else:
            merged.append(g)
    for cid, g in zip(ORDER, merged):
        top = max(g, key=lambda l: l.get("gpu__time_duration.sum", 0))
        out[cid] = int(top.get("dram__bytes_read.sum", 0) + top.get("dram__bytes_write.sum", 0))
        out["_kernel_" + cid] = top["name"][:90]
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--parse":
        print(json.dumps(parse(sys.argv[2]), indent=2))
    else:
        run()
