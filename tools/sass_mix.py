"""Aggregate an ncu source page (--page source --csv --print-source sass) by opcode: executed
warp instructions and stall samples (development aid)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
ex = collections.Counter(); samp = collections.Counter(); stall = collections.defaultdict(collections.Counter)
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot_s = 0
for r in data:
    if len(r) < len(h): continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    op = op.split(".")[0]
    e = float(r[ix["Instructions Executed"]] or 0); s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex[op] += e; samp[op] += s; tot_s += s
    for k in reasons:
        stall[op][k] += float(r[ix[k]] or 0)
tot = sum(ex.values())
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
print(f"total warp instr {tot:.4g}  per unit {tot/div:.1f}   stall samples {tot_s:.4g}")
allr = collections.Counter()
for op in stall:
    allr.update(stall[op])
print("stall reasons:", ", ".join(f"{k[6:]} {v/tot_s*100:.1f}%" for k, v in allr.most_common(8)))
for op, e in ex.most_common(25):
    top = ", ".join(f"{k[6:]} {v/max(samp[op],1)*100:.0f}%" for k, v in stall[op].most_common(3))
    print(f"{op:10s} {e/div:8.1f} /unit  samples {samp[op]/tot_s*100:5.1f}%  [{top}]")
