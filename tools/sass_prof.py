"""Summarise an ncu source page (--page source --csv --print-source sass): stall mix, opcode mix,
and the hottest instructions.  Development aid."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1], errors='replace')))
hdr = next(r for r in rows if r and r[0] == 'Address')
data = [r for r in rows if len(r) == len(hdr) and r[0] not in ('Address', 'Kernel Name')]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
f = lambda r, k: float(r[ix[k]] or 0)
tot = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in data)
print('total samples', tot, 'ninstr', len(data))
agg = Counter()
for r in data:
    for s in stalls: agg[s] += f(r, s)
for s, v in agg.most_common(12): print(f"{s:28s} {v/tot*100:5.1f}%")
c = Counter(); cs = Counter()
for r in data:
    toks = r[ix['Source']].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith('@') else toks[0]
    op = op.split('.')[0]
    c[op] += f(r, 'Instructions Executed'); cs[op] += f(r, 'Warp Stall Sampling (All Samples)')
T = sum(c.values())
print('warp instructions executed', T)
for op, v in c.most_common(25): print(f"{op:10s} exec {v/T*100:5.1f}%  samples {cs[op]/tot*100:5.1f}%")
if len(sys.argv) > 2:
    top = sorted(range(len(data)), key=lambda i: -f(data[i], 'Warp Stall Sampling (All Samples)'))[:int(sys.argv[2])]
    for i in sorted(top):
        r = data[i]
        st = sorted(((f(r, s), s[6:]) for s in stalls), reverse=True)[:3]
        print(f"{i:5d} {r[ix['Address']]:>6s} {f(r,'Warp Stall Sampling (All Samples)'):6.0f} {r[ix['Source']][:60]:60s} " +
              " ".join(f"{n}:{v:.0f}" for v, n in st))
