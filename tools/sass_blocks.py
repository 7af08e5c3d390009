"""Per-basic-block (same execution count, contiguous) summary of an ncu SASS source page:
instructions executed, stall samples, top stall reasons, opcode mix.  Development aid."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1]))); hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
f = lambda r, k: float(r[ix[k]] or 0)
tot = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in data)
blocks = []; cur = None
for i, r in enumerate(data):
    ex = round(f(r, 'Instructions Executed') / 1e5)
    if cur is None or ex != cur['ex']:
        cur = dict(ex=ex, start=i, n=0, smp=0.0, st=Counter(), ops=Counter(), instr=0.0); blocks.append(cur)
    cur['n'] += 1; cur['smp'] += f(r, 'Warp Stall Sampling (All Samples)'); cur['instr'] += f(r, 'Instructions Executed')
    for s in stalls: cur['st'][s[6:]] += f(r, s)
    toks = r[ix['Source']].split()
    if toks:
        op = toks[1] if toks[0].startswith('@') else toks[0]
        cur['ops'][op.split('.')[0] + ('.MOV' if op.startswith('IMAD.MOV') else '')] += 1
minf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for b in blocks:
    if b['smp'] / tot < minf: continue
    st = ", ".join(f"{k}:{v/b['smp']*100:.0f}%" for k, v in b['st'].most_common(4))
    ops = " ".join(f"{k}{v}" for k, v in b['ops'].most_common(6))
    print(f"[{b['start']:5d}+{b['n']:4d}] exec/1e5={b['ex']:4d} samples {b['smp']/tot*100:5.1f}%  instr {b['instr']/1e6:7.1f}M | {st} | {ops}")
