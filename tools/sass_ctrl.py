"""Decode the scheduling control bits (stall, yield, barriers) of every SASS
instruction of one kernel: cuobjdump -sass <cubin> | python sass_ctrl.py <kernel-substring> [op-filter]."""
import re, sys
txt = sys.stdin.read().splitlines()
want = sys.argv[1]; opf = sys.argv[2] if len(sys.argv) > 2 else None
cur = None; out = []
i = 0
while i < len(txt):
    l = txt[i]
    if 'Function :' in l:
        cur = l.split('Function :')[1].strip()
    m = re.search(r'/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;\s*/\* (0x[0-9a-f]+) \*/', l)
    if m and cur and want in cur:
        m2 = re.search(r'/\* (0x[0-9a-f]+) \*/', txt[i + 1])
        lo = int(m.group(3), 16); hi = int(m2.group(1), 16)
        w = (hi << 64) | lo
        stall = (w >> 105) & 0xf; yld = (w >> 109) & 1; wb = (w >> 110) & 7; rb = (w >> 113) & 7; wm = (w >> 116) & 0x3f
        out.append((m.group(1), stall, yld, wb, rb, wm, m.group(2)))
        i += 2; continue
    i += 1
for a, s, y, wb, rb, wm, ins in out:
    if opf is None or opf in ins:
        print(f"{a} s{s:2d} y{y} wb{wb} rb{rb} wm{wm:02x}  {ins[:80]}")
