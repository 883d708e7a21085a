"""Executed warp instructions by opcode from an ncu source-page CSV (--print-source sass)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
isrc, iex = hdr.index('Source'), hdr.index('Instructions Executed')
c = Counter()
for r in rows[2:]:
    if len(r) <= iex or not r[iex]:
        continue
    t = r[isrc].split()
    if not t:
        continue
    op = t[1] if t[0].startswith('@') and len(t) > 1 else t[0]
    c[op.split('.')[0]] += float(r[iex])
tot = sum(c.values())
print(f"total {tot:.3g}")
for op, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{op:10s} {v:10.3g} {v / tot * 100:5.1f}%")
