"""Top SASS lines of an ncu source-page CSV (--print-source sass) by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, ist, iex = (hdr.index(k) for k in ('Address', 'Source', 'Warp Stall Sampling (All Samples)',
                                             'Instructions Executed'))
body = [r for r in rows[2:] if len(r) > iex]
tot = sum(float(r[ist] or 0) for r in body)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
iex_tot = sum(float(r[iex] or 0) for r in body)
print(f"samples {tot:.0f}, warp instructions {iex_tot:.3g}")
for r in sorted(body, key=lambda r: -float(r[ist] or 0))[:n]:
    print(f"{float(r[ist] or 0) / tot * 100:5.1f}% {float(r[iex] or 0):10.3g}  {r[ia]}  {r[isrc][:90]}")
