"""Per-CUDA-line stall samples and executed warp instructions from an ncu
source-page CSV exported with --print-source cuda,sass."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[2]
il, isrc, ia = 0, 1, 2
ist = hdr.index('Warp Stall Sampling (All Samples)')
iex = hdr.index('Instructions Executed')
lines = []
for r in rows[3:]:
    if len(r) > iex and r[ia] == '-' and r[il].isdigit():
        lines.append((int(r[il]), r[isrc], float(r[ist] or 0), float(r[iex] or 0)))
ts = sum(l[2] for l in lines)
te = sum(l[3] for l in lines)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print(f"samples {ts:.0f} instr {te:.3g}")
for ln, src, st, ex in sorted(lines, key=lambda l: -l[2])[:n]:
    print(f"{st / ts * 100:5.1f}% {ex / te * 100:5.1f}%i  L{ln:5d} {src.strip()[:95]}")
