"""Print the key section metrics of an ncu --csv capture (one row per launch)."""
import csv
import sys
from collections import OrderedDict

WANT = ['Duration', 'Achieved Occupancy', 'Registers Per Thread', 'DRAM Throughput', 'L1/TEX Hit Rate',
        'L2 Hit Rate', 'Compute (SM) Throughput', 'Issue Slots Busy', 'L1/TEX Cache Throughput',
        'L2 Cache Throughput', 'Theoretical Occupancy', 'Dynamic Shared Memory Per Block',
        'Warp Cycles Per Issued Instruction', 'Block Limit Shared Mem', 'Grid Size']
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'ID'))
d = OrderedDict()
for r in rows[1:]:
    if r[mi] in WANT:
        d.setdefault((r[ii], r[ki][:44]), {})[r[mi]] = r[vi]
for k, v in d.items():
    print(k, {m: v[m] for m in WANT if m in v})
