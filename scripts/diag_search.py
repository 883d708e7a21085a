"""Search diagnostics on the bench workload: per-query scanned / exact / visited."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import bench
from paper_2006_11851_b200 import api

w = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg, ex, init, sp = bench.stage_inputs(2, w)
ctx = api.Context(0)
t = time.time()
ix = api.make_pca_tree_index(ex, w, d_fixed=32, branching=8, max_depth=4, seed=1, hist_bins=16, ctx=ctx)
print("index build", time.time() - t, "N", ix.count, "leaves", ix.n_leaves, "nodes", ix.n_nodes)
oc = api.OptimizerConfig(max_iterations=100, min_iterations=99, convergence_fraction=1e-9,
                         nbhd_width=w, spacing=sp, budget=api.QueryBudget.exact())
L = api.Level(init, ix, oc)
ctx.profile(True)
L.prime()
def show(tag):
    sc, exv, vi = L.query_stats()
    kt = ctx.kernel_times()
    print(tag, json.dumps({k: round(v[0] / max(v[1], 1), 3) for k, v in kt.items()}))
    for name, v in (("scanned", sc), ("exact", exv), ("visited", vi)):
        print(f"  {name:8s} mean {v.mean():9.1f}  p50 {np.percentile(v,50):8.0f}  p99 {np.percentile(v,99):8.0f}  max {v.max():8d}")
    ctx.profile(True)
show("prime")
for it in range(4):
    st = L.iterate(1)
    show(f"iter{it+1} changed={st[0].changed}")
