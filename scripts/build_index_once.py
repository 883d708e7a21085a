"""Build one BASELINE stage index (for profiling the index build).
usage: python scripts/build_index_once.py <cfg> <level> <w>"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402

cid, level, w = (int(a) for a in sys.argv[1:4])
cfg = wl.CONFIGS[cid]
ex, init, W, H, sp = wl.stage_inputs(cfg, level, w)
ctx = api.Context(0)
for _ in range(2):
    ix = api.make_pca_tree_index(ex, w, variance_target=0.95, d_cap=cfg.d_cap, d_fixed=cfg.d_fixed,
                                 branching=cfg.branching, max_depth=cfg.depth, seed=cfg.seed,
                                 hist_bins=16, ctx=ctx)
print("built", ix.count, ix.n_nodes)
