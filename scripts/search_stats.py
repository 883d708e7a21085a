"""Per-query search statistics of the bench stage (exact mode): points
scanned, exact fp64 evaluations and tree nodes visited, tile vs warp kernels."""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402


def main():
    cfg = wl.CONFIGS[3]
    w = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    ex, init, W, H, sp = wl.stage_inputs(cfg, 2, w)
    ctx = api.Context(0)
    ix = api.make_pca_tree_index(ex, w, d_fixed=cfg.d_fixed or 32, branching=cfg.branching,
                                 max_depth=cfg.depth, seed=cfg.seed, hist_bins=16, ctx=ctx)
    ocfg = api.OptimizerConfig(max_iterations=3, min_iterations=3, convergence_fraction=1e-9,
                               nbhd_width=w, spacing=sp, patch_width=2,
                               budget=api.QueryBudget.exact())
    lv = api.Level(init, ix, ocfg)
    lv.prime()
    lv.iterate(2)
    sc, exv, vi = lv.query_stats()
    out = {"w": w, "anchors": int(sc.size), "n_nodes": ix.n_nodes, "n_leaves": ix.n_leaves,
           "scanned_mean": float(sc.mean()), "exact_mean": float(exv.mean()),
           "visited_mean": float(vi.mean()),
           "scanned_p50_p90_p99": [float(np.percentile(sc, p)) for p in (50, 90, 99)]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
