"""Exact-mode search cost vs k-means tree shape on the bench stage.

Exact answers are tree-independent (lexicographic min), so the tree shape is a
pure performance knob for exact mode.  usage: python scripts/tree_shape_sweep.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402


def main():
    cfg = wl.CONFIGS[3]
    w = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    shapes = [(8, 4), (8, 3), (16, 3), (4, 6), (4, 7), (16, 4), (8, 5), (6, 5), (12, 4), (2, 12)]
    ex, init, W, H, sp = wl.stage_inputs(cfg, 2, w)
    ctx = api.Context(0)
    ref = None
    for b, depth in shapes:
        ix = api.make_pca_tree_index(ex, w, d_fixed=cfg.d_fixed or 32, branching=b,
                                     max_depth=depth, seed=cfg.seed, hist_bins=16, ctx=ctx)
        ocfg = api.OptimizerConfig(max_iterations=10 ** 6, min_iterations=10 ** 6 - 1,
                                   convergence_fraction=1e-9, nbhd_width=w, spacing=sp,
                                   patch_width=2, budget=api.QueryBudget.exact())
        lv = api.Level(init, ix, ocfg)
        lv.prime()
        lv.iterate(2)
        ctx.synchronize()
        ctx.profile(True)
        st = lv.iterate(5)
        ctx.synchronize()
        kt = ctx.kernel_times()
        ctx.profile(False)
        sc, exv, vi = lv.query_stats()
        e = st[-1].energy
        if ref is None:
            ref = e
        print(json.dumps({"b": b, "depth": depth, "nodes": ix.n_nodes, "leaves": ix.n_leaves,
                          "search_ms": round(kt["search_kernel"][0] / 5, 3), "scanned": float(sc.mean()),
                          "visited": float(vi.mean()), "exact": float(exv.mean()),
                          "same_energy": e == ref}), flush=True)


if __name__ == "__main__":
    main()
