"""EM iterations of one BASELINE stage through a device-resident Level.

usage: python scripts/stage_bench.py <cfg> <level> <w> [iters] [budget]
budget: exact (default) | backtrack:m | greedy.  Prints index build time,
ms per EM iteration, per-kernel device times and search statistics.
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402


def main():
    cid, level, w = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    iters = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    bud = sys.argv[5] if len(sys.argv) > 5 else "exact"
    budget = (api.QueryBudget.exact() if bud == "exact" else api.QueryBudget.greedy()
              if bud == "greedy" else api.QueryBudget.backtrack(int(bud.split(":")[1])))
    cfg = wl.CONFIGS[cid]
    ex, init, W, H, sp = wl.stage_inputs(cfg, level, w)
    ctx = api.Context(0)
    t = time.perf_counter()
    ix = api.make_pca_tree_index(ex, w, variance_target=0.95, d_cap=cfg.d_cap,
                                 d_fixed=cfg.d_fixed, branching=cfg.branching,
                                 max_depth=cfg.depth, seed=cfg.seed, hist_bins=16, ctx=ctx)
    ctx.synchronize()
    t_build = time.perf_counter() - t
    ocfg = api.OptimizerConfig(max_iterations=10 ** 6, min_iterations=10 ** 6 - 1,
                               convergence_fraction=1e-9, nbhd_width=w, spacing=sp,
                               patch_width=2, budget=budget)
    lv = api.Level(init, ix, ocfg)
    t = time.perf_counter()
    lv.prime()
    ctx.synchronize()
    t_prime = time.perf_counter() - t
    lv.iterate(2)  # warm-up
    ctx.synchronize()
    ctx.profile(True)
    t = time.perf_counter()
    st = lv.iterate(iters)
    ctx.synchronize()
    t_it = (time.perf_counter() - t) / iters
    kt = ctx.kernel_times()
    ctx.profile(False)
    sc, ex_ev, vi = lv.query_stats()
    print(json.dumps({
        "config": cfg.name, "level": level, "w": w, "W": W, "H": H, "budget": bud,
        "N": ix.count, "D": ix.dim, "d": ix.retained_dim, "tree_nodes": ix.n_nodes,
        "anchors": int(sc.size), "index_build_s": t_build, "prime_ms": 1e3 * t_prime,
        "ms_per_iteration": 1e3 * t_it, "iterations_per_s": 1.0 / t_it,
        "kernels_ms_per_iteration": {k: round(v[0] / iters, 3) for k, v in kt.items()},
        "points_scanned_per_query": float(sc.mean()), "exact_evals_per_query": float(ex_ev.mean()),
        "energy": [s.energy for s in st][-1]}))


if __name__ == "__main__":
    main()
