"""Full coarse-to-fine synthesis of a BASELINE config through psg_synthesize.

usage: python scripts/run_synthesize.py <cfg id> [iterations] [budget] [tree]
  budget: exact (default) | greedy | backtrack:<m>      tree: device (default) | reference
Prints per-stage timings (index build / optimize) and the totals as JSON.
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
    cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    cfg = wl.CONFIGS[cid]
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.iterations
    rgb = wl.sinusoid_exemplar(cfg.ex_size, cfg.n_sin, cfg.ramp, cfg.seed, cfg.lum_gain)
    ex = wl.rgbs_planes(rgb, cfg.G)
    bname = sys.argv[3] if len(sys.argv) > 3 else "exact"
    budget = (api.QueryBudget.exact() if bname == "exact" else api.QueryBudget.greedy()
              if bname == "greedy" else api.QueryBudget.backtrack(int(bname.split(":")[1])))
    tree = sys.argv[4] if len(sys.argv) > 4 else "device"
    ocfg = api.OptimizerConfig(max_iterations=iters, min_iterations=iters,
                               convergence_fraction=1e-9, budget=budget)
    ctx = api.Context(0)
    t = time.perf_counter()
    out, rep = api.synthesize(ex, cfg.out, cfg.out, cfg.levels, cfg.sizes, ocfg,
                              variance_target=0.95, d_cap=cfg.d_cap, d_fixed=cfg.d_fixed,
                              branching=cfg.branching, seed=cfg.seed, ctx=ctx,
                              max_depth=0 if tree == "reference" else cfg.depth,
                              tree_kind=api.TREE_REFERENCE if tree == "reference" else api.TREE_DEVICE)
    wall = time.perf_counter() - t
    n_it = sum(s["iterations"] for s in rep["stages"])
    line = {"config": cfg.name, "budget": bname, "tree": tree, "out": cfg.out, "levels": cfg.levels, "sizes": list(cfg.sizes),
            "wall_s": wall, "em_iterations": n_it,
            "index_build_s": sum(s["index_millis"] for s in rep["stages"]) / 1e3,
            "optimize_s": sum(s["optimize_millis"] for s in rep["stages"]) / 1e3,
            "final_energy": rep["final_energy"], "total_nn_calls": rep["total_nn_calls"],
            "image_range": [float(out.min()), float(out.max())],
            "stages": [{k: (round(v, 2) if isinstance(v, float) else v) for k, v in s.items()
                        if isinstance(v, (int, float, str))} for s in rep["stages"]]}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
