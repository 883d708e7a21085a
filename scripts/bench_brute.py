"""Brute-force index (pixel-brute mode) timing on BASELINE stages.

usage: python scripts/bench_brute.py [cfg] [level] [w] [iters]
Runs `iters` EM iterations of one stage with make_brute_force_index and prints
the per-kernel device times, filter survivors and the tf32 filter throughput.
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
    level = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    cfg = wl.CONFIGS[cid]
    ex, init, W, H, sp = wl.stage_inputs(cfg, level, w)
    ctx = api.Context(0)
    t = time.perf_counter()
    ix = api.make_brute_force_index(ex, w, hist_bins=16, ctx=ctx)
    t_build = time.perf_counter() - t
    ocfg = api.OptimizerConfig(max_iterations=iters, min_iterations=iters,
                               convergence_fraction=1e-9, nbhd_width=w, spacing=sp,
                               patch_width=2, budget=api.QueryBudget.backtrack(4))
    lv = api.Level(init, ix, ocfg)
    lv.prime()
    lv.iterate(1)                      # warm-up
    ctx.profile(True)
    st = lv.iterate(iters)
    times = ctx.kernel_times()
    ctx.profile(False)
    sc, ex_ev, _ = lv.query_stats()
    A = sc.size
    N, D = ix.count, ix.dim
    tot, n_l = times.get("search_kernel", (float("nan"), 1))
    search = {"ms_per_launch": tot / max(n_l, 1)}
    macs = A * N * D
    line = {"config": cfg.name, "level": level, "w": w, "W": W, "H": H, "N": N, "D": D,
            "anchors": A, "index_build_s": t_build, "iterations": len(st),
            "kernels": times,
            "search_ms": search["ms_per_launch"],
            "tf32_tflops": 2 * macs / (search["ms_per_launch"] * 1e-3) / 1e12,
            "exact_evals_per_query": float(ex_ev.mean()),
            "exact_evals_max": int(ex_ev.max()),
            "energy": [s.energy for s in st]}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
