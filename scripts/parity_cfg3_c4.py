"""Full-size parity evidence for the bench stage: BASELINE cfg3 finest stage
(256^2 exemplar, 1024^2 output, w = 8, sp = 2: 259,081 anchors, 4,145,296
plan calls per search) with ONE guidance plane (C = 4, the reference's own
layout), d = 32 injected, exact search, histogram matching on: the device's
optimize_level vs the reference's optimize_level (oracle/_ref, all host
threads) for `iters` EM iterations.  Prints one JSON line (kept under
profiles/).  usage: python scripts/parity_cfg3_c4.py [iters]
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle.oracle import Port, Ref, fit_pca  # noqa: E402  (checker only)
from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    cfg = wl.CONFIGS[3]
    ex, init, W, H, sp = wl.stage_inputs(cfg, 2, 8, G=1)
    port, ref = Port(), Ref()
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=32)
    ctx = api.Context(0)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, max_depth=4,
                                 hist_bins=16, ctx=ctx)
    ocfg = api.OptimizerConfig(max_iterations=iters, min_iterations=iters,
                               convergence_fraction=1e-9, nbhd_width=8, spacing=sp,
                               patch_width=2, budget=api.QueryBudget.exact())
    t = time.perf_counter()
    out, stats = api.optimize_level(init, ix, ocfg)
    t_dev = time.perf_counter() - t
    os.environ.setdefault("PERSYN_THREADS", str(os.cpu_count() or 1))
    h = ref.index_create(ex, 8, mean, basis, kind="tree", branching=8, seed=1)
    t = time.perf_counter()
    out_r, st_r, _ = h.optimize_level(init, 8, sp, 2, max_it=iters, min_it=iters, frac=1e-9,
                                      bins=16, hist_on=True, mode="exact")
    t_ref = time.perf_counter() - t
    q = lambda a: np.rint(np.clip(a, 0, 1) * 255)  # image_io.cpp:18-21
    line = {
        "what": "cfg3 finest stage, C=4, 1024^2, exact, device optimize_level vs reference",
        "iterations": iters, "anchors": int(stats[0].unique_queries),
        "max_abs_diff": float(np.max(np.abs(out - out_r))),
        "pixels_differing_gt_1e-12": int(np.sum(np.abs(out - out_r) > 1e-12)),
        "uint8_rgb_mismatches": int(np.sum(q(out[:3]) != q(out_r[:3]))),
        "stats_device": [[s.iteration, s.energy, s.changed, s.nn_calls] for s in stats],
        "stats_reference": [[int(r[0]), float(r[1]), int(r[2]), int(r[3])] for r in st_r],
        "energy_rel_diff": [abs(s.energy - r[1]) / abs(r[1]) for s, r in zip(stats, st_r)],
        "seconds_device_e2e": t_dev, "seconds_reference": t_ref,
        "reference_threads": int(os.environ["PERSYN_THREADS"]),
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
