"""Where an end-to-end psg_optimize_level call spends its time (cfg3 finest).

usage: python scripts/e2e_parts.py [exact | backtrack:<m>]   (pinned host buffers)"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402


def main():
    bud = sys.argv[1] if len(sys.argv) > 1 else "exact"
    cfg = wl.CONFIGS[3]
    ex, init, W, H, sp = wl.stage_inputs(cfg, 2, 8)
    ctx = api.Context(0)
    if bud == "exact":
        ix = api.make_pca_tree_index(ex, 8, d_fixed=32, branching=8, max_depth=4, seed=1,
                                     hist_bins=16, ctx=ctx)
        budget = api.QueryBudget.exact()
    else:
        ix = api.make_pca_tree_index(ex, 8, d_fixed=32, branching=8, seed=1, hist_bins=16,
                                     tree_kind=api.TREE_REFERENCE, ctx=ctx)
        budget = api.QueryBudget.backtrack(int(bud.split(":")[1]))
    ocfg = api.OptimizerConfig(max_iterations=10, min_iterations=10, convergence_fraction=1e-9,
                               nbhd_width=8, spacing=sp, patch_width=2, budget=budget)
    pin = torch.empty(init.shape, dtype=torch.float64, pin_memory=True)
    pin.numpy()[...] = init
    init_p = pin.numpy()
    for rep in range(3):
        t0 = time.perf_counter()
        lv = api.Level(init_p, ix, ocfg)
        t0b = time.perf_counter()
        ctx.synchronize()
        t1 = time.perf_counter()
        ctx.profile(True)
        lv.prime()
        ctx.synchronize()
        if rep == 2:
            print("prime kernels", {k: round(v[0], 3) for k, v in ctx.kernel_times().items()})
        ctx.profile(False)
        ctx.synchronize()
        t2 = time.perf_counter()
        lv.iterate(10)
        ctx.synchronize()
        t3 = time.perf_counter()
        lv.download()
        t4 = time.perf_counter()
        del lv
        t5 = time.perf_counter()
        print(f"create {1e3*(t1-t0):.2f} ms (host part {1e3*(t0b-t0):.2f}), prime {1e3*(t2-t1):.2f}, "
              f"10 its {1e3*(t3-t2):.2f}, download (pageable) {1e3*(t4-t3):.2f}, destroy {1e3*(t5-t4):.2f}")


if __name__ == "__main__":
    main()
