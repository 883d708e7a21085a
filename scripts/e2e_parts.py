"""Where an end-to-end psg_optimize_level call spends its time (cfg3 finest)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402


def main():
    cfg = wl.CONFIGS[3]
    ex, init, W, H, sp = wl.stage_inputs(cfg, 2, 8)
    ctx = api.Context(0)
    ix = api.make_pca_tree_index(ex, 8, d_fixed=32, branching=8, max_depth=4, seed=1,
                                 hist_bins=16, ctx=ctx)
    ocfg = api.OptimizerConfig(max_iterations=10, min_iterations=10, convergence_fraction=1e-9,
                               nbhd_width=8, spacing=sp, patch_width=2,
                               budget=api.QueryBudget.exact())
    for rep in range(3):
        t0 = time.perf_counter()
        lv = api.Level(init, ix, ocfg)
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
        print(f"create {1e3*(t1-t0):.2f} ms, prime {1e3*(t2-t1):.2f}, 10 its {1e3*(t3-t2):.2f}, "
              f"download {1e3*(t4-t3):.2f}, destroy {1e3*(t5-t4):.2f}")


if __name__ == "__main__":
    main()
