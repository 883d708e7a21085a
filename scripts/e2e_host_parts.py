"""Host-side parts of one psg_optimize_level-equivalent call with pinned buffers
(level create incl. the image copy, prime, 10 iterations, download)."""
import ctypes as ct
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import native as N  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402

cfg = wl.CONFIGS[3]
ex, init, W, H, sp = wl.stage_inputs(cfg, 2, 8)
ctx = api.Context(0)
ix = api.make_pca_tree_index(ex, 8, d_fixed=32, branching=8, max_depth=4, seed=1, hist_bins=16, ctx=ctx)
ocfg = api.OptimizerConfig(max_iterations=10, min_iterations=10, convergence_fraction=1e-9,
                           nbhd_width=8, spacing=sp, patch_width=2, budget=api.QueryBudget.exact())
pin = torch.empty(init.shape, dtype=torch.float64, pin_memory=True)
pin.numpy()[...] = init
outp = torch.empty(init.shape, dtype=torch.float64, pin_memory=True)
for rep in range(4):
    c = ocfg.c()
    h = ct.c_void_p()
    t0 = time.perf_counter()
    N.check(N.lib.psg_level_create(ctx.h, ix.h, ct.c_void_p(pin.data_ptr()), W, H, ct.byref(c),
                                   None, ct.byref(h)))
    ctx.synchronize()
    t1 = time.perf_counter()
    N.check(N.lib.psg_level_prime(h))
    t2 = time.perf_counter()
    st = (N.psg_iter_stats * 10)()
    n = ct.c_int()
    N.check(N.lib.psg_level_iterate(h, 10, 1, ct.cast(st, ct.c_void_p), ct.byref(n)))
    t3 = time.perf_counter()
    N.check(N.lib.psg_level_download(h, ct.c_void_p(outp.data_ptr()), None, None))
    t4 = time.perf_counter()
    N.lib.psg_level_destroy(h)
    ms = [st[i].millis for i in range(n.value)]
    print(f"create {1e3*(t1-t0):.2f} ms, prime {1e3*(t2-t1):.2f}, 10 its {1e3*(t3-t2):.2f} "
          f"(per-iteration ms {[round(m, 2) for m in ms]}), download {1e3*(t4-t3):.2f}")
