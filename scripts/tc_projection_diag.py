import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2006_11851_b200 import api, workloads as wl
cfg = wl.CONFIGS[3]
for G, out, w in [(2, 256, 8), (1, 128, 8), (2, 1024, 8), (2, 256, 16), (1, 96, 4)]:
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(64 if out < 1024 else 256, 16, 3.0, 1), G)
    init = wl.init_output(ex, out, out, G, 1)
    ix = api.make_pca_tree_index(ex, w, d_fixed=32, branching=8, max_depth=4, seed=1)
    sp = max(1, w // 4)
    qt, dl, qe = api.debug_projection(init, ix, sp)
    err = np.sqrt(((qt - qe) ** 2).sum(1))
    print(G, out, w, "max err", err.max(), "delta median", np.median(dl), "max", dl.max(),
          "violations", int((err > dl).sum()), "ratio max", (err / dl).max(), flush=True)
