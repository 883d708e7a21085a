"""Debug: single-device vs row-band results after a multi-resolution synthesize run."""
import os, sys
import numpy as np
sys.path.insert(0, '.')
from paper_2006_11851_b200 import api, sharding as sh, workloads as wl
from oracle.oracle import Port, fit_pca

ctx = api.default_context()
if "--warm" in sys.argv:
    ex0 = wl.rgbs_planes(wl.sinusoid_exemplar(64, 16, 2.0, 1), 1)
    c0 = api.OptimizerConfig(max_iterations=2, min_iterations=2, convergence_fraction=1e-9,
                             budget=api.QueryBudget.exact())
    api.synthesize(ex0, 128, 128, 2, (16, 8), c0, variance_target=0.95, d_cap=32, branching=8,
                   max_depth=3, seed=1)
port = Port()
G, ex_size, out, seed, d = 2, 40, 96, 3, 12
ex = wl.rgbs_planes(wl.sinusoid_exemplar(ex_size, 8, 2.0, seed), G)
init = wl.init_output(ex, out, out, G, seed)
cand = port.extract_all(ex, 8, 1)
mean, basis, _ = fit_pca(cand, d_fixed=d)
proj = port.project_all(cand, mean, basis)
exm = port.build_histograms(ex, 16, 3)
ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, max_depth=4, hist_bins=16, ctx=ctx)
cfg = api.OptimizerConfig(max_iterations=3, min_iterations=3, convergence_fraction=1e-9, nbhd_width=8,
                          spacing=2, patch_width=2, budget=api.QueryBudget.exact())
r1, s1 = api.optimize_level(init, ix, cfg)
out_p, st_p = port.optimize_level(init, 8, 2, 2, cand, proj, mean, basis, max_it=3, min_it=3,
                                  frac=1e-9, bins=16, ex_mass=exm)
print("single vs port maxdiff", np.abs(r1 - out_p).max(), [s.changed for s in s1], [int(r[2]) for r in st_p])
# per-iteration search results of the single-device level vs the port
L = api.Level(init, ix, cfg)
L.prime()
for it in range(3):
    planes, idx, dist = L.download()
    i_p, d_p, _ = port.search_step(planes, 8, 2, 2, cand, proj, mean, basis)
    bad = np.nonzero(idx != i_p)[0]
    print("iter", it, "mismatches", bad.size, bad[:10], "dist mism", int((dist != d_p).sum()))
    L.iterate(1)
for world in ((2, 3) if "--skip" not in sys.argv else ()):
    plans = sh.all_plans(out, out, 8, 2, world)
    bands = [sh.GpuBand(ix, init, p, plans, cfg) for p in plans]
    stats = sh.run_sharded(bands, sh.LoopbackComm(world), 3, 3)
    img = sh.gather_image([b.owned()[0] for b in bands])
    print("world", world, "vs single", np.abs(img - r1).max(), "vs port", np.abs(img - out_p).max())

# per-iteration check of each band's search against the port on the global image
world = 3
plans = sh.all_plans(out, out, 8, 2, world)
bands = [sh.GpuBand(ix, init, p, plans, cfg) for p in plans]
for b in bands:
    b.prime()
nx = plans[0]["nx"]
for it in range(4):
    img = sh.gather_image([b.owned()[0] for b in bands])
    print("image vs port-run at", it, "maxdiff n/a") if it < 3 else print("final vs single", np.abs(img - r1).max())
    if it == 3:
        break
    i_p, d_p, _ = port.search_step(img, 8, 2, 2, cand, proj, mean, basis)
    for r, b in enumerate(bands):
        _, idx, dist = b.owned()
        p = plans[r]
        sl = slice(p["a0"] * nx, p["a1"] * nx)
        bad = np.nonzero(idx != i_p[sl])[0]
        print("iter", it, "rank", r, "idx mismatches", bad.size, (bad[:8] + p["a0"] * nx).tolist(),
              "dist mism", int((dist != d_p[sl]).sum()))
    sh.em_iteration(bands, sh.LoopbackComm(world))
