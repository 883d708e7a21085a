"""Generate the golden parity fixtures from the REFERENCE'S OWN CODE.

Run in the build container (needs oracle/_ref/libpersyn_ref.so, which is
compiled from /root/reference by oracle/Makefile):

    python tests/golden/make_golden.py

Every array in tests/golden/*.npz is an output of the reference's
translation units (neighborhood.cpp, km_tree.cpp, optimizer.cpp, image.cpp)
on seeded synthetic inputs that are stored alongside.  The PCA basis is
injected (the reference's fit_pca needs Eigen3, which is absent — SURVEY §8c).
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Port, Ref, fit_pca  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402

OUT = Path(__file__).resolve().parent


def em_case(ref, port, name, ex_size, out, w, sp, d, iters, hist, seed):
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(ex_size, 8, 2.0, seed), 1)
    init = wl.init_output(ex, out, out, 1, seed)
    cand = ref.extract_all(ex, w, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=d)
    h = ref.index_create(ex, w, mean, basis, kind="tree", branching=4, seed=seed)
    idx, dist, calls, _ = h.search_step(init, w, sp, 2, mode="exact")
    rng = np.random.Generator(np.random.PCG64(seed))
    irls = ref.irls_weights(dist, 0.8, 1e-4)
    pen = rng.uniform(0.0, 0.5, idx.size)
    upd = h.update_step(init, w, sp, idx, irls, pen)
    out_p, stats, _ = h.optimize_level(init, w, sp, 2, max_it=iters, min_it=iters, frac=1e-9,
                                       bins=16, hist_on=hist, mode="exact")
    np.savez_compressed(
        OUT / f"{name}.npz", exemplar=ex, init=init, w=w, sp=sp, d=d, mean=mean, basis=basis,
        projected=h.projected(), search_idx=idx, search_dist=dist, nn_calls=calls,
        irls=irls, pen=pen, update=upd, em_planes=out_p, em_stats=stats, iters=iters,
        hist=int(hist), ex_hist=ref.build_histograms(ex, 16))


def ann_case(ref):
    rng = np.random.Generator(np.random.PCG64(53))
    rows = []
    for count, dim in [(1, 3), (10, 3), (100, 20), (1000, 20), (500, 1)]:
        pts = rng.uniform(-1, 1, (count, dim))
        qs = rng.uniform(-1.2, 1.2, (25, dim))
        h = ref.kmtree_build(pts, 4, 4, 7)
        res = [ref.kmtree_query(h, q, "exact")[:2] for q in qs]
        ref.kmtree_destroy(h)
        rows.append((pts, qs, np.array([r[0] for r in res], np.int32),
                     np.array([r[1] for r in res])))
    np.savez_compressed(OUT / "ann_exact.npz",
                        **{f"pts{i}": r[0] for i, r in enumerate(rows)},
                        **{f"qs{i}": r[1] for i, r in enumerate(rows)},
                        **{f"idx{i}": r[2] for i, r in enumerate(rows)},
                        **{f"dist{i}": r[3] for i, r in enumerate(rows)}, n=len(rows))


def main():
    ref, port = Ref(), Port()
    em_case(ref, port, "em_cfg0_small", 32, 48, 8, 4, 12, 3, True, 1)
    em_case(ref, port, "em_sp2_nohist", 28, 40, 8, 2, 10, 2, False, 2)
    ann_case(ref)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
