"""The E-step's tensor-core projection (kernels_project_tc.cu, north_star:
"PCA ... runs on tensor cores").

q^ is computed exactly in integers on tcgen05.mma kind::i8 from digit slices
of the quantised window and basis; delta bounds |q^ - q| rigorously.  The
search keeps every candidate within the band and settles near-ties with the
reference's exact projection chain, so results stay bit-identical (every
exact-mode parity test runs through this path).  Here: the bound itself, the
out-of-range guard, and the exact fallback on tie-heavy inputs.
"""
import numpy as np
import pytest

from oracle.oracle import fit_pca
from paper_2006_11851_b200 import workloads as wl

pytestmark = pytest.mark.gpu

api = pytest.importorskip("paper_2006_11851_b200.api")


@pytest.mark.parametrize("G,w,d,out,ex_size", [(1, 8, 16, 96, 48), (2, 8, 32, 256, 64),
                                               (2, 16, 32, 128, 64), (1, 4, 12, 64, 32),
                                               (2, 8, 48, 160, 64), (1, 8, 64, 96, 48),
                                               (2, 32, 24, 160, 64),
                                               # spacing 4 / 8: the 5-D TMA tensor-map staging,
                                               # with a clamped (non-uniform) last anchor and
                                               # with several 128-anchor tiles per row
                                               (2, 16, 32, 134, 64), (1, 32, 24, 170, 64),
                                               (1, 16, 32, 600, 64)])
def test_projection_error_within_bound(gpu_ctx, port, G, w, d, out, ex_size):
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(ex_size, 16, 2.0, d), G)
    init = wl.init_output(ex, out, out, G, w)
    cand = port.extract_all(ex, w, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=d)
    ix = api.make_pca_tree_index(ex, w, mean=mean, basis=basis, branching=8, max_depth=3,
                                 ctx=gpu_ctx)
    sp = max(1, w // 4)
    qt, delta, qe = api.debug_projection(init, ix, sp)
    # q_exact is the reference's chain: compare a sample with the oracle
    xs = port.axis_positions(out, w, sp)
    for a in np.linspace(0, qe.shape[0] - 1, 7).astype(int):
        v = port.extract_window(init, xs[a % len(xs)], xs[a // len(xs)], w)
        assert np.array_equal(qe[a], port.project(v, mean, basis))
    err = np.sqrt(((qt - qe) ** 2).sum(axis=1))
    assert np.all(err <= delta), (err.max(), delta.min())
    assert np.all(np.isfinite(delta)) and delta.max() < 1e-4


def test_out_of_range_values_fall_back_exactly(gpu_ctx, port):
    """Values outside [0, 1] cannot be digit-quantised: every query's band is
    infinite and the whole search runs through the exact fallback."""
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(32, 8, 2.0, 5), 1)
    init = wl.init_output(ex, 48, 48, 1, 5)
    init[0, 10, 10] = 1.5
    init[1, 30, 3] = -0.25
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=12)
    proj = port.project_all(cand, mean, basis)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=4, max_depth=3,
                                 ctx=gpu_ctx)
    _, delta, _ = api.debug_projection(init, ix, 2)
    assert np.all(np.isinf(delta))
    idx, dist, calls, _ = api.search_step(init, ix, 2, 2, api.QueryBudget.exact())
    i_p, d_p, c_p = port.search_step(init, 8, 2, 2, cand, proj, mean, basis)
    assert np.array_equal(idx, i_p) and np.array_equal(dist, d_p) and calls == c_p


def test_near_ties_settle_exactly(gpu_ctx, port):
    """A periodic exemplar: every window recurs, so every query has exact
    distance ties -- all of them go through the band fallback, and the lowest
    index must win (km_tree.cpp:134)."""
    tile = wl.sinusoid_exemplar(8, 4, 1.0, 3)
    ex = wl.rgbs_planes(np.tile(tile, (1, 6, 6)), 2)
    ex[3:] = 0.5
    init = wl.init_output(ex, 64, 64, 2, 2)
    init[3:] = 0.5
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=16)
    proj = port.project_all(cand, mean, basis)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, max_depth=3,
                                 ctx=gpu_ctx)
    for planes in (init, ex):
        idx, dist, _, _ = api.search_step(planes, ix, 2, 2, api.QueryBudget.exact())
        i_p, d_p, _ = port.search_step(planes, 8, 2, 2, cand, proj, mean, basis)
        assert np.array_equal(idx, i_p) and np.array_equal(dist, d_p)


def test_exact_projection_knob_same_result(gpu_ctx, port, monkeypatch):
    """PERSYN_EXACT_PROJECTION (the fp64 SIMT projection of every query) and
    the tensor-core path give the same EM run."""
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(40, 8, 2.0, 7), 2)
    init = wl.init_output(ex, 80, 80, 2, 7)
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=20)
    cfg = api.OptimizerConfig(max_iterations=3, min_iterations=3, convergence_fraction=1e-9,
                              nbhd_width=8, spacing=2, patch_width=2,
                              budget=api.QueryBudget.exact())
    runs = []
    for exact in (False, True):
        if exact:
            monkeypatch.setenv("PERSYN_EXACT_PROJECTION", "1")
        ctx = api.Context(0)
        monkeypatch.delenv("PERSYN_EXACT_PROJECTION", raising=False)
        ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, max_depth=4,
                                     hist_bins=16, ctx=ctx)
        runs.append(api.optimize_level(init, ix, cfg))
    (o1, s1), (o2, s2) = runs
    assert np.array_equal(o1, o2)
    assert [s.changed for s in s1] == [s.changed for s in s2]
