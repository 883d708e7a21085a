"""Every device code path that can serve a request gives the same answer.

The library picks a kernel per request (tile search, tcgen05 / mma.sync tile
variants, warp-per-query fallback, thread-per-query budget kernel; subspace
iteration or the direct eigensolver for the PCA fit; device or host tree
build).  Selection can be forced per context with PERSYN_SEARCH /
PERSYN_EIG / PERSYN_TREE; each variant is checked against the oracle here.
"""
import numpy as np
import pytest

from oracle.oracle import fit_pca
from paper_2006_11851_b200 import workloads as wl

pytestmark = pytest.mark.gpu

api = pytest.importorskip("paper_2006_11851_b200.api")


def _stage(size=40, out=56, G=2, seed=4):
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(size, 8, 2.0, seed), G)
    init = wl.init_output(ex, out, out, G, seed)
    return ex, init


@pytest.mark.parametrize("variant", ["default", "warp"])
@pytest.mark.parametrize("d", [16, 32, 48])
def test_exact_search_variants_bit_exact(port, monkeypatch, variant, d):
    if variant != "default":
        monkeypatch.setenv("PERSYN_SEARCH", variant)
    ctx = api.Context(0)
    monkeypatch.delenv("PERSYN_SEARCH", raising=False)
    ex, init = _stage()
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=d)
    proj = port.project_all(cand, mean, basis)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, max_depth=3,
                                 hist_bins=16, ctx=ctx)
    i_p, d_p, c_p = port.search_step(init, 8, 2, 2, cand, proj, mean, basis)
    idx, dist, calls, _ = api.search_step(init, ix, 2, 2, api.QueryBudget.exact())
    assert calls == c_p
    assert np.array_equal(idx, i_p) and np.array_equal(dist, d_p)
    # a seeded (EM) search goes through the same kernels with a previous assignment
    cfg = api.OptimizerConfig(max_iterations=2, min_iterations=2, convergence_fraction=1e-9,
                              nbhd_width=8, spacing=2, patch_width=2,
                              budget=api.QueryBudget.exact())
    out, stats = api.optimize_level(init, ix, cfg)
    exm = port.build_histograms(ex, 16, 3)
    out_p, st_p = port.optimize_level(init, 8, 2, 2, cand, proj, mean, basis, max_it=2,
                                      min_it=2, frac=1e-9, bins=16, ex_mass=exm)
    assert np.max(np.abs(out - out_p)) <= 1.0 / 255
    assert [s.changed for s in stats] == [int(r[2]) for r in st_p]


@pytest.mark.parametrize("m", [1, 2, 3, 8])
def test_budget_kernels_agree(gpu_ctx, port, monkeypatch, m):
    """backtrack(m): thread-per-query kernel (m <= 2) and warp-per-query kernel
    (m > 2, and forced with PERSYN_SEARCH=warp) return identical answers."""
    ex, init = _stage()
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=12)
    monkeypatch.setenv("PERSYN_SEARCH", "warp")
    warp_ctx = api.Context(0)
    monkeypatch.delenv("PERSYN_SEARCH", raising=False)
    res = []
    for ctx in (gpu_ctx, warp_ctx):
        ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=4, max_depth=4,
                                     seed=3, ctx=ctx)
        res.append(api.search_step(init, ix, 2, 2, api.QueryBudget.backtrack(m)))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    assert res[0][3] == res[1][3]  # points scanned


@pytest.mark.parametrize("d,b,m,depth", [(12, 4, 4, 2), (32, 8, 4, 4), (40, 8, 16, 4),
                                         (56, 16, 6, 3), (32, 8, 40, 4), (24, 2, 30, 9),
                                         (13, 3, 5, 5), (64, 8, 4, 4), (25, 5, 7, 4), (1, 4, 4, 3)])
def test_backtrack_lane_group_kernel_equals_warp_kernel(gpu_ctx, port, monkeypatch, d, b, m,
                                                        depth):
    """backtrack(m > 2): the lane-group kernel (8 / 16 lanes per query, rows from
    the pair-interleaved blocks; every width class, leaves larger than a group,
    frontiers that outgrow the pool and are re-run) and the warp-per-query
    kernel (PERSYN_BT_WARP) return identical answers and scan counts."""
    ex, init = _stage()
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=d)
    monkeypatch.setenv("PERSYN_BT_WARP", "1")
    warp_ctx = api.Context(0)
    monkeypatch.delenv("PERSYN_BT_WARP", raising=False)
    res = []
    for ctx in (gpu_ctx, warp_ctx):
        ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=b,
                                     max_depth=depth, seed=3, ctx=ctx)
        res.append(api.search_step(init, ix, 2, 2, api.QueryBudget.backtrack(m)))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    assert res[0][3] == res[1][3]  # points scanned


@pytest.mark.parametrize("kind", ["sinusoid", "periodic"])
@pytest.mark.parametrize("d,b,m", [(16, 8, 4), (32, 4, 8), (40, 16, 4)])
def test_backtrack_tensor_core_projection_equals_exact_projection(gpu_ctx, port, monkeypatch, kind,
                                                                  d, b, m):
    """backtrack(m > 2) with the tensor-core projection (every pop and the final
    winner checked against the projection's error band, uncertain queries re-run
    with the exact fp64 projection) returns what the all-exact path returns --
    also on a periodic exemplar whose duplicate windows tie EVERY decision."""
    if kind == "sinusoid":
        ex, init = _stage()
    else:
        rng = np.random.default_rng(5)
        cell = rng.integers(0, 256, (3, 8, 8)).astype(np.float64) / 255.0
        ex = np.concatenate([np.tile(cell, (1, 5, 5)), np.full((1, 40, 40), 0.5)], 0)
        init = np.concatenate([rng.random((3, 56, 56)), np.full((1, 56, 56), 0.5)], 0)
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=d)
    monkeypatch.setenv("PERSYN_BT_EXACT_PROJECTION", "1")
    exact_ctx = api.Context(0)
    monkeypatch.delenv("PERSYN_BT_EXACT_PROJECTION", raising=False)
    res = []
    for ctx in (gpu_ctx, exact_ctx):
        ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=b, max_depth=4,
                                     seed=3, ctx=ctx)
        res.append(api.search_step(init, ix, 2, 2, api.QueryBudget.backtrack(m)))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    assert res[0][3] == res[1][3]  # points scanned


@pytest.mark.parametrize("budget", ["greedy", "bt1", "bt2"])
@pytest.mark.parametrize("d,b", [(12, 4), (32, 8), (40, 16)])
def test_small_budgets_lane_group_kernel_equals_thread_kernel(gpu_ctx, port, monkeypatch, budget,
                                                              d, b):
    """greedy / backtrack(1) / backtrack(2): the lane-group kernel fed by the
    tensor-core projection and the thread-per-query kernel with the fp64
    projection (PERSYN_BT_THREAD) return identical answers and scan counts."""
    ex, init = _stage()
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=d)
    monkeypatch.setenv("PERSYN_BT_THREAD", "1")
    thread_ctx = api.Context(0)
    monkeypatch.delenv("PERSYN_BT_THREAD", raising=False)
    bud = {"greedy": api.QueryBudget.greedy(), "bt1": api.QueryBudget.backtrack(1),
           "bt2": api.QueryBudget.backtrack(2)}[budget]
    res = []
    for ctx in (gpu_ctx, thread_ctx):
        ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=b, max_depth=4,
                                     seed=3, ctx=ctx)
        res.append(api.search_step(init, ix, 2, 2, bud))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    assert res[0][3] == res[1][3]  # points scanned


def test_eigensolver_paths_agree(gpu_ctx, monkeypatch):
    """Top-d PCA pairs by subspace iteration vs the direct DSYEVDX solver."""
    ex, _ = _stage(size=48, G=2)
    a = api.make_pca_tree_index(ex, 16, d_fixed=24, ctx=gpu_ctx)   # D = 1280: subspace
    monkeypatch.setenv("PERSYN_EIG", "direct")
    b = api.make_pca_tree_index(ex, 16, d_fixed=24, ctx=gpu_ctx)
    monkeypatch.delenv("PERSYN_EIG", raising=False)
    ma, ba, va = a.pca()
    mb, bb, vb = b.pca()
    assert np.array_equal(ma, mb)
    assert np.allclose(va[:24], vb[:24], rtol=1e-10, atol=1e-13)
    gaps = np.abs(np.diff(vb[:25])) / vb[0]
    ok = np.ones(24, bool)
    ok[:-1] &= gaps[:-1] > 1e-6
    ok[1:] &= gaps[:-1] > 1e-6
    ok &= gaps[:24] > 1e-6
    assert np.allclose(np.abs(np.sum(ba * bb, axis=1))[ok], 1.0, atol=1e-8)


@pytest.mark.parametrize("env", [{}, {"PERSYN_SERIAL": "1"}, {"PERSYN_GRAPH": "1"},
                                 {"PERSYN_RESCORE_ALL": "1", "PERSYN_NO_FUSED_HIST": "1",
                                  "PERSYN_PENALTY_PER_ANCHOR": "1"}])
def test_em_scheduling_variants_bit_identical(gpu_ctx, monkeypatch, env):
    """The EM step's scheduling choices -- side-stream overlap (default) or one
    stream, CUDA-graph replay, changed-only rescoring, the M-step's fused
    histogram and the per-candidate penalty table -- never change a bit."""
    ex, init = _stage()
    ix = api.make_pca_tree_index(ex, 8, d_fixed=16, branching=8, max_depth=3, seed=1,
                                 hist_bins=16, ctx=gpu_ctx)
    cfg = api.OptimizerConfig(max_iterations=5, min_iterations=5, convergence_fraction=1e-9,
                              nbhd_width=8, spacing=2, patch_width=2,
                              budget=api.QueryBudget.exact())

    def run():
        lv = api.Level(init, ix, cfg)
        lv.prime()
        st = lv.iterate(5)
        planes, idx, dist = lv.download()
        return planes, idx, dist, [(s.energy, s.changed, s.lsq_energy_after) for s in st]

    ref = run()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    got = run()
    for k in env:
        monkeypatch.delenv(k)
    for a, b in zip(ref[:3], got[:3]):
        assert np.array_equal(a, b)
    assert ref[3] == got[3]


@pytest.mark.parametrize("budget,early_stop", [("exact", False), ("bt4", False), ("exact", True)])
def test_optimize_level_pinned_result_early_download(gpu_ctx, port, budget, early_stop):
    """psg_optimize_level with a page-locked result buffer starts the image's
    download after the last iteration's M-step (copy stream, under that
    iteration's E-step): same image and statistics as with a pageable buffer --
    also when convergence ends the loop before the last possible iteration."""
    import ctypes as ct

    import torch

    from paper_2006_11851_b200 import native as N
    ex, init = _stage()
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=16)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, seed=3, hist_bins=16,
                                 tree_kind=api.TREE_REFERENCE, ctx=gpu_ctx)
    bud = api.QueryBudget.exact() if budget == "exact" else api.QueryBudget.backtrack(4)
    n_it = 30 if early_stop else 4
    cfg = api.OptimizerConfig(max_iterations=n_it, min_iterations=1 if early_stop else n_it,
                              convergence_fraction=0.05 if early_stop else 1e-9, nbhd_width=8,
                              spacing=2, patch_width=2, budget=bud)
    ref_out, ref_st = api.optimize_level(init, ix, cfg)  # pageable result buffer
    if early_stop:
        assert len(ref_st) < n_it
    pin_in = torch.empty(init.shape, dtype=torch.float64, pin_memory=True)
    pin_in.numpy()[...] = init
    pin_out = torch.zeros(init.shape, dtype=torch.float64, pin_memory=True)
    c = cfg.c()
    st = (N.psg_iter_stats * n_it)()
    n = ct.c_int()
    H, W = init.shape[1], init.shape[2]
    for _ in range(2):  # the context and its copy stream are reused
        pin_out.zero_()
        N.check(N.lib.psg_optimize_level(gpu_ctx.h, ix.h, ct.c_void_p(pin_in.data_ptr()), W, H,
                                         ct.byref(c), None, ct.c_void_p(pin_out.data_ptr()),
                                         ct.cast(st, ct.c_void_p), ct.byref(n)))
        assert n.value == len(ref_st)
        assert np.array_equal(pin_out.numpy(), ref_out)
        assert [st[i].changed for i in range(n.value)] == [s.changed for s in ref_st]
