"""Parity of the sm_100a path (through the C ABI) against the CPU checkers.

`ref`: the reference's own TUs (C = 4 only); `port`: our C restatement
(C-generalised, pinned to `ref` in test_oracle_pins.py).  Bars:
  * NN indices and fp64 distances bit-exact (exact search mode);
  * fp64 image planes bit-exact for update_step with injected weights;
  * optimize_level: images within 1/255 (north star) — in practice equal or
    within a few ulp, since only the IRLS pow may round differently from
    glibc (correctly rounded on device vs glibc's < 1 ulp) — energy within
    1e-4 relative, assignment indices equal.
"""
import numpy as np
import pytest

from conftest import random_planes
from oracle.oracle import fit_pca
from paper_2006_11851_b200 import workloads as wl

pytestmark = pytest.mark.gpu

api = pytest.importorskip("paper_2006_11851_b200.api")


def _stage(size=32, out=48, G=1, seed=1, d=12):
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(size, 8, 2.0, seed), G)
    init = wl.init_output(ex, out, out, G, seed)
    return ex, init


def _injected(port, ex, w, d):
    cand = port.extract_all(ex, w, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=d)
    return cand, mean, basis, port.project_all(cand, mean, basis)


# ---- index build ---------------------------------------------------------------
@pytest.mark.parametrize("G,w,d", [(1, 8, 12), (2, 8, 16), (1, 4, 40), (1, 16, 32)])
def test_projected_database_bit_exact(gpu_ctx, port, G, w, d):
    ex, _ = _stage(G=G)
    cand, mean, basis, proj = _injected(port, ex, w, d)
    ix = api.make_pca_tree_index(ex, w, mean=mean, basis=basis, branching=4, max_depth=3,
                                 ctx=gpu_ctx)
    assert ix.count == cand.shape[0] and ix.retained_dim == d
    assert np.array_equal(ix.projected(), proj)
    ids, sizes = ix.leaves()
    assert np.array_equal(np.sort(ids), np.arange(ix.count))
    assert sizes.sum() == ix.count


def test_exemplar_histogram_bit_exact(gpu_ctx, port):
    ex, _ = _stage(size=40)
    ix = api.make_pca_tree_index(ex, 8, d_fixed=8, hist_bins=16, ctx=gpu_ctx)
    assert np.array_equal(ix.histograms(3, 16), port.build_histograms(ex, 16, 3))


def test_device_pca_fit_properties(gpu_ctx, port):
    ex, _ = _stage(size=40)
    ix = api.make_pca_tree_index(ex, 8, variance_target=0.95, ctx=gpu_ctx)
    mean, basis, var = ix.pca()
    cand = port.extract_all(ex, 8, 1)
    m2, b2, v2 = fit_pca(cand, 0.95)
    assert np.allclose(mean, m2, atol=1e-12)
    assert np.allclose(var, v2, rtol=1e-9, atol=1e-12)
    assert basis.shape == b2.shape
    assert np.allclose(basis @ basis.T, np.eye(basis.shape[0]), atol=1e-10)
    # same subspace/sign convention as the numpy restatement (no near-degenerate pairs)
    assert np.allclose(np.abs(np.sum(basis * b2, axis=1)), 1.0, atol=1e-6)
    assert np.all(np.diff(var) <= 1e-12)
    assert var[: basis.shape[0]].sum() >= 0.95 * var.sum()


# ---- E-step -------------------------------------------------------------------------
@pytest.mark.parametrize("G", [1, 2])
def test_search_step_bit_exact(gpu_ctx, port, ref, G):
    ex, init = _stage(G=G)
    cand, mean, basis, proj = _injected(port, ex, 8, 12)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=4, max_depth=3,
                                 ctx=gpu_ctx)
    idx, dist, calls, _ = api.search_step(init, ix, 4, 2, api.QueryBudget.exact())
    i_p, d_p, c_p = port.search_step(init, 8, 4, 2, cand, proj, mean, basis)
    assert calls == c_p
    assert np.array_equal(idx, i_p)
    assert np.array_equal(dist, d_p)
    if G == 1:
        h = ref.index_create(ex, 8, mean, basis, kind="tree", branching=4, seed=7)
        i_r, d_r, c_r, _ = h.search_step(init, 8, 4, 2, mode="exact")
        assert np.array_equal(idx, i_r) and np.array_equal(dist, d_r) and calls == c_r


def test_search_self_image_zero_distance(gpu_ctx, port):
    # optimizer_test.cpp:247-255: querying the exemplar itself gives distance 0
    ex, _ = _stage(size=24)
    ix = api.make_pca_tree_index(ex, 8, d_fixed=10, ctx=gpu_ctx)
    _, dist, _, _ = api.search_step(ex, ix, 2, 2, api.QueryBudget.exact())
    assert np.all(dist == 0.0)


def test_backtrack_all_leaves_equals_exact_and_greedy_runs(gpu_ctx, port):
    ex, init = _stage()
    cand, mean, basis, proj = _injected(port, ex, 8, 12)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=4, max_depth=3,
                                 ctx=gpu_ctx)
    e_idx, e_d, _, _ = api.search_step(init, ix, 4, 2, api.QueryBudget.exact())
    b_idx, b_d, _, _ = api.search_step(init, ix, 4, 2, api.QueryBudget.backtrack(ix.n_leaves))
    assert np.array_equal(e_idx, b_idx) and np.array_equal(e_d, b_d)
    g_idx, g_d, _, _ = api.search_step(init, ix, 4, 2, api.QueryBudget.greedy())
    # greedy is exact only in PCA space order; full-D distances are rescored
    assert np.all((g_idx >= 0) & (g_idx < ix.count)) and np.all(g_d >= 0)
    assert np.mean(g_idx == e_idx) > 0.2


def test_vector_index_exact_equals_bruteforce(gpu_ctx, port, ref):
    # config-2 shape at reduced size: mixture of Gaussians, D = 192, d = 24
    X = wl.gaussian_mixture(4096, 192, 64, 20.0, 1)
    Q = wl.gaussian_mixture(1000, 192, 64, 20.0, 2)
    mean, basis, _ = fit_pca(X, d_fixed=24)
    ix = api.make_vector_index(X, branching=8, max_depth=3, mean=mean, basis=basis, ctx=gpu_ctx)
    idx, dist, dpca, scanned = ix.nearest(Q, api.QueryBudget.exact())
    P = port.project_all(X, mean, basis)
    qp = port.project_all(Q, mean, basis)
    for i in range(0, 1000, 7):
        j, d2 = port.nearest_lexmin(P, qp[i])
        jr, dr = ref.brute_force_nearest(P, qp[i])
        assert idx[i] == j == jr
        assert dpca[i] == np.sqrt(d2) == dr
        assert dist[i] == port.full_distance(Q[i], X[j])
    assert scanned.mean() < X.shape[0]  # the tree prunes


# ---- M-step ---------------------------------------------------------------------------
@pytest.mark.parametrize("G,W,H,sp", [(1, 24, 24, 2), (1, 37, 23, 3), (2, 40, 32, 2)])
def test_update_step_bit_exact(gpu_ctx, port, ref, G, W, H, sp):
    ex, _ = _stage(size=30, G=G)
    ix = api.make_pca_tree_index(ex, 8, d_fixed=8, ctx=gpu_ctx)
    cand = port.extract_all(ex, 8, 1)
    rng = np.random.Generator(np.random.PCG64(W * H))
    A = len(port.axis_positions(W, 8, sp)) * len(port.axis_positions(H, 8, sp))
    idx = rng.integers(0, cand.shape[0], A).astype(np.int32)
    irls = rng.uniform(0.1, 300.0, A)
    pen = rng.uniform(0.0, 0.5, A)
    out = api.update_step(idx, irls, pen, ix, W, H, sp)
    assert np.array_equal(out, port.update_step(3 + G, W, H, 8, sp, cand, idx, irls, pen))
    if G == 1:
        h = ref.index_create(ex, 8, kind="brute")
        assert np.array_equal(out, h.update_step(random_planes(4, H, W, 2), 8, sp, idx, irls, pen))


def test_update_step_rejects_bad_weight(gpu_ctx):
    ex, _ = _stage(size=24)
    ix = api.make_pca_tree_index(ex, 8, d_fixed=8, ctx=gpu_ctx)
    with pytest.raises(api.DomainError):
        api.update_step([0], [0.0], [0.0], ix, 8, 8, 2)


# ---- EM loop -----------------------------------------------------------------------------
@pytest.mark.parametrize("hist", [False, True])
def test_optimize_level_matches_reference(gpu_ctx, port, ref, hist):
    ex, init = _stage()
    cand, mean, basis, proj = _injected(port, ex, 8, 12)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=4, max_depth=3,
                                 hist_bins=16 if hist else 0, ctx=gpu_ctx)
    cfg = api.OptimizerConfig(max_iterations=3, min_iterations=3, convergence_fraction=1e-9,
                              histogram_matching=hist, nbhd_width=8, spacing=4, patch_width=2,
                              budget=api.QueryBudget.exact())
    out, stats = api.optimize_level(init, ix, cfg)
    h = ref.index_create(ex, 8, mean, basis, kind="tree", branching=4, seed=3)
    out_r, st_r, _ = h.optimize_level(init, 8, 4, 2, max_it=3, min_it=3, frac=1e-9, bins=16,
                                      hist_on=hist, mode="exact")
    assert len(stats) == len(st_r)
    assert np.max(np.abs(out - out_r)) <= 1.0 / 255
    q = lambda a: np.rint(np.clip(a, 0, 1) * 255)  # image_io.cpp:18-21
    assert np.array_equal(q(out[:3]), q(out_r[:3]))
    for s, r in zip(stats, st_r):
        assert s.iteration == r[0]
        assert s.nn_calls == r[3]
        assert s.changed == r[2]
        assert abs(s.energy - r[1]) <= 1e-4 * abs(r[1])
        assert abs(s.lsq_energy_before - r[4]) <= 1e-9 * abs(r[4])
        assert abs(s.lsq_energy_after - r[5]) <= 1e-9 * abs(r[5])


def test_optimize_level_c5_matches_port(gpu_ctx, port):
    ex, init = _stage(G=2)
    cand, mean, basis, proj = _injected(port, ex, 8, 16)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, max_depth=4,
                                 hist_bins=16, ctx=gpu_ctx)
    cfg = api.OptimizerConfig(max_iterations=4, min_iterations=4, convergence_fraction=1e-9,
                              nbhd_width=8, spacing=2, patch_width=2,
                              budget=api.QueryBudget.exact())
    out, stats = api.optimize_level(init, ix, cfg)
    exm = port.build_histograms(ex, 16, 3)
    out_p, st_p = port.optimize_level(init, 8, 2, 2, cand, proj, mean, basis, max_it=4, min_it=4,
                                      frac=1e-9, bins=16, ex_mass=exm)
    assert np.max(np.abs(out - out_p)) <= 1.0 / 255
    for s, r in zip(stats, st_p):
        assert s.changed == r[2] and s.nn_calls == r[3]
        assert abs(s.energy - r[1]) <= 1e-4 * abs(r[1])


def test_fixed_point_returns_after_one_iteration(gpu_ctx):
    # optimizer_test.cpp:320-327
    ex, _ = _stage(size=24)
    ix = api.make_pca_tree_index(ex, 8, d_fixed=10, ctx=gpu_ctx)
    cfg = api.OptimizerConfig(histogram_matching=False, nbhd_width=8, spacing=2,
                              budget=api.QueryBudget.exact())
    out, stats = api.optimize_level(ex, ix, cfg)
    assert len(stats) == 1 and stats[0].changed == 0 and abs(stats[0].energy) < 1e-9


def test_level_api_deterministic(gpu_ctx, port):
    ex, init = _stage()
    ix = api.make_pca_tree_index(ex, 8, d_fixed=12, branching=4, ctx=gpu_ctx)
    cfg = api.OptimizerConfig(max_iterations=3, min_iterations=3, convergence_fraction=1e-9,
                              nbhd_width=8, spacing=4, budget=api.QueryBudget.exact())
    runs = []
    for _ in range(2):
        L = api.Level(init, ix, cfg)
        st = L.iterate(3)
        runs.append((L.download(), st))
    (p1, i1, d1), s1 = runs[0]
    (p2, i2, d2), s2 = runs[1]
    assert np.array_equal(p1, p2) and np.array_equal(i1, i2) and np.array_equal(d1, d2)
    assert [s.energy for s in s1] == [s.energy for s in s2]


def test_synthesize_runs_multires(gpu_ctx):
    cfg1 = wl.CONFIGS[1]
    rgb = wl.sinusoid_exemplar(64, 16, 2.0, 1)
    ex = wl.rgbs_planes(rgb, 1)
    cfg = api.OptimizerConfig(max_iterations=2, min_iterations=2, convergence_fraction=1e-9,
                              budget=api.QueryBudget.exact())
    out, rep = api.synthesize(ex, 128, 128, 2, (16, 8), cfg, variance_target=0.95, d_cap=32,
                              branching=8, max_depth=3, seed=1)
    assert out.shape == (4, 128, 128)
    assert np.all((out >= 0) & (out <= 1))
    assert len(rep["stages"]) == 4
    assert rep["total_nn_calls"] > 0


def test_synthesize_carried_seed_is_result_neutral(gpu_ctx, monkeypatch):
    """The driver seeds each stage's first search with the previous stage's
    assignment; exact search is a lexicographic min, so the seed may change the
    work, never the result."""
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(64, 16, 2.0, 3), 2)
    cfg = api.OptimizerConfig(max_iterations=2, min_iterations=2, convergence_fraction=1e-9,
                              budget=api.QueryBudget.exact())
    runs = []
    for carry in (True, False):
        if carry:
            monkeypatch.delenv("PERSYN_NO_CARRY", raising=False)
        else:
            monkeypatch.setenv("PERSYN_NO_CARRY", "1")
        runs.append(api.synthesize(ex, 128, 128, 3, (16, 8), cfg, variance_target=0.95, d_cap=32,
                                   branching=8, max_depth=3, seed=1))
    (o1, r1), (o2, r2) = runs
    assert np.array_equal(o1, o2)
    assert [s["final_energy"] for s in r1["stages"]] == [s["final_energy"] for s in r2["stages"]]
    assert r1["total_nn_calls"] == r2["total_nn_calls"]


@pytest.mark.parametrize("budget,tree", [("exact", "device"), ("bt4", "reference")])
def test_synthesize_index_build_ahead_is_result_neutral(monkeypatch, budget, tree):
    """psg_synthesize builds stage k + 1's index in a worker thread on a second
    context while stage k iterates; the overlap never changes a result (inline
    builds: PERSYN_NO_BUILD_AHEAD).  The same context serves repeated calls."""
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(64, 16, 2.0, 3), 2)
    bud = api.QueryBudget.exact() if budget == "exact" else api.QueryBudget.backtrack(4)
    cfg = api.OptimizerConfig(max_iterations=3, min_iterations=3, convergence_fraction=1e-9,
                              budget=bud)
    kw = dict(variance_target=0.95, d_cap=32, branching=8, seed=1,
              max_depth=3 if tree == "device" else 0,
              tree_kind=api.TREE_DEVICE if tree == "device" else api.TREE_REFERENCE)
    ahead = api.Context(0)
    monkeypatch.setenv("PERSYN_NO_BUILD_AHEAD", "1")
    inline = api.Context(0)
    monkeypatch.delenv("PERSYN_NO_BUILD_AHEAD", raising=False)
    o1, r1 = api.synthesize(ex, 128, 128, 3, (16, 8), cfg, ctx=ahead, **kw)
    o2, r2 = api.synthesize(ex, 128, 128, 3, (16, 8), cfg, ctx=inline, **kw)
    o3, r3 = api.synthesize(ex, 128, 128, 3, (16, 8), cfg, ctx=ahead, **kw)
    assert np.array_equal(o1, o2) and np.array_equal(o1, o3)
    assert len(r1["stages"]) == len(r2["stages"]) == len(r3["stages"]) == 5  # 16^2, w = 16 is skipped
    for a, b, c in zip(r1["stages"], r2["stages"], r3["stages"]):
        assert a["final_energy"] == b["final_energy"] == c["final_energy"]
    assert r1["total_nn_calls"] == r2["total_nn_calls"] == r3["total_nn_calls"]


@pytest.mark.parametrize("size,out,G,d,b,depth", [(128, 256, 2, 32, 8, 4), (256, 1024, 2, 32, 8, 4),
                                                  (96, 192, 1, 48, 16, 3)])
def test_exact_search_full_size_sampled(gpu_ctx, port, size, out, G, d, b, depth):
    """Larger stages (cfg3-like): every anchor's search runs on device, a seeded
    sample of anchors is re-searched by the oracle (exhaustive lexmin)."""
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(size, 32, 3.0, 1), G)
    init = wl.init_output(ex, out, out, G, 1)
    cand, mean, basis, proj = _injected(port, ex, 8, d)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=b, max_depth=depth,
                                 ctx=gpu_ctx)
    idx, dist, calls, _ = api.search_step(init, ix, 2, 2, api.QueryBudget.exact())
    A = idx.size
    rng = np.random.Generator(np.random.PCG64(out))
    only = np.sort(rng.choice(A, size=min(A, 400), replace=False)).astype(np.int32)
    i_p, d_p, c_p = port.search_step(init, 8, 2, 2, cand, proj, mean, basis, only=only)
    assert calls == c_p
    assert np.array_equal(idx[only], i_p)
    assert np.array_equal(dist[only], d_p)


def test_exact_search_ties_and_duplicates(gpu_ctx, port):
    """Exemplar with exactly repeated windows: many exact dist^2 ties, which must
    resolve to the lowest candidate index (km_tree.cpp:134, ann_test.cpp:338-342)."""
    tile = wl.sinusoid_exemplar(8, 4, 1.0, 3)
    rgb = np.tile(tile, (1, 5, 5))  # 40x40, period 8 -> every window appears ~25 times
    ex = wl.rgbs_planes(rgb, 1)
    ex[3] = 0.5  # constant guidance keeps the repeats exact
    init = wl.init_output(ex, 48, 48, 1, 5)
    init[3] = 0.5
    cand, mean, basis, proj = _injected(port, ex, 8, 10)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=4, max_depth=3,
                                 ctx=gpu_ctx)
    idx, dist, calls, _ = api.search_step(init, ix, 2, 2, api.QueryBudget.exact())
    i_p, d_p, c_p = port.search_step(init, 8, 2, 2, cand, proj, mean, basis)
    assert np.array_equal(idx, i_p) and np.array_equal(dist, d_p)
    # querying the exemplar itself: distance 0 and the FIRST occurrence of each window
    idx2, dist2, _, _ = api.search_step(ex, ix, 2, 2, api.QueryBudget.exact())
    i2, d2, _ = port.search_step(ex, 8, 2, 2, cand, proj, mean, basis)
    assert np.all(dist2 == 0.0) and np.array_equal(idx2, i2)


@pytest.mark.parametrize("b,depth", [(4, 3), (8, 4), (16, 0)])
def test_device_tree_build_valid_and_deterministic(gpu_ctx, port, b, depth, monkeypatch):
    """KmTree::build rules on the device: leaves partition the ids, splits stop at
    the depth cap / leaf threshold, identical on rebuild."""
    ex, init = _stage(size=40)
    cand, mean, basis, proj = _injected(port, ex, 8, 12)
    runs = []
    for _ in range(2):
        ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=b, max_depth=depth,
                                     seed=5, ctx=gpu_ctx)
        ids, sizes = ix.leaves()
        assert np.array_equal(np.sort(ids), np.arange(ix.count))
        assert sizes.sum() == ix.count and np.all(sizes > 0)
        if depth:
            assert ix.depth <= depth
        else:
            assert np.all(sizes < b)  # unbounded depth: leaves below the threshold
        runs.append((ids, sizes, ix.n_nodes))
        i_e, d_e, _, _ = api.search_step(init, ix, 4, 2, api.QueryBudget.exact())
        i_p, d_p, _ = port.search_step(init, 8, 4, 2, cand, proj, mean, basis)
        assert np.array_equal(i_e, i_p) and np.array_equal(d_e, d_p)
    assert all(np.array_equal(a, c) for a, c in zip(runs[0][:2], runs[1][:2]))


@pytest.mark.parametrize("G,w,kw", [(1, 8, dict(d_cap=12)), (2, 16, dict(d_fixed=20)),
                                    (2, 4, dict(variance_target=0.9))])
def test_device_pca_fit_matches_numpy(gpu_ctx, port, G, w, kw):
    """Window covariance from box sums (no N x D matrix) + top-d eigensolver vs
    the numpy restatement of fit_pca on the materialised windows."""
    ex, _ = _stage(size=40, G=G)
    ix = api.make_pca_tree_index(ex, w, ctx=gpu_ctx, **kw)
    mean, basis, var = ix.pca()
    cand = port.extract_all(ex, w, 1)
    m2, b2, v2 = fit_pca(cand, kw.get("variance_target", 0.95), kw.get("d_fixed", 0),
                         kw.get("d_cap", 0))
    k = basis.shape[0]
    assert k == b2.shape[0]
    assert np.allclose(mean, m2, atol=1e-12)
    assert np.allclose(var[:k], v2[:k], rtol=1e-9, atol=1e-12)
    assert np.allclose(basis @ basis.T, np.eye(k), atol=1e-10)
    gaps = np.abs(np.diff(v2[: k + 1])) / v2[0]
    ok = np.ones(k, bool)                     # well-separated components only
    ok[:-1] &= gaps[:-1] > 1e-6
    ok[1:] &= gaps[:-1] > 1e-6
    ok &= gaps[:k] > 1e-6
    assert np.allclose(np.abs(np.sum(basis * b2, axis=1))[ok], 1.0, atol=1e-6)


@pytest.mark.slow
def test_optimize_level_cfg1_finest_stage_matches_reference(gpu_ctx, port, ref):
    """BASELINE cfg1 finest stage at full size with one guidance plane (C = 4,
    the reference's own channel layout): 128^2 exemplar, 256^2 output, w = 8,
    sp = 2 (15,625 anchors, 250,000 plan calls per search), d = 32 injected,
    exact search, histogram matching on, 3 EM iterations — device vs the
    reference's optimize_level (oracle/_ref, all host threads)."""
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(128, 16, 2.0, 1), 1)
    init = wl.init_output(ex, 256, 256, 1, 1)
    cand, mean, basis, proj = _injected(port, ex, 8, 32)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, max_depth=3,
                                 hist_bins=16, ctx=gpu_ctx)
    cfg = api.OptimizerConfig(max_iterations=3, min_iterations=3, convergence_fraction=1e-9,
                              nbhd_width=8, spacing=2, patch_width=2,
                              budget=api.QueryBudget.exact())
    out, stats = api.optimize_level(init, ix, cfg)
    h = ref.index_create(ex, 8, mean, basis, kind="tree", branching=8, seed=1)
    out_r, st_r, _ = h.optimize_level(init, 8, 2, 2, max_it=3, min_it=3, frac=1e-9, bins=16,
                                      hist_on=True, mode="exact")
    assert len(stats) == len(st_r) == 3
    assert np.max(np.abs(out - out_r)) <= 1.0 / 255
    q = lambda a: np.rint(np.clip(a, 0, 1) * 255)  # image_io.cpp:18-21
    assert np.mean(q(out[:3]) != q(out_r[:3])) < 1e-4
    for s, r in zip(stats, st_r):
        assert s.changed == r[2] and s.nn_calls == r[3]
        assert abs(s.energy - r[1]) <= 1e-4 * abs(r[1])


@pytest.mark.parametrize("d", [80, 128])
def test_retained_dim_above_64(gpu_ctx, port, ref, d):
    """d in (64, 128]: the warp search kernel and the fp64 projection (the tile
    kernel and the tensor-core projection take d <= 64): still bit-exact."""
    ex, init = _stage(size=40, out=56)
    cand, mean, basis, proj = _injected(port, ex, 8, d)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, max_depth=3,
                                 hist_bins=16, ctx=gpu_ctx)
    assert ix.retained_dim == d and np.array_equal(ix.projected(), proj)
    idx, dist, calls, _ = api.search_step(init, ix, 2, 2, api.QueryBudget.exact())
    i_p, d_p, c_p = port.search_step(init, 8, 2, 2, cand, proj, mean, basis)
    assert calls == c_p and np.array_equal(idx, i_p) and np.array_equal(dist, d_p)
    b_idx, b_d, _, _ = api.search_step(init, ix, 2, 2, api.QueryBudget.backtrack(ix.n_leaves))
    assert np.array_equal(b_idx, i_p)
    h = ref.index_create(ex, 8, mean, basis, kind="tree", branching=8, seed=1)
    cfg = api.OptimizerConfig(max_iterations=2, min_iterations=2, convergence_fraction=1e-9,
                              nbhd_width=8, spacing=2, patch_width=2,
                              budget=api.QueryBudget.exact())
    out, stats = api.optimize_level(init, ix, cfg)
    out_r, st_r, _ = h.optimize_level(init, 8, 2, 2, max_it=2, min_it=2, frac=1e-9, bins=16,
                                      hist_on=True, mode="exact")
    assert np.max(np.abs(out - out_r)) <= 1.0 / 255
    assert [s.changed for s in stats] == [int(r[2]) for r in st_r]


def test_variance_rule_may_retain_more_than_64(gpu_ctx, port):
    """A high variance target on a 16x16 window keeps more than 64 components
    (the reference has no cap): the device fit and search follow."""
    ex, init = _stage(size=48, out=64)
    ix = api.make_pca_tree_index(ex, 16, variance_target=0.98, branching=8, max_depth=3,
                                 ctx=gpu_ctx)
    assert 64 < ix.retained_dim <= 128
    mean, basis, _ = ix.pca()
    cand = port.extract_all(ex, 16, 1)
    proj = port.project_all(cand, mean, basis)
    idx, dist, _, _ = api.search_step(init, ix, 4, 2, api.QueryBudget.exact())
    i_p, d_p, _ = port.search_step(init, 16, 4, 2, cand, proj, mean, basis)
    assert np.array_equal(idx, i_p) and np.array_equal(dist, d_p)
