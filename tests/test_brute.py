"""BruteForceIndex on the tensor cores (optimizer.cpp:168-212) vs the reference.

The reference scans all candidates with an fp64 j-sequential dist^2 and keeps
the first index of the minimum; it ignores the QueryBudget and counts every
candidate as scanned.  The device index filters with a tf32 UMMA distance
bound and settles the survivors with the same fp64 chain, so index and
distance must match bit for bit.
"""
import numpy as np
import pytest

from paper_2006_11851_b200 import workloads as wl

pytestmark = pytest.mark.gpu

api = pytest.importorskip("paper_2006_11851_b200.api")


def _stage(size=32, out=48, seed=1):
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(size, 8, 2.0, seed), 1)
    init = wl.init_output(ex, out, out, 1, seed)
    return ex, init


@pytest.mark.parametrize("w", [4, 8, 16])
def test_brute_window_queries_match_reference(gpu_ctx, port, ref, w):
    ex, init = _stage()
    cand = port.extract_all(ex, w, 1)
    ix = api.make_brute_force_index(ex, w, ctx=gpu_ctx)
    assert ix.count == cand.shape[0] and ix.dim == cand.shape[1]
    rng = np.random.default_rng(w)
    outw = port.extract_all(init, w, 1)
    Q = np.concatenate([
        outw[rng.choice(outw.shape[0], 120, replace=False)],
        cand[rng.choice(cand.shape[0], 40)],                                   # exact hits
        cand[rng.choice(cand.shape[0], 40)] +
        rng.normal(0, 1e-4, (40, cand.shape[1])).astype(np.float32),           # near ties
    ]).astype(np.float32)
    idx, dist, _, scanned = ix.nearest(Q, api.QueryBudget.backtrack(4))
    h = ref.index_create(ex, w, kind="brute")
    for i in range(Q.shape[0]):
        ri, rd, rs = h.nearest(Q[i])
        assert (idx[i], dist[i]) == (ri, rd), i
        assert scanned[i] == rs == cand.shape[0]


def test_brute_vectors_ties_and_mixture(gpu_ctx, port):
    # config-2 shaped candidates (values ~[0, 255], D = 192) plus duplicated
    # rows: the lowest index of an exact tie must win (optimizer.cpp:197-200)
    X = wl.gaussian_mixture(3000, 192, 32, 20.0, 1)
    X = np.concatenate([X, X[:500], X[100:200]]).astype(np.float32)
    Q = np.concatenate([wl.gaussian_mixture(400, 192, 32, 20.0, 2), X[2900:3100]]).astype(np.float32)
    ix = api.make_brute_force_vector_index(X, ctx=gpu_ctx)
    idx, dist, _, scanned = ix.nearest(Q)
    X64 = X.astype(np.float64)
    for i in range(Q.shape[0]):
        pi, pd2 = port.nearest_lexmin(X64, Q[i].astype(np.float64))
        assert idx[i] == pi, i
        assert dist[i] == np.sqrt(pd2), i
    assert np.all(scanned == X.shape[0])
    r = np.arange(2900, 3100)
    assert np.array_equal(idx[400:], np.where(r >= 3000, r - 3000, r))


def test_brute_search_step_matches_reference(gpu_ctx, port, ref):
    ex, init = _stage()
    ix = api.make_brute_force_index(ex, 8, ctx=gpu_ctx)
    h = ref.index_create(ex, 8, kind="brute")
    for sp in (2, 4):
        idx, dist, calls, scanned = api.search_step(init, ix, sp, 2, api.QueryBudget.exact())
        i_r, d_r, c_r, s_r = h.search_step(init, 8, sp, 2, mode="backtrack", max_leaves=4)
        assert calls == c_r and scanned == s_r
        assert np.array_equal(idx, i_r) and np.array_equal(dist, d_r)


@pytest.mark.parametrize("hist", [True, False])
def test_brute_optimize_level_matches_reference(gpu_ctx, ref, hist):
    ex, init = _stage()
    ix = api.make_brute_force_index(ex, 8, hist_bins=16 if hist else 0, ctx=gpu_ctx)
    cfg = api.OptimizerConfig(max_iterations=3, min_iterations=3, convergence_fraction=1e-9,
                              histogram_matching=hist, nbhd_width=8, spacing=4, patch_width=2,
                              budget=api.QueryBudget.backtrack(4))
    out, stats = api.optimize_level(init, ix, cfg)
    h = ref.index_create(ex, 8, kind="brute")
    out_r, st_r, _ = h.optimize_level(init, 8, 4, 2, max_it=3, min_it=3, frac=1e-9, bins=16,
                                      hist_on=hist, mode="backtrack", max_leaves=4)
    assert len(stats) == len(st_r)
    assert np.max(np.abs(out - out_r)) <= 1.0 / 255
    for s, r in zip(stats, st_r):
        assert s.changed == r[2] and s.nn_calls == r[3] and s.points_scanned == r[6]
        assert abs(s.energy - r[1]) <= 1e-4 * abs(r[1])


def test_brute_self_image_zero_distance(gpu_ctx):
    ex, _ = _stage(size=24)
    ix = api.make_brute_force_index(ex, 8, ctx=gpu_ctx)
    idx, dist, _, _ = api.search_step(ex, ix, 2, 2, api.QueryBudget.exact())
    assert np.all(dist == 0.0)


def test_brute_many_ties_spill_the_survivor_lists(gpu_ctx, port):
    # 300 identical rows and 300 near-identical ones around each query: far
    # more survivors than a (query, split) list holds -> overflow buffer path
    rng = np.random.default_rng(5)
    base = rng.uniform(0, 1, (4, 256)).astype(np.float32)
    rows = [base[i % 4] + (rng.normal(0, 1e-6, 256).astype(np.float32) if i % 2 else 0)
            for i in range(1200)]
    X = np.concatenate([rng.uniform(0, 1, (500, 256)).astype(np.float32), np.stack(rows)])
    Q = np.concatenate([base, base + 1e-7]).astype(np.float32)
    ix = api.make_brute_force_vector_index(X, ctx=gpu_ctx)
    idx, dist, _, _ = ix.nearest(Q)
    X64 = X.astype(np.float64)
    for i in range(Q.shape[0]):
        pi, pd2 = port.nearest_lexmin(X64, Q[i].astype(np.float64))
        assert idx[i] == pi and dist[i] == np.sqrt(pd2), i
