"""Greedy / backtrack(m) parity through the reference's own tree.

The reference's default budget is backtrack(4) (optimizer.hpp:48), whose
answer depends on the tree.  The reference's KmTree is rebuilt on the device
from its public structure_json() + leaves() (psg_index_import_tree), after
which greedy and backtrack queries must reproduce KmTree::query
(km_tree.cpp:213-250) exactly: index, distance and points scanned — including
the frontier tie-break on the reference's post-order node ids.  The same tree is
also rebuilt by the library itself (tree_kind=TREE_REFERENCE, a replica of
KmTree::build with the same std::mt19937_64 stream), with no import.
"""
import json

import numpy as np
import pytest

from oracle.oracle import fit_pca
from paper_2006_11851_b200 import workloads as wl

api = pytest.importorskip("paper_2006_11851_b200.api")


def _stage(size=32, out=48, seed=1):
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(size, 8, 2.0, seed), 1)
    init = wl.init_output(ex, out, out, 1, seed)
    return ex, init


def _ref_tree(ref, ex, w, mean, basis, b, seed):
    h = ref.index_create(ex, w, mean, basis, kind="tree", branching=b, seed=seed)
    t = h.tree()
    sj = ref.kmtree_structure_json(t)
    ids, sizes = ref.kmtree_leaves(t, h.count)
    leaves = np.split(ids, np.cumsum(sizes)[:-1])
    return h, sj, leaves


# ---- host-side structure conversion (CPU) ----------------------------------------------
def test_preorder_child_counts_matches_reference_structure(port, ref):
    ex, _ = _stage(size=24)
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=8)
    _, sj, leaves = _ref_tree(ref, ex, 8, mean, basis, 4, 5)
    nc = api.preorder_child_counts(sj)
    j = json.loads(sj)
    assert nc[0] == len(j["root"]["children"])
    assert int(np.sum(nc == 0)) == len(leaves)          # one zero per leaf
    assert int(nc.sum()) == nc.size - 1                 # every node but the root is a child
    assert sum(len(l) for l in leaves) == cand.shape[0]
    for l in leaves:                                    # clusters keep ascending ids
        assert np.all(np.diff(l) > 0)


# ---- device parity -----------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("b,seed", [(4, 7), (8, 3), (16, 11)])
def test_replayed_tree_queries_bit_exact(gpu_ctx, port, ref, b, seed):
    ex, init = _stage()
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=12)
    h, sj, leaves = _ref_tree(ref, ex, 8, mean, basis, b, seed)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=b, ctx=gpu_ctx)
    ix.import_reference_tree(sj, leaves)
    assert ix.n_leaves == len(leaves)
    ids, sizes = ix.leaves()
    assert sorted(map(tuple, np.split(ids, np.cumsum(sizes)[:-1]))) == \
        sorted(map(tuple, leaves))
    rng = np.random.default_rng(seed)
    # queries: output windows (near the data) and noisy exemplar windows (ties/near-ties)
    Q = port.extract_all(init, 8, 1)[rng.choice(41 * 41, 150, replace=False)]
    Q = np.concatenate([Q, cand[rng.choice(cand.shape[0], 50)] +
                        rng.normal(0, 1e-3, (50, cand.shape[1])).astype(np.float32)])
    budgets = [("greedy", 1, api.QueryBudget.greedy())] + \
        [("backtrack", m, api.QueryBudget.backtrack(m)) for m in (1, 2, 4, 8)] + \
        [("exact", 1, api.QueryBudget.exact())]
    for mode, m, bud in budgets:
        idx, dist, _, scanned = ix.nearest(Q, bud)
        for i in range(Q.shape[0]):
            ri, rd, rs = h.nearest(Q[i], mode=mode, max_leaves=m)
            assert (idx[i], dist[i]) == (ri, rd), (mode, m, i)
            if mode != "exact":  # exact-mode scan counts depend on the traversal order
                assert scanned[i] == rs, (mode, m, i)


@pytest.mark.gpu
def test_replayed_tree_search_step_backtrack4(gpu_ctx, port, ref):
    ex, init = _stage()
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=12)
    h, sj, leaves = _ref_tree(ref, ex, 8, mean, basis, 4, 7)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=4, ctx=gpu_ctx)
    ix.import_reference_tree(sj, leaves)
    for sp in (2, 4):
        idx, dist, calls, scanned = api.search_step(init, ix, sp, 2, api.QueryBudget.backtrack(4))
        i_r, d_r, c_r, s_r = h.search_step(init, 8, sp, 2, mode="backtrack", max_leaves=4)
        assert calls == c_r and scanned == s_r
        assert np.array_equal(idx, i_r) and np.array_equal(dist, d_r)


@pytest.mark.gpu
@pytest.mark.parametrize("hist", [True, False])
def test_replayed_tree_optimize_level_backtrack4(gpu_ctx, port, ref, hist):
    """cfg-0 secondary parity mode: the reference's default budget end to end."""
    ex, init = _stage()
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=12)
    h, sj, leaves = _ref_tree(ref, ex, 8, mean, basis, 4, 3)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=4,
                                 hist_bins=16 if hist else 0, ctx=gpu_ctx)
    ix.import_reference_tree(sj, leaves)
    cfg = api.OptimizerConfig(max_iterations=4, min_iterations=4, convergence_fraction=1e-9,
                              histogram_matching=hist, nbhd_width=8, spacing=4, patch_width=2,
                              budget=api.QueryBudget.backtrack(4))
    out, stats = api.optimize_level(init, ix, cfg)
    out_r, st_r, _ = h.optimize_level(init, 8, 4, 2, max_it=4, min_it=4, frac=1e-9, bins=16,
                                      hist_on=hist, mode="backtrack", max_leaves=4)
    assert len(stats) == len(st_r)
    assert np.max(np.abs(out - out_r)) <= 1.0 / 255
    for s, r in zip(stats, st_r):
        assert s.changed == r[2] and s.nn_calls == r[3]
        assert abs(s.energy - r[1]) <= 1e-4 * abs(r[1])
        assert s.points_scanned == r[6]


# ---- the host replica of KmTree::build, on the CPU ------------------------------------
@pytest.mark.parametrize("size,b,seed,d", [(32, 4, 7, 12), (40, 8, 3, 16), (40, 16, 11, 8),
                                           (80, 8, 5, 24)])
def test_host_tree_replica_equals_reference_tree_cpu(port, ref, size, b, seed, d):
    """psg_reference_tree_host (vectorised, threaded k-means; the RNG walk
    sequential) builds the reference's own KmTree: same pre-order structure,
    same leaves in the same order.  (80^2 exemplar: 5,329 points -- the thread
    pool and every vector clone's code path run.)"""
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(size, 8, 2.0, seed), 1)
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=d)
    h, sj, leaves = _ref_tree(ref, ex, 8, mean, basis, b, seed)
    nc, lv = api.reference_tree_host(port.project_all(cand, mean, basis), b, seed)
    assert len(lv) == len(leaves)
    assert all(np.array_equal(a, np.asarray(r)) for a, r in zip(lv, leaves))
    assert np.array_equal(nc, api.preorder_child_counts(sj))


# ---- the library's own replica of KmTree::build (no import) -----------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("b,seed,d", [(4, 7, 12), (8, 3, 16), (16, 11, 8)])
def test_reference_tree_kind_equals_reference_tree(gpu_ctx, port, ref, b, seed, d):
    """make_pca_tree_index(tree_kind=TREE_REFERENCE) builds the reference's tree
    (same leaves, same post-order tie ids): every budget answers like
    KmTree::query on the reference's own PcaTreeIndex."""
    ex, init = _stage()
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=d)
    h, sj, leaves = _ref_tree(ref, ex, 8, mean, basis, b, seed)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=b, seed=seed,
                                 tree_kind=api.TREE_REFERENCE, ctx=gpu_ctx)
    assert ix.n_leaves == len(leaves)
    ids, sizes = ix.leaves()
    assert sorted(map(tuple, np.split(ids, np.cumsum(sizes)[:-1]))) == \
        sorted(map(tuple, leaves))
    rng = np.random.default_rng(seed)
    Q = port.extract_all(init, 8, 1)[rng.choice(41 * 41, 120, replace=False)]
    for mode, m, bud in [("greedy", 1, api.QueryBudget.greedy()),
                         ("backtrack", 4, api.QueryBudget.backtrack(4)),
                         ("backtrack", 8, api.QueryBudget.backtrack(8))]:
        idx, dist, _, scanned = ix.nearest(Q, bud)
        for i in range(Q.shape[0]):
            ri, rd, rs = h.nearest(Q[i], mode=mode, max_leaves=m)
            assert (idx[i], dist[i], scanned[i]) == (ri, rd, rs), (mode, m, i)
    idx, dist, calls, scanned = api.search_step(init, ix, 2, 2, api.QueryBudget.backtrack(4))
    i_r, d_r, c_r, s_r = h.search_step(init, 8, 2, 2, mode="backtrack", max_leaves=4)
    assert (calls, scanned) == (c_r, s_r)
    assert np.array_equal(idx, i_r) and np.array_equal(dist, d_r)


@pytest.mark.gpu
@pytest.mark.parametrize("b,m", [(16, 400), (8, 250)])
def test_wide_frontiers_spill_past_shared_memory(gpu_ctx, port, ref, b, m):
    """backtrack(m) with hundreds of leaves on a wide tree: the frontier (one
    entry per child of every expanded node) outgrows the lane-group pool AND the
    deep-stack kernel's shared-memory pool (512 entries), and continues in the
    warp's global scratch -- the reference's priority queue is unbounded
    (km_tree.cpp:206-208).  Same answers and scan counts as KmTree::query."""
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(72, 8, 2.0, 9), 1)
    init = wl.init_output(ex, 40, 40, 1, 9)
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=10)
    h, sj, leaves = _ref_tree(ref, ex, 8, mean, basis, b, 5)
    assert len(leaves) > m  # the budget, not the tree, ends the walk
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=b, seed=5,
                                 tree_kind=api.TREE_REFERENCE, ctx=gpu_ctx)
    rng = np.random.default_rng(b)
    Q = port.extract_all(init, 8, 1)[rng.choice(33 * 33, 40, replace=False)]
    idx, dist, _, scanned = ix.nearest(Q, api.QueryBudget.backtrack(m))
    for i in range(Q.shape[0]):
        ri, rd, rs = h.nearest(Q[i], mode="backtrack", max_leaves=m)
        assert (idx[i], dist[i], scanned[i]) == (ri, rd, rs), i
    i2, d2, _, _ = api.search_step(init, ix, 2, 2, api.QueryBudget.backtrack(m))
    i_r, d_r, _, _ = h.search_step(init, 8, 2, 2, mode="backtrack", max_leaves=m)
    assert np.array_equal(i2, i_r) and np.array_equal(d2, d_r)


@pytest.mark.gpu
def test_reference_tree_kind_rejects_depth_cap(gpu_ctx, port):
    ex, _ = _stage(size=24)
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=8)
    with pytest.raises(api.DomainError):
        api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=4, max_depth=3,
                                tree_kind=api.TREE_REFERENCE, ctx=gpu_ctx)
