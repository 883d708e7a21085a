"""Pin the C restatement (oracle/oracle.c) against the reference's OWN code.

`ref` is the reference's neighborhood/km_tree/optimizer/image translation
units compiled unmodified from /root/reference (oracle/Makefile).  Every test
here compares the port with the reference bit-for-bit (==, not approx) on
seeded inputs, plus the known answers of the reference's own unit tests
(ann_test.cpp, optimizer_test.cpp, neighborhood_test.cpp).
"""
import numpy as np
import pytest

from conftest import random_planes
from oracle.oracle import fit_pca
from paper_2006_11851_b200 import workloads as wl

pytestmark = pytest.mark.ref


# ---- geometry (neighborhood.cpp) ------------------------------------------
@pytest.mark.parametrize("W,H,w,sp", [(128, 128, 8, 4), (64, 64, 8, 2), (24, 24, 8, 2),
                                      (10, 8, 8, 2), (37, 23, 8, 3), (256, 256, 32, 8),
                                      (16, 16, 16, 4), (9, 9, 2, 1)])
def test_grid_axes_match_reference(port, ref, W, H, w, sp):
    xs, ys = ref.grid_axes(W, H, w, sp)
    assert np.array_equal(port.axis_positions(W, w, sp), xs)
    assert np.array_equal(port.axis_positions(H, w, sp), ys)


def test_containing_known_answers(ref):
    # neighborhood_test.cpp:138-155
    assert ref.containing_anchors(64, 64, 8, 2, 30, 30, 1).size == 16
    assert ref.containing_anchors(64, 64, 8, 2, 31, 31, 1).size == 16
    assert ref.containing_anchors(64, 64, 8, 2, 31, 31, 2).size == 9
    assert ref.containing_anchors(64, 64, 8, 2, 30, 30, 2).size == 16
    assert ref.containing_anchors(64, 64, 8, 2, 0, 0, 1).size == 1


@pytest.mark.parametrize("W,H,w,sp,p", [(128, 128, 8, 4, 2), (24, 24, 8, 2, 2), (24, 24, 8, 2, 1),
                                        (37, 23, 8, 3, 2), (64, 48, 16, 4, 2), (33, 33, 8, 2, 2),
                                        (256, 256, 32, 8, 2)])
def test_plan_closed_form_matches_reference_plan(port, ref, W, H, w, sp, p):
    """nn_calls = |plan| (optimizer.cpp:288-296,333); multiplicity per anchor."""
    calls, mult = port.plan(W, H, w, sp, p)
    tiles = ref.patch_tiles(W, H, p)
    xs, ys = ref.grid_axes(W, H, w, sp)
    expect = np.zeros(len(xs) * len(ys), np.int64)
    for tx, ty in tiles:
        ids = ref.containing_anchors(W, H, w, sp, int(tx), int(ty), p)
        np.add.at(expect, ids, 1)
    assert calls == expect.sum()
    assert np.array_equal(mult, expect)


def test_plan_probe_counts(port):
    # SURVEY §8(a) A3 probe: cfg0 15,376; cfg3 finest w8 4,145,296; w32 4,000,000
    assert port.plan(128, 128, 8, 4, 2)[0] == 15376
    assert port.plan(1024, 1024, 8, 2, 2)[0] == 4145296
    assert port.plan(1024, 1024, 32, 8, 2)[0] == 4000000


def test_extract_all_matches_reference(port, ref):
    planes = random_planes(4, 21, 19, 3)
    for w, sp in [(8, 1), (8, 2), (4, 3)]:
        assert np.array_equal(port.extract_all(planes, w, sp), ref.extract_all(planes, w, sp))


# ---- index math (pca.cpp restated, km_tree.cpp) -----------------------------
def test_projection_matches_reference_injected(port, ref):
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(32, 8, 2.0, 5), 1)
    X = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(X, d_fixed=12)
    idx = ref.index_create(ex, 8, mean, basis, kind="pca_brute")
    assert np.array_equal(port.project_all(X, mean, basis), idx.projected())


def test_lexmin_equals_reference_brute_and_exact_tree(port, ref):
    rng = np.random.Generator(np.random.PCG64(53))
    for count in (1, 10, 100, 1000):
        for dim in (1, 3, 20):
            pts = rng.uniform(-1, 1, (count, dim))
            h = ref.kmtree_build(pts, 4, 4, int(rng.integers(1 << 30)))
            for _ in range(15):
                q = rng.uniform(-1.2, 1.2, dim)
                i_ref, d_ref = ref.brute_force_nearest(pts, q)
                i_tree, d_tree, _, _ = ref.kmtree_query(h, q, "exact")
                i_port, d2 = port.nearest_lexmin(pts, q)
                assert i_port == i_ref == i_tree
                assert np.sqrt(d2) == d_ref == d_tree
            ref.kmtree_destroy(h)


def test_ties_go_to_lowest_index(port, ref):
    # ann_test.cpp:338-342 and :204-212
    pts = np.array([[10.0], [20.0], [1.0], [30.0], [40.0], [-1.0]])
    assert port.nearest_lexmin(pts, np.array([0.0]))[0] == 2 == ref.brute_force_nearest(pts, [0.0])[0]
    same = np.full((20, 3), 1.25)
    h = ref.kmtree_build(same, 4, 4, 3)
    assert ref.kmtree_query(h, [1.25] * 3, "exact")[0] == 0 == port.nearest_lexmin(same, [1.25] * 3)[0]
    ref.kmtree_destroy(h)


# ---- weights / energy / histograms (optimizer.cpp:44-131) -------------------
def test_irls_and_energy_known_answers(port, ref):
    assert abs(port.irls_weight(0.0, 0.8, 1e-4) - 251.18864) < 1e-2   # optimizer_test.cpp:29-32
    assert abs(port.irls_weight(1.0, 0.8, 1e-12) - 1.0) < 1e-9
    assert abs(port.energy([2.0, 3.0], 0.8) - 4.14932) < 1e-4          # optimizer_test.cpp:45-52
    rng = np.random.Generator(np.random.PCG64(71))
    d = rng.uniform(0, 5, 5000)
    w_ref = ref.irls_weights(d, 0.8, 1e-4)
    w_port = np.array([port.irls_weight(v, 0.8, 1e-4) for v in d])
    assert np.array_equal(w_ref, w_port)
    assert ref.energy(d, 0.8) == port.energy(d, 0.8)


@pytest.mark.parametrize("bins", [2, 8, 16, 64])
def test_histograms_match_reference(port, ref, bins):
    planes = random_planes(4, 17, 23, bins)
    planes[0, 0, :5] = [0.0, 1.0, 0.5, 1.0 / bins, 1 - 1e-17]
    assert np.array_equal(port.build_histograms(planes, bins, 3), ref.build_histograms(planes, bins))
    assert np.array_equal(port.build_histograms(planes, bins, 4),
                          ref.build_histograms(planes, bins, include_scale=True))


def test_penalty_matches_reference(port, ref):
    assert abs(ref.histogram_penalty(np.full(16, 0.1, np.float32), 2, [[0.8, 0.2]] * 3,
                                     [[0.5, 0.5]] * 3) - 0.9) < 1e-12
    rng = np.random.Generator(np.random.PCG64(72))
    for rep in range(30):
        bins = int(rng.choice([2, 16, 64]))
        om = rng.dirichlet(np.ones(bins), 3)
        em = rng.dirichlet(np.ones(bins), 3)
        nb = rng.uniform(0, 1, 64 * 4).astype(np.float32)
        nb[:8] = [0.0, 1.0, 0.5, 0.999999, 0.0625, 0.1875, 1e-8, 0.3]
        assert port.histogram_penalty(nb, 4, 3, bins, om, em) == \
            ref.histogram_penalty(nb, bins, om, em)


def test_penalty_hand_computed():
    # optimizer_test.cpp:124-131: one channel, two bins, over-representation 0.3
    from oracle.oracle import Port
    p = Port()
    nb = np.full(4 * 4, 0.1, np.float32)
    pen = p.histogram_penalty(nb, 4, 1, 2, np.array([[0.8, 0.2]]), np.array([[0.5, 0.5]]))
    assert abs(pen - 0.3) < 1e-12


# ---- M-step (optimizer.cpp:350-401) ------------------------------------------
def test_update_known_answers(port):
    # optimizer_test.cpp:167-190: 10x8 grid, two windows, all-zero / all-one
    cand = np.zeros((2, 256), np.float32)
    cand[1] = 1.0
    out = port.update_step(4, 10, 8, 8, 2, cand, [0, 1], [1.0, 3.0], [0.0, 0.0])
    assert np.all(out[:, :, 0] == 0.0)
    assert np.allclose(out[:, :, 5], 0.75)
    assert np.all(out[:, :, 9] == 1.0)


def test_update_matches_reference(port, ref):
    ex = random_planes(4, 30, 28, 9)
    idx_h = ref.index_create(ex, 8, kind="brute")
    cand = port.extract_all(ex, 8, 1)
    rng = np.random.Generator(np.random.PCG64(10))
    for (W, H, sp) in [(24, 24, 2), (37, 23, 3), (16, 16, 8)]:
        A = len(port.axis_positions(W, 8, sp)) * len(port.axis_positions(H, 8, sp))
        idx = rng.integers(0, cand.shape[0], A).astype(np.int32)
        irls = rng.uniform(0.1, 300.0, A)
        pen = rng.uniform(0.0, 0.5, A)
        a = port.update_step(4, W, H, 8, sp, cand, idx, irls, pen)
        b = idx_h.update_step(random_planes(4, H, W, 1), 8, sp, idx, irls, pen)
        assert np.array_equal(a, b)


def test_update_rejects_nonpositive_weight(port):
    from oracle.oracle import OracleError
    cand = np.zeros((1, 256), np.float32)
    with pytest.raises(OracleError):
        port.update_step(4, 8, 8, 8, 2, cand, [0], [0.0], [0.0])


# ---- search + EM loop ----------------------------------------------------------
def _cfg0_like(size=32, out=48, d=12, seed=1):
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(size, 8, 2.0, seed), 1)
    init = wl.init_output(ex, out, out, 1, seed)
    return ex, init


def test_search_step_matches_reference(port, ref):
    ex, init = _cfg0_like()
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=12)
    proj = port.project_all(cand, mean, basis)
    for kind in ("tree", "pca_brute"):
        h = ref.index_create(ex, 8, mean, basis, kind=kind, branching=4, seed=7)
        i_ref, d_ref, calls_ref, _ = h.search_step(init, 8, 4, 2, mode="exact")
        i_p, d_p, calls_p = port.search_step(init, 8, 4, 2, cand, proj, mean, basis)
        assert calls_p == calls_ref
        assert np.array_equal(i_p, i_ref)
        assert np.array_equal(d_p, d_ref)


@pytest.mark.parametrize("hist", [False, True])
def test_optimize_level_matches_reference(port, ref, hist):
    ex, init = _cfg0_like()
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=12)
    proj = port.project_all(cand, mean, basis)
    h = ref.index_create(ex, 8, mean, basis, kind="tree", branching=4, seed=3)
    out_r, st_r, _ = h.optimize_level(init, 8, 4, 2, max_it=3, min_it=3, frac=1e-9, bins=16,
                                      hist_on=hist, mode="exact")
    exm = port.build_histograms(ex, 16, 3) if hist else None
    out_p, st_p = port.optimize_level(init, 8, 4, 2, cand, proj, mean, basis, max_it=3, min_it=3,
                                      frac=1e-9, bins=16, ex_mass=exm)
    assert np.array_equal(out_p, out_r)
    assert np.array_equal(st_p[:, :6], st_r[:, :6])   # iter, energy, changed, calls, lsq x2


def test_resampling_matches_reference(port, ref):
    rgb = random_planes(3, 20, 24, 4)
    for f in (2, 3):
        d_r = ref.downsample(rgb, f)
        for c in range(3):
            assert np.array_equal(port.downsample(rgb[c], f), d_r[c])
    u_r = ref.upsample_bilinear(rgb, 2)
    for c in range(3):
        assert np.array_equal(port.upsample_bilinear(rgb[c], 2), u_r[c])
