"""Parity at the BASELINE configs' own sizes (BASELINE.json configs[0..4]).

Bars (north_star): NN indices bit-exact (exact mode: the lexicographic
(fp64 dist^2, id) minimum, km_tree.cpp:251-278), images within 1/255,
energies within 1e-4 relative.  Every EM test asserts the assignments of
EVERY iteration, not only the final image:

* cfg0 exactly as stated (64^2 -> 128^2, C = 4, w = 8, sp = 4, d = 16,
  b = 4 depth 3, 5 iterations, hist on and off): device iterations in lock
  step with the reference's loop body (oracle/_ref em_iteration = the
  reference's own search_step / update_step / weights), plus the reference's
  own optimize_level end to end;
* cfg2 at full size: 1,048,576 queries x 65,536 database vectors, D = 192,
  d = 24, b = 8 depth 3; a seeded 2,000-query sample re-searched by the port's
  exhaustive lexmin and 200 by the reference's brute_force_nearest;
* the bench stage itself (cfg3 finest, C = 5, 1024^2, d = 32, b = 8 depth 4)
  after 3 seeded EM iterations -- the code paths bench.py times (tile order,
  changed-only rescoring, fused histogram) -- re-searched on the downloaded
  state at 2,000 sampled anchors by the port;
* cfg4's finest stage (512^2 exemplar, 4096^2 output, d = 48, b = 16 depth 3)
  after the priming search and one EM iteration, 1,000 sampled anchors;
* the pyramid: device downsample / upsample / fit_to against image.cpp and
  the port's fit_to; a 2-level x 2-size psg_synthesize against a chain of the
  reference's own initialize_output / upsample_bilinear / optimize_level.
"""
import numpy as np
import pytest

from oracle.oracle import fit_pca
from paper_2006_11851_b200 import workloads as wl

pytestmark = pytest.mark.gpu

api = pytest.importorskip("paper_2006_11851_b200.api")


def _q255(a):  # image_io.cpp:18-21
    return np.rint(np.clip(a, 0.0, 1.0) * 255.0)


# ---- cfg0 -------------------------------------------------------------------------------
@pytest.mark.parametrize("hist", [True, False])
def test_cfg0_as_stated_lockstep_with_reference(gpu_ctx, port, ref, hist):
    cfg0 = wl.CONFIGS[0]
    rgb = wl.sinusoid_exemplar(cfg0.ex_size, cfg0.n_sin, cfg0.ramp, cfg0.seed)
    ex = wl.rgbs_planes(rgb, 1)                       # guidance = row / 63 as fp32
    init = wl.init_output(ex, cfg0.out, cfg0.out, 1, cfg0.seed)
    w, sp, its = 8, 4, cfg0.iterations
    cand = port.extract_all(ex, w, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=cfg0.d_fixed)
    ix = api.make_pca_tree_index(ex, w, mean=mean, basis=basis, branching=cfg0.branching,
                                 max_depth=cfg0.depth, hist_bins=16 if hist else 0, ctx=gpu_ctx)
    h = ref.index_create(ex, w, mean, basis, kind="tree", branching=cfg0.branching, seed=1)
    cfg = api.OptimizerConfig(max_iterations=its, min_iterations=its, convergence_fraction=1e-9,
                              histogram_matching=hist, nbhd_width=w, spacing=sp, patch_width=2,
                              budget=api.QueryBudget.exact())
    # lock step: the priming search, then every EM iteration
    L = api.Level(init, ix, cfg)
    L.prime()
    _, idx, dist = L.download()
    i_r, d_r, _, _ = h.search_step(init, w, sp, 2, mode="exact")
    assert np.array_equal(idx, i_r) and np.array_equal(dist, d_r)
    state = {"planes": init.copy()}
    for t in range(its):
        st = L.iterate(1)[0]
        planes, idx, dist = L.download()
        energy, changed = h.em_iteration(state, w, sp, 2, bins=16, hist_on=hist, mode="exact")
        assert np.array_equal(idx, state["idx"]), f"assignments differ at iteration {t + 1}"
        assert np.max(np.abs(planes - state["planes"])) <= 1e-12
        assert np.allclose(dist, state["dist"], rtol=1e-12, atol=1e-14)
        assert st.changed == changed
        assert abs(st.energy - energy) <= 1e-9 * abs(energy)
    # the reference's own optimize_level end to end
    out, stats = api.optimize_level(init, ix, cfg)
    out_r, st_r, _ = h.optimize_level(init, w, sp, 2, max_it=its, min_it=its, frac=1e-9, bins=16,
                                      hist_on=hist, mode="exact")
    assert len(stats) == len(st_r) == its
    assert np.max(np.abs(out - out_r)) <= 1.0 / 255
    assert np.array_equal(_q255(out[:3]), _q255(out_r[:3]))
    for s, r in zip(stats, st_r):
        assert (s.iteration, s.changed, s.nn_calls) == (r[0], r[2], r[3])
        assert abs(s.energy - r[1]) <= 1e-4 * abs(r[1])
        assert abs(s.lsq_energy_before - r[4]) <= 1e-9 * abs(r[4])
        assert abs(s.lsq_energy_after - r[5]) <= 1e-9 * abs(r[5])


# ---- cfg2 -------------------------------------------------------------------------------
def test_cfg2_full_size_sampled(gpu_ctx, port, ref):
    X = wl.gaussian_mixture(65536, 192, 64, 20.0, 1)
    Q = wl.gaussian_mixture(1 << 20, 192, 64, 20.0, 2)
    mean, basis, _ = fit_pca(X, d_fixed=24)
    ix = api.make_vector_index(X, branching=8, max_depth=3, mean=mean, basis=basis, ctx=gpu_ctx)
    idx, dist, dpca, scanned = ix.nearest(Q, api.QueryBudget.exact())
    assert idx.size == Q.shape[0]
    P = port.project_all(X, mean, basis)
    rng = np.random.Generator(np.random.PCG64(2))
    sample = np.sort(rng.choice(Q.shape[0], 2000, replace=False))
    qp = port.project_all(Q[sample], mean, basis)
    for k, i in enumerate(sample):
        j, d2 = port.nearest_lexmin(P, qp[k])
        assert idx[i] == j and dpca[i] == np.sqrt(d2), i
        assert dist[i] == port.full_distance(Q[i], X[j])
        if k % 10 == 0:
            jr, dr = ref.brute_force_nearest(P, qp[k])
            assert (idx[i], dpca[i]) == (jr, dr)
    assert scanned.mean() < X.shape[0] / 4  # the tree prunes


# ---- cfg3: the bench stage --------------------------------------------------------------
def test_cfg3_bench_stage_after_seeded_iterations(gpu_ctx, port):
    cfg3 = wl.CONFIGS[3]
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(cfg3.ex_size, cfg3.n_sin, cfg3.ramp, cfg3.seed), 2)
    init = wl.init_output(ex, cfg3.out, cfg3.out, 2, cfg3.seed)
    w, sp = 8, 2
    cand = port.extract_all(ex, w, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=32)
    proj = port.project_all(cand, mean, basis)
    ix = api.make_pca_tree_index(ex, w, mean=mean, basis=basis, branching=8, max_depth=4,
                                 seed=1, hist_bins=16, ctx=gpu_ctx)
    cfg = api.OptimizerConfig(max_iterations=100, min_iterations=99, convergence_fraction=1e-9,
                              histogram_bins=16, histogram_matching=True, nbhd_width=w,
                              spacing=sp, patch_width=2, budget=api.QueryBudget.exact())
    L = api.Level(init, ix, cfg)
    L.prime()
    stats = L.iterate(3)
    assert len(stats) == 3 and stats[-1].changed > 0
    planes, idx, dist = L.download()
    A = idx.size
    assert A == 509 * 509
    rng = np.random.Generator(np.random.PCG64(3))
    only = np.sort(rng.choice(A, 2000, replace=False)).astype(np.int32)
    i_p, d_p, c_p = port.search_step(planes, w, sp, 2, cand, proj, mean, basis, only=only,
                                     threads=0)
    assert c_p == 4145296 == stats[-1].nn_calls
    assert np.array_equal(idx[only], i_p)
    assert np.array_equal(dist[only], d_p)


# ---- cfg4: the finest stage --------------------------------------------------------------
def test_cfg4_finest_stage_sampled(gpu_ctx, port):
    cfg4 = wl.CONFIGS[4]
    ex, init, W, H, sp = wl.stage_inputs(cfg4, cfg4.levels - 1, 8)
    assert (W, H, sp) == (4096, 4096, 2) and ex.shape == (5, 512, 512)
    w = 8
    cand = port.extract_all(ex, w, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=48)
    proj = port.project_all(cand, mean, basis)
    ix = api.make_pca_tree_index(ex, w, mean=mean, basis=basis, branching=16, max_depth=3,
                                 seed=1, hist_bins=16, ctx=gpu_ctx)
    cfg = api.OptimizerConfig(max_iterations=100, min_iterations=99, convergence_fraction=1e-9,
                              histogram_bins=16, histogram_matching=True, nbhd_width=w,
                              spacing=sp, patch_width=2, budget=api.QueryBudget.exact())
    L = api.Level(init, ix, cfg)
    L.prime()
    st = L.iterate(1)
    planes, idx, dist = L.download()
    A = idx.size
    assert A == 2045 * 2045 == 4182025
    rng = np.random.Generator(np.random.PCG64(4))
    only = np.sort(rng.choice(A, 1000, replace=False)).astype(np.int32)
    i_p, d_p, c_p = port.search_step(planes, w, sp, 2, cand, proj, mean, basis, only=only,
                                     threads=0)
    assert c_p == 66912400 and st[0].nn_calls == 2 * c_p  # iteration 1 includes the priming search
    assert np.array_equal(idx[only], i_p)
    assert np.array_equal(dist[only], d_p)


# ---- pyramid ------------------------------------------------------------------------------
@pytest.mark.parametrize("W,H,f", [(64, 64, 2), (67, 45, 2), (256, 256, 4), (37, 91, 3)])
def test_downsample_bit_exact(gpu_ctx, ref, W, H, f):
    rng = np.random.Generator(np.random.PCG64(W * H + f))
    rgb = rng.uniform(0.0, 1.0, (3, H, W))
    assert np.array_equal(api.downsample(rgb, f, ctx=gpu_ctx), ref.downsample(rgb, f))


@pytest.mark.parametrize("W,H,f", [(32, 32, 2), (17, 29, 2), (8, 5, 3), (64, 48, 1)])
def test_upsample_bilinear_bit_exact(gpu_ctx, ref, W, H, f):
    rng = np.random.Generator(np.random.PCG64(W * H + 7 * f))
    rgb = rng.uniform(0.0, 1.0, (3, H, W))
    assert np.array_equal(api.upsample_bilinear(rgb, f, ctx=gpu_ctx), ref.upsample_bilinear(rgb, f))


@pytest.mark.parametrize("W,H,ow,oh", [(64, 64, 65, 63), (10, 12, 10, 12), (30, 20, 33, 17)])
def test_fit_to_bit_exact(gpu_ctx, port, W, H, ow, oh):
    rng = np.random.Generator(np.random.PCG64(W + ow))
    x = rng.uniform(0.0, 1.0, (4, H, W))
    out = api.fit_to(x, ow, oh, ctx=gpu_ctx)
    assert np.array_equal(out, np.stack([port.fit_to(p, ow, oh) for p in x]))


def test_resampling_errors(gpu_ctx):
    with pytest.raises(api.DomainError):
        api.downsample(np.zeros((3, 4, 4)), 5, ctx=gpu_ctx)
    with pytest.raises(api.DomainError):
        api.upsample_bilinear(np.zeros((3, 4, 4)), 0, ctx=gpu_ctx)


def test_synthesize_matches_reference_chain(gpu_ctx, port, ref):
    """psg_synthesize, 2 levels x sizes {16, 8}, C = 4, hist on, exact, with
    injected per-stage PCA, against the reference's own pieces chained the way
    synthesize (pipeline.cpp:216-315) chains them: initialize_output at the
    coarsest level, then per level upsample_bilinear(x2) + fit_to with the
    level's S re-imposed, and optimize_level per stage."""
    levels, sizes, out_w, seed, its = 2, (16, 8), 128, 5, 3
    rgb = wl.sinusoid_exemplar(64, 16, 2.0, seed).astype(np.float64) / 255.0
    ex_full = np.concatenate([rgb, wl.guidance_planes(64, 64, 1)], 0)
    ex_lv, stage_pca = [], []
    for l in range(levels):
        f = 1 << (levels - 1 - l)
        e = ref.downsample(rgb, f) if f > 1 else rgb
        e = np.concatenate([e, wl.guidance_planes(e.shape[2], e.shape[1], 1)], 0)
        ex_lv.append(e)
        for w in sizes:
            mean, basis, _ = fit_pca(port.extract_all(e, w, 1), d_fixed=12)
            stage_pca.append((mean, basis))
    cfg = api.OptimizerConfig(max_iterations=its, min_iterations=its, convergence_fraction=1e-9,
                              histogram_bins=16, histogram_matching=True,
                              budget=api.QueryBudget.exact())
    out, rep = api.synthesize(ex_full, out_w, out_w, levels, sizes, cfg, branching=4,
                              max_depth=3, seed=seed, stage_pca=stage_pca, ctx=gpu_ctx)
    # the reference chain
    W0 = out_w >> (levels - 1)
    x = ref.initialize_output(ex_lv[0], wl.guidance_planes(W0, W0, 1)[0].astype(np.float32),
                              0.0, 1.0, seed)
    stages_r = []
    for l in range(levels):
        W = out_w >> (levels - 1 - l)
        if l > 0:
            up = ref.upsample_bilinear(x[:3], 2)
            x = np.concatenate([np.stack([port.fit_to(p, W, W) for p in up]),
                                wl.guidance_planes(W, W, 1)], 0)
        for si, w in enumerate(sizes):
            mean, basis = stage_pca[l * len(sizes) + si]
            h = ref.index_create(ex_lv[l], w, mean, basis, kind="tree", branching=4, seed=1)
            sp = max(1, w // 4)
            x, st, _ = h.optimize_level(x, w, sp, min(2, sp), max_it=its, min_it=its,
                                        frac=1e-9, bins=16, hist_on=True, mode="exact")
            stages_r.append(st)
    assert len(rep["stages"]) == len(stages_r) == levels * len(sizes)
    for s, st in zip(rep["stages"], stages_r):
        assert s["iterations"] == len(st)
        assert s["nn_calls"] == int(st[:, 3].sum())
        assert abs(s["final_energy"] - st[-1, 1]) <= 1e-4 * abs(st[-1, 1])
    assert np.max(np.abs(out - x)) <= 1.0 / 255
    assert np.mean(_q255(out[:3]) != _q255(x[:3])) < 1e-4
