"""Seeded exact searches settled by the database-side certificate
(kernels_cert.cu) give exactly the tile search's answers.

KmTree::query(exact) is the lexicographic minimum of (fp64 dist^2, id) over
all points (km_tree.cpp:251-278); the certificate settles a seeded query from
its seed's neighbour list when that provably contains the minimum.  Every EM
iteration's assignments, distances and images must be bit-identical with the
certificate on (several list lengths) and off (PERSYN_CERT_K=0), with the
tensor-core projection and with the exact fp64 projection.
"""
import numpy as np
import pytest

from paper_2006_11851_b200 import workloads as wl

pytestmark = pytest.mark.gpu

api = pytest.importorskip("paper_2006_11851_b200.api")


def _ctx(monkeypatch, k=None, exact_projection=False):
    if k is not None:
        monkeypatch.setenv("PERSYN_CERT_K", str(k))
    if exact_projection:
        monkeypatch.setenv("PERSYN_EXACT_PROJECTION", "1")
    ctx = api.Context(0)
    monkeypatch.delenv("PERSYN_CERT_K", raising=False)
    monkeypatch.delenv("PERSYN_EXACT_PROJECTION", raising=False)
    return ctx


def _em(ctx, ex, init, w, sp, d, iters, mean=None, basis=None, b=8, depth=4):
    kw = dict(mean=mean, basis=basis) if mean is not None else dict(d_fixed=d)
    ix = api.make_pca_tree_index(ex, w, branching=b, max_depth=depth, seed=1, hist_bins=16,
                                 ctx=ctx, **kw)
    cfg = api.OptimizerConfig(max_iterations=10 ** 6, min_iterations=10 ** 6 - 1,
                              convergence_fraction=1e-9, histogram_bins=16, nbhd_width=w,
                              spacing=sp, patch_width=2, budget=api.QueryBudget.exact())
    L = api.Level(init, ix, cfg)
    L.prime()
    out = []
    for _ in range(iters):
        L.iterate(1)
        planes, idx, dist = L.download()
        _, _, visited = L.query_stats()
        out.append((planes, idx, dist, float(np.mean(visited == 0))))
    return ix, out


def _same(a, b):
    for t, (x, y) in enumerate(zip(a, b)):
        assert np.array_equal(x[1], y[1]), f"iteration {t + 1}: assignments differ"
        assert np.array_equal(x[2], y[2]), f"iteration {t + 1}: distances differ"
        assert np.array_equal(x[0], y[0]), f"iteration {t + 1}: images differ"


def test_cert_bench_stage_bit_exact(monkeypatch):
    """The bench stage (BASELINE cfg3 finest, C = 5, 1024^2): certificate on
    (K = 128 default, K = 16) vs off, 4 seeded EM iterations."""
    cfg = wl.CONFIGS[3]
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(cfg.ex_size, cfg.n_sin, cfg.ramp, cfg.seed), 2)
    init = wl.init_output(ex, cfg.out, cfg.out, 2, cfg.seed)
    ix, on = _em(_ctx(monkeypatch), ex, init, 8, 2, 32, 4)
    mean, basis, _ = ix.pca()
    _, off = _em(_ctx(monkeypatch, k=0), ex, init, 8, 2, 32, 4, mean, basis)
    _same(on, off)
    assert on[-1][3] > 0.3, f"certificate settled only {on[-1][3]:.3f} of the anchors"
    assert off[-1][3] == 0.0
    _, short = _em(_ctx(monkeypatch, k=16), ex, init, 8, 2, 32, 4, mean, basis)
    _same(short, off)


@pytest.mark.parametrize("d", [12, 48])
@pytest.mark.parametrize("exact_projection", [False, True])
def test_cert_small_stage_bit_exact(monkeypatch, d, exact_projection):
    """d <= 32 and d in (32, 64] list layouts, both projections, short lists."""
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(48, 8, 2.0, 3), 1)
    init = wl.init_output(ex, 96, 96, 1, 3)
    ix, off = _em(_ctx(monkeypatch, k=0, exact_projection=exact_projection), ex, init, 8, 2, d, 5)
    mean, basis, _ = ix.pca()
    for k in (4, 64, 256):
        _, on = _em(_ctx(monkeypatch, k=k, exact_projection=exact_projection), ex, init, 8, 2, d,
                    5, mean, basis)
        _same(on, off)


def test_cert_duplicate_windows(monkeypatch):
    """An exemplar with flat areas: many identical database windows (distance
    0, ties broken by the lowest id) and near-empty histograms."""
    rgb = wl.sinusoid_exemplar(48, 8, 2.0, 5).copy()
    rgb[:, :20, :20] = rgb[:, :1, :1]
    rgb[:, 30:, 10:40] = 128
    ex = wl.rgbs_planes(rgb, 1)
    init = wl.init_output(ex, 80, 80, 1, 5)
    ix, off = _em(_ctx(monkeypatch, k=0), ex, init, 8, 2, 16, 5)
    mean, basis, _ = ix.pca()
    for k in (8, 128):
        _, on = _em(_ctx(monkeypatch, k=k), ex, init, 8, 2, 16, 5, mean, basis)
        _same(on, off)
