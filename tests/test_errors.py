"""Error contract of the C ABI: every precondition the reference checks on the
path raises the same persyn exception class (errors.hpp:26-36) through
psg_status + psg_last_error, and the reference itself (oracle/_ref) agrees
where it exposes the check.

  OptimizerConfig::validate      optimizer.cpp:24-42
  GridSpec::validate             neighborhood.cpp:22-35
  search_step shape checks       optimizer.cpp:278-286
  update_step weight check       optimizer.cpp:366-369
  irls_weight                    optimizer.cpp:112-115
  KmTree::build / fit_pca        km_tree.cpp:145-150, pca.cpp:52
  BruteForceIndex                optimizer.cpp:170-172, 177-179
"""
import numpy as np
import pytest

from oracle.oracle import fit_pca
from paper_2006_11851_b200 import workloads as wl

pytestmark = pytest.mark.gpu

api = pytest.importorskip("paper_2006_11851_b200.api")


@pytest.fixture(scope="module")
def stage(port):
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(32, 8, 2.0, 1), 1)
    init = wl.init_output(ex, 40, 40, 1, 1)
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=8)
    return ex, init, mean, basis


@pytest.fixture(scope="module")
def index(gpu_ctx, stage):
    ex, _, mean, basis = stage
    return api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=4, max_depth=3,
                                   hist_bins=16, ctx=gpu_ctx)


def _cfg(**kw):
    base = dict(max_iterations=2, min_iterations=1, convergence_fraction=0.01, nbhd_width=8,
                spacing=4, patch_width=2, budget=api.QueryBudget.exact())
    base.update(kw)
    return api.OptimizerConfig(**base)


@pytest.mark.parametrize("kw", [
    dict(robust_exponent=0.0), dict(robust_exponent=2.0), dict(distance_epsilon=0.0),
    dict(max_iterations=0), dict(min_iterations=0), dict(min_iterations=3),
    dict(convergence_fraction=0.0), dict(convergence_fraction=1.0), dict(histogram_bins=1),
    dict(patch_width=0), dict(patch_width=5), dict(spacing=0), dict(spacing=9),
])
def test_optimizer_config_validation_domain_errors(stage, index, kw):
    _, init, _, _ = stage
    with pytest.raises(api.DomainError):
        api.optimize_level(init, index, _cfg(**kw))


def test_grid_smaller_than_window_is_domain_error(index):
    tiny = np.full((4, 6, 6), 0.5)
    with pytest.raises(api.DomainError):
        api.search_step(tiny, index, 2, 2, api.QueryBudget.exact())


def test_search_step_channel_mismatch_is_shape_error(stage, index):
    _, init, _, _ = stage
    with pytest.raises(api.ShapeError):
        api.search_step(np.concatenate([init, init[3:]]), index, 4, 2, api.QueryBudget.exact())


def test_backtrack_budget_must_be_positive(stage, index):
    _, init, _, _ = stage
    with pytest.raises(api.DomainError):
        api.search_step(init, index, 4, 2, api.QueryBudget.backtrack(0))


def test_update_step_rejects_non_positive_weights(stage, index, ref):
    ex, init, mean, basis = stage
    idx, _, _, _ = api.search_step(init, index, 4, 2, api.QueryBudget.exact())
    irls = np.ones(idx.size)
    pen = np.zeros(idx.size)
    irls[idx.size // 2] = 0.0
    with pytest.raises(api.DomainError):
        api.update_step(idx, irls, pen, index, 40, 40, 4)
    irls[idx.size // 2] = np.nan
    with pytest.raises(api.DomainError):
        api.update_step(idx, irls, pen, index, 40, 40, 4)
    h = ref.index_create(ex, 8, mean, basis, kind="tree", branching=4, seed=1)
    from oracle.oracle import OracleError
    with pytest.raises(OracleError):
        h.update_step(init, 8, 4, idx, irls, pen)


def test_index_preconditions(gpu_ctx, stage):
    ex, _, _, _ = stage
    with pytest.raises(api.DomainError):       # odd window (neighborhood.cpp:24)
        api.make_pca_tree_index(ex, 7, d_fixed=4, ctx=gpu_ctx)
    with pytest.raises(api.DomainError):       # branching < 2 (km_tree.cpp:146)
        api.make_pca_tree_index(ex, 8, d_fixed=4, branching=1, ctx=gpu_ctx)
    with pytest.raises(api.DomainError):       # window larger than the exemplar
        api.make_pca_tree_index(ex[:, :6, :6], 8, d_fixed=4, ctx=gpu_ctx)
    with pytest.raises(api.DomainError):       # fit_pca needs n >= 2 (pca.cpp:52)
        api.make_pca_tree_index(ex[:, :8, :8], 8, d_fixed=4, ctx=gpu_ctx)
    with pytest.raises(api.ShapeError):        # channels outside 3 + G
        api.make_pca_tree_index(ex[:3], 8, d_fixed=4, ctx=gpu_ctx)
    with pytest.raises(api.DomainError):       # empty candidate set (optimizer.cpp:171)
        api.make_brute_force_vector_index(np.zeros((0, 16), np.float32), ctx=gpu_ctx)


def test_query_dimension_mismatch_is_shape_error(gpu_ctx, index):
    with pytest.raises(api.ShapeError):
        index.nearest(np.zeros((3, index.dim + 1), np.float32))
    bi = api.make_brute_force_vector_index(np.ones((10, 8), np.float32), ctx=gpu_ctx)
    with pytest.raises(api.ShapeError):
        bi.nearest(np.zeros((2, 9), np.float32))


def test_irls_negative_distance_domain_error(port, ref):
    # irls_weight (optimizer.cpp:113): the host restatement and the reference agree
    from oracle.oracle import OracleError
    with pytest.raises(OracleError):
        ref.irls_weights(np.array([1.0, -1.0]), 0.8, 1e-4)
