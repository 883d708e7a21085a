"""Row-band sharding orchestrated by the library itself (shard.cpp): NCCL
collectives / send-recv on the context stream, or the in-process loopback
with the same exchange buffers.  Bit-identical to one device."""
import numpy as np
import pytest

from oracle.oracle import fit_pca
from paper_2006_11851_b200 import workloads as wl

api = pytest.importorskip("paper_2006_11851_b200.api")


def _case(port, G=2, ex_size=40, out=96, d=12, seed=3, hist=True, iters=3):
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(ex_size, 8, 2.0, seed), G)
    init = wl.init_output(ex, out, out, G, seed)
    cand = port.extract_all(ex, 8, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=d)
    cfg = api.OptimizerConfig(max_iterations=iters, min_iterations=iters,
                              convergence_fraction=1e-9, histogram_matching=hist, nbhd_width=8,
                              spacing=2, patch_width=2, budget=api.QueryBudget.exact())
    return ex, init, mean, basis, cfg


def test_nccl_unique_id_without_gpu_or_with():
    """NCCL is loaded at run time (no link dependency); a unique id is 128 bytes."""
    try:
        uid = api.comm_unique_id()
    except api.PersynError as e:  # no libnccl on this host
        pytest.skip(str(e))
    assert isinstance(uid, bytes) and len(uid) == 128


@pytest.mark.gpu
@pytest.mark.parametrize("world,hist", [(1, True), (2, True), (3, True), (4, False)])
def test_loopback_bands_equal_single_device(gpu_ctx, port, world, hist):
    ex, init, mean, basis, cfg = _case(port, hist=hist)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, max_depth=4,
                                 hist_bins=16 if hist else 0, ctx=gpu_ctx)
    ref, st_ref = api.optimize_level(init, ix, cfg)
    out, st = api.optimize_level_loopback(init, ix, cfg, world)
    assert np.array_equal(out, ref)
    assert [s.changed for s in st] == [s.changed for s in st_ref]
    assert [s.nn_calls for s in st] == [s.nn_calls for s in st_ref]
    for a, b in zip(st, st_ref):
        assert abs(a.energy - b.energy) <= 1e-12 * abs(b.energy)


@pytest.mark.gpu
@pytest.mark.parametrize("world,budget", [(2, "bt4"), (3, "greedy"), (3, "bt4")])
def test_loopback_bands_budget_searches_equal_single_device(gpu_ctx, port, world, budget):
    """Row bands with the reference's default budget: the bands' lane-group
    searches (tensor-core projection + band checks, per band) reproduce the
    single-device assignments bit for bit."""
    ex, init, mean, basis, cfg = _case(port)
    cfg.budget = api.QueryBudget.backtrack(4) if budget == "bt4" else api.QueryBudget.greedy()
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, seed=5,
                                 tree_kind=api.TREE_REFERENCE, hist_bins=16, ctx=gpu_ctx)
    ref, st_ref = api.optimize_level(init, ix, cfg)
    out, st = api.optimize_level_loopback(init, ix, cfg, world)
    assert np.array_equal(out, ref)
    assert [s.changed for s in st] == [s.changed for s in st_ref]
    assert [s.nn_calls for s in st] == [s.nn_calls for s in st_ref]


@pytest.mark.gpu
def test_nccl_world1_band_equals_single_device(gpu_ctx, port):
    """A real NCCL communicator (world 1: the exchanges degenerate, the
    collectives still run) through psg_optimize_level_sharded and the
    iterate API."""
    ex, init, mean, basis, cfg = _case(port)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, max_depth=4,
                                 hist_bins=16, ctx=gpu_ctx)
    ref, st_ref = api.optimize_level(init, ix, cfg)
    comm = api.Communicator(gpu_ctx, api.comm_unique_id(), 1, 0)
    out, plan, st = api.optimize_level_sharded(init, ix, cfg, comm)
    assert plan["p0"] == 0 and plan["p1"] == init.shape[1]
    assert np.array_equal(out, ref)
    assert [s.changed for s in st] == [s.changed for s in st_ref]
    band = api.Band(init, ix, cfg, comm)
    band.prime()
    st2 = band.iterate(3)
    assert [s.changed for s in st2] == [s.changed for s in st_ref]


@pytest.mark.gpu
def test_band_plan_mismatch_is_shape_error(gpu_ctx, port):
    ex, init, mean, basis, cfg = _case(port)
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, max_depth=4,
                                 hist_bins=16, ctx=gpu_ctx)
    comm = api.Communicator(gpu_ctx, api.comm_unique_id(), 1, 0)
    import paper_2006_11851_b200.sharding as sh
    plans = sh.all_plans(96, 96, 8, 2, 2)
    gb = sh.GpuBand(ix, init, plans[0], plans, cfg)
    with pytest.raises(api.ShapeError):
        api.N.check(api.N.lib.psg_band_iterate(gb.h, comm.h, 1, 0, None, None))
