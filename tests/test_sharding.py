"""Row-sharded EM: plan invariants, and the production
orchestrator (paper_2006_11851_b200/sharding.py) run over world sizes 2 and 3
with gloo on CPU (oracle band backend) and in-process on one GPU (library band
backend), checked bit-for-bit against the unsharded computation."""
import os
import socket

import numpy as np
import pytest

from oracle.oracle import Port, fit_pca
from paper_2006_11851_b200 import sharding as sh
from paper_2006_11851_b200 import workloads as wl


@pytest.mark.parametrize("W,H,w,sp,world", [(64, 64, 8, 2, 2), (64, 64, 8, 2, 3), (40, 96, 8, 4, 4),
                                            (48, 200, 16, 4, 5), (1024, 1024, 8, 2, 8),
                                            (1024, 1024, 32, 8, 8), (37, 53, 8, 3, 2)])
def test_shard_plan_partitions(W, H, w, sp, world):
    port = Port()
    ys = port.axis_positions(H, w, sp)
    plans = sh.all_plans(W, H, w, sp, world)
    assert plans[0]["p0"] == 0 and plans[-1]["p1"] == H
    assert plans[0]["a0"] == 0 and plans[-1]["a1"] == len(ys)
    for g, p in enumerate(plans):
        if g:
            assert p["p0"] == plans[g - 1]["p1"] and p["a0"] == plans[g - 1]["a1"]
        assert p["p0"] <= p["p1"] <= p["e1"] <= H and p["hlo"] <= p["a0"] < p["a1"]
        # every window of an owned anchor lies in the local rows
        assert ys[p["a1"] - 1] + w <= p["e1"] and ys[p["a0"]] >= p["p0"]
        # every anchor covering an owned pixel row is owned or in the halo
        for y in range(p["p0"], p["p1"]):
            cov = [i for i, a in enumerate(ys) if a <= y < a + w]
            assert all(p["hlo"] <= i < p["a1"] for i in cov)
        if g:
            assert p["hlo"] >= plans[g - 1]["a0"]              # halo anchors: rank g-1 only
        if g + 1 < world:
            assert p["e1"] <= plans[g + 1]["p1"]               # halo rows: rank g+1 only


def _case(G=1, ex_size=32, out=64, w=8, sp=2, d=12, seed=3):
    port = Port()
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(ex_size, 8, 2.0, seed), G)
    init = wl.init_output(ex, out, out, G, seed)
    cand = port.extract_all(ex, w, 1)
    mean, basis, _ = fit_pca(cand, d_fixed=d)
    proj = port.project_all(cand, mean, basis)
    exm = port.build_histograms(ex, 16, 3)
    return port, ex, init, cand, mean, basis, proj, exm


def _unsharded(port, init, cand, proj, mean, basis, exm, w, sp, iters):
    return port.optimize_level(init, w, sp, 2, cand, proj, mean, basis, max_it=iters, min_it=iters,
                               frac=1e-9, bins=16, ex_mass=exm)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_loopback_cpu_bands_equal_unsharded(world):
    from oracle.sharded_cpu import CpuBand
    port, ex, init, cand, mean, basis, proj, exm = _case()
    H = W = init.shape[1]
    plans = sh.all_plans(W, H, 8, 2, world)
    bands = [CpuBand(port, cand, proj, mean, basis, init, p, plans, 8, 2, 2, ex_mass=exm)
             for p in plans]
    stats = sh.run_sharded(bands, sh.LoopbackComm(world), 2, 2)
    img = sh.gather_image([b.owned()[0] for b in bands])
    ref, rstats = _unsharded(port, init, cand, proj, mean, basis, exm, 8, 2, 2)
    assert np.array_equal(img, ref)
    for g, r in zip(stats, rstats):
        assert g[3] == r[2]                      # changed (exact)
        assert g[6] + g[7] == r[3]               # nn_calls incl. priming
        assert abs(g[2] - r[1]) <= 1e-12 * abs(r[1])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port_no, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.sharded_cpu import CpuBand
        port, ex, init, cand, mean, basis, proj, exm = _case()
        H = W = init.shape[1]
        plans = sh.all_plans(W, H, 8, 2, world)
        band = CpuBand(port, cand, proj, mean, basis, init, plans[rank], plans, 8, 2, 2,
                       ex_mass=exm)
        stats = sh.run_sharded([band], sh.DistComm(), 2, 2)
        q.put((rank, band.owned()[0], [s.tolist() for s in stats]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_bands_equal_unsharded(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port_no, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict()
    for _ in range(world):
        r, img, st = q.get(timeout=240)
        got[r] = (img, st)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    port, ex, init, cand, mean, basis, proj, exm = _case()
    ref, rstats = _unsharded(port, init, cand, proj, mean, basis, exm, 8, 2, 2)
    img = sh.gather_image([got[r][0] for r in range(world)])
    assert np.array_equal(img, ref)
    for r in range(world):  # every rank sees the same global stats
        assert got[r][1] == got[0][1]
    for g, rr in zip(got[0][1], rstats):
        assert g[3] == rr[2] and g[6] + g[7] == rr[3]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_gpu_bands_loopback_equal_single_device(gpu_ctx, world):
    import torch  # noqa: F401
    from paper_2006_11851_b200 import api
    port, ex, init, cand, mean, basis, proj, exm = _case(G=2, ex_size=40, out=96)
    H = W = init.shape[1]
    ix = api.make_pca_tree_index(ex, 8, mean=mean, basis=basis, branching=8, max_depth=4,
                                 hist_bins=16, ctx=gpu_ctx)
    cfg = api.OptimizerConfig(max_iterations=3, min_iterations=3, convergence_fraction=1e-9,
                              nbhd_width=8, spacing=2, patch_width=2,
                              budget=api.QueryBudget.exact())
    ref_img, ref_stats = api.optimize_level(init, ix, cfg)
    plans = sh.all_plans(W, H, 8, 2, world)
    bands = [sh.GpuBand(ix, init, p, plans, cfg) for p in plans]
    stats = sh.run_sharded(bands, sh.LoopbackComm(world), 3, 3)
    img = sh.gather_image([b.owned()[0] for b in bands])
    assert np.array_equal(img, ref_img)          # bit-identical to one device
    for g, r in zip(stats, ref_stats):
        assert g[3] == r.changed
        assert g[6] + g[7] == r.nn_calls
        assert abs(g[2] - r.energy) <= 1e-10 * abs(r.energy)
