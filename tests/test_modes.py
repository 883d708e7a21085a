"""compare_modes and the `persyn bench` table (pipeline.cpp:317-357,
persyn_main.cpp:196-272) over the device brute-force and tree indexes."""
import numpy as np
import pytest

from paper_2006_11851_b200 import workloads as wl

pytestmark = pytest.mark.gpu

api = pytest.importorskip("paper_2006_11851_b200.api")


def _ex():
    return wl.rgbs_planes(wl.sinusoid_exemplar(48, 8, 2.0, 2), 1)


def test_compare_modes_runs_every_mode(gpu_ctx):
    cfg = api.OptimizerConfig(max_iterations=2, min_iterations=1, convergence_fraction=1e-6)
    runs = api.compare_modes(_ex(), 64, 64, 2, (8,), cfg, api.BENCH_MODES, seed=3, ctx=gpu_ctx)
    assert [r.name for r in runs] == ["pixel-brute", "pixel-tree", "patch-tree"]
    for r in runs:
        assert r.nn_calls > 0 and r.part2_millis > 0 and r.wall_millis >= r.part2_millis
        assert np.isfinite(r.final_energy)
    # acceptance #7 (acceptance_main.cpp:324-356): patches issue fewer calls than pixels
    assert runs[2].nn_calls < runs[1].nn_calls
    assert runs[0].nn_calls == runs[1].nn_calls  # same plan (patch width 1) in both pixel modes
    csv = api.modes_to_csv(runs)
    assert csv.splitlines()[0] == "mode,wall_millis,part2_millis,nn_calls,final_energy"
    assert len(csv.splitlines()) == 4


def test_brute_force_synthesis_matches_tree_exact(gpu_ctx):
    """The device BruteForceIndex inside synthesize: an exact full-D search;
    the tree in exact mode returns the PCA-space nearest -- both are valid
    stages (pipeline.cpp:278-284); the brute-force stages report `brute-force`."""
    cfg = api.OptimizerConfig(max_iterations=2, min_iterations=2, convergence_fraction=1e-9,
                              budget=api.QueryBudget.exact())
    out, rep = api.synthesize(_ex(), 64, 64, 1, (8,), cfg, index_kind=api.INDEX_BRUTE_FORCE,
                              ctx=gpu_ctx)
    assert rep["index"] == "brute-force" and out.shape == (4, 64, 64)
    assert len(rep["stages"][0]["trace"]) == 2
    assert all(t.nn_calls > 0 for t in rep["stages"][0]["trace"])


def test_bench_table_shape(gpu_ctx):
    js, csv = api.bench_table(_ex(), [(64, 64), (80, 64)], 1, (8,), 2, 2, seed=1, ctx=gpu_ctx)
    lines = csv.splitlines()
    assert lines[0] == "size,mode,reps,mean_ms,stddev_ms,mean_nn_calls"
    assert len(lines) == 1 + 2 * 3  # sizes x modes (cli_test.cpp:152-168)
    assert lines[1].startswith("64x64,pixel-brute,2,")
    import json
    cells = json.loads(js)
    assert [c["mode"] for c in cells[:3]] == ["pixel-brute", "pixel-tree", "patch-tree"]
    assert all(c["reps"] == 2 and c["mean_ms"] > 0 for c in cells)
