"""Wire formats next to the hot path, pinned to the reference's own code.

EnergyTrace::to_jsonl (optimizer.cpp:411-424): the per-iteration trace a
caller of optimize_level / synthesize writes.  api.trace_jsonl formats the
device path's IterationStats; the reference's serializer (compiled into
oracle/_ref) formats the same records; the strings must be identical.
"""
import numpy as np
import pytest

from paper_2006_11851_b200 import api


class _It:
    def __init__(self, it, e, ch, calls, ms):
        self.iteration, self.energy, self.changed, self.nn_calls, self.millis = it, e, ch, calls, ms


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_trace_jsonl_matches_reference_serializer(ref, seed):
    rng = np.random.default_rng(seed)
    n = 12
    energy = np.concatenate([[5.0, 0.0, 1e-5, 1e22, 123456789.0, 2.5e-300],
                             rng.uniform(0, 1e5, n - 6) * 10.0 ** rng.integers(-8, 8, n - 6)])
    millis = np.concatenate([[0.0, 1.0, 12.5, 1e-7, 3e4, 7.25],
                             rng.exponential(5.0, n - 6)])
    changed = rng.integers(0, 10 ** 6, n)
    calls = rng.integers(0, 10 ** 9, n)
    stats = [_It(i + 1, float(energy[i]), int(changed[i]), int(calls[i]), float(millis[i]))
             for i in range(n)]
    st7 = np.zeros((n, 7))
    st7[:, 0] = np.arange(1, n + 1)
    st7[:, 1] = energy
    st7[:, 2] = changed
    st7[:, 3] = calls
    assert api.trace_jsonl(stats) == ref.trace_jsonl(st7, millis)


def test_trace_jsonl_empty(ref):
    assert api.trace_jsonl([]) == ref.trace_jsonl(np.zeros((0, 7)), np.zeros(0)) == ""


# ---- SynthesisReport::to_json and the compare_modes formats (pipeline.cpp:182-214, :336-357)
def _values(rng, n):
    v = np.concatenate([[5.0, 0.0, 1e-5, 1e22, 123456789.0, 2.5e-300, 0.1, 1.0 / 3.0],
                        rng.uniform(0, 1e5, max(0, n - 8)) * 10.0 ** rng.integers(-8, 8, max(0, n - 8))])
    return v[:n]


@pytest.mark.parametrize("seed", [0, 1])
def test_synthesis_report_json_matches_reference(ref, seed):
    import json
    rng = np.random.default_rng(seed)
    config = {"sigma": 40.0, "tau": 90.0, "out_width": 256, "out_height": 128, "levels": 2,
              "nbhd_width": 8, "spacing": 2, "patch_width": 2, "robust_exponent": 0.8,
              "epsilon": 0.0001, "max_iterations": 5, "min_iterations": 1,
              "convergence_fraction": 0.01, "histogram_matching": True, "histogram_bins": 16,
              "histogram_include_scale": False, "index": "pca-tree", "pca_variance": 0.95,
              "tree_branching": 4, "budget": "backtrack:4", "seed": 7}
    stages, levels = [], []
    for s, (W, H, n) in enumerate([(64, 32, 3), (128, 64, 0), (256, 128, 5)]):
        e = _values(rng, max(n, 1))
        ms = rng.exponential(3.0, max(n, 1))
        tr = [_It(i + 1, float(e[i]), int(rng.integers(0, 10 ** 5)), int(rng.integers(0, 10 ** 8)),
                  float(ms[i])) for i in range(n)]
        stages.append({"W": W, "H": H, "trace": tr})
        levels.append((W, H, "pca-tree", [(t.iteration, t.energy, t.changed, t.nn_calls, t.millis)
                                          for t in tr]))
    rep = {"part1_millis": 1.25, "part2_millis": float(rng.uniform(1, 1e4)),
           "total_nn_calls": 123456, "stages": stages, "index": "pca-tree"}
    mine = api.synthesis_report_json(rep, config)
    theirs = ref.report_json(json.dumps(config, separators=(",", ":")), rep["part1_millis"],
                             rep["part2_millis"], rep["total_nn_calls"], levels)
    assert mine == theirs


def test_modes_json_csv_match_reference(ref):
    rng = np.random.default_rng(3)
    runs = [api.ModeRun(name, float(w), float(p), int(c), float(e)) for name, w, p, c, e in
            zip(["pixel-brute", "pixel-tree", "patch-tree"], _values(rng, 3) + 1.0,
                rng.uniform(0, 1e4, 3), rng.integers(0, 10 ** 9, 3), _values(rng, 8)[5:])]
    tup = [(r.name, r.wall_millis, r.part2_millis, r.nn_calls, r.final_energy) for r in runs]
    assert api.modes_to_json(runs) == ref.modes_format(tup, 0)
    assert api.modes_to_csv(runs) == ref.modes_format(tup, 1)


# ---- PSM1 scale-map container (scale_map.cpp:125-201) ---------------------------------
@pytest.mark.parametrize("slant,tilt,W,H", [(40.0, 90.0, 33, 17), (0.0, 0.0, 8, 8),
                                            (75.5, 271.25, 64, 40)])
def test_psm1_bytes_match_reference(ref, tmp_path, slant, tilt, W, H):
    vals, b = ref.scale_map(W, H, slant, tilt)
    a, r = tmp_path / "mine.psm", tmp_path / "ref.psm"
    api.save_scale_map(a, vals, slant, tilt, b[1], b[0])
    ref.save_scale_map(vals, slant, tilt, b[1], b[0], r)
    assert a.read_bytes() == r.read_bytes()
    v2, view = api.load_scale_map(r)
    v3, view3 = ref.load_scale_map(a)
    assert np.array_equal(v2, vals) and np.array_equal(v3, vals)
    assert view == view3 == (slant, tilt, b[1], b[0])


def test_psm1_format_errors(tmp_path):
    p = tmp_path / "bad.psm"
    p.write_bytes(b"PSM2\n{}\n")
    with pytest.raises(api.FormatError):
        api.load_scale_map(p)
    api.save_scale_map(p, np.full((2, 3), 0.5, np.float32), 10.0, 0.0, 0.0, 1.0)
    p.write_bytes(p.read_bytes() + b"x")
    with pytest.raises(api.FormatError):
        api.load_scale_map(p)
    p.write_bytes(p.read_bytes()[:-6])
    with pytest.raises(api.FormatError):
        api.load_scale_map(p)
