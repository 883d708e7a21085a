"""Part 1 of the pipeline: initialize_output (pipeline.cpp:96-175).

The library's psg_initialize_output is host code (one engine drawn in pixel
order, like the reference); it is compared here with the reference's own
initialize_output (pipeline.cpp compiled from oracle/Makefile's one-token-fixed
copy) on perspective scale maps from the reference's compute_scale_map and on
the guidance-ramp maps psg_synthesize uses.  No GPU needed.
"""
import numpy as np
import pytest

from paper_2006_11851_b200 import workloads as wl

api = pytest.importorskip("paper_2006_11851_b200.api")


@pytest.mark.parametrize("slant,tilt,ew,ow,oh,seed", [(40.0, 90.0, 32, 48, 40, 1),
                                                      (60.0, 30.0, 24, 64, 64, 7),
                                                      (0.0, 0.0, 16, 20, 12, 3),
                                                      (75.0, 270.0, 40, 33, 57, 11)])
def test_initialize_output_matches_reference(ref, slant, tilt, ew, ow, oh, seed):
    rgb = wl.sinusoid_exemplar(ew, 8, 2.0, seed).astype(np.float64) / 255.0
    ex4 = ref.attach_scale(rgb, slant, tilt)
    vals, b = ref.scale_map(ow, oh, slant, tilt)
    s_max, s_min = b[0], b[1]
    mine = api.initialize_output(ex4, vals, s_min, s_max, seed)
    theirs = ref.initialize_output(ex4, vals, s_min, s_max, seed)
    assert np.array_equal(mine, theirs)


@pytest.mark.parametrize("ew,ow,seed", [(16, 32, 1), (32, 64, 5), (64, 128, 9)])
def test_initialize_output_ramp_maps_match_reference(ref, ew, ow, seed):
    """The maps psg_synthesize uses: the row ramp as normalised scale, bounds [0, 1]."""
    ex = wl.rgbs_planes(wl.sinusoid_exemplar(ew, 8, 2.0, seed), 1)
    vals = wl.guidance_planes(ow, ow, 1)[0].astype(np.float32)
    mine = api.initialize_output(ex, vals, 0.0, 1.0, seed)
    theirs = ref.initialize_output(ex, vals, 0.0, 1.0, seed)
    assert np.array_equal(mine, theirs)
    # every output pixel copies an exemplar pixel of (nearly) the same scale
    assert set(np.unique(mine[0])) <= set(np.unique(ex[0]))


def test_initialize_output_rejects_missing_scale():
    with pytest.raises(api.ShapeError):
        api.initialize_output(np.zeros((3, 8, 8)), np.zeros((4, 4), np.float32), 0.0, 1.0, 0)
