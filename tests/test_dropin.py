"""The C++ drop-in binding (include/persyn_gpu.hpp) inside the reference.

oracle/_ref/dropin_demo is compiled against the reference's headers and
library (oracle/Makefile `dropin`).  It plugs persyn::gpu::GpuSearchIndex
into the REFERENCE's own search_step and optimize_level (per-query plug-in
path, optimizer.hpp:111-119) and compares with the batched device path
persyn::gpu::search_step / optimize_level: identical assignments, distances
and call counts, identical per-iteration stats, images within 1/255, and
psg_status errors rethrown as the reference's exception classes.
"""
import json
import subprocess
from pathlib import Path

import pytest

DEMO = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "dropin_demo"

pytestmark = pytest.mark.gpu


def test_reference_loop_with_device_index_matches_batched_path():
    if not DEMO.exists():
        pytest.skip("oracle/_ref/dropin_demo not built (needs /root/reference)")
    out = subprocess.run([str(DEMO)], capture_output=True, text=True, timeout=600, check=True)
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["search_equal"] is True
    assert r["optimize_stats_equal"] is True and r["iterations"] == 3
    assert r["optimize_max_abs_diff"] <= 1.0 / 255
    assert r["energy_rel_diff"] <= 1e-4
    assert r["domain_error_mapped"] is True
    assert "B200" in r["describe"]
