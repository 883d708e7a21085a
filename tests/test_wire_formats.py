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
