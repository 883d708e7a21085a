"""CPU-side checks of the C-ABI library (no GPU needed).

* the in-tree libpersyn_b200.so loads and exports every function declared in
  include/persyn_b200.h;
* host-side logic behind the ABI (grid axes, the search plan closed form, the
  exact histogram fold, the correctly rounded pow) agrees with the oracle;
* without a GPU the context fails loudly (no CPU fallback).
"""
import ctypes as ct
import math
import subprocess
from decimal import Decimal, getcontext

import numpy as np
import pytest

from paper_2006_11851_b200 import native as N
from paper_2006_11851_b200 import api


def test_library_exports_every_header_symbol():
    syms = N.header_symbols()
    assert len(syms) >= 29
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert N.lib.psg_abi_version() == 2


def test_library_is_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("extent,window,step", [(128, 8, 4), (24, 8, 2), (37, 8, 3), (8, 8, 2),
                                                (1024, 32, 8), (9, 2, 1)])
def test_axis_positions_match_oracle(port, extent, window, step):
    assert np.array_equal(api.axis_positions(extent, window, step),
                          port.axis_positions(extent, window, step))


@pytest.mark.parametrize("W,H,w,sp,p", [(128, 128, 8, 4, 2), (24, 24, 8, 2, 1), (37, 23, 8, 3, 2),
                                        (1024, 1024, 8, 2, 2), (1024, 1024, 32, 8, 2)])
def test_plan_matches_oracle(port, W, H, w, sp, p):
    c1, m1 = api.plan(W, H, w, sp, p)
    c2, m2 = port.plan(W, H, w, sp, p)
    assert c1 == c2 and np.array_equal(m1, m2)


def _seq_mass(count, P):
    inv = 1.0 / float(P)
    m = 0.0
    for _ in range(count):
        m += inv
    return m


@pytest.mark.parametrize("P", [16384, 65536, 3249, 1000, 12345, 7, 3 * 17 * 31, 1048576, 262143])
def test_hist_mass_equals_sequential_sum(P):
    rng = np.random.Generator(np.random.PCG64(P))
    counts = sorted(set([0, 1, 2, 3, P // 2, P, P - 1] +
                        list(rng.integers(0, P + 1, 40))))
    for c in counts:
        assert api.hist_mass(int(c), P) == _seq_mass(int(c), P), (c, P)


def test_pow_cr_close_to_glibc_and_correctly_rounded():
    getcontext().prec = 60
    rng = np.random.Generator(np.random.PCG64(5))
    xs = np.concatenate([1e-4 + rng.uniform(0, 5, 4000) ** 2, [1e-4, 1.0, 2.0, 1e4]])
    e = (0.8 - 2.0) / 2.0
    mism_glibc = 0
    for x in xs:
        got = api.pow_cr(float(x), e)
        exact = Decimal(float(x)) ** Decimal(e)
        # correctly rounded: |got - exact| <= half ulp
        ulp = math.ulp(got)
        assert abs(Decimal(got) - exact) <= Decimal(ulp) / 2 * Decimal("1.0000001"), x
        mism_glibc += got != math.pow(float(x), e)
    # glibc pow is < 1 ulp and nearly always correctly rounded
    assert mism_glibc <= len(xs) * 0.01


def test_context_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ct.c_void_p()
    st = N.lib.psg_ctx_create(0, None, ct.byref(h))
    assert st == N.PSG_E_CUDA
    assert "device" in N.lib.psg_last_error().decode().lower()
