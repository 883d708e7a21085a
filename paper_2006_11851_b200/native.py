"""ctypes binding of the in-tree C-ABI library ``libpersyn_b200.so``.

The library is the product: every call lands in hand-written sm_100a kernels.
There is no fallback — if the shared object is missing this module raises at
import, and without a B200 ``psg_ctx_create`` returns PSG_E_CUDA.
"""
from __future__ import annotations

import ctypes as ct
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libpersyn_b200.so"
HEADER = PKG.parent / "include" / "persyn_b200.h"

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(make -C paper_2006_11851_b200/csrc). There is no CPU fallback.")

lib = ct.CDLL(str(LIB_PATH))

# ---- status codes (include/persyn_b200.h) -----------------------------------
PSG_OK, PSG_E_DOMAIN, PSG_E_SHAPE, PSG_E_LOGIC, PSG_E_IO, PSG_E_FORMAT, PSG_E_CUDA, PSG_E_NCCL = \
    range(8)
PSG_GREEDY, PSG_BACKTRACK, PSG_EXACT = 0, 1, 2


class psg_tree_import(ct.Structure):
    _fields_ = [("n_nodes", ct.c_int64), ("n_children", ct.c_void_p), ("n_leaves", ct.c_int64),
                ("leaf_sizes", ct.c_void_p), ("leaf_ids", ct.c_void_p)]


class psg_budget(ct.Structure):
    _fields_ = [("mode", ct.c_int), ("max_leaves", ct.c_int)]


class psg_index_cfg(ct.Structure):
    _fields_ = [("variance_target", ct.c_double), ("d_cap", ct.c_int), ("d_fixed", ct.c_int),
                ("branching", ct.c_int), ("max_depth", ct.c_int), ("leaf_threshold", ct.c_int),
                ("seed", ct.c_uint64), ("hist_bins", ct.c_int), ("hist_include_scale", ct.c_int),
                ("tree_kind", ct.c_int)]


class psg_opt_cfg(ct.Structure):
    _fields_ = [("robust_exponent", ct.c_double), ("distance_epsilon", ct.c_double),
                ("max_iterations", ct.c_int), ("min_iterations", ct.c_int),
                ("convergence_fraction", ct.c_double), ("histogram_bins", ct.c_int),
                ("histogram_matching", ct.c_int), ("histogram_include_scale", ct.c_int),
                ("spacing", ct.c_int), ("patch_width", ct.c_int), ("budget", psg_budget)]


class psg_iter_stats(ct.Structure):
    _fields_ = [("iteration", ct.c_int), ("energy", ct.c_double), ("changed", ct.c_int64),
                ("nn_calls", ct.c_int64), ("millis", ct.c_double),
                ("lsq_energy_before", ct.c_double), ("lsq_energy_after", ct.c_double),
                ("points_scanned", ct.c_int64), ("unique_queries", ct.c_int64),
                ("unique_points_scanned", ct.c_int64)]


class psg_band(ct.Structure):
    _fields_ = [(n, ct.c_int) for n in ("W", "H", "w", "spacing", "rank", "world", "p0", "p1",
                                        "e1", "hlo", "a0", "a1", "nx", "ny")]


class psg_stage_list(ct.Structure):
    _fields_ = [("n_sizes", ct.c_int), ("sizes", ct.c_int * 4)]


class psg_request(ct.Structure):
    _fields_ = [("exemplar", ct.POINTER(ct.c_double)), ("C", ct.c_int), ("ew", ct.c_int),
                ("eh", ct.c_int), ("out_guidance", ct.POINTER(ct.c_double)), ("out_w", ct.c_int),
                ("out_h", ct.c_int), ("levels", ct.c_int), ("stages", psg_stage_list),
                ("cfg", psg_opt_cfg), ("index", psg_index_cfg), ("seed", ct.c_uint64),
                ("guidance_kind", ct.c_int), ("stage_mean", ct.POINTER(ct.c_void_p)),
                ("stage_basis", ct.POINTER(ct.c_void_p)), ("stage_d", ct.POINTER(ct.c_int)),
                ("index_kind", ct.c_int), ("trace", ct.c_void_p), ("trace_cap", ct.c_int)]


class psg_stage_report(ct.Structure):
    _fields_ = [("level", ct.c_int), ("w", ct.c_int), ("W", ct.c_int), ("H", ct.c_int),
                ("ew", ct.c_int), ("eh", ct.c_int), ("d", ct.c_int), ("iterations", ct.c_int),
                ("final_energy", ct.c_double), ("nn_calls", ct.c_int64),
                ("index_millis", ct.c_double), ("optimize_millis", ct.c_double),
                ("trace_first", ct.c_int), ("trace_count", ct.c_int)]


class psg_report(ct.Structure):
    _fields_ = [("n_stages", ct.c_int), ("stages", psg_stage_report * 16),
                ("part1_millis", ct.c_double), ("part2_millis", ct.c_double),
                ("total_nn_calls", ct.c_int64), ("final_energy", ct.c_double),
                ("n_trace", ct.c_int)]


VP = ct.c_void_p
I = ct.c_int
I64 = ct.c_int64
D = ct.c_double
PP = ct.POINTER(ct.c_void_p)

_SIGS = {
    "psg_last_error": (ct.c_char_p, []),
    "psg_abi_version": (I, []),
    "psg_ctx_create": (I, [I, VP, PP]),
    "psg_ctx_destroy": (None, [VP]),
    "psg_ctx_synchronize": (I, [VP]),
    "psg_ctx_launch_count": (I64, [VP]),
    "psg_ctx_profile": (I, [VP, I]),
    "psg_ctx_kernel_times": (I, [VP, VP, VP, VP, I]),
    "psg_index_create": (I, [VP, VP, I, I, I, I, VP, VP, I, ct.POINTER(psg_index_cfg), PP]),
    "psg_index_create_vectors": (I, [VP, VP, I64, I, VP, VP, I, ct.POINTER(psg_index_cfg), PP]),
    "psg_index_destroy": (None, [VP]),
    "psg_index_info": (I, [VP, VP]),
    "psg_index_pca": (I, [VP, VP, VP, VP]),
    "psg_index_projected": (I, [VP, VP]),
    "psg_index_leaves": (I, [VP, VP, VP, VP]),
    "psg_index_histograms": (I, [VP, VP]),
    "psg_index_import_tree": (I, [VP, VP, VP]),
    "psg_reference_tree_host": (I, [VP, I64, I, I, I, ct.c_uint64, VP, VP, VP, VP, VP]),
    "psg_index_create_brute": (I, [VP, VP, I, I, I, I, I, I, PP]),
    "psg_index_create_brute_vectors": (I, [VP, VP, I64, I, PP]),
    "psg_index_query": (I, [VP, VP, VP, I64, psg_budget, VP, VP, VP, VP]),
    "psg_search_step": (I, [VP, VP, VP, I, I, I, I, psg_budget, VP, VP, VP, VP]),
    "psg_update_step": (I, [VP, VP, VP, VP, VP, I, I, I, VP]),
    "psg_optimize_level": (I, [VP, VP, VP, I, I, ct.POINTER(psg_opt_cfg), VP, VP, VP, VP]),
    "psg_level_create": (I, [VP, VP, VP, I, I, ct.POINTER(psg_opt_cfg), VP, PP]),
    "psg_level_prime": (I, [VP]),
    "psg_level_iterate": (I, [VP, I, I, VP, VP]),
    "psg_level_download": (I, [VP, VP, VP, VP]),
    "psg_level_state_dev": (I, [VP, PP, PP, PP]),
    "psg_level_query_stats": (I, [VP, VP, VP, VP]),
    "psg_level_destroy": (None, [VP]),
    "psg_synthesize": (I, [VP, ct.POINTER(psg_request), VP, ct.POINTER(psg_report)]),
    "psg_shard_plan": (I, [I, I, I, I, I, I, ct.POINTER(psg_band)]),
    "psg_band_create": (I, [VP, VP, VP, ct.POINTER(psg_band), ct.POINTER(psg_opt_cfg), VP, PP]),
    "psg_band_phase1": (I, [VP, VP]),
    "psg_band_phase2": (I, [VP, VP, I, VP]),
    "psg_band_phase3": (I, [VP, VP, I, VP]),
    "psg_band_phase4": (I, [VP, VP, VP]),
    "psg_band_commit": (I, [VP, VP, VP]),
    "psg_axis_positions": (I, [I, I, I, VP]),
    "psg_plan": (I64, [I, I, I, I, I, VP]),
    "psg_pow_cr": (D, [D, D]),
    "psg_hist_mass": (D, [I64, I64]),
    "psg_initialize_output": (I, [VP, I, I, I, VP, I, I, D, D, ct.c_uint64, VP]),
    "psg_downsample": (I, [VP, VP, I, I, I, I, VP]),
    "psg_upsample_bilinear": (I, [VP, VP, I, I, I, I, VP]),
    "psg_fit_to": (I, [VP, VP, I, I, I, I, I, VP]),
    "psg_debug_projection": (I, [VP, VP, VP, I, I, I, VP, VP, VP]),
    "psg_comm_unique_id": (I, [VP]),
    "psg_comm_create": (I, [VP, VP, I, I, PP]),
    "psg_comm_destroy": (None, [VP]),
    "psg_band_iterate": (I, [VP, VP, I, I, VP, VP]),
    "psg_optimize_level_sharded": (I, [VP, VP, VP, VP, I, I, ct.POINTER(psg_opt_cfg), VP, VP,
                                       VP, VP]),
    "psg_optimize_level_loopback": (I, [VP, VP, VP, I, I, ct.POINTER(psg_opt_cfg), VP, I, VP,
                                        VP, VP]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def header_symbols() -> list[str]:
    """Function names declared in include/persyn_b200.h."""
    import re
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(psg_[a-z0-9_]+)\s*\(", text)))


class PersynError(RuntimeError):
    """Base of the mapped reference exceptions (errors.hpp:8-36)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class DomainError(PersynError):
    pass


class ShapeError(PersynError):
    pass


class LogicError(PersynError):
    pass


class CudaError(PersynError):
    pass


_EXC = {PSG_E_DOMAIN: DomainError, PSG_E_SHAPE: ShapeError, PSG_E_LOGIC: LogicError,
        PSG_E_CUDA: CudaError, PSG_E_NCCL: CudaError}


def check(status: int) -> None:
    if status != PSG_OK:
        msg = lib.psg_last_error().decode(errors="replace")
        raise _EXC.get(status, PersynError)(status, msg)


def loaded_path() -> str:
    return os.path.realpath(str(LIB_PATH))
