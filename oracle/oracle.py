"""TEST INFRASTRUCTURE ONLY — ctypes wrappers of the two CPU checkers.

* :class:`Port` — our C restatement (oracle/oracle.c), C-generalised.
* :class:`Ref`  — the reference's own TUs (image, neighborhood, km_tree,
  optimizer .cpp) compiled from /root/reference plus oracle/ref_shim.cpp.

Images are numpy float64 arrays of shape (C, H, W), row 0 = bottom
(image.hpp:11-12).  Features are float32 rows, pixel-major, channel-minor
(neighborhood.cpp:128-135).
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "_build" / "liboracle.so"
REF_SO = HERE / "_ref" / "libpersyn_ref.so"

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_VP = ct.c_void_p
_I = ct.c_int
_I64 = ct.c_int64
_D = ct.c_double

MODES = {"greedy": 0, "backtrack": 1, "exact": 2}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def build(ref: bool = True) -> None:
    """Compile the C restatement and (when /root/reference exists) the reference TUs."""
    targets = ["oracle"]
    if ref and Path("/root/reference/proj/core/src").is_dir():
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _ptr(a):
    return a.ctypes.data_as(ct.c_void_p)


def _dptr(a):
    return a.ctypes.data_as(ct.POINTER(ct.c_double)) if a is not None else None


# ---------------------------------------------------------------------------
class Port:
    """Our C restatement (generalised C = 3 + G channels)."""

    _lib = None

    def __init__(self):
        if Port._lib is None:
            if not PORT_SO.exists():
                build(ref=False)
            Port._lib = ct.CDLL(str(PORT_SO))
            L = Port._lib
            L.or_axis_positions.restype = _I
            L.or_plan.restype = _I64
            L.or_plan.argtypes = [_I, _I, _I, _I, _I, _VP]
            L.or_project.argtypes = [_VP, _I64, _VP, _VP, _I, _VP]
            L.or_extract_window.argtypes = [_VP, _I, _I, _I, _I, _I, _I, _VP]
            L.or_project_all.argtypes = [_VP, _I64, _I64, _VP, _VP, _I, _VP]
            L.or_dist2.restype = _D
            L.or_nearest_lexmin.restype = ct.c_int32
            L.or_nearest_lexmin.argtypes = [_VP, _I64, _I, _VP, _VP]
            L.or_full_distance.restype = _D
            L.or_full_distance.argtypes = [_VP, _VP, _I64]
            L.or_extract_all.restype = _I64
            L.or_extract_all.argtypes = [_VP, _I, _I, _I, _I, _I, _VP]
            L.or_search_step.restype = _I
            L.or_search_step.argtypes = [_VP, _I, _I, _I, _I, _I, _I, _VP, _VP, _I64, _VP, _VP, _I,
                                         _VP, _I64, _I, _VP, _VP, _VP]
            L.or_irls_weight.restype = _D
            L.or_irls_weight.argtypes = [_D, _D, _D]
            L.or_energy.restype = _D
            L.or_energy.argtypes = [_VP, _I64, _D]
            L.or_build_histograms.argtypes = [_VP, _I, _I, _I, _I, _VP]
            L.or_bin_of.restype = _I
            L.or_bin_of.argtypes = [ct.c_float, _I]
            L.or_histogram_penalty.restype = _D
            L.or_histogram_penalty.argtypes = [_VP, _I64, _I, _I, _I, _VP, _VP]
            L.or_update_step.restype = _I
            L.or_update_step.argtypes = [_I, _I, _I, _I, _I, _VP, _VP, _VP, _VP, _VP]
            L.or_assignment_distances.argtypes = [_VP, _I, _I, _I, _I, _I, _VP, _VP, _VP]
            L.or_optimize_level.restype = _I
            L.or_optimize_level.argtypes = [_VP, _I, _I, _I, _I, _I, _I, _VP, _VP, _I64, _VP, _VP,
                                            _I, _D, _D, _I, _I, _D, _I, _I, _VP, _I, _VP, _VP,
                                            _VP]
            L.or_downsample_plane.argtypes = [_VP, _I, _I, _I, _VP]
            L.or_upsample_bilinear_plane.argtypes = [_VP, _I, _I, _I, _VP]
            L.or_fit_to_plane.argtypes = [_VP, _I, _I, _I, _I, _VP]
        self.L = Port._lib

    # geometry ---------------------------------------------------------------
    def axis_positions(self, extent, window, step):
        out = np.zeros(extent + 2, np.int32)
        n = self.L.or_axis_positions(extent, window, step, _ptr(out))
        return out[:n].copy()

    def plan(self, W, H, w, sp, p):
        nx = len(self.axis_positions(W, w, sp))
        ny = len(self.axis_positions(H, w, sp))
        mult = np.zeros(nx * ny, np.int32)
        calls = self.L.or_plan(W, H, w, sp, p, _ptr(mult))
        return int(calls), mult

    def extract_all(self, planes, w, sp=1):
        planes = _c(planes, np.float64)
        C, H, W = planes.shape
        n = self.L.or_extract_all(_ptr(planes), C, W, H, w, sp, None)
        out = np.zeros((n, w * w * C), np.float32)
        self.L.or_extract_all(_ptr(planes), C, W, H, w, sp, _ptr(out))
        return out

    def extract_window(self, planes, ax, ay, w):
        """neighborhood.cpp:120-137 on a (C, H, W) image (C-generalised)."""
        C, H, W = planes.shape
        out = np.zeros(w * w * C, np.float32)
        self.L.or_extract_window(_ptr(planes), C, W, H, ax, ay, w, _ptr(out))
        return out

    def project(self, v, mean, basis):
        v = _c(v, np.float32)
        out = np.zeros(basis.shape[0], np.float64)
        self.L.or_project(_ptr(v), v.size, _ptr(mean), _ptr(basis), basis.shape[0], _ptr(out))
        return out

    # index math -------------------------------------------------------------
    def project_all(self, X, mean, basis):
        X = _c(X, np.float32)
        mean = _c(mean, np.float64)
        basis = _c(basis, np.float64)
        d = basis.shape[0]
        out = np.zeros((X.shape[0], d), np.float64)
        self.L.or_project_all(_ptr(X), X.shape[0], X.shape[1], _ptr(mean), _ptr(basis), d,
                              _ptr(out))
        return out

    def nearest_lexmin(self, pts, q):
        pts = _c(pts, np.float64)
        q = _c(q, np.float64)
        d2 = np.zeros(1, np.float64)
        i = self.L.or_nearest_lexmin(_ptr(pts), pts.shape[0], pts.shape[1], _ptr(q), _ptr(d2))
        return int(i), float(d2[0])

    def full_distance(self, a, b):
        a = _c(a, np.float32)
        b = _c(b, np.float32)
        return self.L.or_full_distance(_ptr(a), _ptr(b), a.size)

    # optimizer ----------------------------------------------------------------
    def search_step(self, planes, w, sp, p, cand, proj, mean, basis, only=None, threads=0):
        planes = _c(planes, np.float64)
        C, H, W = planes.shape
        cand = _c(cand, np.float32)
        proj = _c(proj, np.float64)
        mean = _c(mean, np.float64)
        basis = _c(basis, np.float64)
        nx = len(self.axis_positions(W, w, sp))
        ny = len(self.axis_positions(H, w, sp))
        if only is not None:
            only = _c(only, np.int32)
            n = only.size
        else:
            n = nx * ny
        idx = np.zeros(n, np.int32)
        dist = np.zeros(n, np.float64)
        calls = np.zeros(1, np.int64)
        st = self.L.or_search_step(_ptr(planes), C, W, H, w, sp, p, _ptr(cand), _ptr(proj),
                                   cand.shape[0], _ptr(mean), _ptr(basis), basis.shape[0],
                                   _ptr(only) if only is not None else None, n, threads,
                                   _ptr(idx), _ptr(dist), _ptr(calls))
        if st:
            raise OracleError(st, "search_step")
        return idx, dist, int(calls[0])

    def irls_weight(self, d, r=0.8, eps=1e-4):
        return self.L.or_irls_weight(float(d), r, eps)

    def energy(self, d, r=0.8):
        d = _c(d, np.float64)
        return self.L.or_energy(_ptr(d), d.size, r)

    def build_histograms(self, planes, bins, nslots=3):
        planes = _c(planes, np.float64)
        C, H, W = planes.shape
        out = np.zeros((nslots, bins), np.float64)
        self.L.or_build_histograms(_ptr(planes), W, H, bins, nslots, _ptr(out))
        return out

    def bin_of(self, v, bins):
        return self.L.or_bin_of(float(v), bins)

    def histogram_penalty(self, nb, C, nslots, bins, out_mass, ex_mass):
        nb = _c(nb, np.float32)
        om = _c(out_mass, np.float64)
        em = _c(ex_mass, np.float64)
        return self.L.or_histogram_penalty(_ptr(nb), nb.size // C, C, nslots, bins, _ptr(om),
                                           _ptr(em))

    def update_step(self, C, W, H, w, sp, cand, idx, irls, pen):
        cand = _c(cand, np.float32)
        idx = _c(idx, np.int32)
        irls = _c(irls, np.float64)
        pen = _c(pen, np.float64)
        out = np.zeros((C, H, W), np.float64)
        st = self.L.or_update_step(C, W, H, w, sp, _ptr(cand), _ptr(idx), _ptr(irls), _ptr(pen),
                                   _ptr(out))
        if st:
            raise OracleError(st, "update_step")
        return out

    def assignment_distances(self, planes, w, sp, cand, idx):
        planes = _c(planes, np.float64)
        C, H, W = planes.shape
        idx = _c(idx, np.int32)
        cand = _c(cand, np.float32)
        out = np.zeros(idx.size, np.float64)
        self.L.or_assignment_distances(_ptr(planes), C, W, H, w, sp, _ptr(cand), _ptr(idx),
                                       _ptr(out))
        return out

    def optimize_level(self, init, w, sp, p, cand, proj, mean, basis, r=0.8, eps=1e-4,
                       max_it=20, min_it=1, frac=0.01, bins=16, nslots=3, ex_mass=None,
                       threads=0):
        init = _c(init, np.float64)
        C, H, W = init.shape
        cand = _c(cand, np.float32)
        proj = _c(proj, np.float64)
        mean = _c(mean, np.float64)
        basis = _c(basis, np.float64)
        out = np.zeros_like(init)
        stats = np.zeros((max_it, 7), np.float64)
        n = np.zeros(1, np.int32)
        em = _c(ex_mass, np.float64) if ex_mass is not None else None
        st = self.L.or_optimize_level(_ptr(init), C, W, H, w, sp, p, _ptr(cand), _ptr(proj),
                                      cand.shape[0], _ptr(mean), _ptr(basis), basis.shape[0],
                                      r, eps, max_it, min_it, frac, bins, nslots,
                                      _ptr(em) if em is not None else None, threads, _ptr(out),
                                      _ptr(stats), _ptr(n))
        if st:
            raise OracleError(st, "optimize_level")
        return out, stats[: int(n[0])]

    # resampling ----------------------------------------------------------------
    def downsample(self, plane, f):
        plane = _c(plane, np.float64)
        H, W = plane.shape
        out = np.zeros((H // f, W // f), np.float64)
        self.L.or_downsample_plane(_ptr(plane), W, H, f, _ptr(out))
        return out

    def upsample_bilinear(self, plane, f):
        plane = _c(plane, np.float64)
        H, W = plane.shape
        out = np.zeros((H * f, W * f), np.float64)
        self.L.or_upsample_bilinear_plane(_ptr(plane), W, H, f, _ptr(out))
        return out

    def fit_to(self, plane, ow, oh):
        plane = _c(plane, np.float64)
        H, W = plane.shape
        out = np.zeros((oh, ow), np.float64)
        self.L.or_fit_to_plane(_ptr(plane), W, H, ow, oh, _ptr(out))
        return out


# ---------------------------------------------------------------------------
class Ref:
    """The reference's own TUs (C = 4 only, image.hpp:70)."""

    _lib = None

    def __init__(self):
        if Ref._lib is None:
            if not REF_SO.exists():
                build(ref=True)
            Ref._lib = ct.CDLL(str(REF_SO))
            L = Ref._lib
            L.ref_last_error.restype = ct.c_char_p
            L.ref_kmtree_build.restype = _VP
            L.ref_kmtree_build.argtypes = [_VP, _I64, _I, _I, _I64, ct.c_uint64]
            L.ref_kmtree_destroy.argtypes = [_VP]
            L.ref_kmtree_query.argtypes = [_VP, _VP, _I, _I, _I, _VP, _VP, _VP, _VP]
            L.ref_kmtree_leaves.argtypes = [_VP, _VP, _VP, _VP]
            L.ref_kmtree_structure_json.argtypes = [_VP, ct.c_char_p, _I64, _VP]
            L.ref_trace_jsonl.argtypes = [_VP, _VP, _I, ct.c_char_p, _I64, _VP]
            L.ref_brute_force_nearest.argtypes = [_VP, _I64, _I, _VP, _VP, _VP]
            L.ref_index_create.restype = _VP
            L.ref_index_create.argtypes = [_VP, _I, _I, _I, _VP, _VP, _I, _I, _I, ct.c_uint64]
            L.ref_index_destroy.argtypes = [_VP]
            L.ref_index_count.restype = _I64
            L.ref_index_count.argtypes = [_VP]
            L.ref_index_projected.argtypes = [_VP, _VP]
            L.ref_index_tree.restype = _VP
            L.ref_index_tree.argtypes = [_VP]
            L.ref_index_nearest.argtypes = [_VP, _VP, _I, _I, _I, _VP, _VP, _VP]
            L.ref_search_step.argtypes = [_VP, _VP, _I, _I, _I, _I, _I, _I, _I, _I, _VP, _VP,
                                          _VP, _VP]
            L.ref_update_step.argtypes = [_VP, _I, _I, _I, _I, _VP, _VP, _VP, _VP, _VP]
            L.ref_assignment_distances.argtypes = [_VP, _VP, _I, _I, _I, _I, _VP, _VP]
            L.ref_index_histograms.argtypes = [_VP, _I, _I, _VP]
            L.ref_optimize_level.argtypes = [_VP, _VP, _I, _I, _I, _I, _I, _D, _D, _I, _I, _D, _I,
                                             _I, _I, _I, _I, _VP, _VP, _VP, _VP]
            L.ref_build_histograms.argtypes = [_VP, _I, _I, _I, _I, _VP]
            L.ref_histogram_penalty.argtypes = [_VP, _I64, _I, _I, _VP, _VP, _VP]
            L.ref_irls_weights.argtypes = [_VP, _I64, _D, _D, _VP]
            L.ref_energy_from_distances.argtypes = [_VP, _I64, _D, _VP]
            L.ref_full_distance.argtypes = [_VP, _VP, _I64, _VP]
            L.ref_extract_all.argtypes = [_VP, _I, _I, _I, _I, _VP, _VP]
            L.ref_grid_axes.argtypes = [_I, _I, _I, _I, _VP, _VP, _VP, _VP]
            L.ref_containing_anchors.argtypes = [_I, _I, _I, _I, _I, _I, _I, _VP, _VP]
            L.ref_patch_tiles.argtypes = [_I, _I, _I, _VP, _VP]
            L.ref_downsample.argtypes = [_VP, _I, _I, _I, _VP, _VP, _VP]
            L.ref_upsample_bilinear.argtypes = [_VP, _I, _I, _I, _VP]
            L.ref_scale_map.argtypes = [_I, _I, _D, _D, _VP, _VP]
            L.ref_attach_scale.argtypes = [_VP, _I, _I, _D, _D, _VP]
            L.ref_initialize_output.argtypes = [_VP, _I, _I, _VP, _I, _I, _D, _D, ct.c_uint64,
                                                _VP]
            L.ref_report_json.argtypes = [ct.c_char_p, _D, _D, _I64, _I, _VP, _VP, ct.c_char_p,
                                          _VP, _VP, ct.c_char_p, _I64, _VP]
            L.ref_modes_format.argtypes = [ct.c_char_p, _VP, _VP, _VP, _VP, _I, _I, ct.c_char_p,
                                           _I64, _VP]
            L.ref_save_scale_map.argtypes = [_VP, _I, _I, _D, _D, _D, _D, ct.c_char_p]
            L.ref_load_scale_map.argtypes = [ct.c_char_p, _VP, _VP, _VP]
        self.L = Ref._lib

    def _check(self, st, what=""):
        if st:
            raise OracleError(st, f"{what}: {self.L.ref_last_error().decode()}")

    # geometry
    def grid_axes(self, W, H, w, sp):
        xs = np.zeros(W + 2, np.int32)
        ys = np.zeros(H + 2, np.int32)
        nx = np.zeros(1, np.int32)
        ny = np.zeros(1, np.int32)
        self._check(self.L.ref_grid_axes(W, H, w, sp, _ptr(xs), _ptr(nx), _ptr(ys), _ptr(ny)),
                    "grid")
        return xs[: nx[0]].copy(), ys[: ny[0]].copy()

    def containing_anchors(self, W, H, w, sp, ox, oy, region):
        out = np.zeros(4096, np.int32)
        n = np.zeros(1, np.int32)
        self._check(self.L.ref_containing_anchors(W, H, w, sp, ox, oy, region, _ptr(out), _ptr(n)),
                    "containing_anchors")
        return out[: n[0]].copy()

    def patch_tiles(self, W, H, p):
        n = np.zeros(1, np.int64)
        self._check(self.L.ref_patch_tiles(W, H, p, None, _ptr(n)), "patch_tiles")
        xy = np.zeros(2 * n[0], np.int32)
        self.L.ref_patch_tiles(W, H, p, _ptr(xy), _ptr(n))
        return xy.reshape(-1, 2)

    def extract_all(self, planes, w, sp=1):
        planes = _c(planes, np.float64)
        C, H, W = planes.shape
        assert C == 4
        n = np.zeros(1, np.int64)
        self._check(self.L.ref_extract_all(_ptr(planes), W, H, w, sp, None, _ptr(n)), "extract")
        out = np.zeros((n[0], w * w * 4), np.float32)
        self.L.ref_extract_all(_ptr(planes), W, H, w, sp, _ptr(out), _ptr(n))
        return out

    # km tree
    def kmtree_build(self, pts, branching=4, leaf_threshold=4, seed=0):
        pts = _c(pts, np.float64)
        n, d = pts.shape
        h = self.L.ref_kmtree_build(_ptr(pts), n, d, branching, leaf_threshold, seed)
        if not h:
            raise OracleError(9, self.L.ref_last_error().decode())
        return h

    def kmtree_destroy(self, h):
        self.L.ref_kmtree_destroy(h)

    def kmtree_query(self, h, q, mode="exact", max_leaves=4):
        q = _c(q, np.float64)
        idx = np.zeros(1, np.int32)
        dist = np.zeros(1, np.float64)
        sc = np.zeros(1, np.int64)
        vi = np.zeros(1, np.int64)
        self._check(self.L.ref_kmtree_query(h, _ptr(q), q.size, MODES[mode], max_leaves, _ptr(idx),
                                            _ptr(dist), _ptr(sc), _ptr(vi)), "query")
        return int(idx[0]), float(dist[0]), int(sc[0]), int(vi[0])

    def kmtree_leaves(self, h, count):
        ids = np.zeros(count, np.int32)
        sizes = np.zeros(count, np.int32)
        nl = np.zeros(1, np.int64)
        self._check(self.L.ref_kmtree_leaves(h, _ptr(ids), _ptr(sizes), _ptr(nl)), "leaves")
        return ids, sizes[: nl[0]].copy()

    def trace_jsonl(self, stats7, millis):
        """EnergyTrace::to_jsonl of the given records (ref_trace_jsonl)."""
        st = _c(stats7, np.float64)
        ms = _c(millis, np.float64)
        n = np.zeros(1, np.int64)
        self._check(self.L.ref_trace_jsonl(_ptr(st), _ptr(ms), len(ms), None, 0, _ptr(n)),
                    "trace_jsonl")
        buf = ct.create_string_buffer(int(n[0]) + 1)
        self._check(self.L.ref_trace_jsonl(_ptr(st), _ptr(ms), len(ms), buf, int(n[0]) + 1,
                                           _ptr(n)), "trace_jsonl")
        return buf.value.decode()

    def kmtree_structure_json(self, h):
        n = np.zeros(1, np.int64)
        self.L.ref_kmtree_structure_json(h, None, 0, _ptr(n))
        buf = ct.create_string_buffer(int(n[0]) + 1)
        self.L.ref_kmtree_structure_json(h, buf, int(n[0]) + 1, _ptr(n))
        return buf.value.decode()

    def brute_force_nearest(self, pts, q):
        pts = _c(pts, np.float64)
        q = _c(q, np.float64)
        idx = np.zeros(1, np.int32)
        dist = np.zeros(1, np.float64)
        self._check(self.L.ref_brute_force_nearest(_ptr(pts), pts.shape[0], pts.shape[1], _ptr(q),
                                                   _ptr(idx), _ptr(dist)), "brute")
        return int(idx[0]), float(dist[0])

    # index + optimizer
    def index_create(self, ex_planes, w, mean=None, basis=None, kind="tree", branching=4,
                     seed=0):
        ex = _c(ex_planes, np.float64)
        C, EH, EW = ex.shape
        assert C == 4, "the reference hard-codes C = 4 (image.hpp:70)"
        k = {"tree": 0, "pca_brute": 1, "brute": 2}[kind]
        mean = _c(mean, np.float64) if mean is not None else np.zeros(1)
        basis = _c(basis, np.float64) if basis is not None else np.zeros((1, 1))
        d = basis.shape[0] if k != 2 else 0
        h = self.L.ref_index_create(_ptr(ex), EW, EH, w, _ptr(mean), _ptr(basis), d, k, branching,
                                    seed)
        if not h:
            raise OracleError(9, self.L.ref_last_error().decode())
        return RefIndex(self, h, d)

    def build_histograms(self, planes, bins, include_scale=False):
        planes = _c(planes, np.float64)
        C, H, W = planes.shape
        ns = 4 if include_scale else 3
        out = np.zeros((ns, bins), np.float64)
        self._check(self.L.ref_build_histograms(_ptr(planes), W, H, bins, int(include_scale),
                                                _ptr(out)), "hist")
        return out

    def histogram_penalty(self, nb, bins, out_mass, ex_mass, include_scale=False):
        nb = _c(nb, np.float32)
        om = _c(out_mass, np.float64)
        em = _c(ex_mass, np.float64)
        pen = np.zeros(1, np.float64)
        self._check(self.L.ref_histogram_penalty(_ptr(nb), nb.size, bins, int(include_scale),
                                                 _ptr(om), _ptr(em), _ptr(pen)), "penalty")
        return float(pen[0])

    def irls_weights(self, d, r=0.8, eps=1e-4):
        d = _c(d, np.float64)
        out = np.zeros_like(d)
        self._check(self.L.ref_irls_weights(_ptr(d), d.size, r, eps, _ptr(out)), "irls")
        return out

    def energy(self, d, r=0.8):
        d = _c(d, np.float64)
        out = np.zeros(1, np.float64)
        self._check(self.L.ref_energy_from_distances(_ptr(d), d.size, r, _ptr(out)), "energy")
        return float(out[0])

    def full_distance(self, a, b):
        a = _c(a, np.float32)
        b = _c(b, np.float32)
        out = np.zeros(1, np.float64)
        self._check(self.L.ref_full_distance(_ptr(a), _ptr(b), a.size, _ptr(out)), "full_distance")
        return float(out[0])

    def downsample(self, rgb, f):
        rgb = _c(rgb, np.float64)
        _, H, W = rgb.shape
        ow = np.zeros(1, np.int32)
        oh = np.zeros(1, np.int32)
        out = np.zeros((3, H // f, W // f), np.float64)
        self._check(self.L.ref_downsample(_ptr(rgb), W, H, f, _ptr(out), _ptr(ow), _ptr(oh)),
                    "downsample")
        return out

    def upsample_bilinear(self, rgb, f):
        rgb = _c(rgb, np.float64)
        _, H, W = rgb.shape
        out = np.zeros((3, H * f, W * f), np.float64)
        self._check(self.L.ref_upsample_bilinear(_ptr(rgb), W, H, f, _ptr(out)), "upsample")
        return out


    # part 1 (scale_map.cpp, pipeline.cpp:96-175; pipeline.cpp built with the
    # one-token fix of :118, oracle/Makefile)
    def scale_map(self, W, H, slant, tilt):
        """compute_scale_map: (raw float32 values (H, W), (s_max, s_min, s_delta))."""
        vals = np.zeros((H, W), np.float32)
        b = np.zeros(3, np.float64)
        self._check(self.L.ref_scale_map(W, H, slant, tilt, _ptr(vals), _ptr(b)), "scale_map")
        return vals, b

    def attach_scale(self, rgb, slant, tilt):
        rgb = _c(rgb, np.float64)
        _, H, W = rgb.shape
        out = np.zeros((4, H, W), np.float64)
        self._check(self.L.ref_attach_scale(_ptr(rgb), W, H, slant, tilt, _ptr(out)), "attach")
        return out

    def initialize_output(self, ex4, out_vals, s_min, s_max, seed):
        ex4 = _c(ex4, np.float64)
        _, eh, ew = ex4.shape
        v = _c(out_vals, np.float32)
        oh, ow = v.shape
        out = np.zeros((4, oh, ow), np.float64)
        self._check(self.L.ref_initialize_output(_ptr(ex4), ew, eh, _ptr(v), ow, oh, s_min, s_max,
                                                 seed, _ptr(out)), "initialize_output")
        return out


    def _text(self, fn, *args):
        n = np.zeros(1, np.int64)
        self._check(fn(*args, None, 0, _ptr(n)), "format")
        buf = ct.create_string_buffer(int(n[0]) + 1)
        self._check(fn(*args, buf, int(n[0]) + 1, _ptr(n)), "format")
        return buf.value.decode()

    def report_json(self, config_echo, part1, part2, total_calls, levels):
        """levels: [(width, height, index name, [(iter, energy, changed, nn_calls, millis)])]"""
        w = np.array([l[0] for l in levels], np.int32)
        h = np.array([l[1] for l in levels], np.int32)
        names = "\n".join(l[2] for l in levels).encode()
        ni = np.array([len(l[3]) for l in levels], np.int32)
        st = np.array([list(t) for l in levels for t in l[3]] or [[0] * 5], np.float64)
        return self._text(self.L.ref_report_json, config_echo.encode(), part1, part2, total_calls,
                          len(levels), _ptr(w), _ptr(h), names, _ptr(ni), _ptr(st))

    def save_scale_map(self, values, slant, tilt, s_min, s_max, path):
        v = _c(values, np.float32)
        H, W = v.shape
        self._check(self.L.ref_save_scale_map(_ptr(v), W, H, slant, tilt, s_min, s_max,
                                              str(path).encode()), "save_scale_map")

    def load_scale_map(self, path):
        wh = np.zeros(2, np.int32)
        vb = np.zeros(4, np.float64)
        self._check(self.L.ref_load_scale_map(str(path).encode(), _ptr(wh), _ptr(vb), None), "load")
        v = np.zeros((wh[1], wh[0]), np.float32)
        self._check(self.L.ref_load_scale_map(str(path).encode(), _ptr(wh), _ptr(vb), _ptr(v)),
                    "load")
        return v, tuple(vb)

    def modes_format(self, runs, which):
        names = "\n".join(r[0] for r in runs).encode()
        cols = [np.array([r[k] for r in runs], np.float64) for k in (1, 2, 4)]
        calls = np.array([r[3] for r in runs], np.int64)
        return self._text(self.L.ref_modes_format, names, _ptr(cols[0]), _ptr(cols[1]),
                          _ptr(calls), _ptr(cols[2]), len(runs), which)


class RefIndex:
    def __init__(self, ref: Ref, h, d):
        self.ref, self.h, self.d = ref, h, d
        self.count = int(ref.L.ref_index_count(h))

    def __del__(self):
        try:
            self.ref.L.ref_index_destroy(self.h)
        except Exception:
            pass

    def projected(self):
        out = np.zeros((self.count, self.d), np.float64)
        self.ref._check(self.ref.L.ref_index_projected(self.h, _ptr(out)), "projected")
        return out

    def tree(self):
        return self.ref.L.ref_index_tree(self.h)

    def nearest(self, q, mode="exact", max_leaves=4):
        q = _c(q, np.float32)
        idx = np.zeros(1, np.int32)
        dist = np.zeros(1, np.float64)
        sc = np.zeros(1, np.int64)
        self.ref._check(self.ref.L.ref_index_nearest(self.h, _ptr(q), q.size, MODES[mode],
                                                     max_leaves, _ptr(idx), _ptr(dist), _ptr(sc)),
                        "nearest")
        return int(idx[0]), float(dist[0]), int(sc[0])

    def search_step(self, planes, w, sp, p=2, mode="exact", max_leaves=4, workers=0):
        planes = _c(planes, np.float64)
        C, H, W = planes.shape
        xs, ys = self.ref.grid_axes(W, H, w, sp)
        A = len(xs) * len(ys)
        idx = np.zeros(A, np.int32)
        dist = np.zeros(A, np.float64)
        calls = np.zeros(1, np.int64)
        sc = np.zeros(1, np.int64)
        self.ref._check(self.ref.L.ref_search_step(self.h, _ptr(planes), W, H, w, sp, p,
                                                   MODES[mode], max_leaves, workers, _ptr(idx),
                                                   _ptr(dist), _ptr(calls), _ptr(sc)),
                        "search_step")
        return idx, dist, int(calls[0]), int(sc[0])

    def update_step(self, planes, w, sp, idx, irls, pen):
        planes = _c(planes, np.float64)
        C, H, W = planes.shape
        out = np.zeros_like(planes)
        self.ref._check(self.ref.L.ref_update_step(self.h, W, H, w, sp, _ptr(_c(idx, np.int32)),
                                                   _ptr(_c(irls, np.float64)),
                                                   _ptr(_c(pen, np.float64)), _ptr(planes),
                                                   _ptr(out)), "update_step")
        return out

    def assignment_distances(self, planes, w, sp, idx):
        planes = _c(planes, np.float64)
        C, H, W = planes.shape
        idx = _c(idx, np.int32)
        out = np.zeros(idx.size, np.float64)
        self.ref._check(self.ref.L.ref_assignment_distances(self.h, _ptr(planes), W, H, w, sp,
                                                            _ptr(idx), _ptr(out)), "assign")
        return out

    def em_iteration(self, state, w, sp, p=2, r=0.8, eps=1e-4, bins=16, hist_on=True,
                     mode="exact", max_leaves=4, workers=0):
        """One optimize_level loop body through the reference's functions.
        state: dict with 'planes' (C,H,W) updated in place, 'idx', 'dist',
        'primed'.  Returns (energy, changed)."""
        planes = state["planes"]
        C, H, W = planes.shape
        if "idx" not in state:
            xs, ys = self.ref.grid_axes(W, H, w, sp)
            state["idx"] = np.zeros(len(xs) * len(ys), np.int32)
            state["dist"] = np.zeros(len(xs) * len(ys), np.float64)
            state["primed"] = np.zeros(1, np.int32)
        en = np.zeros(1, np.float64)
        ch = np.zeros(1, np.int64)
        L = self.ref.L
        if not getattr(L.ref_em_iteration, "_typed", False):
            L.ref_em_iteration.argtypes = [_VP, _VP, _I, _I, _I, _I, _I, _D, _D, _I, _I, _I, _I,
                                           _I, _VP, _VP, _VP, _VP, _VP]
            L.ref_em_iteration._typed = True
        self.ref._check(L.ref_em_iteration(self.h, _ptr(planes), W, H, w, sp, p, r, eps, bins,
                                           int(hist_on), MODES[mode], max_leaves, workers,
                                           _ptr(state["idx"]), _ptr(state["dist"]),
                                           _ptr(state["primed"]), _ptr(en), _ptr(ch)),
                        "em_iteration")
        return float(en[0]), int(ch[0])

    def histograms(self, bins, include_scale=False):
        out = np.zeros((4 if include_scale else 3, bins), np.float64)
        self.ref._check(self.ref.L.ref_index_histograms(self.h, bins, int(include_scale),
                                                        _ptr(out)), "hist")
        return out

    def optimize_level(self, init, w, sp, p=2, r=0.8, eps=1e-4, max_it=20, min_it=1, frac=0.01,
                       bins=16, hist_on=True, include_scale=False, mode="exact", max_leaves=4):
        init = _c(init, np.float64)
        C, H, W = init.shape
        out = np.zeros_like(init)
        stats = np.zeros((max_it, 7), np.float64)
        millis = np.zeros(max_it, np.float64)
        n = np.zeros(1, np.int32)
        self.ref._check(self.ref.L.ref_optimize_level(self.h, _ptr(init), W, H, w, sp, p, r, eps,
                                                      max_it, min_it, frac, bins, int(hist_on),
                                                      int(include_scale), MODES[mode],
                                                      max_leaves, _ptr(out), _ptr(stats),
                                                      _ptr(millis), _ptr(n)),
                        "optimize_level")
        k = int(n[0])
        return out, stats[:k], millis[:k]


def available() -> dict:
    return {"port": PORT_SO.exists(), "ref": REF_SO.exists()}


def host_cores() -> int:
    return os.cpu_count() or 1


def fit_pca(X, variance_target=0.95, d_fixed=0, d_cap=0):
    """numpy restatement of fit_pca (pca.cpp:49-101) used to make injected
    bases for parity tests: mean, cov = Xc^T Xc / (n-1), symmetric eigen-
    decomposition, descending clamped variances, smallest prefix reaching the
    target (optionally fixed / capped), sign = largest-|.| entry positive.
    Eigen3 is absent, so bit-parity of the fit with the reference is unpinned;
    the basis is injected into both sides."""
    X = np.asarray(X, np.float64)
    n, D = X.shape
    if n < 2:
        raise OracleError(1, "PCA needs at least 2 points")
    mean = X.mean(axis=0)
    Xc = X - mean
    cov = Xc.T @ Xc / (n - 1)
    evals, evecs = np.linalg.eigh(cov)
    var = np.maximum(0.0, evals[::-1])
    total = var.sum()
    if d_fixed:
        d = min(d_fixed, D)
    elif total > 0:
        cum = np.cumsum(var)
        d = int(np.searchsorted(cum >= variance_target * total, True)) + 1
        d = min(d, D)
        if d_cap:
            d = min(d, d_cap)
    else:
        d = 0
    basis = np.zeros((d, D))
    for k in range(d):
        comp = evecs[:, D - 1 - k].copy()
        arg = int(np.argmax(np.abs(comp)))
        if comp[arg] < 0:
            comp = -comp
        basis[k] = comp
    return mean, basis, var
