"""Python mirror of the reference's ``persyn::`` hot-path API over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/core/include/persyn/{optimizer,km_tree,pipeline}.hpp:

* :class:`QueryBudget` (km_tree.hpp:13-25), :class:`OptimizerConfig`
  (optimizer.hpp:37-52), :class:`IterationStats` (optimizer.hpp:153-163);
* :func:`make_pca_tree_index` (optimizer.hpp:126-129) -> :class:`SearchIndex`
  with a batched ``nearest`` (optimizer.hpp:111-119);
* :func:`search_step` (optimizer.hpp:141-143), :func:`update_step`
  (optimizer.hpp:149-151), :func:`optimize_level` (optimizer.hpp:181-183),
  :func:`synthesize` (pipeline.hpp:69).

Images are numpy float64 arrays shaped (C, H, W), row 0 = bottom.  Errors
raise DomainError / ShapeError / LogicError like the reference.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import native as N
from .native import DomainError, LogicError, ShapeError, CudaError, PersynError  # noqa: F401


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _p(a):
    return a.ctypes.data_as(ct.c_void_p) if a is not None else None


# ---------------------------------------------------------------------------
@dataclass
class QueryBudget:
    mode: str = "backtrack"
    max_leaves: int = 4

    @staticmethod
    def greedy():
        return QueryBudget("greedy", 1)

    @staticmethod
    def backtrack(max_leaves: int):
        if max_leaves < 1:
            raise DomainError(N.PSG_E_DOMAIN, "backtrack budget must be >= 1")
        return QueryBudget("backtrack", max_leaves)

    @staticmethod
    def exact():
        return QueryBudget("exact", 0)

    def c(self) -> N.psg_budget:
        m = {"greedy": N.PSG_GREEDY, "backtrack": N.PSG_BACKTRACK, "exact": N.PSG_EXACT}[self.mode]
        return N.psg_budget(m, self.max_leaves)


@dataclass
class OptimizerConfig:
    robust_exponent: float = 0.8
    distance_epsilon: float = 1e-4
    max_iterations: int = 20
    min_iterations: int = 1
    convergence_fraction: float = 0.01
    histogram_bins: int = 16
    histogram_matching: bool = True
    histogram_include_scale: bool = False
    nbhd_width: int = 8
    spacing: int = 2
    patch_width: int = 2
    budget: QueryBudget = field(default_factory=lambda: QueryBudget.backtrack(4))

    def c(self) -> N.psg_opt_cfg:
        return N.psg_opt_cfg(self.robust_exponent, self.distance_epsilon, self.max_iterations,
                             self.min_iterations, self.convergence_fraction, self.histogram_bins,
                             int(self.histogram_matching), int(self.histogram_include_scale),
                             self.spacing, self.patch_width, self.budget.c())


@dataclass
class IterationStats:
    iteration: int
    energy: float
    changed: int
    nn_calls: int
    millis: float
    lsq_energy_before: float
    lsq_energy_after: float
    points_scanned: int
    unique_queries: int
    unique_points_scanned: int

    @staticmethod
    def of(s: N.psg_iter_stats) -> "IterationStats":
        return IterationStats(s.iteration, s.energy, s.changed, s.nn_calls, s.millis,
                              s.lsq_energy_before, s.lsq_energy_after, s.points_scanned,
                              s.unique_queries, s.unique_points_scanned)


# ---------------------------------------------------------------------------
class Context:
    """One device + one CUDA stream (``stream``: a cudaStream_t int or None)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        h = ct.c_void_p()
        N.check(N.lib.psg_ctx_create(device, ct.c_void_p(stream) if stream else None,
                                     ct.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            N.lib.psg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def synchronize(self):
        N.check(N.lib.psg_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        return int(N.lib.psg_ctx_launch_count(self.h))

    def profile(self, enable: bool = True):
        N.check(N.lib.psg_ctx_profile(self.h, int(enable)))

    def kernel_times(self) -> dict:
        """{kernel: (total ms, launches)} of event-timed launches since profile(True)."""
        n = 16
        names = (ct.c_char_p * n)()
        ms = np.zeros(n)
        cnt = np.zeros(n, np.int64)
        k = N.lib.psg_ctx_kernel_times(self.h, ct.cast(names, ct.c_void_p), _p(ms), _p(cnt), n)
        return {names[i].decode(): (float(ms[i]), int(cnt[i])) for i in range(k) if cnt[i]}


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


TREE_DEVICE, TREE_REFERENCE = 0, 1  # psg_tree_kind


def index_cfg(variance_target=0.95, d_cap=0, d_fixed=0, branching=4, max_depth=0,
              leaf_threshold=0, seed=0, hist_bins=0, hist_include_scale=False,
              tree_kind=TREE_DEVICE) -> N.psg_index_cfg:
    return N.psg_index_cfg(variance_target, d_cap, d_fixed, branching, max_depth, leaf_threshold,
                           seed, hist_bins, int(hist_include_scale), int(tree_kind))


class SearchIndex:
    """PCA + k-means tree over an exemplar's dense windows (or a vector set)."""

    def __init__(self, ctx: Context, handle, keep):
        self.ctx = ctx
        self.h = handle
        self._keep = keep
        dims = np.zeros(10, np.int64)
        N.check(N.lib.psg_index_info(self.h, _p(dims)))
        (self.count, self.dim, self.retained_dim, self.channels, self.window, self.ew, self.eh,
         self.n_nodes, self.n_leaves, self.depth) = (int(v) for v in dims)

    def __del__(self):
        if getattr(self, "h", None):
            N.lib.psg_index_destroy(self.h)
            self.h = None

    # PcaModel accessors (pca.hpp:21-31)
    def pca(self):
        mean = np.zeros(self.dim)
        basis = np.zeros((self.retained_dim, self.dim))
        var = np.zeros(self.dim)
        N.check(N.lib.psg_index_pca(self.h, _p(mean), _p(basis), _p(var)))
        return mean, basis, var

    def projected(self) -> np.ndarray:
        out = np.zeros((self.count, self.retained_dim))
        N.check(N.lib.psg_index_projected(self.h, _p(out)))
        return out

    def leaves(self):
        ids = np.zeros(self.count, np.int32)
        sizes = np.zeros(self.count, np.int32)
        nl = ct.c_int64()
        N.check(N.lib.psg_index_leaves(self.h, _p(ids), _p(sizes), ct.byref(nl)))
        return ids, sizes[: nl.value].copy()

    def import_tree(self, n_children, leaf_sizes, leaf_ids):
        """Replace the tree by an external one (psg_index_import_tree): child
        counts in pre-order DFS and KmTree::leaves() (km_tree.cpp:286-318)."""
        nc = _c(n_children, np.int32)
        ls = _c(leaf_sizes, np.int32)
        li = _c(leaf_ids, np.int32)
        t = N.psg_tree_import(nc.size, nc.ctypes.data, ls.size, ls.ctypes.data, li.ctypes.data)
        N.check(N.lib.psg_index_import_tree(self.ctx.h, self.h, ct.byref(t)))
        dims = np.zeros(10, np.int64)
        N.check(N.lib.psg_index_info(self.h, _p(dims)))
        self.n_nodes, self.n_leaves, self.depth = (int(v) for v in dims[7:10])

    def import_reference_tree(self, structure_json, leaves):
        """Import the reference's KmTree from structure_json() (str or dict) and
        leaves() (a list of id lists)."""
        n_children = preorder_child_counts(structure_json)
        sizes = np.array([len(l) for l in leaves], np.int32)
        ids = np.concatenate([np.asarray(l, np.int32) for l in leaves])
        self.import_tree(n_children, sizes, ids)

    def histograms(self, slots=3, bins=16) -> np.ndarray:
        out = np.zeros((slots, bins))
        N.check(N.lib.psg_index_histograms(self.h, _p(out)))
        return out

    def nearest(self, Q: np.ndarray, budget: QueryBudget = QueryBudget.exact()):
        """Batched SearchIndex::nearest: (idx, full-D dist, PCA dist, points scanned)."""
        Q = _c(Q, np.float32)
        if Q.ndim == 1:
            Q = Q[None, :]
        if Q.shape[1] != self.dim:
            raise ShapeError(N.PSG_E_SHAPE, "query dim does not match the candidates")
        n = Q.shape[0]
        idx = np.zeros(n, np.int32)
        dist = np.zeros(n)
        dpca = np.zeros(n)
        sc = np.zeros(n, np.int64)
        N.check(N.lib.psg_index_query(self.ctx.h, self.h, _p(Q), n, budget.c(), _p(idx), _p(dist),
                                      _p(dpca), _p(sc)))
        return idx, dist, dpca, sc


def preorder_child_counts(structure_json) -> np.ndarray:
    """Child counts in pre-order DFS from KmTree::structure_json()
    (km_tree.cpp:300-318: {"root": {"size", "children": [...]}})."""
    import json as _json
    j = _json.loads(structure_json) if isinstance(structure_json, (str, bytes)) else structure_json
    out = []
    stack = [j["root"]]
    while stack:
        node = stack.pop()
        kids = node.get("children", [])
        out.append(len(kids))
        stack.extend(reversed(kids))
    return np.array(out, np.int32)


def make_pca_tree_index(exemplar: np.ndarray, window: int, variance_target: float = 0.95,
                        branching: int = 4, seed: int = 0, *, mean=None, basis=None,
                        d_cap: int = 0, d_fixed: int = 0, max_depth: int = 0,
                        hist_bins: int = 0, hist_include_scale: bool = False,
                        tree_kind: int = TREE_DEVICE,
                        ctx: Optional[Context] = None) -> SearchIndex:
    """make_pca_tree_index(extract_all(exemplar, {w,1,..}), variance, b, seed).
    tree_kind=TREE_REFERENCE builds the reference's own KmTree (same greedy /
    backtrack answers as the reference); the default is the device tree."""
    ctx = ctx or default_context()
    ex = _c(exemplar, np.float64)
    C, eh, ew = ex.shape
    cfg = index_cfg(variance_target, d_cap, d_fixed, branching, max_depth, 0, seed, hist_bins,
                    hist_include_scale, tree_kind)
    m = _c(mean, np.float64) if mean is not None else None
    b = _c(basis, np.float64) if basis is not None else None
    d = b.shape[0] if b is not None else 0
    h = ct.c_void_p()
    N.check(N.lib.psg_index_create(ctx.h, _p(ex), C, ew, eh, window, _p(m), _p(b), d,
                                   ct.byref(cfg), ct.byref(h)))
    return SearchIndex(ctx, h, None)


def make_brute_force_index(exemplar: np.ndarray, window: int, *, hist_bins: int = 0,
                           hist_include_scale: bool = False,
                           ctx: Optional[Context] = None) -> SearchIndex:
    """make_brute_force_index(extract_all(exemplar, {w,1,..})) (optimizer.cpp:168-212)."""
    ctx = ctx or default_context()
    ex = _c(exemplar, np.float64)
    C, eh, ew = ex.shape
    h = ct.c_void_p()
    N.check(N.lib.psg_index_create_brute(ctx.h, _p(ex), C, ew, eh, window, hist_bins,
                                         int(hist_include_scale), ct.byref(h)))
    return SearchIndex(ctx, h, None)


def make_brute_force_vector_index(X: np.ndarray, *, ctx: Optional[Context] = None) -> SearchIndex:
    """make_brute_force_index over an explicit candidate matrix X[n][D]."""
    ctx = ctx or default_context()
    X = _c(X, np.float32)
    h = ct.c_void_p()
    N.check(N.lib.psg_index_create_brute_vectors(ctx.h, _p(X), X.shape[0], X.shape[1],
                                                 ct.byref(h)))
    return SearchIndex(ctx, h, None)


def reference_tree_host(proj: np.ndarray, branching: int, seed: int = 0, leaf_threshold: int = 0):
    """The library's host replica of KmTree::build (km_tree.cpp:141-195) over
    projected points [N][d] -- no device needed.  Returns (pre-order child
    counts, list of the leaves' id arrays in DFS order): psg_tree_import's form."""
    P = _c(proj, np.float64)
    n, d = P.shape
    nc = np.zeros(2 * n, np.int32)
    ls = np.zeros(n, np.int32)
    li = np.zeros(n, np.int32)
    nn, nl = ct.c_int64(), ct.c_int64()
    N.check(N.lib.psg_reference_tree_host(_p(P), n, d, branching, leaf_threshold, seed, _p(nc),
                                          ct.byref(nn), _p(ls), ct.byref(nl), _p(li)))
    sizes = ls[: nl.value]
    return nc[: nn.value].copy(), np.split(li, np.cumsum(sizes)[:-1])


def make_vector_index(X: np.ndarray, variance_target: float = 0.95, branching: int = 8,
                      seed: int = 0, *, mean=None, basis=None, d_fixed: int = 0,
                      max_depth: int = 0, tree_kind: int = TREE_DEVICE,
                      ctx: Optional[Context] = None) -> SearchIndex:
    ctx = ctx or default_context()
    X = _c(X, np.float32)
    cfg = index_cfg(variance_target, 0, d_fixed, branching, max_depth, 0, seed,
                    tree_kind=tree_kind)
    m = _c(mean, np.float64) if mean is not None else None
    b = _c(basis, np.float64) if basis is not None else None
    d = b.shape[0] if b is not None else 0
    h = ct.c_void_p()
    N.check(N.lib.psg_index_create_vectors(ctx.h, _p(X), X.shape[0], X.shape[1], _p(m), _p(b), d,
                                           ct.byref(cfg), ct.byref(h)))
    return SearchIndex(ctx, h, None)


# ---------------------------------------------------------------------------
def trace_jsonl(stats) -> str:
    """EnergyTrace::to_jsonl (optimizer.cpp:411-424): one compact
    {"iter","energy","changed","nn_calls","millis"} object per line, keys in
    that order, numbers in shortest round-trip form (as nlohmann::json)."""
    import json as _json
    out = []
    for s in stats:
        out.append(_json.dumps({"iter": int(s.iteration), "energy": float(s.energy),
                                "changed": int(s.changed), "nn_calls": int(s.nn_calls),
                                "millis": float(s.millis)}, separators=(",", ":")))
        out.append("\n")
    return "".join(out)


def search_step(out: np.ndarray, index: SearchIndex, spacing: int, patch_width: int,
                budget: QueryBudget):
    """(assignments, distances, nn_calls, points_scanned) — optimizer.cpp:275-348."""
    x = _c(out, np.float64)
    C, H, W = x.shape
    if C != index.channels:
        raise ShapeError(N.PSG_E_SHAPE, "candidate dim does not match the grid window")
    nx = N.lib.psg_axis_positions(W, index.window, spacing, None) or 1
    ny = N.lib.psg_axis_positions(H, index.window, spacing, None) or 1
    idx = np.zeros(nx * ny, np.int32)
    dist = np.zeros(nx * ny)
    calls = ct.c_int64()
    sc = ct.c_int64()
    N.check(N.lib.psg_search_step(index.ctx.h, index.h, _p(x), W, H, spacing, patch_width,
                                  budget.c(), _p(idx), _p(dist), ct.byref(calls), ct.byref(sc)))
    return idx, dist, calls.value, sc.value


def update_step(idx, irls, pen, index: SearchIndex, W: int, H: int, spacing: int) -> np.ndarray:
    """update_step with WeightMap{irls, hist_penalty} — optimizer.cpp:350-401."""
    idx = _c(idx, np.int32)
    irls = _c(irls, np.float64)
    pen = _c(pen, np.float64)
    out = np.zeros((index.channels, H, W))
    nx = N.lib.psg_axis_positions(W, index.window, spacing, None)
    ny = N.lib.psg_axis_positions(H, index.window, spacing, None)
    if idx.size != nx * ny or irls.size != nx * ny or pen.size != nx * ny:
        raise ShapeError(N.PSG_E_SHAPE, "assignments/weights do not cover the grid")
    N.check(N.lib.psg_update_step(index.ctx.h, index.h, _p(idx), _p(irls), _p(pen), W, H, spacing,
                                  _p(out)))
    return out


def _check_level_inputs(x: np.ndarray, index: SearchIndex, cfg: OptimizerConfig,
                        exemplar_hist: Optional[np.ndarray]):
    """The C ABI reads C*H*W doubles of the image and bins*slots doubles of the
    exemplar histogram (C = index.channels): validate before handing it raw
    pointers (optimizer.cpp:278-286, :93 HistogramSet::compatible)."""
    if x.ndim != 3 or x.shape[0] != index.channels:
        raise ShapeError(N.PSG_E_SHAPE, "image channels do not match the index")
    if cfg.nbhd_width != index.window:
        raise ShapeError(N.PSG_E_SHAPE, "candidate dim does not match the grid window")
    if exemplar_hist is not None:
        slots = index.channels if cfg.histogram_include_scale else 3
        if np.asarray(exemplar_hist).size != cfg.histogram_bins * slots:
            raise ShapeError(N.PSG_E_SHAPE, "histogram sets are not compatible")


def optimize_level(init: np.ndarray, index: SearchIndex, cfg: OptimizerConfig,
                   exemplar_hist: Optional[np.ndarray] = None):
    """(image, [IterationStats]) — optimizer.cpp:426-516."""
    x = _c(init, np.float64)
    _check_level_inputs(x, index, cfg, exemplar_hist)
    C, H, W = x.shape
    c = cfg.c()
    out = np.zeros_like(x)
    stats = (N.psg_iter_stats * max(cfg.max_iterations, 1))()
    n = ct.c_int()
    eh = _c(exemplar_hist, np.float64) if exemplar_hist is not None else None
    N.check(N.lib.psg_optimize_level(index.ctx.h, index.h, _p(x), W, H, ct.byref(c), _p(eh),
                                     _p(out), ct.cast(stats, ct.c_void_p), ct.byref(n)))
    return out, [IterationStats.of(stats[i]) for i in range(n.value)]


class Level:
    """Device-resident optimize_level state (benchmark / driver use)."""

    def __init__(self, init: np.ndarray, index: SearchIndex, cfg: OptimizerConfig,
                 exemplar_hist: Optional[np.ndarray] = None):
        x = _c(init, np.float64)
        _check_level_inputs(x, index, cfg, exemplar_hist)
        self.C, self.H, self.W = x.shape
        self.index = index
        self.cfg = cfg
        c = cfg.c()
        eh = _c(exemplar_hist, np.float64) if exemplar_hist is not None else None
        h = ct.c_void_p()
        N.check(N.lib.psg_level_create(index.ctx.h, index.h, _p(x), self.W, self.H, ct.byref(c),
                                       _p(eh), ct.byref(h)))
        self.h = h
        self.nx = N.lib.psg_axis_positions(self.W, index.window, cfg.spacing, None)
        self.ny = N.lib.psg_axis_positions(self.H, index.window, cfg.spacing, None)

    def __del__(self):
        if getattr(self, "h", None):
            N.lib.psg_level_destroy(self.h)
            self.h = None

    def prime(self):
        N.check(N.lib.psg_level_prime(self.h))

    def iterate(self, n: int, honor_convergence: bool = False):
        stats = (N.psg_iter_stats * max(n, 1))()
        done = ct.c_int()
        N.check(N.lib.psg_level_iterate(self.h, n, int(honor_convergence),
                                        ct.cast(stats, ct.c_void_p), ct.byref(done)))
        return [IterationStats.of(stats[i]) for i in range(done.value)]

    def query_stats(self):
        """Per-anchor (points_scanned, exact fp64 evaluations, nodes_visited) of the last search."""
        A = self.nx * self.ny
        sc = np.zeros(A, np.int64)
        ex = np.zeros(A, np.int64)
        vi = np.zeros(A, np.int32)
        N.check(N.lib.psg_level_query_stats(self.h, _p(sc), _p(ex), _p(vi)))
        return sc, ex, vi

    def download(self):
        planes = np.zeros((self.C, self.H, self.W))
        A = self.nx * self.ny
        idx = np.zeros(A, np.int32)
        dist = np.zeros(A)
        N.check(N.lib.psg_level_download(self.h, _p(planes), _p(idx), _p(dist)))
        return planes, idx, dist


# ---- multi-GPU row bands (shard.cpp: NCCL inside the library) ---------------------
def _nccl_first():
    """The library dlopens libnccl.so.2 on first use; when torch is importable,
    let torch load ITS NCCL first (one libnccl.so.2 per process: the library
    then reuses it instead of pulling in an older system copy)."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def comm_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 makes it, the caller distributes it)."""
    _nccl_first()
    buf = ct.create_string_buffer(128)
    N.check(N.lib.psg_comm_unique_id(buf))
    return buf.raw


class Communicator:
    """One rank of a row-band job (psg_comm_create); `ctx` is this GPU's context."""

    def __init__(self, ctx: Context, unique_id: bytes, world: int, rank: int):
        if len(unique_id) != 128:
            raise ShapeError(N.PSG_E_SHAPE, "an NCCL unique id is 128 bytes")
        self.ctx, self.world, self.rank = ctx, world, rank
        _nccl_first()
        h = ct.c_void_p()
        N.check(N.lib.psg_comm_create(ctx.h, ct.create_string_buffer(unique_id, 128), world, rank,
                                      ct.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            N.lib.psg_comm_destroy(self.h)
            self.h = None


def shard_plan(W: int, H: int, w: int, spacing: int, rank: int, world: int) -> dict:
    b = N.psg_band()
    N.check(N.lib.psg_shard_plan(W, H, w, spacing, rank, world, ct.byref(b)))
    return {f: getattr(b, f) for f, _ in N.psg_band._fields_}


class Band:
    """This rank's row band of a Level (psg_band_create), iterated over NCCL
    by the library (psg_band_iterate)."""

    def __init__(self, init_full: np.ndarray, index: SearchIndex, cfg: OptimizerConfig,
                 comm: Communicator, exemplar_hist: Optional[np.ndarray] = None):
        x = _c(init_full, np.float64)
        _check_level_inputs(x, index, cfg, exemplar_hist)
        C, H, W = x.shape
        self.plan = shard_plan(W, H, index.window, cfg.spacing, comm.rank, comm.world)
        p = self.plan
        rows = np.ascontiguousarray(x[:, p["p0"]:p["e1"], :])
        b = N.psg_band(*[p[f] for f, _ in N.psg_band._fields_])
        c = cfg.c()
        eh = _c(exemplar_hist, np.float64) if exemplar_hist is not None else None
        h = ct.c_void_p()
        N.check(N.lib.psg_band_create(index.ctx.h, index.h, _p(rows), ct.byref(b), ct.byref(c),
                                      _p(eh), ct.byref(h)))
        self.h, self.comm, self.index, self.C, self.W = h, comm, index, C, W

    def __del__(self):
        if getattr(self, "h", None):
            N.lib.psg_level_destroy(self.h)
            self.h = None

    def prime(self):
        N.check(N.lib.psg_level_prime(self.h))

    def iterate(self, n: int, honor_convergence: bool = False):
        stats = (N.psg_iter_stats * max(n, 1))()
        done = ct.c_int()
        N.check(N.lib.psg_band_iterate(self.h, self.comm.h, n, int(honor_convergence),
                                       ct.cast(stats, ct.c_void_p), ct.byref(done)))
        return [IterationStats.of(stats[i]) for i in range(done.value)]


def optimize_level_sharded(init_full: np.ndarray, index: SearchIndex, cfg: OptimizerConfig,
                           comm: Communicator, exemplar_hist: Optional[np.ndarray] = None):
    """(owned rows [C][p1-p0][W], plan, [IterationStats]) of this rank's band."""
    x = _c(init_full, np.float64)
    _check_level_inputs(x, index, cfg, exemplar_hist)
    C, H, W = x.shape
    p = shard_plan(W, H, index.window, cfg.spacing, comm.rank, comm.world)
    rows = np.ascontiguousarray(x[:, p["p0"]:p["e1"], :])
    out = np.zeros((C, p["p1"] - p["p0"], W))
    c = cfg.c()
    stats = (N.psg_iter_stats * max(cfg.max_iterations, 1))()
    n = ct.c_int()
    eh = _c(exemplar_hist, np.float64) if exemplar_hist is not None else None
    N.check(N.lib.psg_optimize_level_sharded(index.ctx.h, comm.h, index.h, _p(rows), W, H,
                                             ct.byref(c), _p(eh), _p(out),
                                             ct.cast(stats, ct.c_void_p), ct.byref(n)))
    return out, p, [IterationStats.of(stats[i]) for i in range(n.value)]


def optimize_level_loopback(init: np.ndarray, index: SearchIndex, cfg: OptimizerConfig,
                            world: int, exemplar_hist: Optional[np.ndarray] = None):
    """The row-band schedule for `world` bands in this process (exchanges as
    device copies): (image, [IterationStats]); bit-identical to optimize_level."""
    x = _c(init, np.float64)
    _check_level_inputs(x, index, cfg, exemplar_hist)
    C, H, W = x.shape
    out = np.zeros_like(x)
    c = cfg.c()
    stats = (N.psg_iter_stats * max(cfg.max_iterations, 1))()
    n = ct.c_int()
    eh = _c(exemplar_hist, np.float64) if exemplar_hist is not None else None
    N.check(N.lib.psg_optimize_level_loopback(index.ctx.h, index.h, _p(x), W, H, ct.byref(c),
                                              _p(eh), world, _p(out),
                                              ct.cast(stats, ct.c_void_p), ct.byref(n)))
    return out, [IterationStats.of(stats[i]) for i in range(n.value)]


def synthesize(exemplar: np.ndarray, out_w: int, out_h: int, levels: int, sizes, cfg: OptimizerConfig,
               variance_target=0.95, d_cap=0, d_fixed=0, branching=4, max_depth=0, seed=0,
               out_guidance: Optional[np.ndarray] = None, stage_pca=None,
               tree_kind: int = TREE_DEVICE, index_kind: int = 0,
               ctx: Optional[Context] = None):
    """Coarse-to-fine driver (pipeline.cpp:216-315) over stages (level x size).
    stage_pca: optional list over stages (level-major, then sizes) of
    (mean, basis) or None -- injected PCA models (fit on the device otherwise)."""
    ctx = ctx or default_context()
    ex = _c(exemplar, np.float64)
    C, eh, ew = ex.shape
    req = N.psg_request()
    req.exemplar = ex.ctypes.data_as(ct.POINTER(ct.c_double))
    req.C, req.ew, req.eh = C, ew, eh
    og = None
    if out_guidance is not None:
        og = _c(out_guidance, np.float64)
        req.out_guidance = og.ctypes.data_as(ct.POINTER(ct.c_double))
        req.guidance_kind = 1
    req.out_w, req.out_h, req.levels = out_w, out_h, levels
    sizes = list(sizes)
    req.stages.n_sizes = len(sizes)
    for i, s in enumerate(sizes):
        req.stages.sizes[i] = s
    req.cfg = cfg.c()
    req.index = index_cfg(variance_target, d_cap, d_fixed, branching, max_depth, 0, seed,
                          tree_kind=tree_kind)
    req.seed = seed
    keep = []
    if stage_pca is not None:
        ns = levels * len(sizes)
        if len(stage_pca) != ns:
            raise ShapeError(N.PSG_E_SHAPE, "stage_pca needs one entry per (level, size)")
        means = (ct.c_void_p * ns)()
        bases = (ct.c_void_p * ns)()
        ds = (ct.c_int * ns)()
        for s, mb in enumerate(stage_pca):
            if mb is None:
                continue
            m, b = _c(mb[0], np.float64), _c(mb[1], np.float64)
            keep += [m, b]
            means[s], bases[s], ds[s] = m.ctypes.data, b.ctypes.data, b.shape[0]
        keep += [means, bases, ds]
        req.stage_mean = ct.cast(means, ct.POINTER(ct.c_void_p))
        req.stage_basis = ct.cast(bases, ct.POINTER(ct.c_void_p))
        req.stage_d = ct.cast(ds, ct.POINTER(ct.c_int))
    req.index_kind = int(index_kind)
    cap = levels * len(sizes) * max(cfg.max_iterations, 1)
    trace = (N.psg_iter_stats * cap)()
    req.trace = ct.cast(trace, ct.c_void_p)
    req.trace_cap = cap
    out = np.zeros((C, out_h, out_w))
    rep = N.psg_report()
    N.check(N.lib.psg_synthesize(ctx.h, ct.byref(req), _p(out), ct.byref(rep)))
    stages = [rep.stages[i] for i in range(rep.n_stages)]
    report = {
        "part1_millis": rep.part1_millis, "part2_millis": rep.part2_millis,
        "total_nn_calls": rep.total_nn_calls, "final_energy": rep.final_energy,
        "stages": [dict(level=s.level, w=s.w, W=s.W, H=s.H, ew=s.ew, eh=s.eh, d=s.d,
                        iterations=s.iterations, final_energy=s.final_energy,
                        nn_calls=s.nn_calls, index_millis=s.index_millis,
                        optimize_millis=s.optimize_millis,
                        trace=[IterationStats.of(trace[i]) for i in
                               range(s.trace_first, min(cap, s.trace_first + s.trace_count))])
                   for s in stages],
        "index": "brute-force" if index_kind == INDEX_BRUTE_FORCE else "pca-tree",
    }
    return out, report


INDEX_PCA_TREE, INDEX_BRUTE_FORCE = 0, 1  # psg_index_kind (IndexKind, pipeline.hpp)


# ---- compare_modes / the bench table (pipeline.cpp:317-357, persyn_main.cpp:196-272) ----
@dataclass
class ModeSpec:
    """pipeline.hpp ModeSpec: name, patch width, index kind, budget."""
    name: str
    patch_width: int = 2
    index: int = INDEX_PCA_TREE
    budget: QueryBudget = field(default_factory=lambda: QueryBudget.backtrack(4))


@dataclass
class ModeRun:
    name: str
    wall_millis: float
    part2_millis: float
    nn_calls: int
    final_energy: float


# the modes of `persyn bench` (persyn_main.cpp:205-212)
BENCH_MODES = (ModeSpec("pixel-brute", 1, INDEX_BRUTE_FORCE, QueryBudget.exact()),
               ModeSpec("pixel-tree", 1, INDEX_PCA_TREE, QueryBudget.backtrack(4)),
               ModeSpec("patch-tree", 2, INDEX_PCA_TREE, QueryBudget.backtrack(4)))


def compare_modes(exemplar: np.ndarray, out_w: int, out_h: int, levels: int, sizes,
                  cfg: OptimizerConfig, modes, *, seed: int = 0, variance_target: float = 0.95,
                  branching: int = 4, d_cap: int = 0, ctx: Optional[Context] = None):
    """compare_modes (pipeline.cpp:317-334): the same request under each mode
    (patch width, index kind, budget) with identical seeds.  Tree budgets run
    on the reference's own KmTree construction (tree_kind=TREE_REFERENCE)."""
    if not modes:
        raise DomainError(N.PSG_E_DOMAIN, "no modes to compare")
    runs = []
    import time as _time
    for m in modes:
        c = OptimizerConfig(**{**cfg.__dict__, "patch_width": m.patch_width, "budget": m.budget})
        t0 = _time.perf_counter()
        _, rep = synthesize(exemplar, out_w, out_h, levels, sizes, c,
                            variance_target=variance_target, d_cap=d_cap, branching=branching,
                            max_depth=0, seed=seed, tree_kind=TREE_REFERENCE, index_kind=m.index,
                            ctx=ctx)
        wall = (_time.perf_counter() - t0) * 1e3
        # ModeRun{name, part1 + part2, part2, total_nn_calls, final_energy}
        # (pipeline.cpp:327-331); `wall` (host time of the call) is returned too
        runs.append(ModeRun(m.name, rep["part1_millis"] + rep["part2_millis"],
                            rep["part2_millis"], int(rep["total_nn_calls"]),
                            float(rep["final_energy"])))
        runs[-1].host_millis = wall
    return runs


def synthesis_report_json(rep: dict, config: dict) -> str:
    """SynthesisReport::to_json (pipeline.cpp:182-208): {config, part1_millis,
    part2_millis, total_nn_calls, final_energy, levels: [{width, height, index,
    iterations: [{iter, energy, changed, nn_calls, millis}]}]} -- one entry per
    stage (a level x neighbourhood size), nlohmann dump(2) formatting.
    `config` is the request echo (config_json, pipeline.cpp:58-88)."""
    import json as _json
    stages = rep["stages"]
    final = stages[-1]["trace"][-1].energy if stages and stages[-1]["trace"] else 0.0
    j = {"config": config, "part1_millis": float(rep["part1_millis"]),
         "part2_millis": float(rep["part2_millis"]), "total_nn_calls": int(rep["total_nn_calls"]),
         "final_energy": float(final), "levels": []}
    for s in stages:
        j["levels"].append({"width": int(s["W"]), "height": int(s["H"]),
                            "index": rep.get("index_describe", rep.get("index", "pca-tree")),
                            "iterations": [{"iter": int(t.iteration), "energy": float(t.energy),
                                            "changed": int(t.changed),
                                            "nn_calls": int(t.nn_calls),
                                            "millis": float(t.millis)} for t in s["trace"]]})
    return _json.dumps(j, indent=2)


class FormatError(PersynError):
    """errors.hpp FormatError (a malformed file)."""


def save_scale_map(path, values: np.ndarray, slant_deg: float, tilt_deg: float, s_min: float,
                   s_max: float) -> None:
    """save_scale_map (scale_map.cpp:125-145): "PSM1\\n", a compact JSON header
    {width, height, sigma, tau, smin, smax}, "\\n", then width*height
    little-endian float32 values, row-major, bottom row first."""
    import json as _json
    v = np.ascontiguousarray(values, dtype="<f4")
    H, W = v.shape
    head = _json.dumps({"width": W, "height": H, "sigma": float(slant_deg),
                        "tau": float(tilt_deg), "smin": float(s_min), "smax": float(s_max)},
                       separators=(",", ":"))
    with open(path, "wb") as f:
        f.write(b"PSM1\n" + head.encode() + b"\n" + v.tobytes())


def load_scale_map(path):
    """load_scale_map (scale_map.cpp:147-201): (values (H, W) float32,
    (slant, tilt, smin, smax)); FormatError on any malformed container."""
    import json as _json
    data = open(path, "rb").read()
    nl = data.find(b"\n")
    if nl < 0 or data[:nl] != b"PSM1":
        raise FormatError(N.PSG_E_FORMAT, f"{path}: missing PSM1 magic line")
    nl2 = data.find(b"\n", nl + 1)
    if nl2 < 0:
        raise FormatError(N.PSG_E_FORMAT, f"{path}: missing PSM1 header line")
    try:
        h = _json.loads(data[nl + 1:nl2])
        W, H = int(h["width"]), int(h["height"])
        view = (float(h["sigma"]), float(h["tau"]), float(h["smin"]), float(h["smax"]))
    except (ValueError, KeyError, TypeError) as e:
        raise FormatError(N.PSG_E_FORMAT, f"{path}: bad PSM1 header: {e}")
    if W < 1 or H < 1:
        raise FormatError(N.PSG_E_FORMAT, f"{path}: PSM1 header has empty dimensions")
    payload = data[nl2 + 1:]
    if len(payload) < 4 * W * H:
        raise FormatError(N.PSG_E_FORMAT, f"{path}: truncated PSM1 payload")
    if len(payload) > 4 * W * H:
        raise FormatError(N.PSG_E_FORMAT, f"{path}: trailing bytes after PSM1 payload")
    v = np.frombuffer(payload, dtype="<f4").reshape(H, W).copy()
    if not np.all((v >= view[2] - 1e-9) & (v <= view[3] + 1e-9)):
        raise FormatError(N.PSG_E_FORMAT, f"{path}: scale value outside the header bounds")
    return v, view


def _cpp_to_string(v: float) -> str:
    """std::to_string(double): printf("%f")."""
    return "%f" % v


def modes_to_json(runs) -> str:
    """modes_to_json (pipeline.cpp:336-346): nlohmann ordered_json dump(2)."""
    import json as _json
    return _json.dumps([{"mode": r.name, "wall_millis": r.wall_millis,
                         "part2_millis": r.part2_millis, "nn_calls": int(r.nn_calls),
                         "final_energy": r.final_energy} for r in runs], indent=2)


def modes_to_csv(runs) -> str:
    """modes_to_csv (pipeline.cpp:348-357)."""
    out = "mode,wall_millis,part2_millis,nn_calls,final_energy\n"
    for r in runs:
        out += (f"{r.name},{_cpp_to_string(r.wall_millis)},{_cpp_to_string(r.part2_millis)},"
                f"{int(r.nn_calls)},{_cpp_to_string(r.final_energy)}\n")
    return out


def bench_table(exemplar: np.ndarray, sizes_wh, levels: int, nbhd_sizes, iterations: int,
                reps: int, seed: int = 0, modes=BENCH_MODES, ctx: Optional[Context] = None):
    """`persyn bench` (persyn_main.cpp:196-272): per output size and mode,
    mean / stddev of part-2 milliseconds and mean nn_calls over `reps` seeds;
    returns (json, csv) in the reference's formats."""
    import json as _json
    import math as _math
    if reps < 1:
        raise DomainError(N.PSG_E_DOMAIN, "bench needs at least 1 repetition")
    if not sizes_wh:
        raise DomainError(N.PSG_E_DOMAIN, "no benchmark sizes given")
    cfg = OptimizerConfig(max_iterations=iterations, convergence_fraction=1e-6)
    cells = []
    for (w, h) in sizes_wh:
        for m in modes:
            part2, calls = [], []
            for rep in range(reps):
                r = compare_modes(exemplar, w, h, levels, nbhd_sizes, cfg, [m], seed=seed + rep,
                                  ctx=ctx)[0]
                part2.append(r.part2_millis)
                calls.append(float(r.nn_calls))
            mean = sum(part2) / len(part2)
            var = sum((v - mean) ** 2 for v in part2)
            sd = _math.sqrt(var / (len(part2) - 1)) if len(part2) > 1 else 0.0
            cells.append((f"{w}x{h}", m.name, mean, sd, sum(calls) / len(calls)))
    js = _json.dumps([{"size": c[0], "mode": c[1], "reps": reps, "mean_ms": c[2],
                       "stddev_ms": c[3], "mean_nn_calls": c[4]} for c in cells], indent=2) + "\n"
    csv = "size,mode,reps,mean_ms,stddev_ms,mean_nn_calls\n"
    for c in cells:
        csv += (f"{c[0]},{c[1]},{reps},{_cpp_to_string(c[2])},{_cpp_to_string(c[3])},"
                f"{_cpp_to_string(c[4])}\n")
    return js, csv


def initialize_output(exemplar: np.ndarray, out_scale: np.ndarray, s_min: float, s_max: float,
                      seed: int) -> np.ndarray:
    """initialize_output (pipeline.cpp:96-175): exemplar (C >= 4, plane 3 = S),
    out_scale = the output ScaleMap's raw float values (oh, ow) with bounds
    [s_min, s_max]; returns RGB + normalised S, (4, oh, ow)."""
    ex = _c(exemplar, np.float64)
    C, eh, ew = ex.shape
    sc = _c(out_scale, np.float32)
    oh, ow = sc.shape
    out = np.zeros((4, oh, ow))
    N.check(N.lib.psg_initialize_output(_p(ex), C, ew, eh, _p(sc), ow, oh, float(s_min),
                                        float(s_max), int(seed), _p(out)))
    return out


def debug_projection(planes: np.ndarray, index: SearchIndex, spacing: int):
    """(q_tc, delta, q_exact) at every anchor: the E-step's tensor-core
    projection, its error bound and the reference's fp64 chain."""
    x = _c(planes, np.float64)
    C, H, W = x.shape
    nx = N.lib.psg_axis_positions(W, index.window, spacing, None)
    ny = N.lib.psg_axis_positions(H, index.window, spacing, None)
    qt = np.zeros((nx * ny, index.retained_dim))
    qe = np.zeros_like(qt)
    dl = np.zeros(nx * ny, np.float32)
    N.check(N.lib.psg_debug_projection(index.ctx.h, index.h, _p(x), W, H, spacing, _p(qt),
                                       _p(dl), _p(qe)))
    return qt, dl, qe


def downsample(planes: np.ndarray, factor: int, ctx: Optional[Context] = None) -> np.ndarray:
    """Block-mean downsample of every plane (image.cpp:38-62), on the device."""
    ctx = ctx or default_context()
    x = _c(planes, np.float64)
    C, H, W = x.shape
    out = np.zeros((C, H // factor if factor > 0 else 0, W // factor if factor > 0 else 0))
    N.check(N.lib.psg_downsample(ctx.h, _p(x), C, W, H, factor, _p(out)))
    return out


def upsample_bilinear(planes: np.ndarray, factor: int, ctx: Optional[Context] = None) -> np.ndarray:
    """Half-pixel bilinear upsample of every plane (image.cpp:64-109), on the device."""
    ctx = ctx or default_context()
    x = _c(planes, np.float64)
    C, H, W = x.shape
    out = np.zeros((C, H * max(factor, 0), W * max(factor, 0)))
    N.check(N.lib.psg_upsample_bilinear(ctx.h, _p(x), C, W, H, factor, _p(out)))
    return out


def fit_to(planes: np.ndarray, width: int, height: int, ctx: Optional[Context] = None) -> np.ndarray:
    """Crop / edge-replicate every plane to width x height (pipeline.cpp:39-52), on the device."""
    ctx = ctx or default_context()
    x = _c(planes, np.float64)
    C, H, W = x.shape
    out = np.zeros((C, max(height, 0), max(width, 0)))
    N.check(N.lib.psg_fit_to(ctx.h, _p(x), C, W, H, width, height, _p(out)))
    return out


# ---- host helpers -----------------------------------------------------------------
def axis_positions(extent: int, window: int, step: int) -> np.ndarray:
    n = N.lib.psg_axis_positions(extent, window, step, None)
    out = np.zeros(max(n, 1), np.int32)
    N.lib.psg_axis_positions(extent, window, step, _p(out))
    return out[:n]


def plan(W: int, H: int, w: int, spacing: int, patch_width: int):
    nx = N.lib.psg_axis_positions(W, w, spacing, None)
    ny = N.lib.psg_axis_positions(H, w, spacing, None)
    mult = np.zeros(max(nx * ny, 1), np.int32)
    calls = N.lib.psg_plan(W, H, w, spacing, patch_width, _p(mult))
    return int(calls), mult[: nx * ny]


def pow_cr(x: float, y: float) -> float:
    return N.lib.psg_pow_cr(x, y)


def hist_mass(count: int, pixels: int) -> float:
    return N.lib.psg_hist_mass(count, pixels)
