"""Row-sharded multi-GPU EM iterations.

The output is split into row bands (``psg_shard_plan``): rank g owns anchor
rows [a0, a1) and pixel rows [p0, p1).  One EM iteration is the library's
four phases with three exchanges in between (optimizer.cpp:453-497 order):

  phase1  IRLS weights, owned-row histogram counts
          -> all-reduce(sum) of the int64 counts (exact)
  phase2  penalties + effective weights; pack (eff, idx) of the anchor rows
          rank g+1 needs   -> send up / receive rank g-1's rows
  phase3  M-step of the owned pixel rows (halo anchors accumulated in
          ascending id: bit-identical to one device); pack the first rows of
          the updated fp32 mirror -> send down / receive rank g+1's rows
  phase4  lsq diagnostic + E-step of the owned anchors -> telemetry partials
          -> gathered and summed in rank order (deterministic)

The orchestration is written once against two small interfaces: a *band*
backend (the GPU library, or the CPU oracle in tests) and a *comm*
(torch.distributed — NCCL on GPUs, gloo on CPU — or an in-process loopback
that moves buffers between several bands of one process).  The loopback
never runs kernels that wait on one another: phases are host-synchronous.
"""
from __future__ import annotations

import ctypes as ct
from typing import List, Optional, Sequence

import numpy as np

PARTIALS = 9  # lsq_before, lsq_after, energy, changed, scanned, unique scanned,
#               nn_calls, priming nn_calls, unique queries


def shard_plan(W: int, H: int, w: int, spacing: int, rank: int, world: int) -> dict:
    """Band of `rank` (pure host logic of the library, psg_shard_plan)."""
    from . import native as N
    b = N.psg_band()
    N.check(N.lib.psg_shard_plan(W, H, w, spacing, rank, world, ct.byref(b)))
    return {f: getattr(b, f) for f, _ in N.psg_band._fields_}


def all_plans(W, H, w, spacing, world) -> List[dict]:
    return [shard_plan(W, H, w, spacing, r, world) for r in range(world)]


# ---------------------------------------------------------------------------
# communicators
class LoopbackComm:
    """All ranks' bands live in this process; exchanges are buffer moves."""

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))

    def allreduce_sum(self, xs: Sequence):
        cuda = getattr(xs[0], "is_cuda", False)
        if cuda:
            # the counts were written on the library's stream; the sum runs on
            # torch's: order both ways (the library reads the sum in phase 2)
            import torch
            torch.cuda.synchronize()
        tot = xs[0].clone() if hasattr(xs[0], "clone") else xs[0].copy()
        for x in xs[1:]:
            tot += x
        if cuda:
            torch.cuda.synchronize()
        return [tot for _ in xs]

    def shift_up(self, sends: Sequence):
        """rank r receives what rank r-1 sent (rank 0 receives None)."""
        return [None] + list(sends[:-1])

    def shift_down(self, sends: Sequence):
        """rank r receives what rank r+1 sent (the last rank receives None)."""
        return list(sends[1:]) + [None]

    def sum_partials(self, parts: Sequence[np.ndarray]) -> List[np.ndarray]:
        tot = np.zeros(PARTIALS)
        for p in parts:  # rank order
            tot = tot + p
        return [tot for _ in parts]


class DistComm:
    """One band per process over torch.distributed (NCCL: CUDA tensors; gloo: CPU).

    stream_ordered (NCCL): the library's context stream IS torch's current
    stream, so every collective / P2P op is ordered after the kernels that
    produced its buffer and before the kernels that consume it (torch makes
    the NCCL stream wait on the current stream and `wait()` makes the current
    stream wait on NCCL) -- no host synchronisation between phases.  Otherwise
    each exchange is bracketed by a device synchronisation."""

    def __init__(self, stream_ordered: bool = False):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.ranks = [self.rank]
        self.cuda = dist.get_backend() == "nccl"
        self.device = torch.device("cuda", torch.cuda.current_device()) if self.cuda else None
        self.stream_ordered = bool(stream_ordered) and self.cuda

    def _settle(self):
        # library kernels on a stream of their own: make every exchange
        # complete before the next phase reads or overwrites its buffers
        if self.cuda and not self.stream_ordered:
            import torch
            torch.cuda.synchronize()

    def allreduce_sum(self, xs):
        (x,) = xs
        self._settle()
        self.dist.all_reduce(x, op=self.dist.ReduceOp.SUM)
        self._settle()
        return [x]

    def _shift(self, send, dst, src, recv_like):
        import torch
        ops = []
        recv = None
        if send is not None and dst is not None:
            ops.append(self.dist.P2POp(self.dist.isend, send, dst))
        if recv_like is not None and src is not None:
            recv = torch.empty_like(recv_like)
            ops.append(self.dist.P2POp(self.dist.irecv, recv, src))
        self._settle()
        if ops:
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()
        self._settle()
        return recv

    def shift_up(self, sends, recv_likes):
        (s,) = sends
        (rl,) = recv_likes
        dst = self.rank + 1 if self.rank + 1 < self.world else None
        src = self.rank - 1 if self.rank > 0 else None
        return [self._shift(s if dst is not None else None, dst, src, rl)]

    def shift_down(self, sends, recv_likes):
        (s,) = sends
        (rl,) = recv_likes
        dst = self.rank - 1 if self.rank > 0 else None
        src = self.rank + 1 if self.rank + 1 < self.world else None
        return [self._shift(s if dst is not None else None, dst, src, rl)]

    def sum_partials(self, parts):
        import torch
        (p,) = parts
        t = torch.tensor(p, dtype=torch.float64, device=self.device)
        if self.cuda:  # one gather, one device->host copy
            flat = torch.empty(self.world * PARTIALS, dtype=torch.float64, device=self.device)
            self.dist.all_gather_into_tensor(flat, t)
            rows = flat.cpu().numpy().reshape(self.world, PARTIALS)
        else:
            out = [torch.zeros_like(t) for _ in range(self.world)]
            self.dist.all_gather(out, t)
            rows = [o.numpy() for o in out]
        tot = np.zeros(PARTIALS)
        for r in rows:  # rank order: the same sum on every rank
            tot = tot + r
        return [tot]


# ---------------------------------------------------------------------------
def em_iteration(bands: Sequence, comm) -> np.ndarray:
    """One EM iteration over the bands of this process; returns the global
    partials (identical on every rank)."""
    counts = [b.phase1() for b in bands]
    totals = comm.allreduce_sum(counts) if counts[0] is not None else counts
    sends = [b.phase2(t) for b, t in zip(bands, totals)]
    if isinstance(comm, LoopbackComm):
        recvs = comm.shift_up(sends)
    else:
        recvs = comm.shift_up(sends, [b.halo_anchor_like() for b in bands])
    rows = [b.phase3(r) for b, r in zip(bands, recvs)]
    if isinstance(comm, LoopbackComm):
        rrecv = comm.shift_down(rows)
    else:
        rrecv = comm.shift_down(rows, [b.halo_rows_like() for b in bands])
    parts = [b.phase4(r) for b, r in zip(bands, rrecv)]
    glob = comm.sum_partials(parts)
    for b, g in zip(bands, glob):
        b.commit(g)
    return glob[0]


def run_sharded(bands: Sequence, comm, iterations: int, min_iterations: int = 1,
                convergence_fraction: float = 1e-9, total_anchors: Optional[int] = None):
    """optimize_level's loop over row bands (convergence rule optimizer.cpp:509-513,
    decided on the global `changed`, so every rank stops together)."""
    for b in bands:
        b.prime()
    stats = []
    for it in range(1, iterations + 1):
        g = em_iteration(bands, comm)
        stats.append(g)
        A = total_anchors if total_anchors is not None else bands[0].total_anchors
        if it >= min_iterations and g[3] < convergence_fraction * A:
            break
    return stats


# ---------------------------------------------------------------------------
class GpuBand:
    """A band level of the sm_100a library; exchange payloads are CUDA tensors."""

    def __init__(self, index, init_full: np.ndarray, plan: dict, plans: List[dict], cfg,
                 ctx=None, exemplar_hist=None):
        import torch
        from . import native as N
        self.N = N
        self.torch = torch
        self.plan, self.plans = plan, plans
        self.index = index
        from .api import _check_level_inputs
        _check_level_inputs(np.asarray(init_full), index, cfg, exemplar_hist)
        self.C = init_full.shape[0]
        self.W, self.H = plan["W"], plan["H"]
        rows = np.ascontiguousarray(init_full[:, plan["p0"]:plan["e1"], :], dtype=np.float64)
        b = N.psg_band(*[plan[f] for f, _ in N.psg_band._fields_])
        c = cfg.c()
        eh = np.ascontiguousarray(exemplar_hist, np.float64) if exemplar_hist is not None else None
        h = ct.c_void_p()
        N.check(N.lib.psg_band_create(index.ctx.h, index.h, rows.ctypes.data_as(ct.c_void_p),
                                      ct.byref(b), ct.byref(c),
                                      eh.ctypes.data_as(ct.c_void_p) if eh is not None else None,
                                      ct.byref(h)))
        self.h = h
        self.hist = bool(cfg.histogram_matching)
        slots = self.C if cfg.histogram_include_scale else 3
        self.ncounts = cfg.histogram_bins * slots
        dev = torch.device("cuda", torch.cuda.current_device())
        self.counts = torch.zeros(self.ncounts, dtype=torch.int64, device=dev)
        r, w = plan["rank"], plan["world"]
        nx = plan["nx"]
        self.send_row0 = plans[r + 1]["hlo"] if r + 1 < w else plan["a1"]
        n_up = (plan["a1"] - self.send_row0) * nx
        self.send_ae = torch.zeros(n_up * 12, dtype=torch.uint8, device=dev)
        self.n_halo_ae = (plan["a0"] - plan["hlo"]) * nx
        self.n_send_rows = (plans[r - 1]["e1"] - plans[r - 1]["p1"]) if r > 0 else 0
        self.send_rows = torch.zeros(max(1, self.n_send_rows * self.W * self.C), dtype=torch.float32,
                                     device=dev)
        self.n_halo_rows = plan["e1"] - plan["p1"]
        self.total_anchors = plan["nx"] * plan["ny"]
        self.dev = dev
        # the buffers above were zero-filled on torch's stream; the library
        # writes them on its own
        torch.cuda.synchronize()

    def __del__(self):
        if getattr(self, "h", None):
            self.N.lib.psg_level_destroy(self.h)
            self.h = None

    def _p(self, t):
        return ct.c_void_p(t.data_ptr()) if t is not None else None

    def prime(self):
        self.N.check(self.N.lib.psg_level_prime(self.h))

    def phase1(self):
        self.N.check(self.N.lib.psg_band_phase1(self.h, self._p(self.counts) if self.hist else None))
        return self.counts if self.hist else None

    def phase2(self, total):
        self.N.check(self.N.lib.psg_band_phase2(self.h, self._p(total) if self.hist else None,
                                                self.send_row0, self._p(self.send_ae)))
        return self.send_ae if self.send_ae.numel() else None

    def halo_anchor_like(self):
        return self.torch.empty(self.n_halo_ae * 12, dtype=self.torch.uint8, device=self.dev) \
            if self.n_halo_ae else None

    def halo_rows_like(self):
        return self.torch.empty(self.n_halo_rows * self.W * self.C, dtype=self.torch.float32,
                                device=self.dev) if self.n_halo_rows else None

    def phase3(self, recv):
        self.N.check(self.N.lib.psg_band_phase3(self.h, self._p(recv), self.n_send_rows,
                                                self._p(self.send_rows)))
        return self.send_rows[: self.n_send_rows * self.W * self.C] if self.n_send_rows else None

    def phase4(self, recv_rows):
        parts = np.zeros(PARTIALS)
        self.N.check(self.N.lib.psg_band_phase4(self.h, self._p(recv_rows),
                                                parts.ctypes.data_as(ct.c_void_p)))
        return parts

    def commit(self, glob):
        g = np.ascontiguousarray(glob, np.float64)
        self.N.check(self.N.lib.psg_band_commit(self.h, g.ctypes.data_as(ct.c_void_p), None))

    def owned(self):
        """(planes of the owned rows [C][p1-p0][W], owned assignments, distances)."""
        p = self.plan
        Hl = p["e1"] - p["p0"]
        A = (p["a1"] - p["hlo"]) * p["nx"]
        planes = np.zeros((self.C, Hl, self.W))
        idx = np.zeros(A, np.int32)
        dist = np.zeros(A)
        self.N.check(self.N.lib.psg_level_download(self.h, planes.ctypes.data_as(ct.c_void_p),
                                                   idx.ctypes.data_as(ct.c_void_p),
                                                   dist.ctypes.data_as(ct.c_void_p)))
        off = (p["a0"] - p["hlo"]) * p["nx"]
        return planes[:, : p["p1"] - p["p0"]], idx[off:], dist[off:]


def gather_image(parts: Sequence[np.ndarray]) -> np.ndarray:
    """Concatenate owned row blocks in rank order."""
    return np.concatenate(list(parts), axis=1)
