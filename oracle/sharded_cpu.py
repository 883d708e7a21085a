"""TEST INFRASTRUCTURE ONLY — CPU band backend for the row-sharded protocol.

Implements the same four phases as the library's psg_band_* functions with
the oracle's arithmetic (oracle/oracle.c primitives + ordered numpy), so the
production orchestrator (paper_2006_11851_b200/sharding.py) can be exercised
with torch.distributed/gloo on CPU (world_size 2, 3) and checked against the
unsharded oracle bit-for-bit.  Exchange payloads are torch CPU tensors in the
library's formats: (eff f64[n], idx i32[n]) as bytes, mirror rows f32 [r][W][C].
"""
from __future__ import annotations

import math

import numpy as np
import torch

from oracle.oracle import Port


def hist_mass_seq(count: int, P: int) -> float:
    inv = 1.0 / float(P)
    m = 0.0
    for _ in range(int(count)):
        m += inv
    return m


class CpuBand:
    def __init__(self, port: Port, cand, proj, mean, basis, init_full, plan, plans, w, sp, patch,
                 r=0.8, eps=1e-4, bins=16, ex_mass=None):
        self.port = port
        self.cand, self.proj, self.mean, self.basis = cand, proj, mean, basis
        self.plan, self.plans = plan, plans
        self.w, self.sp, self.r, self.eps, self.bins = w, sp, r, eps, bins
        self.ex_mass = ex_mass
        self.hist = ex_mass is not None
        self.C = init_full.shape[0]
        self.W, self.H = plan["W"], plan["H"]
        p0, p1, e1 = plan["p0"], plan["p1"], plan["e1"]
        self.Hu, self.Hl = p1 - p0, e1 - p0
        self.rows = np.array(init_full[:, p0:e1, :], dtype=np.float64, copy=True)
        xs = port.axis_positions(self.W, w, sp)
        ysg = port.axis_positions(self.H, w, sp)
        self.xs = xs
        self.ys_loc = ysg[plan["hlo"]:plan["a1"]] - p0
        self.nx = len(xs)
        self.nh = plan["a0"] - plan["hlo"]
        self.A = self.nx * len(self.ys_loc)
        self.off = self.nh * self.nx
        calls, mult = port.plan(self.W, self.H, w, sp, patch)
        self.mult = mult.reshape(len(ysg), self.nx)[plan["a0"]:plan["a1"]].reshape(-1)
        self.nn_calls = int(self.mult.sum())
        self.idx = np.zeros(self.A, np.int32)
        self.dist = np.zeros(self.A)
        self.eff = np.zeros(self.A)
        self.irls = np.zeros(self.A)
        self.total_anchors = self.nx * plan["ny"]
        rk, wd = plan["rank"], plan["world"]
        self.send_row0 = plans[rk + 1]["hlo"] if rk + 1 < wd else plan["a1"]
        self.n_send_rows = (plans[rk - 1]["e1"] - plans[rk - 1]["p1"]) if rk > 0 else 0
        self.n_halo_rows = e1 - p1
        self.pending_calls = 0
        self.lsq_before = 0.0

    # -- helpers ----------------------------------------------------------------
    def _anchor(self, a):
        return int(self.xs[a % self.nx]), int(self.ys_loc[a // self.nx])

    def _search_owned(self):
        idx = np.zeros(self.A - self.off, np.int32)
        dist = np.zeros(self.A - self.off)
        for k, a in enumerate(range(self.off, self.A)):
            ax, ay = self._anchor(a)
            v = self.port.extract_window(self.rows, ax, ay, self.w)
            q = self.port.project(v, self.mean, self.basis)
            j, _ = self.port.nearest_lexmin(self.proj, q)
            idx[k] = j
            dist[k] = self.port.full_distance(v, self.cand[j])
        return idx, dist

    # -- phases (same contract as psg_band_phase*) ---------------------------------
    def prime(self):
        i, d = self._search_owned()
        self.idx[self.off:], self.dist[self.off:] = i, d
        self.pending_calls = self.nn_calls

    def phase1(self):
        o = slice(self.off, self.A)
        self.irls[o] = [self.port.irls_weight(d, self.r, self.eps) for d in self.dist[o]]
        self.eff[o] = self.irls[o]
        if not self.hist:
            return None
        own = self.rows[:3, : self.Hu, :]
        b = np.clip(np.floor(own * self.bins).astype(np.int64), 0, self.bins - 1)
        counts = np.stack([np.bincount(b[s].ravel(), minlength=self.bins) for s in range(3)])
        return torch.tensor(counts.ravel(), dtype=torch.int64)

    def phase2(self, total):
        o = slice(self.off, self.A)
        pen = np.zeros(self.A)
        if self.hist:
            tot = total.numpy().reshape(3, self.bins)
            P = self.W * self.H
            out_mass = np.array([[hist_mass_seq(c, P) for c in row] for row in tot])
            for a in range(self.off, self.A):
                pen[a] = self.port.histogram_penalty(self.cand[self.idx[a]], self.C, 3, self.bins,
                                                     out_mass, self.ex_mass)
            self.eff[o] = self.irls[o] / (1.0 + pen[o])
        lb = 0.0
        for a in range(self.off, self.A):  # optimizer.cpp:470-474 order within the band
            lb += self.eff[a] * self.dist[a] * self.dist[a]
        self.lsq_before = lb
        if self.send_row0 >= self.plan["a1"]:
            return None
        first = (self.send_row0 - self.plan["hlo"]) * self.nx
        eff = self.eff[first:].astype(np.float64).tobytes()
        idx = self.idx[first:].astype(np.int32).tobytes()
        return torch.frombuffer(bytearray(eff + idx), dtype=torch.uint8)

    def halo_anchor_like(self):
        return torch.empty(self.off * 12, dtype=torch.uint8) if self.off else None

    def halo_rows_like(self):
        return torch.empty(self.n_halo_rows * self.W * self.C, dtype=torch.float32) \
            if self.n_halo_rows else None

    def phase3(self, recv):
        if self.off:
            raw = recv.numpy().tobytes()
            n = self.off
            self.eff[:n] = np.frombuffer(raw[: 8 * n], np.float64)
            self.idx[:n] = np.frombuffer(raw[8 * n:], np.int32)
        # M-step of the owned rows, anchors in ascending (global) id (optimizer.cpp:365-399)
        acc = np.zeros((self.C, self.Hu, self.W))
        wsum = np.zeros((self.Hu, self.W))
        w, C = self.w, self.C
        for a in range(self.A):
            ax, ay = self._anchor(a)
            we = self.eff[a]
            if not (we > 0.0) or not math.isfinite(we):
                raise ValueError("non-positive or non-finite update weight")
            z = self.cand[self.idx[a]].reshape(w, w, C)
            for dy in range(w):
                y = ay + dy
                if 0 <= y < self.Hu:
                    for c in range(C):
                        acc[c, y, ax:ax + w] = acc[c, y, ax:ax + w] + we * z[dy, :, c].astype(np.float64)
                    wsum[y, ax:ax + w] = wsum[y, ax:ax + w] + we
        inv = 1.0 / wsum
        self.rows[:, : self.Hu, :] = np.clip(acc * inv[None], 0.0, 1.0)
        if not self.n_send_rows:
            return None
        mir = self.rows[:, : self.n_send_rows, :].astype(np.float32).transpose(1, 2, 0).copy()
        return torch.from_numpy(mir.reshape(-1))

    def phase4(self, recv_rows):
        if self.n_halo_rows:
            m = recv_rows.numpy().reshape(self.n_halo_rows, self.W, self.C)
            self.rows[:, self.Hu:, :] = m.transpose(2, 0, 1).astype(np.float64)
        la = 0.0
        for a in range(self.off, self.A):
            ax, ay = self._anchor(a)
            v = self.port.extract_window(self.rows, ax, ay, self.w)
            d = self.port.full_distance(v, self.cand[self.idx[a]])
            la += self.eff[a] * d * d
        ni, nd = self._search_owned()
        oi = self.idx[self.off:]
        changed = int(np.sum(ni != oi))
        energy = 0.0
        for d in nd:
            energy += math.pow(d, self.r)
        self._next = (ni, nd)
        return np.array([self.lsq_before, la, energy, changed, 0.0, 0.0, self.nn_calls,
                         self.pending_calls, 0.0])

    def commit(self, glob):
        ni, nd = self._next
        self.idx[self.off:], self.dist[self.off:] = ni, nd
        self.pending_calls = 0

    def owned(self):
        return self.rows[:, : self.Hu, :].copy(), self.idx[self.off:].copy(), self.dist[self.off:].copy()
