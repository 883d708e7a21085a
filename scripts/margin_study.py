"""Feasibility study (not product code): how often could an exact E-step skip a
query because its window moved less than the margin between its previous best
and second-best distances?  Skip test (triangle inequality in PCA space):
    sqrt(d(q_k, p*_{k-1})) < sqrt(d2_{k-1}) - |q_k - q_{k-1}|
Prints, per EM iteration of the bench stage, the fraction of anchors passing.
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402


def windows(planes, w, step):
    t = torch.as_tensor(planes, device="cuda", dtype=torch.float64)[None]
    u = torch.nn.functional.unfold(t, w, stride=step)  # [1, C*w*w, L]
    return u[0].T.contiguous()


def main():
    cfg = wl.CONFIGS[3]
    w = 8
    ex, init, W, H, sp = wl.stage_inputs(cfg, 2, w)
    ctx = api.Context(0)
    ix = api.make_pca_tree_index(ex, w, d_fixed=32, branching=8, max_depth=4, seed=1,
                                 hist_bins=16, ctx=ctx)
    X = windows(ex, w, 1)
    mu = X.mean(0)
    cov = (X - mu).T @ (X - mu)
    evals, evecs = torch.linalg.eigh(cov)
    B = evecs[:, -32:]
    P = ((X - mu) @ B).float()
    pn = (P * P).sum(1)
    ocfg = api.OptimizerConfig(max_iterations=10 ** 6, min_iterations=10 ** 6 - 1,
                               convergence_fraction=1e-9, nbhd_width=w, spacing=sp,
                               patch_width=2, budget=api.QueryBudget.exact())
    lv = api.Level(init, ix, ocfg)
    lv.prime()
    prev = None
    for k in range(12):
        lv.iterate(1)
        img = lv.download()[0]
        Q = ((windows(img, w, sp) - mu) @ B).float()
        d1 = torch.empty(Q.shape[0], device="cuda")
        d2 = torch.empty_like(d1)
        i1 = torch.empty(Q.shape[0], dtype=torch.long, device="cuda")
        for s in range(0, Q.shape[0], 8192):
            q = Q[s:s + 8192]
            dd = (q * q).sum(1, keepdim=True) + pn[None] - 2 * q @ P.T
            v, i = torch.topk(dd, 2, dim=1, largest=False)
            d1[s:s + 8192], d2[s:s + 8192], i1[s:s + 8192] = v[:, 0], v[:, 1], i[:, 0]
        if prev is not None:
            Qp, d2p, i1p = prev
            dq = (Q - Qp).norm(dim=1)
            seed = ((Q - P[i1p]) ** 2).sum(1)
            ok = seed.clamp_min(0).sqrt() < d2p.clamp_min(0).sqrt() - dq
            print(json.dumps({"iter": k, "skip_frac": float(ok.float().mean()),
                              "same_nn_frac": float((i1 == i1p).float().mean()),
                              "median_dq": float(dq.median()),
                              "median_gap": float((d2p.sqrt() - d1.sqrt()).median())}), flush=True)
        prev = (Q, d2, i1)


if __name__ == "__main__":
    main()
