"""Study: how often does a database-side kNN certificate settle a seeded query?

For every database point s keep its K nearest other database points (PCA
space) and the distance r_K(s) to the (K+1)-th.  A query q seeded with s at
distance delta = |q - s|: every point p outside the list has
|q - p| >= |s - p| - delta >= r_K(s) - delta, so when 2 delta < r_K(s) the
exact winner is s or a list point with |s - p| <= 2 delta.

On the bench stage (cfg3 finest, C = 5) run the library's EM loop one
iteration at a time and report, per iteration, the fraction of anchors the
certificate settles for several K and the mean number of list points that
would need an exact evaluation.  Study only: nothing here is product code.
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402


def main(iters=6):
    cfg = wl.CONFIGS[3]
    G, w, sp = 2, 8, 2
    rgb = wl.sinusoid_exemplar(cfg.ex_size, cfg.n_sin, cfg.ramp, cfg.seed)
    ex = wl.rgbs_planes(rgb, G)
    init = wl.init_output(ex, cfg.out, cfg.out, G, cfg.seed)
    ctx = api.Context(0)
    ix = api.make_pca_tree_index(ex, w, d_fixed=32, branching=8, max_depth=4, seed=1,
                                 hist_bins=16, ctx=ctx)
    mean, basis, _ = ix.pca()
    P = torch.tensor(ix.projected(), device="cuda")
    pn = (P * P).sum(1)
    N = P.shape[0]
    Ks = [8, 16, 32, 64, 128]
    KM = max(Ks) + 1
    nd, ni = [], []
    for s in range(0, N, 2048):
        pp = P[s:s + 2048]
        d2 = ((pp * pp).sum(1, keepdim=True) + pn[None] - 2.0 * pp @ P.T).clamp_min(0)
        d2[torch.arange(pp.shape[0], device="cuda"), torch.arange(s, s + pp.shape[0], device="cuda")] = float("inf")
        v, i = torch.topk(d2, KM, largest=False)
        nd.append(v.sqrt())
        ni.append(i)
    nd = torch.cat(nd)  # (N, KM) ascending neighbour distances
    qs = torch.tensor([0.1, 0.5, 0.9], device="cuda", dtype=torch.float64)
    for K in Ks:
        print(f"r_{K} p10/50/90 {torch.quantile(nd[:, K], qs).cpu().numpy()}")

    ocfg = api.OptimizerConfig(max_iterations=10 ** 6, min_iterations=10 ** 6 - 1,
                               convergence_fraction=1e-9, histogram_bins=16,
                               histogram_matching=True, nbhd_width=w, spacing=sp, patch_width=2,
                               budget=api.QueryBudget.exact())
    L = api.Level(init, ix, ocfg)
    L.prime()
    xs = torch.tensor(api.axis_positions(cfg.out, w, sp), device="cuda")
    ys = xs.clone()
    dy, dx = torch.meshgrid(torch.arange(w, device="cuda"), torch.arange(w, device="cuda"),
                            indexing="ij")
    mean_t = torch.tensor(mean, device="cuda")
    basis_t = torch.tensor(basis, device="cuda")

    def queries(planes):
        m = torch.tensor(planes, device="cuda").float()
        Y = ys[:, None, None, None] + dy[None, None]
        X = xs[None, :, None, None] + dx[None, None]
        win = m[:, Y, X].permute(1, 2, 3, 4, 0).reshape(len(ys) * len(xs), -1)
        return (win.double() - mean_t) @ basis_t.T

    _, idx_prev, _ = L.download()
    for t in range(1, iters + 1):
        L.iterate(1)
        planes, idx, _ = L.download()
        # the search of iteration t ran on these planes, seeded with idx_prev
        q = queries(planes)
        seed = torch.tensor(idx_prev, device="cuda").long()
        delta = (q - P[seed]).norm(dim=1)
        line = f"it {t}: delta p10/50/90 {torch.quantile(delta, qs).cpu().numpy()}"
        for K in Ks:
            rk = nd[seed, K]
            cert = 2.0 * delta * (1 + 1e-9) + 1e-9 < rk
            nlist = (nd[seed, :K] <= (2.0 * delta)[:, None]).sum(1).float()
            line += (f" | K={K}: cert {cert.float().mean().item():.3f}"
                     f" evals {nlist[cert].mean().item() if cert.any() else 0:.1f}")
        print(line, flush=True)
        idx_prev = idx


if __name__ == "__main__":
    main()
