"""Study: how many E-step searches could a provable "winner unchanged" test skip?

On the bench stage (cfg3 finest, C=5), run the library's EM loop one iteration
at a time; after each, project every anchor's window in fp64 (torch) and find
its exact two nearest database points in PCA space.  Report the movement
delta = |q_t - q_ref| against the gap sqrt(d2) - sqrt(d1), and the fraction of
anchors for which d(q_t, p*) < sqrt(sec_ref) - delta (a skip is provable).
Also simulates Verlet-style candidate lists: at a (re)build the list holds every
point within d1 + 2m of q_ref; while |q - q_ref| <= m the nearest point of q is
provably in the list.  Reports rebuild fractions and list sizes per margin m.
Study only: nothing here is product code.
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402


def main(iters=10, hist=True):
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
    mean_t = torch.tensor(mean, device="cuda")
    basis_t = torch.tensor(basis, device="cuda")
    ocfg = api.OptimizerConfig(max_iterations=10 ** 6, min_iterations=10 ** 6 - 1,
                               convergence_fraction=1e-9, histogram_bins=16,
                               histogram_matching=hist, nbhd_width=w, spacing=sp, patch_width=2,
                               budget=api.QueryBudget.exact())
    L = api.Level(init, ix, ocfg)
    L.prime()
    xs = torch.tensor(api.axis_positions(cfg.out, w, sp), device="cuda")
    ys = xs.clone()
    dy, dx = torch.meshgrid(torch.arange(w, device="cuda"), torch.arange(w, device="cuda"),
                            indexing="ij")

    def queries(planes):
        m = torch.tensor(planes, device="cuda").float()  # (C, H, W) fp32 features
        Y = ys[:, None, None, None] + dy[None, None]      # (ny, 1, w, w)
        X = xs[None, :, None, None] + dx[None, None]      # (1, nx, w, w)
        win = m[:, Y, X]                                  # (C, ny, nx, w, w)
        win = win.permute(1, 2, 3, 4, 0).reshape(len(ys) * len(xs), -1)
        return (win.double() - mean_t) @ basis_t.T

    Pf = P.float()
    pnf = pn.float()
    margins = [0.02, 0.05, 0.1, 0.2]

    def top2(q, refd1=None):
        out_d, out_i, cnt = [], [], []
        for s in range(0, q.shape[0], 4096):
            qq = q[s:s + 4096]
            d2 = (qq * qq).sum(1, keepdim=True) + pn[None] - 2.0 * qq @ P.T
            v, i = torch.topk(d2, 2, largest=False)
            out_d.append(v.clamp_min(0))
            out_i.append(i)
            # list sizes: points within (d1 + 2m)
            qf = qq.float()
            d2f = ((qf * qf).sum(1, keepdim=True) + pnf[None] - 2.0 * qf @ Pf.T).clamp_min(0)
            r1 = v[:, 0].clamp_min(0).sqrt().float()
            cnt.append(torch.stack([(d2f <= ((r1 + 2 * m) ** 2)[:, None]).sum(1)
                                    for m in margins], 1))
        return torch.cat(out_d), torch.cat(out_i), torch.cat(cnt)

    ref_q = ref_sec = ref_id = None
    prev_q = None
    vq = [None] * len(margins)  # Verlet reference queries per margin
    vcnt = [None] * len(margins)
    for t in range(iters + 1):
        if t > 0:
            L.iterate(1)
        planes, idx, _ = L.download()
        q = queries(planes)
        d, i, cnt = top2(q)
        vl = []
        for k, m in enumerate(margins):
            if vq[k] is None:
                vq[k], vcnt[k] = q.clone(), cnt[:, k].clone()
                vl.append("init")
                continue
            rebuild = (q - vq[k]).norm(dim=1) > m
            vq[k] = torch.where(rebuild[:, None], q, vq[k])
            vcnt[k] = torch.where(rebuild, cnt[:, k], vcnt[k])
            vl.append(f"m={m}: rebuild {rebuild.float().mean().item():.3f} "
                      f"list mean {vcnt[k].float().mean().item():.1f} "
                      f"p90 {torch.quantile(vcnt[k][:200000].float(), 0.9).item():.0f}")
        lib_idx = torch.tensor(idx, device="cuda")
        agree = (lib_idx == i[:, 0]).float().mean().item()
        line = f"it {t}: top1 agrees with library {agree:.5f}"
        if ref_q is not None:
            delta = (q - ref_q).norm(dim=1)
            dp = (q - P[ref_id]).norm(dim=1)
            skip = dp < ref_sec.sqrt() - delta
            ok = (i[:, 0][skip] == ref_id[skip]).float().mean().item() if skip.any() else 1.0
            gap = d[:, 1].sqrt() - d[:, 0].sqrt()
            dlt = (q - prev_q).norm(dim=1)
            qs = torch.tensor([0.1, 0.5, 0.9], device="cuda", dtype=torch.float64)
            line += (f" | skip {skip.float().mean().item():.3f} (sound {ok:.4f})"
                     f" | delta p10/50/90 {torch.quantile(dlt[:200000], qs).cpu().numpy()}"
                     f" | gap p10/50/90 {torch.quantile(gap[:200000], qs).cpu().numpy()}"
                     f" | d1 p50 {torch.quantile(d[:200000, 0].sqrt(), 0.5).item():.4f}")
            # stale references: keep the reference of skipped anchors
            upd = ~skip
            ref_q = torch.where(upd[:, None], q, ref_q)
            ref_sec = torch.where(upd, d[:, 1], ref_sec)
            ref_id = torch.where(upd, i[:, 0], ref_id)
        else:
            ref_q, ref_sec, ref_id = q.clone(), d[:, 1].clone(), i[:, 0].clone()
        prev_q = q
        print(line, flush=True)
        print("    verlet: " + " | ".join(vl), flush=True)


if __name__ == "__main__":
    main(hist="--nohist" not in sys.argv)
