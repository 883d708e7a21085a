"""BASELINE config 2 (search-only, 1,048,576 x 65,536, d = 24) under the budget
searches: greedy / backtrack(m) through psg_index_query on the device tree and
on the library's replica of the reference tree.  Prints one JSON line per run.

usage: python scripts/budget_cfg2.py [n_queries]"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402


def main():
    nq = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    X = wl.gaussian_mixture(65536, 192, 64, 20.0, 1)
    Q = wl.gaussian_mixture(nq, 192, 64, 20.0, 2)
    ctx = api.Context(0)
    for tree, kw in (("device", dict(max_depth=3)), ("reference", dict(tree_kind=api.TREE_REFERENCE))):
        t = time.perf_counter()
        ix = api.make_vector_index(X, branching=8, d_fixed=24, seed=1, ctx=ctx, **kw)
        t_build = time.perf_counter() - t
        ix.nearest(Q[:4096], api.QueryBudget.backtrack(4))  # warm-up
        e_idx = None
        for name, bud in (("exact", api.QueryBudget.exact()), ("greedy", api.QueryBudget.greedy()),
                          ("backtrack:4", api.QueryBudget.backtrack(4)),
                          ("backtrack:16", api.QueryBudget.backtrack(16))):
            ctx.profile(True)
            t = time.perf_counter()
            idx, dist, dpca, scanned = ix.nearest(Q, bud)
            dt = time.perf_counter() - t
            kern = ctx.kernel_times()
            ctx.profile(False)
            if name == "exact":
                e_idx = idx
            print(json.dumps({"tree": tree, "budget": name, "queries": nq, "index_build_s": t_build,
                              "queries_per_s_e2e": nq / dt,
                              "search_ms": kern.get("search_kernel", (0, 0))[0],
                              "recall_vs_exact": float((idx == e_idx).mean()),
                              "points_scanned_per_query": float(scanned.mean())}))


if __name__ == "__main__":
    main()
