"""BASELINE config 2: search-only microbenchmark.

1,048,576 queries and 65,536 database vectors, D = 192 fp32, mixture of 64
isotropic Gaussians (means ~U[0,255], sigma = 20); PCA to d = 24 (fitted on
the DB, on device); k-means tree b = 8 depth 3; exact search.  Checked against
exhaustive search in PCA space (the oracle port) on a sample of queries and
against the reference's brute_force_nearest when oracle/_ref is present.

Prints one JSON line: queries/s through psg_index_query (host buffers in/out,
i.e. including the 805 MB H2D of the queries) and the device search time.
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2006_11851_b200 import api  # noqa: E402
from paper_2006_11851_b200 import workloads as wl  # noqa: E402


def main():
    nq = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    X = wl.gaussian_mixture(65536, 192, 64, 20.0, 1)
    Q = wl.gaussian_mixture(nq, 192, 64, 20.0, 2)
    ctx = api.Context(0)
    t = time.perf_counter()
    ix = api.make_vector_index(X, branching=8, max_depth=3, d_fixed=24, seed=1, ctx=ctx)
    t_build = time.perf_counter() - t
    ix.nearest(Q[:4096])  # warm-up
    ctx.profile(True)
    t = time.perf_counter()
    idx, dist, dpca, scanned = ix.nearest(Q)
    t_query = time.perf_counter() - t
    kern = ctx.kernel_times()
    # exactness on a sample: exhaustive lexicographic min in PCA space
    from oracle.oracle import Port
    port = Port()
    mean, basis, _ = ix.pca()
    P = ix.projected()
    rng = np.random.Generator(np.random.PCG64(7))
    sample = rng.choice(nq, size=min(nq, 1000), replace=False)
    qp = port.project_all(Q[sample], mean, basis)
    bad = 0
    for k, i in enumerate(sample):
        j, d2 = port.nearest_lexmin(P, qp[k])
        bad += (j != idx[i]) or (np.sqrt(d2) != dpca[i])
    ref_bad = None
    try:
        from oracle.oracle import Ref, REF_SO
        if REF_SO.exists():
            ref = Ref()
            ref_bad = 0
            for k, i in enumerate(sample[:200]):
                jr, dr = ref.brute_force_nearest(P, qp[k])
                ref_bad += (jr != idx[i]) or (dr != dpca[i])
    except Exception as e:  # noqa: BLE001
        ref_bad = f"unavailable: {e}"
    search_ms = kern.get("search_kernel", (0.0, 0))[0]
    line = {
        "workload": "cfg2 search-only: 1M queries x 65,536 DB, D=192, d=24, tree b=8 depth 3, exact",
        "queries": nq, "index_build_s": t_build,
        "queries_per_s_e2e": nq / t_query,
        "queries_per_s_device_search": nq / (search_ms / 1e3) if search_ms else None,
        "kernels_ms": {k: round(v[0], 3) for k, v in kern.items()},
        "points_scanned_per_query": float(scanned.mean()),
        "tree": {"leaves": ix.n_leaves, "nodes": ix.n_nodes, "depth": ix.depth},
        "exact_mismatches_vs_port_of_1000": int(bad),
        "mismatches_vs_reference_of_200": int(ref_bad) if isinstance(ref_bad, (int, np.integer)) else ref_bad,
    }
    print(json.dumps(line, default=float))


if __name__ == "__main__":
    main()
