"""Per-iteration cost of the persistent small-n fit (min over repeats), or
one fit for ncu with --once.  GMDS_NO_SMALL_FIT=1 times the host-driven
engine instead."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2605_25124_b200 import gmds as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="*", default=[200, 1000, 2000])
ap.add_argument("--kinds", nargs="*", default=["kruskal", "smacof"])
ap.add_argument("--iters", type=int, default=300)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--once", action="store_true")
a = ap.parse_args()
for n in a.n:
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, 20))
    Dm = G.dmat_from_host(G.pairwise_matrix(X, 2.0))
    Y0 = rng.normal(0.0, 0.1, (n, 2))
    for kind in a.kinds:
        G.minimize_stress(Dm, 2, kind, max_iters=5, rel_tol=1e-300, Y0=Y0)
        best = 1e9
        for _ in range(1 if a.once else a.reps):
            t0 = time.perf_counter()
            e = G.minimize_stress(Dm, 2, kind, max_iters=a.iters, rel_tol=1e-300, Y0=Y0)
            best = min(best, time.perf_counter() - t0)
        print(f"n={n} {kind}: {best / e['iterations'] * 1e6:.1f} us/iter  ({e['iterations']} it, {e['passes']} passes,"
              f" stress {e['stress']:.6g})", flush=True)
