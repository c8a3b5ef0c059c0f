"""Small fixed workloads for ncu captures (one GPU): `distance` runs the
metric-config generator at a reduced n; `stress` runs a few Kruskal
iterations at the full metric n.  Not a benchmark (numbers printed under a
profiler are never reported)."""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import make_image_like  # noqa: E402
from paper_2605_25124_b200 import gmds as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["distance", "stress", "both"])
    ap.add_argument("--n", type=int, default=4000)
    ap.add_argument("--p", type=int, default=784)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--q", type=int, default=2)
    a = ap.parse_args()
    import torch

    X = make_image_like(a.n, a.p)
    dX = torch.from_numpy(X).cuda()
    if a.mode in ("distance", "both"):
        pe = G.packed_elems(a.n)
        dD = torch.zeros(pe, dtype=torch.float32, device="cuda")
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            G.pairwise_gini_device(dX.data_ptr(), G.F32, a.n, a.p, [2.0], G.F32, True, dD.data_ptr())
            torch.cuda.synchronize()
            print(f"distance n={a.n} p={a.p}: {time.perf_counter() - t0:.4f} s", flush=True)
    if a.mode in ("stress", "both"):
        Dm = G.dmat_gini_device(dX.data_ptr(), G.F32, a.n, a.p, 2.0, G.F32)
        Y0 = np.random.default_rng(1).normal(0, 0.1, (a.n, a.q))
        for _ in range(a.reps):
            t0 = time.perf_counter()
            r = G.minimize_stress(Dm, a.q, "kruskal", max_iters=a.iters, rel_tol=1e-300, Y0=Y0)
            print(f"stress n={a.n}: {a.iters} iters {time.perf_counter() - t0:.4f} s passes={r['passes']}", flush=True)


if __name__ == "__main__":
    main()
