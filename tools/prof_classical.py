"""Classical-MDS init at large n: device subspace iteration vs
the dense cuSOLVER path, on the metric-config generator."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import make_image_like  # noqa: E402
from paper_2605_25124_b200 import gmds as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="*", default=[5000, 20000])
ap.add_argument("--dense-max", type=int, default=8000)
ap.add_argument("--q", type=int, default=2)
a = ap.parse_args()
import torch  # noqa: E402

for n in a.n:
    X = make_image_like(n, 784, seed=11)
    dX = torch.from_numpy(X).cuda()
    Dm = G.dmat_gini_device(dX.data_ptr(), G.F32, n, 784, 2.0, G.F32)
    G.classical_mds_topq(G.dmat_from_host(G.pairwise_matrix(X[:300], 2.0)), a.q)  # warm-up
    t0 = time.perf_counter()
    t = G.classical_mds_topq(Dm, a.q)
    tt = time.perf_counter() - t0
    out = {"n": n, "q": a.q, "topq_s": tt, "iterations": t["iterations"], "eigenvalues": list(t["eigenvalues"])}
    if n <= a.dense_max:
        t0 = time.perf_counter()
        r = G.classical_mds(Dm, a.q)
        out["dense_s"] = time.perf_counter() - t0
        out["max_coord_dev_rel"] = float(np.max(np.abs(t["coords"] - r["coords"])) / np.max(np.abs(r["coords"])))
        out["eig_rel_dev"] = float(np.max(np.abs(t["eigenvalues"] - r["eigenvalues"]) / np.abs(r["eigenvalues"])))
    print(json.dumps(out), flush=True)
    del Dm, dX
