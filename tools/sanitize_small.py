"""Small invocations of the hot kernels for compute-sanitizer (racecheck / memcheck):
gini_gmd_kernel (nu = 2, sparse fp32), gini_gen_kernel (nu = 2.5), the split and merge
kernels, the TMA stress passes (fused / gradient / difference, device gd_step loop; the
small-fit kernel is bypassed with GMDS_NO_SMALL_FIT), the Lanczos classical init and the
sharded fit through a local rank group."""
import os
import sys

os.environ["GMDS_NO_SMALL_FIT"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2605_25124_b200 import gmds as G  # noqa: E402

rng = np.random.default_rng(0)
n, p = 300, 200
X = rng.integers(0, 256, size=(n, p)).astype(np.float32) / 255.0
X[rng.random(X.shape) < 0.8] = 0.0
D2 = G.pairwise_gini(X, [2.0])[0]           # gini_gmd_kernel
D25 = G.pairwise_gini(X, [2.5])[0]          # gini_gen_kernel
Dm = G.pairwise_gini(X, list(np.linspace(1.2, 6.0, 6)))  # merge kernel (> 4 nu)
Xd = rng.standard_normal((200, 40))
Ds = G.pairwise_gini(Xd, [1.5, 3.0])        # split kernel (dense, p <= 512)
print("distance kernels ok", float(D2.sum()), float(D25.sum()), float(Dm.sum()), float(Ds.sum()))
Y0 = rng.normal(0.0, 0.1, (n, 2))
e = G.minimize_stress(D2, 2, "kruskal", max_iters=12, rel_tol=1e-300, Y0=Y0, storage=G.F32)
print("stress fit ok", e["iterations"], e["passes"])
c = G.classical_mds_topq(G.dmat_from_host(D2, G.F32), 2)
print("lanczos ok", c["iterations"])
