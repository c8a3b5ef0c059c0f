"""bench.py's stress step alone (n = 20000 metric data, packed fp32 D, seeded N(0, 0.1^2)
init, Kruskal x ITERS) -- for launch lists and kernel profiles of the fit."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import make_image_like  # noqa: E402
from paper_2605_25124_b200 import gmds as G  # noqa: E402

n = int(os.environ.get("FIT_N", "20000"))
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
q = int(os.environ.get("FIT_Q", "2"))
X = make_image_like(n, 784)
dX = torch.from_numpy(X).cuda()
D = G.dmat_gini_device(dX.data_ptr(), G.F32, n, 784, 2.0, G.F32)
Y0 = np.random.default_rng(2605).normal(0.0, 0.1, (n, q))
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    e = G.minimize_stress(D, q, "kruskal", max_iters=iters, rel_tol=1e-300, Y0=Y0)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(e["iterations"], e["passes"], e["stress"], f"ms={min(ts[1:]):.3f}")
