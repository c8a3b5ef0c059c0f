"""Phase trace of the drop-in pairwise_matrix call at the metric shape (host
fp32 X -> pinned host fp64 n x n D): GMDS_TRACE phases plus the wall time."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ.setdefault("GMDS_TRACE", "1")
from bench import make_image_like, N, P  # noqa: E402
from paper_2605_25124_b200 import gmds as G  # noqa: E402

X = make_image_like(N, P)
Xh = torch.from_numpy(X).pin_memory().numpy()
Dh = torch.empty((1, N, N), dtype=torch.float64).pin_memory().numpy()
for k in range(3):
    t0 = time.perf_counter()
    G.lib().gmds_pairwise_gini(G._vp(Xh), G._i32(G.F32), G._i32(G.ROW_MAJOR), G._i64(N), G._i64(P),
                               G._p(np.array([2.0])), G._i32(1), G._i32(G.F64), G._vp(Dh))
    print(f"e2e call {k}: {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)
