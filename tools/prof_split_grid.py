"""Split-kernel occupancy grid: dense inputs, p x dtype x nnu, time per matrix."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_25124_b200 import gmds as G  # noqa: E402

n = int(os.environ.get("PSG_N", "12000"))
OT = G.F64 if os.environ.get("PSG_OUT") == "f64" else G.F32
PS = [int(v) for v in os.environ.get("PSG_P", "32,64,128,256").split(",")]
g = np.random.default_rng(4)
for p in PS:
    for dt in (np.float32, np.float64):
        X = np.exp(g.standard_normal((n, p))).astype(dt)
        dX = torch.from_numpy(X).cuda()
        xt = G.F32 if dt == np.float32 else G.F64
        for nus in ([2.0], [1.5, 2.0, 3.0, 5.0]):
            out = torch.zeros(len(nus) * G.packed_elems(n), dtype=torch.float32 if OT == G.F32 else torch.float64,
                              device="cuda")
            best = 1e9
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                G.pairwise_gini_device(dX.data_ptr(), xt, n, p, nus, OT, True, out.data_ptr())
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            print(f"p={p:4d} {np.dtype(dt).name:8s} nnu={len(nus)}: {best * 1e3:8.1f} ms", flush=True)
