"""Split-kernel workloads (dense inputs): C4 (n=20000, p=128 log-normal, 4 nu,
fp32 full matrices), dense normal p=64 fp64 (packed), dense normal p=400 fp32."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_25124_b200 import gmds as G  # noqa: E402


def run(name, X, nus, ot, packed, reps=2):
    n, p = X.shape
    dX = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    xt = G.F32 if X.dtype == np.float32 else G.F64
    elems = G.packed_elems(n) if packed else n * n
    out = torch.zeros(len(nus) * elems, dtype=torch.float32 if ot == G.F32 else torch.float64, device="cuda")
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        G.pairwise_gini_device(dX.data_ptr(), xt, n, p, nus, ot, packed, out.data_ptr())
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    print(f"{name}: {t * 1e3:.1f} ms  ({n * (n - 1) / 2 / t / 1e6:.1f} M pairs/s)", flush=True)


g = np.random.default_rng(4)
run("C4 n=20000 p=128 lognormal 4nu f32 full", np.exp(g.standard_normal((20000, 128))).astype(np.float32),
    [1.5, 2.0, 3.0, 5.0], G.F32, False)
run("dense n=20000 p=64 f64 packed", g.standard_normal((20000, 64)), [2.0], G.F64, True)
run("dense n=8000 p=400 f32 packed", g.standard_normal((8000, 400)).astype(np.float32), [2.0], G.F32, True)
