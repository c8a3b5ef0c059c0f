"""Fit sanity at a given n (image-like data, nu = 2, seeded N(0, 0.1^2) init): iterations,
first losses, final stress -- for bisecting fit regressions and the fp32-resolution regime."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import make_image_like  # noqa: E402
from paper_2605_25124_b200 import gmds as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 60
storage = G.F64 if (len(sys.argv) > 3 and sys.argv[3] == "f64") else G.F32
X = make_image_like(n, 784, seed=3)
dX = torch.from_numpy(X).cuda()
Dm = G.dmat_gini_device(dX.data_ptr(), G.F32, n, 784, 2.0, storage)
Y0 = np.random.default_rng(3).normal(0.0, 0.1, (n, 2))
G.minimize_stress(Dm, 2, "kruskal", max_iters=2, rel_tol=1e-300, Y0=Y0)
torch.cuda.synchronize()
t0 = time.perf_counter()
e = G.minimize_stress(Dm, 2, "kruskal", max_iters=iters, rel_tol=1e-300, Y0=Y0)
dt = time.perf_counter() - t0
h = np.array(e["stress_history"])
print(f"n={n} {'f64' if storage == G.F64 else 'f32'} env={ {k: v for k, v in os.environ.items() if k.startswith('GMDS')} } "
      f"iters={e['iterations']} passes={e['passes']} {dt:.3f}s h[0,10,20,30,40,-1]={[float(h[i]) for i in (0, 10, 20, 30, 40, -1) if i < len(h)]}",
      flush=True)
np.save(f"gpurun_out/hist_{n}_{'f64' if storage == G.F64 else 'f32'}.npy", h)
