"""Acceptance C10 shape (acceptance_main.cpp:498-509): tune_nu on a
seeded 1372 x 4 matrix, q = 3, 30-point nu grid in [1.1, 5], K = 5 folds,
classical embedding.  Times the engine, and the compiled reference when present."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2605_25124_b200 import gmds as G  # noqa: E402

rng = np.random.default_rng(10)
X = rng.standard_normal((1372, 4))
grid = list(np.linspace(1.1, 5.0, 30))
G.tune_nu(X, 3, grid[:2], 5)  # warm-up at the same fold size (module loads, cuSOLVER)
out = {}
for rep in range(2):
    t0 = time.perf_counter()
    r = G.tune_nu(X, 3, grid, 5)
    out[f"engine_s_{rep}"] = time.perf_counter() - t0
out["nu_star"] = r["nu_star"]
out["stress"] = r["stress"]
try:
    from oracle import ref_lib as R
    if R.load() is not None and hasattr(R, "tune_nu"):
        t0 = time.perf_counter()
        rr = R.tune_nu(X, 3, grid, 5)
        out["reference_s"] = time.perf_counter() - t0
        out["reference_nu_star"] = rr["nu_star"]
        out["mean_stress_max_rel_dev"] = float(np.max(np.abs(np.array(r["mean_stress"]) - np.array(rr["mean_stress"]))
                                                     / np.array(rr["mean_stress"])))
except Exception as e:  # noqa: BLE001
    out["reference_error"] = str(e)
print(json.dumps(out))
