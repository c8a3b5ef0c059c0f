"""All five BASELINE.json configs on one B200 (SURVEY 8(d) generators), each
with a parity spot-check against the oracle and the reference CPU time on a
bounded sample.  Prints one JSON object per config.  Secondary to bench.py
(the headline metric); used for DESIGN.md's per-config table.

  C1  n=200,   p=8,   fp64 N(0,1), nu=2, q=2, 500 iterations, every stress kind,
      classical init and seeded N(0, 0.1^2) init
  C2  n=1000,  p=20,  fp64 3-component mixture, 5% of rows x10 (contaminate),
      8 nu log-spaced in [1.1, 8] (nu <= 1 is invalid in the reference, F5), Kruskal x1000 per nu
  C3  n=5000,  p=784, fp32 image-like, nu=2, q=2, Kruskal x2000
  C4  n=20000, p=128, fp32 log-normal(0,1), 1% duplicated rows, 4 nu in {1.5,2,3,5}, full matrices
  C5  n=60000, p=784, fp32 image-like, q=3, ONE nu of the 16-value sweep (the per-GPU share
      on 8 GPUs is 2), 500 Kruskal iterations, seeded init (F4)
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import make_image_like  # noqa: E402
from oracle import gini_oracle as O  # noqa: E402
from oracle import ref_lib as R  # noqa: E402
from paper_2605_25124_b200 import gmds as G  # noqa: E402


def timed(fn):
    import torch

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def ref_time(fn, budget=20.0):
    if R.load() is None:
        return None
    t0 = time.perf_counter()
    fn()
    return time.perf_counter() - t0


def c1():
    rng = np.random.default_rng(1)
    X = rng.standard_normal((200, 8))
    D = G.pairwise_matrix(X, 2.0)
    Dm = G.dmat_from_host(D)
    res = {"config": "C1", "n": 200, "p": 8}
    Y0 = rng.normal(0.0, 0.1, (200, 2))
    for kind in ("kruskal", "sammon", "smacof", "huber"):
        hd = 0.5 * float(np.median(D[np.triu_indices(200, 1)])) if kind == "huber" else None
        e, t = timed(lambda: G.minimize_stress(Dm, 2, kind, huber_delta=hd, max_iters=500, rel_tol=1e-300))
        e2, t2 = timed(lambda: G.minimize_stress(Dm, 2, kind, huber_delta=hd, max_iters=500, rel_tol=1e-300, Y0=Y0))
        tr = ref_time(lambda: R.minimize_stress(D, 2, kind, huber_delta=hd, max_iters=500, rel_tol=1e-300))
        ref = O.minimize_stress(D, 2, kind, huber_delta=hd, max_iters=60, rel_tol=1e-300)
        dev = float(np.max(np.abs(np.array(e["stress_history"][:51]) - ref.stress_history[:51]) / ref.stress_history[0]))
        res[kind] = {"fit_s": t, "seeded_fit_s": t2, "iterations": e["iterations"], "ref_cpu_s": tr,
                     "traj50_max_rel_dev": dev}
    _, td = timed(lambda: G.pairwise_matrix(X, 2.0))
    res["distance_s_e2e"] = td
    return res


def c2():
    rng = np.random.default_rng(2)
    n, p = 1000, 20
    means = rng.normal(0.0, 3.0, (3, p))
    X = means[rng.integers(0, 3, n)] + rng.standard_normal((n, p))
    rows = rng.choice(n, int(round(0.05 * n)), replace=False)
    X[rows] *= 10.0 * X.std(axis=0)  # contaminate(multiply_by_factor_sigma, factor=10)
    grid = list(np.exp(np.linspace(np.log(1.1), np.log(8.0), 8)))
    Ds, td = timed(lambda: G.pairwise_gini(X, grid))
    fits = []
    t_fit = 0.0
    for k, nu in enumerate(grid):
        Dm = G.dmat_from_host(Ds[k])
        e, t = timed(lambda: G.minimize_stress(Dm, 2, "kruskal", max_iters=1000, rel_tol=1e-300))
        fits.append(e["stress"])
        t_fit += t
    err = max(float(np.max(np.abs(Ds[k] - O.pairwise_matrix(X, nu))) / np.max(Ds[k])) for k, nu in enumerate(grid[:2]))
    tr = ref_time(lambda: R.pairwise_matrix(X, grid[0]))
    return {"config": "C2", "n": n, "p": p, "nus": grid, "distance_all_nu_s": td, "fits_s": t_fit,
            "kruskal_per_nu": fits, "nu_star": grid[int(np.argmin(fits))], "D_maxnorm_err": err,
            "ref_cpu_distance_one_nu_s": tr}


def c3():
    X = make_image_like(5000, 784, seed=3)
    import torch

    dX = torch.from_numpy(X).cuda()
    Dm, td = timed(lambda: G.dmat_gini_device(dX.data_ptr(), G.F32, 5000, 784, 2.0, G.F32))
    Y0 = np.random.default_rng(3).normal(0.0, 0.1, (5000, 2))
    e, tf = timed(lambda: G.minimize_stress(Dm, 2, "kruskal", max_iters=2000, rel_tol=1e-300, Y0=Y0))
    # the same fit with fp64 storage of D (parity mode): the reference's first iterations
    # change the loss by ~1e-13 relative, below fp32 storage's resolution
    Dm64 = G.dmat_gini_device(dX.data_ptr(), G.F32, 5000, 784, 2.0, G.F64)
    e64, tf64 = timed(lambda: G.minimize_stress(Dm64, 2, "kruskal", max_iters=2000, rel_tol=1e-300, Y0=Y0))
    I = np.random.default_rng(4).integers(0, 5000, 2000)
    J = np.random.default_rng(5).integers(0, 5000, 2000)
    keep = I < J
    Xd = X.astype(np.float64)
    ref = O.gini_pairs(Xd, I[keep], J[keep], 2.0)
    full = G.pairwise_gini(X[:600], [2.0])[0]
    err = float(np.max(np.abs(full - O.pairwise_matrix(Xd[:600], 2.0))) / np.max(full))
    # the sampled pairs against the GPU's own full matrix (the fit's D, unpacked)
    Dfull = Dm64.download()
    pair_err = float(np.max(np.abs(Dfull[I[keep], J[keep]] - ref)) / np.max(Dfull))
    rows = 8
    tr = None
    if R.load() is not None:
        t0 = time.perf_counter()
        R.gini_rows(Xd, 2.0, 0, rows)
        tr = (time.perf_counter() - t0) / sum(4999 - i for i in range(rows)) * (5000 * 4999 / 2)
    return {"config": "C3", "n": 5000, "p": 784, "distance_s": td, "pairs_per_s": 5000 * 4999 / 2 / td,
            "fit_2000_iters_s": tf, "iters_per_s": e["iterations"] / tf, "final_stress": e["stress"],
            "fit_iterations": e["iterations"],
            "fp64_storage": {"fit_s": tf64, "iterations": e64["iterations"], "final_stress": e64["stress"],
                             "iters_per_s": e64["iterations"] / tf64},
            "D_maxnorm_err_600rows": err, "ref_cpu_distance_s_extrapolated": tr, "checked_pairs": int(keep.sum()),
            "checked_pairs_maxnorm_err": pair_err,
            "ref_pairs_mean": float(np.mean(ref))}


def c4():
    g = np.random.default_rng(4)
    n, p = 20000, 128
    X = np.exp(g.standard_normal((n, p))).astype(np.float32)
    dup = g.choice(n, 200, replace=False)
    X[dup] = X[g.choice(n, 200, replace=False)]
    import torch

    dX = torch.from_numpy(X).cuda()
    nus = [1.5, 2.0, 3.0, 5.0]
    out = torch.zeros((4, n, n), dtype=torch.float32, device="cuda")
    _, td = timed(lambda: G.pairwise_gini_device(dX.data_ptr(), G.F32, n, p, nus, G.F32, False, out.data_ptr()))
    sub = out[:, :300, :300].cpu().numpy()
    err = max(float(np.max(np.abs(sub[k] - O.pairwise_matrix(X[:300].astype(np.float64), nu))) / np.max(sub[k]))
              for k, nu in enumerate(nus))
    tr = None
    if R.load() is not None:
        t0 = time.perf_counter()
        R.gini_rows(X.astype(np.float64), 2.0, 0, 16)
        per_pair = (time.perf_counter() - t0) / sum(n - 1 - i for i in range(16))
        tr = per_pair * n * (n - 1) / 2 * 4  # 4 nu, each a separate reference pass
    return {"config": "C4", "n": n, "p": p, "nus": nus, "distance_all_nu_s": td,
            "pairs_per_s_all_nu": n * (n - 1) / 2 / td, "D_maxnorm_err_300rows": err,
            "ref_cpu_s_extrapolated": tr}


def c5():
    n, p = 60000, 784
    X = make_image_like(n, p, seed=5)
    import torch

    dX = torch.from_numpy(X).cuda()
    nu = float(np.exp(np.linspace(np.log(1.1), np.log(8.0), 16))[5])
    Dm, td = timed(lambda: G.dmat_gini_device(dX.data_ptr(), G.F32, n, p, nu, G.F32))
    Y0 = np.random.default_rng(5).normal(0.0, 0.1, (n, 3))
    e, tf = timed(lambda: G.minimize_stress(Dm, 3, "kruskal", max_iters=500, rel_tol=1e-300, Y0=Y0))
    Dm.free()
    # one GPU's share of the 16-value sweep on 8 GPUs: two nu from ONE launch (packed fp32, 2 x 7.2 GB)
    grid = np.exp(np.linspace(np.log(1.1), np.log(8.0), 16))
    two = [float(grid[5]), float(grid[6])]
    out = torch.empty(2 * G.packed_elems(n), dtype=torch.float32, device="cuda")
    _, t2 = timed(lambda: G.pairwise_gini_device(dX.data_ptr(), G.F32, n, p, two, G.F32, True, out.data_ptr()))
    return {"config": "C5 (one nu; 2 per GPU on 8 GPUs)", "n": n, "p": p, "q": 3, "nu": nu, "distance_s": td,
            "pairs_per_s": n * (n - 1) / 2 / td, "fit_500_iters_s": tf, "iters_per_s": e["iterations"] / tf,
            "final_stress": e["stress"], "distance_two_nu_one_launch_s": t2,
            "pairs_per_s_two_nu": n * (n - 1) / 2 / t2}


def warmup():
    # first calls load kernels / cuSOLVER lazily: keep that out of the timings
    rng = np.random.default_rng(0)
    X = rng.standard_normal((256, 40))
    D = G.pairwise_matrix(X, 2.0)
    for kind in ("kruskal", "smacof"):
        G.minimize_stress(D, 2, kind, max_iters=3)
        G.minimize_stress(D, 3, kind, max_iters=3)
    G.pairwise_gini(X.astype(np.float32), [2.0])
    Xs = (np.abs(X) * (rng.random(X.shape) < 0.25)).astype(np.float32)  # sparse, non-negative, p > 32
    G.pairwise_gini(Xs, [2.0])   # gini_gmd2_kernel (lazy kernel load)
    G.pairwise_gini(Xs, [2.5])   # gini_gen2_kernel


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c1", "c2", "c3", "c4", "c5"])
    a = ap.parse_args()
    warmup()
    for c in a.configs:
        print(json.dumps(globals()[c]()), flush=True)


if __name__ == "__main__":
    main()
