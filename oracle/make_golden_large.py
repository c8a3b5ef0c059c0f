"""Golden fixtures at BASELINE.json's shapes, from the UNMODIFIED reference --
TEST INFRASTRUCTURE (VERDICT r1 "next" #1-#2).

Every expected value comes from the reference compiled by oracle/Makefile:
``pairwise_matrix`` / ``gen_gini_distance`` / ``midrank`` / ``minimize_stress``
(oracle/_ref/libginimds_ref.so) and, for seeded starts, the
reference's own ``gradient_descent`` loop entered with Y0
(oracle/_ref/libginimds_ref_seeded.so, oracle/ref_seeded.cpp).  Inputs are the
seeded generators of oracle/synth.py (numpy PCG64: a GPU box regenerates the same
bytes).  Matrices are too large to commit at these sizes, so the fixtures hold
trajectories, final stresses, coordinates and seeded samples of D entries /
per-pair rank fingerprints.

    make -C oracle && python oracle/make_golden_large.py [metric c3 img2600 c2 c4]

Runtimes on 8 host cores: metric ~35 min (the reference builds the full
20000 x 20000 Gini matrix), c3 ~25 min, the others a few minutes.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import ref_lib as R  # noqa: E402
from oracle import synth as S  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)", flush=True)


def log(msg, t0):
    print(f"[{time.perf_counter() - t0:8.1f} s] {msg}", flush=True)


def seeded_traj(name, n, p, xseed, yseed, iters, t0):
    """Kruskal from Y0 ~ N(0, 0.1^2) on image-like data: the path bench.py measures."""
    X = S.image_like(n, p, xseed)
    D = R.pairwise_matrix(X.astype(np.float64), 2.0)
    log(f"{name}: reference D ({n} x {n})", t0)
    Y0 = np.random.default_rng(yseed).normal(0.0, 0.1, (n, 2))
    r = R.seeded_fit(D.T, Y0, "kruskal", max_iters=iters, rel_tol=1e-300)
    log(f"{name}: reference seeded Kruskal x{iters}", t0)
    return X, D, dict(history=np.array(r["stress_history"]), iterations=r["iterations"], stress=r["stress"],
                      coords=r["coords"], n=n, p=p, xseed=xseed, yseed=yseed)


def metric(t0):
    # BASELINE metric shape = bench.py's workload (bench.make_image_like(N, P) with SEED = 2605,
    # Y0 = default_rng(SEED).normal(0, 0.1, (N, 2)), 50 Kruskal iterations)
    n, p, seed = 20000, 784, 2605
    X, D, fit = seeded_traj("metric", n, p, seed, seed, 50, t0)
    # >= 1e6 sampled entries (+ the zero diagonal is not sampled), stored fp32 (1e-6 max-normalised bar)
    I, J = S.sample_pairs(n, 1_000_000, seed=11)
    vals = D[I, J]
    # >= 1e4 per-pair rank fingerprints (reference midrank of x_i - x_j)
    Ir, Jr = S.sample_pairs(n, 10_000, seed=12)
    w = S.rank_weights(p)
    Xd = X.astype(np.float64)
    fp = np.zeros(Ir.size, dtype=np.int64)
    for k in range(Ir.size):
        fp[k] = int(S.rank_fingerprints(R.midrank(Xd[Ir[k]] - Xd[Jr[k]])[None, :], w)[0])
    log("metric: samples + rank fingerprints", t0)
    save("large_metric", D_sample=vals.astype(np.float32), D_max=np.float64(D.max()), pair_seed=11,
         npairs=I.size, rank_seed=12, nrank=Ir.size, rank_fp=fp, rank_w_seed=99,
         D_sum=np.float64(D.sum()), D_sumsq=np.float64(np.sum(D * D)), **{"fit_" + k: v for k, v in fit.items()})


def c3(t0):
    # C3 (n = 5000, p = 784 image-like, nu = 2, q = 2): (a) the bench path's regime -- seeded
    # N(0, 0.1^2) init, 50 iterations; (b) parity mode -- the reference's own minimize_stress
    # (classical init) for 2000 iterations
    n, p = 5000, 784
    X, D, fit = seeded_traj("c3", n, p, 3, 3, 50, t0)
    e = R.minimize_stress(D, 2, "kruskal", max_iters=2000, rel_tol=1e-300)
    log("c3: reference minimize_stress (classical init) x2000", t0)
    I, J = S.sample_pairs(n, 200_000, seed=31)
    save("large_c3", D_sample=D[I, J], D_max=np.float64(D.max()), pair_seed=31, npairs=I.size,
         D_rowsum=D.sum(axis=1), cls_history=np.array(e["stress_history"]), cls_iterations=e["iterations"],
         cls_stress=e["stress"], cls_coords=e["coords"], **{"fit_" + k: v for k, v in fit.items()})


def img2600(t0):
    # above the persistent small-fit size (n <= 2048): the TMA fp32 passes + difference passes +
    # device gd_step loop; 60 iterations, seeded N(0, 0.1^2) init
    X, D, fit = seeded_traj("img2600", 2600, 784, 78, 78, 60, t0)
    save("large_img2600", D_rowsum=D.sum(axis=1), **{"fit_" + k: v for k, v in fit.items()})


def cls1500(t0):
    # the reference's classical_mds (dense SelfAdjointEigenSolver, embed.cpp:415-460) at n = 1500,
    # image-like data: pins the engine's top-q Lanczos solver (no dense B) directly
    X = S.image_like(1500, 784, 9)
    D = R.pairwise_matrix(X.astype(np.float64), 2.0)
    out = {}
    for q in (1, 2, 3):
        e = R.classical_mds(D, q)
        out[f"coords{q}"] = e["coords"]
        out[f"eig{q}"] = e["eigenvalues"]
        out[f"stress{q}"] = e["stress"]
    log("cls1500: reference classical_mds q = 1, 2, 3", t0)
    save("large_cls1500", D_rowsum=D.sum(axis=1), **out)


def c2(t0):
    # C2: 8 nu in [1.1, 8]; per nu the reference pairwise_matrix and minimize_stress(Kruskal,
    # classical init, 1000 iterations)
    X = S.mixture_contaminated()
    grid = S.c2_grid()
    n = X.shape[0]
    I, J = S.sample_pairs(n, 50_000, seed=21)
    out = dict(grid=np.array(grid), pair_seed=21, npairs=I.size)
    samples, rowsums, hists, stresses, iters, coords = [], [], [], [], [], []
    for nu in grid:
        D = R.pairwise_matrix(X, nu)
        samples.append(D[I, J])
        rowsums.append(D.sum(axis=1))
        e = R.minimize_stress(D, 2, "kruskal", max_iters=1000, rel_tol=1e-300)
        hists.append(e["stress_history"])
        stresses.append(e["stress"])
        iters.append(e["iterations"])
        coords.append(e["coords"])
        log(f"c2: nu = {nu:.4f}: D + Kruskal x1000 (iterations {e['iterations']})", t0)
    m = max(len(h) for h in hists)
    H = np.full((len(grid), m), np.nan)
    for k, h in enumerate(hists):
        H[k, : len(h)] = h
    save("large_c2", D_sample=np.array(samples), D_rowsum=np.array(rowsums), history=H, stress=np.array(stresses),
         iterations=np.array(iters), coords=np.array(coords), **out)


def c4(t0):
    # C4: n = 20000, p = 128 log-normal, 1% duplicated rows, 4 nu; 250k sampled pairs (all
    # duplicate pairs included: exact zeros) x 4 nu = 1e6 entries
    X, dup, src = S.lognormal_dup()
    Xd = X.astype(np.float64)
    I, J = S.sample_pairs(X.shape[0], 250_000 - dup.size, seed=41, extra=(dup, src))
    vals = np.stack([R.gini_pairs(Xd, I, J, nu) for nu in S.C4_NUS])
    log("c4: 4 x 250k reference gen_gini_distance", t0)
    Ir, Jr = S.sample_pairs(X.shape[0], 10_000, seed=42)
    w = S.rank_weights(X.shape[1])
    fp = np.array([int(S.rank_fingerprints(R.midrank(Xd[i] - Xd[j])[None, :], w)[0]) for i, j in zip(Ir, Jr)])
    save("large_c4", D_sample=vals.astype(np.float32), pair_seed=41, npairs=I.size, nus=np.array(S.C4_NUS),
         rank_seed=42, nrank=Ir.size, rank_fp=fp)


def main():
    if R.load() is None or R.load_seeded() is None:
        sys.exit("oracle/_ref not built: make -C oracle")
    which = sys.argv[1:] or ["img2600", "cls1500", "c2", "c4", "c3", "metric"]
    t0 = time.perf_counter()
    for w in which:
        globals()[w](t0)


if __name__ == "__main__":
    main()
