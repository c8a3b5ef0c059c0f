"""Generate tests/golden/*.npz from the UNMODIFIED reference -- TEST INFRASTRUCTURE.

Every expected value below is produced by ``oracle/_ref/libginimds_ref.so``
(the reference's own proj/core sources compiled by oracle/Makefile); inputs
are regenerated with the reference's own Rng (mt19937_64) exactly as the
reference tests build them (test_util.hpp:15-39, test_metrics.cpp,
test_embed.cpp, acceptance_main.cpp).  Run from the repo root:

    make -C oracle && python oracle/make_golden.py

The fixtures travel with the repo, so GPU boxes (which have no
/root/reference) can check the CUDA path against the reference's outputs.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import gini_oracle as O  # noqa: E402  (input generators only)
from oracle import ref_lib as R  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def pad_rows(rows, fill=np.nan):
    m = max(len(r) for r in rows)
    out = np.full((len(rows), m), fill)
    for k, r in enumerate(rows):
        out[k, : len(r)] = r
    return out


def midrank_cases():
    # test_metrics.cpp:121-149 -- Rng(2024), 300 vectors with ties, d in [1,12]
    rng = O.Rng(2024)
    vecs = []
    for _ in range(300):
        d = 1 + rng.uniform_below(12)
        vecs.append(O.random_vector_with_ties(rng, d))
    # plus larger heavy-tie vectors (signed zeros, lattice values), p up to 1100
    g = np.random.default_rng(11)
    for d in (31, 32, 33, 64, 127, 128, 200, 784, 1025):
        v = g.integers(-3, 4, size=d).astype(np.float64)
        v[g.random(d) < 0.3] = -0.0
        vecs.append(v)
    ranks = [R.midrank(v) for v in vecs]
    save("midrank", values=pad_rows(vecs), ranks=pad_rows(ranks), lengths=np.array([len(v) for v in vecs]))


def distance_cases():
    # test_metrics.cpp:281-300 inputs (Rng(404)) at nu in {1.5, 2, 3, 5}, and
    # the nu=2 reduction inputs of acceptance C3 (Rng(333), with ties).
    xs, ys, nus, fwd, dist = [], [], [], [], []
    rng = O.Rng(404)
    for nu in (1.5, 2.0, 3.0, 5.0):
        for _ in range(200):
            d = 2 + rng.uniform_below(8)
            x = O.random_vector(rng, d, 10.0)
            y = O.random_vector(rng, d, 10.0)
            _ = O.random_vector(rng, d, 10.0)
            xs.append(x), ys.append(y), nus.append(nu)
    rng = O.Rng(333)
    for _ in range(200):
        d = 1 + rng.uniform_below(10)
        rv = O.random_vector_with_ties
        xs.append(rv(rng, d)), ys.append(rv(rng, d)), nus.append(2.0)
    for x, y, nu in zip(xs, ys, nus):
        fwd.append(R.gen_gini_directed(x, y, nu))
        dist.append(R.gen_gini_distance(x, y, nu))
    save("distance", x=pad_rows(xs), y=pad_rows(ys), lengths=np.array([len(x) for x in xs]), nu=np.array(nus),
         directed=np.array(fwd), distance=np.array(dist))


def pairwise_cases():
    # test_metrics.cpp:318-348 inputs, C1 (n=200, p=8, N(0,1)) and a tie-heavy
    # case with duplicated rows and a constant column.
    cases = {}
    rng = O.Rng(888)
    cases["t888"] = (O.random_matrix(rng, 5, 3, 4.0), [2.7])
    rng = O.Rng(321)
    cases["t321"] = (O.random_matrix(rng, 24, 4, 2.0), [1.8])
    rng = O.Rng(1)
    X = np.array([[rng.normal() for _ in range(8)] for _ in range(200)])
    cases["c1"] = (X, [2.0, 1.5, 3.0])
    g = np.random.default_rng(5)
    T = g.integers(0, 4, size=(64, 40)).astype(np.float64)
    T[7] = T[3]
    T[:, 5] = 1.0
    T[g.random(T.shape) < 0.5] = 0.0
    cases["ties"] = (T, [1.1, 2.0, 7.5])
    arrays = {}
    for name, (X, nus) in cases.items():
        arrays[f"{name}_X"] = X
        arrays[f"{name}_nus"] = np.array(nus)
        for k, nu in enumerate(nus):
            D = R.pairwise_matrix(X, nu)
            iu = np.triu_indices(X.shape[0], 1)
            arrays[f"{name}_D{k}"] = D[iu]
        arrays[f"{name}_E"] = R.pairwise_matrix(X, None)[np.triu_indices(X.shape[0], 1)]
    save("pairwise", **arrays)


def random_dissimilarity(rng, n, offset=0.1, sqrt=True):
    pts = O.random_matrix(rng, n, 5, 2.0)
    D = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1, n):
            v = np.linalg.norm(pts[i] - pts[j])
            v = (np.sqrt(v) if sqrt else v) + offset
            D[i, j] = D[j, i] = v
    return D


def stress_cases():
    # Fits on the C1 shape (n=200, p=8, N(0,1), nu=2, q=2): classical init
    # (the reference's minimize_stress exactly), every kind, 500 iterations,
    # rel_tol=1e-300 so every run is a fixed-length trajectory.
    rng = O.Rng(1)
    X = np.array([[rng.normal() for _ in range(8)] for _ in range(200)])
    D = R.pairwise_matrix(X, 2.0)
    arrays = {"c1_X": X, "c1_D": D[np.triu_indices(200, 1)]}
    cm = R.classical_mds(D, 2)
    arrays.update(cmds_coords=cm["coords"], cmds_eig=cm["eigenvalues"], cmds_clamped_mass=cm["clamped_mass"],
                  cmds_clamped_count=cm["clamped_count"], cmds_stress=cm["stress"])
    for kind in ("kruskal", "sammon", "smacof", "huber"):
        hd = 0.5 * np.median(D[np.triu_indices(200, 1)]) if kind == "huber" else None
        e = R.minimize_stress(D, 2, kind, huber_delta=hd, max_iters=500, rel_tol=1e-300)
        arrays[f"{kind}_history"] = np.array(e["stress_history"])
        arrays[f"{kind}_coords"] = e["coords"]
        arrays[f"{kind}_iterations"] = e["iterations"]
        arrays[f"{kind}_huber_delta"] = e["huber_delta"]
        if kind != "smacof":
            Y = cm["coords"]
            arrays[f"{kind}_loss0"] = R.stress_loss(kind, Y, D, hd)
            arrays[f"{kind}_grad0"] = R.stress_gradient(kind, Y, D, hd)
    # default-config fits on random dissimilarities (test_embed.cpp:301-314 style)
    rng = O.Rng(55)
    for kind in ("kruskal", "huber", "sammon", "smacof"):
        Dk = random_dissimilarity(rng, 15)
        hd = 0.5 if kind == "huber" else None
        e = R.minimize_stress(Dk, 2, kind, huber_delta=hd)
        arrays[f"rd_{kind}_D"] = Dk
        arrays[f"rd_{kind}_history"] = np.array(e["stress_history"])
        arrays[f"rd_{kind}_iterations"] = e["iterations"]
        arrays[f"rd_{kind}_converged"] = int(e["converged"])
        arrays[f"rd_{kind}_stress"] = e["stress"]
    # Huber auto-delta (test_embed.cpp:333-341)
    rng = O.Rng(3)
    Dh = random_dissimilarity(rng, 12)
    e = R.minimize_stress(Dh, 2, "huber")
    arrays.update(auto_D=Dh, auto_huber_delta=e["huber_delta"], auto_stress=e["stress"])
    save("stress", **arrays)


def tune_cases():
    arrays = {}
    rng = O.Rng(3)
    X = O.random_matrix(rng, 24, 3, 1.5)
    grid = O.nugrid_linspace(1.5, 4.0, 6)
    r = R.tune_nu(X, 2, grid, 3, "classical", 42)
    arrays.update(t_X=X, t_grid=np.array(grid), t_mean=np.array(r["mean_stress"]), t_nu_star=r["nu_star"],
                  t_coords=r["coords"])
    # p=6 features so the grid values are genuinely separated (with p=3 every
    # D_nu is a multiple of D_2 and the argmin is decided by round-off).
    rng = O.Rng(12)
    X = O.random_matrix(rng, 30, 6, 2.0)
    X[:, 2] = np.exp(X[:, 2] * 2.0)
    r = R.tune_nu(X, 2, [1.2, 2.0, 3.5, 6.0], 3, "classical", 4)
    arrays.update(u_X=X, u_grid=np.array([1.2, 2.0, 3.5, 6.0]), u_mean=np.array(r["mean_stress"]),
                  u_nu_star=r["nu_star"], u_coords=r["coords"])
    rng = O.Rng(6)
    X = O.random_matrix(rng, 16, 3, 1.0)
    r = R.tune_nu(X, 2, [1.8, 3.0], 2, "smacof", 11)
    arrays.update(s_X=X, s_grid=np.array([1.8, 3.0]), s_mean=np.array(r["mean_stress"]), s_nu_star=r["nu_star"])
    rng = O.Rng(8)
    X = O.random_matrix(rng, 16, 3, 2.0)
    grid = O.nugrid_linspace(1.4, 4.0, 5)
    a = R.alternating_tune(X, 2, 3, grid, 17)
    arrays.update(a_X=X, a_grid=np.array(grid), a_path=np.array(a["nu_path"]), a_nu_star=a["nu_star"],
                  a_stress=a["stress"], a_coords=a["coords"])
    save("tune", **arrays)


if __name__ == "__main__":
    if R.load() is None:
        sys.exit("oracle/_ref/libginimds_ref.so missing: run `make -C oracle` first")
    midrank_cases()
    distance_cases()
    pairwise_cases()
    stress_cases()
    tune_cases()
