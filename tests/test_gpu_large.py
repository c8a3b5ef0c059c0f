"""CUDA path vs the REFERENCE at BASELINE.json's shapes (golden fixtures from
oracle/make_golden_large.py: the unmodified reference's pairwise_matrix,
gen_gini_distance, midrank, minimize_stress and -- for seeded starts, SURVEY F4 --
its own gradient_descent loop entered with Y0).

Contract (BASELINE.json north_star): ranks bit-exact; D within 1e-6 relative,
max-normalised; the per-iteration stress trajectory within 1e-4 relative for the
first 50 iterations; the final stress within 1%.  The fits below run the path
bench.py measures: fp32 packed-triangle storage of D above the small-fit size
(TMA passes, difference passes in the sub-resolution phase, device-resident
gd_step loop).
"""
import numpy as np
import pytest

from oracle import synth as S
from paper_2605_25124_b200 import gmds as G

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

D_TOL = 1e-6  # relative, max-normalised
TRAJ = 1e-4  # relative, first 50 iterations
FINAL = 0.01  # final stress


def _device_X(X):
    return torch.from_numpy(np.ascontiguousarray(X)).cuda()


def _full_f32(dX, n, p, nus):
    out = torch.zeros((len(nus), n, n), dtype=torch.float32, device="cuda")
    G.pairwise_gini_device(dX.data_ptr(), G.F32, n, p, nus, G.F32, False, out.data_ptr())
    torch.cuda.synchronize()
    return out


def _take(Dfull, I, J):
    ii = torch.from_numpy(I).cuda()
    jj = torch.from_numpy(J).cuda()
    return Dfull[ii, jj].double().cpu().numpy(), Dfull[jj, ii].double().cpu().numpy()


def _traj_check(h, ref_h, iters_ref, iters):
    h, ref_h = np.asarray(h), np.asarray(ref_h)
    assert iters == iters_ref
    assert h.shape == ref_h.shape
    m = min(51, h.size)
    rel = np.abs(h[:m] - ref_h[:m]) / ref_h[:m]
    assert np.max(rel) <= TRAJ, f"trajectory deviates by {np.max(rel):.3e} at iteration {int(np.argmax(rel))}"
    assert abs(h[-1] - ref_h[-1]) <= FINAL * ref_h[-1]
    return float(np.max(rel))


def _seeded_fit(g, storage):
    n, p = int(g["fit_n"]), int(g["fit_p"])
    X = S.image_like(n, p, int(g["fit_xseed"]))
    dX = _device_X(X)
    Dm = G.dmat_gini_device(dX.data_ptr(), G.F32, n, p, 2.0, storage)
    Y0 = np.random.default_rng(int(g["fit_yseed"])).normal(0.0, 0.1, (n, 2))
    iters = int(g["fit_iterations"])
    e = G.minimize_stress(Dm, 2, "kruskal", max_iters=iters, rel_tol=1e-300, Y0=Y0)
    return e, Dm


@pytest.mark.parametrize("name", ["large_img2600", "large_c3"])
@pytest.mark.parametrize("storage", [G.F32, G.F64])
def test_seeded_image_trajectory_vs_reference(golden, name, storage):
    # image-like data, Kruskal from Y0 ~ N(0, 0.1^2): the reference's first ~25 iterations
    # change the loss by 1e-13..1e-7 relative (below fp32 storage's resolution) -- the
    # regime of bench.py's fit; n > 2048, so the tiled fp32 TMA passes run (F32)
    g = golden(name)
    e, _ = _seeded_fit(g, storage)
    _traj_check(e["stress_history"], g["fit_history"], int(g["fit_iterations"]), e["iterations"])
    ref_c = g["fit_coords"]
    assert np.max(np.abs(e["coords"] - ref_c)) <= 1e-3 * np.max(np.abs(ref_c))


def test_c3_classical_init_2000_iterations(golden):
    # C3 parity mode: the reference's own minimize_stress (classical init, embed.cpp:495) for
    # 2000 Kruskal iterations; the engine's classical init at n = 5000 is the top-q subspace solver
    g = golden("large_c3")
    n, p = 5000, 784
    X = S.image_like(n, p, 3)
    dX = _device_X(X)
    ref_h = g["cls_history"]
    for storage in (G.F64, G.F32):
        Dm = G.dmat_gini_device(dX.data_ptr(), G.F32, n, p, 2.0, storage)
        e = G.minimize_stress(Dm, 2, "kruskal", max_iters=2000, rel_tol=1e-300)
        _traj_check(e["stress_history"], ref_h, int(g["cls_iterations"]), e["iterations"])
        Dm.free()


def test_c3_distance_samples(golden):
    g = golden("large_c3")
    n, p = 5000, 784
    X = S.image_like(n, p, 3)
    Dfull = _full_f32(_device_X(X), n, p, [2.0])[0]
    I, J = S.sample_pairs(n, int(g["npairs"]), int(g["pair_seed"]))
    a, b = _take(Dfull, I, J)
    scale = float(g["D_max"])
    assert np.max(np.abs(a - g["D_sample"])) <= D_TOL * scale
    assert np.array_equal(a, b)  # both triangles written, symmetric
    rows = Dfull.double().sum(dim=1).cpu().numpy()
    assert np.max(np.abs(rows - g["D_rowsum"])) <= D_TOL * scale * n


def test_c2_distances_and_fits(golden):
    # C2: 8 nu in [1.1, 8] (F5), mixture data with 5% x10 outliers; all 8 matrices from one
    # launch; per nu the Kruskal fit from the classical init, 1000 iterations
    g = golden("large_c2")
    X = S.mixture_contaminated()
    grid = list(g["grid"])
    n = X.shape[0]
    Ds = G.pairwise_gini(X, grid)
    I, J = S.sample_pairs(n, int(g["npairs"]), int(g["pair_seed"]))
    for k, nu in enumerate(grid):
        scale = np.max(Ds[k])
        assert np.max(np.abs(Ds[k][I, J] - g["D_sample"][k])) <= D_TOL * scale
        assert np.max(np.abs(Ds[k].sum(axis=1) - g["D_rowsum"][k])) <= D_TOL * scale * n
    stresses = []
    for k, nu in enumerate(grid):
        Dm = G.dmat_from_host(Ds[k])
        e = G.minimize_stress(Dm, 2, "kruskal", max_iters=1000, rel_tol=1e-300)
        ref_h = g["history"][k]
        ref_h = ref_h[~np.isnan(ref_h)]
        _traj_check(e["stress_history"], ref_h, int(g["iterations"][k]), e["iterations"])
        stresses.append(e["stress"])
    assert int(np.argmin(stresses)) == int(np.argmin(g["stress"]))


def _rank_fp_check(X, g):
    n, p = X.shape
    Ir, Jr = S.sample_pairs(n, int(g["nrank"]), int(g["rank_seed"]))
    R = G.pair_midranks(X, Ir, Jr)
    fp = S.rank_fingerprints(R, S.rank_weights(p, int(g["rank_w_seed"]) if "rank_w_seed" in g else 99))
    assert np.array_equal(fp, g["rank_fp"])
    assert np.all(R * 2 == np.rint(R * 2))  # half-integers, exactly


def test_c4_distance_samples_and_ranks(golden):
    # C4: n = 20000, p = 128 log-normal, 1% duplicated rows, 4 nu from one launch; 1e6 sampled
    # entries (every duplicate pair included: exact zeros), 1e4 per-pair rank fingerprints
    g = golden("large_c4")
    X, dup, src = S.lognormal_dup()
    n, p = X.shape
    nus = list(g["nus"])
    Dfull = _full_f32(_device_X(X), n, p, nus)
    I, J = S.sample_pairs(n, int(g["npairs"]) - int(np.sum(dup != src)), int(g["pair_seed"]), extra=(dup, src))
    assert I.size == int(g["npairs"])
    for k in range(len(nus)):
        a, b = _take(Dfull[k], I, J)
        ref = g["D_sample"][k].astype(np.float64)
        assert np.max(np.abs(a - ref)) <= D_TOL * float(Dfull[k].max())
        assert np.array_equal(a, b)
        same = np.all(X[I] == X[J], axis=1)
        assert same.sum() > 0 and np.all(a[same] == 0.0)
    _rank_fp_check(X, g)


def test_metric_distance_samples_and_ranks(golden):
    # the BASELINE metric shape (bench.py's workload): 1e6 sampled entries of the full
    # 20000 x 20000 matrix and 1e4 per-pair rank fingerprints vs the reference
    g = golden("large_metric")
    n, p = 20000, 784
    X = S.image_like(n, p, 2605)
    Dfull = _full_f32(_device_X(X), n, p, [2.0])[0]
    I, J = S.sample_pairs(n, int(g["npairs"]), int(g["pair_seed"]))
    a, b = _take(Dfull, I, J)
    ref = g["D_sample"].astype(np.float64)
    assert np.max(np.abs(a - ref)) <= D_TOL * float(g["D_max"])
    assert np.array_equal(a, b)
    total = float(Dfull.double().sum())
    assert abs(total - float(g["D_sum"])) <= 1e-6 * float(g["D_sum"])
    del Dfull
    torch.cuda.empty_cache()
    _rank_fp_check(X, g)


def test_metric_fit_trajectory_vs_reference(golden):
    # bench.py's own stress fit (fp32 packed storage, Y0 = default_rng(2605) N(0, 0.1^2),
    # 50 Kruskal iterations) against the reference's gradient_descent on the reference D
    g = golden("large_metric")
    e, Dm = _seeded_fit(g, G.F32)
    _traj_check(e["stress_history"], g["fit_history"], int(g["fit_iterations"]), e["iterations"])
    assert abs(G.kruskal_stress(e["coords"], Dm) - e["stress"]) <= 1e-6 * e["stress"]


@pytest.mark.parametrize("q", [1, 2, 3])
@pytest.mark.parametrize("storage", [G.F64, G.F32])
def test_classical_topq_vs_reference(golden, q, storage):
    # the top-q classical init without a dense B (Lanczos over the packed
    # triangle, hand-written kernels) against the reference's own classical_mds (dense
    # SelfAdjointEigenSolver, embed.cpp:415-460) at n = 1500
    g = golden("large_cls1500")
    X = S.image_like(1500, 784, 9)
    dX = _device_X(X)
    Dm = G.dmat_gini_device(dX.data_ptr(), G.F32, 1500, 784, 2.0, storage)
    t = G.classical_mds_topq(Dm, q, tol=1e-12)
    ev, ref_c = g[f"eig{q}"], g[f"coords{q}"]
    rel = 1e-9 if storage == G.F64 else 1e-6  # fp32 storage rounds D (and so B) at 6e-8
    assert np.allclose(t["eigenvalues"], ev, rtol=rel, atol=0)
    assert np.max(np.abs(t["coords"] - ref_c)) <= (1e-7 if storage == G.F64 else 1e-4) * np.max(np.abs(ref_c))
    assert t["iterations"] < 400
