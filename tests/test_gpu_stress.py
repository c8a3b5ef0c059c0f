"""GPU parity: stress losses / gradients, classical MDS, minimize_stress
trajectories and the nu-tuning callers vs the oracle and the reference's
golden outputs.  Contract (north_star): stress trajectory within 1e-4
relative for the first 50 iterations, final stress within 1%."""
import math

import numpy as np
import pytest

from oracle import gini_oracle as O

pytestmark = pytest.mark.gpu
G = pytest.importorskip("paper_2605_25124_b200.gmds")

TRAJ = 1e-4
FINAL = 1e-2


def c1(golden):
    g = golden("stress")
    n = 200
    D = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    D[iu] = g["c1_D"]
    return g, D + D.T


def rand_dissim(seed, n, dim=5):
    rng = np.random.default_rng(seed)
    P = rng.uniform(-2, 2, (n, dim))
    D = np.sqrt(np.linalg.norm(P[:, None] - P[None], axis=2)) + 0.1
    np.fill_diagonal(D, 0.0)
    return D


@pytest.mark.parametrize("kind", ["kruskal", "huber", "sammon", "smacof"])
@pytest.mark.parametrize("q", [1, 2, 3, 5])
def test_loss_and_gradient(kind, q):
    D = rand_dissim(q, 150)
    rng = np.random.default_rng(10 + q)
    Y = rng.standard_normal((150, q))
    hd = 0.7 if kind == "huber" else None
    Dm = G.dmat_from_host(D)
    assert G.stress_loss(kind, Y, Dm, hd) == pytest.approx(O.stress_loss(kind, Y, D, hd), rel=1e-12)
    g = G.stress_gradient(kind, Y, Dm, hd)
    gr = O.stress_gradient(kind, Y, D, hd)
    assert np.max(np.abs(g - gr)) <= 1e-11 * np.max(np.abs(gr))


def test_kruskal_and_golden_gradients(golden):
    g, D = c1(golden)
    Y = g["cmds_coords"]
    assert G.kruskal_stress(Y, D) == pytest.approx(float(g["cmds_stress"]), rel=1e-12)
    for kind in ("kruskal", "sammon", "huber"):
        hd = float(g["huber_history"][0] * 0 + g["huber_huber_delta"]) if kind == "huber" else None
        assert G.stress_loss(kind, Y, D, hd) == pytest.approx(float(g[f"{kind}_loss0"]), rel=1e-12)
        gg = G.stress_gradient(kind, Y, D, hd)
        assert np.max(np.abs(gg - g[f"{kind}_grad0"])) <= 1e-10 * np.max(np.abs(g[f"{kind}_grad0"]))


def test_fp32_storage_loss():
    D = rand_dissim(3, 300)
    Y = np.random.default_rng(1).standard_normal((300, 2))
    assert G.kruskal_stress(Y, G.dmat_from_host(D, G.F32)) == pytest.approx(O.kruskal_stress(Y, D), rel=1e-6)


def test_classical_mds_golden(golden):
    g, D = c1(golden)
    r = G.classical_mds(D, 2)
    assert np.allclose(r["coords"], g["cmds_coords"], atol=1e-9)
    assert np.allclose(r["eigenvalues"], g["cmds_eig"], rtol=1e-11)
    assert r["clamped_mass"] == pytest.approx(float(g["cmds_clamped_mass"]), rel=1e-9)
    assert r["stress"] == pytest.approx(float(g["cmds_stress"]), rel=1e-10)


def test_classical_known_answers():
    # test_embed.cpp:90-98: two points at distance 2 -> +1 / -1, eigenvalue 2
    r = G.classical_mds(np.array([[0.0, 2.0], [2.0, 0.0]]), 1)
    assert r["coords"][0, 0] == pytest.approx(1.0, rel=1e-12) and r["coords"][1, 0] == pytest.approx(-1.0, rel=1e-12)
    assert r["eigenvalues"][0] == pytest.approx(2.0, rel=1e-12)
    sq = G.pairwise_matrix(np.array([[0, 0], [1, 0], [1, 1], [0, 1.0]]), None)
    assert G.classical_mds(sq, 2)["stress"] < 1e-8
    with pytest.raises(G.InvalidInput):
        G.classical_mds(sq, 4)
    with pytest.raises(G.InvalidInput):
        G.classical_mds(sq, 0)


def test_classical_clamped_indefinite():
    # test_embed.cpp:100-122: a Gini metric whose Gram matrix is indefinite
    for seed in range(64):
        rng = O.Rng(seed)
        X = O.random_matrix(rng, 8, 3, 5.0)
        D = O.pairwise_matrix(X, 3.0)
        lam = np.linalg.eigvalsh(O.double_center(D * D))
        if lam[0] < -1e-9 * np.max(np.abs(lam)):
            r = G.classical_mds(D, 7)
            ref = O.classical_mds(D, 7)
            assert r["clamped_count"] == ref.clamped_count > 0
            assert r["clamped_mass"] == pytest.approx(ref.clamped_mass, rel=1e-9)
            assert r["eigenvalues"][6] < 0 and np.max(np.abs(r["coords"][:, 6])) == 0.0
            assert r["stress"] == pytest.approx(ref.stress, rel=1e-9)
            return
    pytest.fail("no indefinite instance found")


@pytest.mark.parametrize("kind", ["kruskal", "sammon", "smacof", "huber"])
def test_minimize_stress_c1_golden(golden, kind):
    # config 1 (n=200, p=8, nu=2, q=2), classical init, 500 iterations, vs the reference run
    g, D = c1(golden)
    hd = float(g["huber_huber_delta"]) if kind == "huber" else None
    e = G.minimize_stress(D, 2, kind, huber_delta=hd, max_iters=500, rel_tol=1e-300)
    ref = g[f"{kind}_history"]
    h = np.array(e["stress_history"])
    k = min(51, len(ref))
    assert len(h) >= k
    assert np.max(np.abs(h[:k] - ref[:k]) / ref[:k]) <= TRAJ
    assert abs(e["stress"] - ref[-1]) <= FINAL * ref[-1]
    assert e["iterations"] == int(g[f"{kind}_iterations"])


@pytest.mark.parametrize("kind", ["kruskal", "sammon", "smacof"])
def test_minimize_stress_fp32_storage(golden, kind):
    g, D = c1(golden)
    e = G.minimize_stress(D, 2, kind, max_iters=200, rel_tol=1e-300, storage=G.F32)
    ref = g[f"{kind}_history"]
    h = np.array(e["stress_history"])
    assert np.max(np.abs(h[:51] - ref[:51]) / ref[:51]) <= TRAJ
    assert abs(e["stress"] - ref[200]) <= FINAL * ref[200]


@pytest.mark.parametrize("kind", ["kruskal", "sammon", "smacof"])
def test_minimize_stress_seeded_init(kind):
    # config 1's seeded N(0, 1e-2) init vs the oracle fed the same Y0
    rng = np.random.default_rng(1)
    X = rng.standard_normal((120, 8))
    D = O.pairwise_matrix(X, 2.0)
    Y0 = rng.normal(0.0, 0.1, (120, 2))
    e = G.minimize_stress(D, 2, kind, max_iters=60, rel_tol=1e-300, Y0=Y0)
    r = O.minimize_stress(D, 2, kind, max_iters=60, rel_tol=1e-300, Y0=Y0)
    h, hr = np.array(e["stress_history"]), np.array(r.stress_history)
    assert len(h) == len(hr)
    assert np.max(np.abs(h[:51] - hr[:51]) / hr[:51]) <= TRAJ


@pytest.mark.parametrize("kind", ["kruskal", "huber", "sammon", "smacof"])
def test_default_config_fits_golden(golden, kind):
    g = golden("stress")
    D = g[f"rd_{kind}_D"]
    e = G.minimize_stress(D, 2, kind, huber_delta=(0.5 if kind == "huber" else None))
    assert e["iterations"] == int(g[f"rd_{kind}_iterations"])
    assert e["converged"] == bool(g[f"rd_{kind}_converged"])
    assert e["stress"] == pytest.approx(float(g[f"rd_{kind}_stress"]), rel=1e-6)


def test_huber_auto_delta(golden):
    g = golden("stress")
    e = G.minimize_stress(g["auto_D"], 2, "huber")
    assert e["huber_delta"] == pytest.approx(float(g["auto_huber_delta"]), rel=1e-15)
    assert e["stress"] == pytest.approx(float(g["auto_stress"]), rel=1e-6)


def test_unit_square_all_kinds():
    # test_embed.cpp:272-284
    sq = G.pairwise_matrix(np.array([[0, 0], [1, 0], [1, 1], [0, 1.0]]), None)
    for kind in ("kruskal", "huber", "sammon", "smacof"):
        e = G.minimize_stress(sq, 2, kind, huber_delta=(1.0 if kind == "huber" else None))
        assert e["stress"] < 1e-6 and e["converged"]


def test_smacof_monotone_and_weighted():
    for seed in range(5):
        D = rand_dissim(100 + seed, 20)
        h = G.minimize_stress(D, 2, "smacof")["stress_history"]
        assert all(h[t] <= h[t - 1] * (1 + 1e-12) + 1e-15 for t in range(1, len(h)))
    D = rand_dissim(7, 25)
    W = np.random.default_rng(3).uniform(0.5, 2.0, (25, 25))
    W = (W + W.T) / 2
    e = G.minimize_stress(D, 2, "smacof", weights=W, max_iters=40, rel_tol=1e-300)
    r = O.minimize_stress(D, 2, "smacof", weights=W, max_iters=40, rel_tol=1e-300)
    assert np.max(np.abs(np.array(e["stress_history"]) - r.stress_history) / r.stress_history[0]) <= 1e-8


def test_stress_error_contract():
    D = np.array([[0, 0, 1], [0, 0, 1], [1, 1, 0.0]])
    with pytest.raises(G.DegenerateInput):
        G.stress_loss("sammon", np.zeros((3, 2)), D)
    with pytest.raises(G.InvalidConfig):
        G.stress_loss("huber", np.zeros((3, 2)), D)
    with pytest.raises(G.InvalidConfig):
        G.stress_loss("huber", np.zeros((3, 2)), D, huber_delta=-1.0)
    with pytest.raises(G.DegenerateInput):
        G.kruskal_stress(np.zeros((2, 1)), np.zeros((2, 2)))
    with pytest.raises(G.InvalidConfig):
        G.minimize_stress(D, 2, "kruskal", max_iters=0)
    with pytest.raises(G.InvalidConfig):
        G.minimize_stress(D, 2, "kruskal", rel_tol=0.0)
    with pytest.raises(G.InvalidInput):
        G.dmat_from_host(np.array([[0.0, 1.0], [2.0, 0.0]]))
    Y = np.zeros((3, 2))
    Y[0, 0] = np.nan
    with pytest.raises(G.InvalidInput):
        G.kruskal_stress(Y, D)


def test_nonconvergence_flag():
    # test_embed.cpp:343-358
    D = rand_dissim(21, 14)
    a = G.minimize_stress(D, 2, "sammon")
    b = G.minimize_stress(D, 2, "sammon")
    assert np.array_equal(a["coords"], b["coords"]) and a["stress"] == b["stress"]  # deterministic
    t = G.minimize_stress(D, 2, "sammon", max_iters=1, rel_tol=1e-14)
    assert not t["converged"] and t["iterations"] == 1


def test_tune_golden(golden):
    g = golden("tune")
    r = G.tune_nu(g["u_X"], 2, g["u_grid"], 3, "classical", 4)
    assert np.allclose(r["mean_stress"], g["u_mean"], rtol=1e-9)
    assert r["nu_star"] == float(g["u_nu_star"])
    assert np.allclose(r["coords"], g["u_coords"], atol=1e-8)
    r = G.tune_nu(g["s_X"], 2, g["s_grid"], 2, "smacof", 11)
    assert np.allclose(r["mean_stress"], g["s_mean"], rtol=1e-6)
    a = G.alternating_tune(g["a_X"], 2, 3, g["a_grid"], 17)
    assert a["nu_path"] == list(g["a_path"]) and a["nu_star"] == float(g["a_nu_star"])
    assert a["stress"] == pytest.approx(float(g["a_stress"]), rel=1e-6)


def test_tune_contract():
    X = np.full((12, 3), 4.2)
    r = G.tune_nu(X, 1, O.nugrid_linspace(1.5, 3.5, 4), 3, "classical", 5)
    assert r["nu_star"] == 1.5 and all(s == 0.0 for s in r["mean_stress"])
    X = np.random.default_rng(5).uniform(-1, 1, (9, 3))
    with pytest.raises(G.InvalidConfig):
        G.tune_nu(X, 3, [2.0], 3)
    with pytest.raises(G.InvalidConfig):
        G.tune_nu(X, 2, [2.0], 0)
    with pytest.raises(G.InvalidConfig):
        G.tune_nu(X, 2, [2.0], 10)
    with pytest.raises(G.InvalidConfig):
        G.tune_nu(X, 2, [2.0, 2.0], 2)
    with pytest.raises(G.InvalidConfig):
        G.alternating_tune(X, 2, 0, [2.0])
    # one fold + singleton grid == direct pipeline (test_tune.cpp:36-46)
    X = O.random_matrix(O.Rng(2), 15, 4, 2.0)
    r = G.tune_nu(X, 2, [2.4], 1, "classical", 9)
    D = G.pairwise_matrix(X, 2.4)
    direct = G.classical_mds(D, 2)
    assert r["mean_stress"][0] == pytest.approx(G.kruskal_stress(direct["coords"], D), rel=1e-12)
    assert np.allclose(r["coords"], direct["coords"], atol=1e-12)


@pytest.mark.parametrize("kind", ["kruskal", "huber", "sammon", "smacof"])
@pytest.mark.parametrize("n,q", [(2, 1), (37, 3), (300, 2), (1024, 4), (2048, 2)])
def test_small_fit_matches_pass_engine(monkeypatch, kind, n, q):
    # n <= 2048, q <= 4 fits run as one cooperative persistent kernel (small_fit.cu); the
    # multi-kernel pass engine (GMDS_NO_SMALL_FIT) is the same algorithm
    D = rand_dissim(n + q, n)
    hd = 0.6 if kind == "huber" else None
    Y0 = np.random.default_rng(n).normal(0.0, 0.1, (n, q))
    e = G.minimize_stress(D, q, kind, huber_delta=hd, max_iters=120, rel_tol=1e-300, Y0=Y0)
    monkeypatch.setenv("GMDS_NO_SMALL_FIT", "1")
    r = G.minimize_stress(D, q, kind, huber_delta=hd, max_iters=120, rel_tol=1e-300, Y0=Y0)
    h, hr = np.array(e["stress_history"]), np.array(r["stress_history"])
    k = min(len(h), len(hr), 51)
    assert k >= min(len(hr), 2)
    assert np.max(np.abs(h[:k] - hr[:k]) / np.maximum(hr[:k], 1e-8 * hr[0])) <= 1e-9
    assert abs(e["stress"] - r["stress"]) <= FINAL * max(r["stress"], 1e-8 * hr[0])
    if n <= 300:
        o = O.minimize_stress(D, q, kind, huber_delta=hd, max_iters=60, rel_tol=1e-300, Y0=Y0)
        ho = np.array(o.stress_history)
        k = min(len(h), len(ho), 51)
        assert np.max(np.abs(h[:k] - ho[:k]) / np.maximum(ho[:k], 1e-8 * ho[0])) <= TRAJ


@pytest.mark.parametrize("q", [1, 2, 3])
def test_classical_topq_matches_dense(q):
    # top-q subspace iteration == the dense eigensolver's top q
    rng = np.random.default_rng(7 + q)
    X = rng.standard_normal((700, 12)) * np.linspace(3.0, 0.5, 12)
    D = G.pairwise_matrix(X, 2.0)
    Dm = G.dmat_from_host(D)
    r = G.classical_mds(Dm, q)
    t = G.classical_mds_topq(Dm, q, tol=1e-12)
    assert t["iterations"] >= 1
    assert np.allclose(t["eigenvalues"], r["eigenvalues"], rtol=1e-10)
    assert np.max(np.abs(t["coords"] - r["coords"])) <= 1e-7 * np.max(np.abs(r["coords"]))
    assert t["clamped_count"] == r["clamped_count"]


def test_classical_topq_full_subspace_indefinite():
    # k == n (tiny n): the subspace is the whole space, clamped eigenvalues included
    for seed in range(64):
        rng = O.Rng(seed)
        X = O.random_matrix(rng, 8, 3, 5.0)
        D = O.pairwise_matrix(X, 3.0)
        lam = np.linalg.eigvalsh(O.double_center(D * D))
        if lam[0] < -1e-9 * np.max(np.abs(lam)):
            r = G.classical_mds(D, 7)
            t = G.classical_mds_topq(D, 7, tol=1e-13)
            # B's exact null eigenvalue (J 1 = 0) has a round-off sign in both solvers:
            # count clamps only for eigenvalues clearly below zero
            big = 1e-9 * np.max(np.abs(lam))
            assert np.sum(t["eigenvalues"] < -big) == np.sum(r["eigenvalues"] < -big) > 0
            assert np.allclose(t["eigenvalues"], r["eigenvalues"], rtol=1e-8, atol=1e-9 * np.max(np.abs(lam)))
            assert np.max(np.abs(t["coords"] - r["coords"])) <= 1e-6 * np.max(np.abs(r["coords"]))
            return
    pytest.fail("no indefinite instance found")


def test_classical_topq_errors():
    D = rand_dissim(1, 50)
    with pytest.raises(G.InvalidInput):
        G.classical_mds_topq(D, 0)
    with pytest.raises(G.InvalidConfig):
        G.classical_mds_topq(D, 2, tol=0.0)
    with pytest.raises(G.NumericFailure):
        G.classical_mds_topq(D, 2, tol=1e-300, max_iters=2)


def test_minimize_stress_subspace_classical_init(monkeypatch):
    # the classical init of minimize_stress switches to the subspace solver above
    # n = 4096; both inits must give the same trajectory
    rng = np.random.default_rng(3)
    X = rng.standard_normal((900, 10)) * np.linspace(2.0, 0.5, 10)
    D = G.pairwise_matrix(X, 2.0)
    monkeypatch.setenv("GMDS_CLASSICAL", "dense")
    a = G.minimize_stress(D, 2, "kruskal", max_iters=60, rel_tol=1e-300)
    monkeypatch.setenv("GMDS_CLASSICAL", "subspace")
    b = G.minimize_stress(D, 2, "kruskal", max_iters=60, rel_tol=1e-300)
    ha, hb = np.array(a["stress_history"]), np.array(b["stress_history"])
    assert len(ha) == len(hb)
    assert np.max(np.abs(ha - hb) / ha) <= 1e-8


@pytest.mark.parametrize("kind,q", [("kruskal", 2), ("kruskal", 3), ("huber", 2), ("sammon", 1)])
def test_speculative_trial_gradient_identical(monkeypatch, kind, q):
    # fp32 storage above the small-fit size: the trial pass also carries the
    # gradient of the predicted acceptance; the arithmetic per trial point is the
    # same as separate loss / gradient passes, so trajectories are bit-identical
    monkeypatch.setenv("GMDS_NO_TINY", "1")  # the tiny phase's single pass: test_tiny_phase_one_pass
    rng = np.random.default_rng(11)
    n = 2600
    X = rng.standard_normal((n, 6)) * np.linspace(2.0, 0.5, 6)
    D = G.pairwise_matrix(X, 2.0)
    Y0 = rng.normal(0.0, 0.1, (n, q))
    hd = 0.5 * float(np.median(D)) if kind == "huber" else None
    a = G.minimize_stress(D, q, kind, huber_delta=hd, max_iters=40, rel_tol=1e-300, Y0=Y0, storage=G.F32)
    monkeypatch.setenv("GMDS_NO_SPECULATION", "1")
    b = G.minimize_stress(D, q, kind, huber_delta=hd, max_iters=40, rel_tol=1e-300, Y0=Y0, storage=G.F32)
    assert np.array_equal(np.array(a["stress_history"]), np.array(b["stress_history"]))
    assert np.array_equal(a["coords"], b["coords"])
    assert a["passes"] < b["passes"]
    o = O.minimize_stress(D, q, kind, huber_delta=hd, max_iters=10, rel_tol=1e-300, Y0=Y0)
    h, ho = np.array(a["stress_history"][:11]), np.array(o.stress_history[:11])
    assert np.max(np.abs(h - ho) / ho) <= TRAJ


@pytest.mark.parametrize("kind,rel_tol,iters", [("kruskal", 1e-300, 60), ("kruskal", 1e-4, 500),
                                                ("sammon", 1e-300, 37), ("huber", 1e-5, 300)])
def test_device_resident_descent_identical(monkeypatch, kind, rel_tol, iters):
    # gd_step_kernel decides accepted iterations on the device (no host round
    # trip) with the host loop's arithmetic: same history, coordinates,
    # iteration count and converged flag as GMDS_HOST_GD=1, through the
    # max_iters and rel_tol exits and the hand-backs to the host
    monkeypatch.setenv("GMDS_NO_TINY", "1")  # the tiny phase's single pass: test_tiny_phase_one_pass
    rng = np.random.default_rng(21)
    n = 2400
    X = rng.standard_normal((n, 5)) * np.linspace(2.0, 0.5, 5)
    D = G.pairwise_matrix(X, 2.0)
    Y0 = rng.normal(0.0, 0.1, (n, 2))
    hd = 0.5 * float(np.median(D)) if kind == "huber" else None
    a = G.minimize_stress(D, 2, kind, huber_delta=hd, max_iters=iters, rel_tol=rel_tol, Y0=Y0, storage=G.F32)
    monkeypatch.setenv("GMDS_HOST_GD", "1")
    b = G.minimize_stress(D, 2, kind, huber_delta=hd, max_iters=iters, rel_tol=rel_tol, Y0=Y0, storage=G.F32)
    assert a["iterations"] == b["iterations"] and a["converged"] == b["converged"]
    assert np.array_equal(np.array(a["stress_history"]), np.array(b["stress_history"]))
    assert np.array_equal(a["coords"], b["coords"])
    # a solo pass (slot 0 only, GdState::solo) that misses costs one extra pass; further halvings
    # decided on the device (GdState::rt) save the host loop's separate gradient pass
    assert a["passes"] <= b["passes"] + max(3, iters // 20)
    monkeypatch.delenv("GMDS_HOST_GD")
    monkeypatch.setenv("GMDS_NO_SOLO", "1")
    monkeypatch.setenv("GMDS_NO_ONDEV", "1")
    c = G.minimize_stress(D, 2, kind, huber_delta=hd, max_iters=iters, rel_tol=rel_tol, Y0=Y0, storage=G.F32)
    assert np.array_equal(np.array(c["stress_history"]), np.array(b["stress_history"]))
    assert np.array_equal(c["coords"], b["coords"])
    assert c["passes"] == b["passes"]


@pytest.mark.parametrize("kind,q,iters", [("kruskal", 1, 150), ("kruskal", 3, 150), ("kruskal", 4, 120),
                                          ("sammon", 3, 120), ("huber", 1, 120), ("huber", 4, 100)])
def test_device_loop_identical_to_host_loop_other_q(monkeypatch, kind, q, iters):
    # the on-device fix / re-trial units (GdState::fix, rt) and solo passes at q = 1, 3, 4 and for
    # the kinds without a difference pass: same history and coordinates, bit for bit, as the
    # host loop (GMDS_HOST_GD=1); the tiny phase is off on both sides as in the q = 2 test above
    monkeypatch.setenv("GMDS_NO_TINY", "1")
    rng = np.random.default_rng(100 + 7 * q + len(kind))
    n = 2300 + 37 * q
    X = rng.standard_normal((n, 6)) * np.linspace(2.0, 0.5, 6)
    D = G.pairwise_matrix(X, 2.0)
    Y0 = rng.normal(0.0, 0.1, (n, q))
    hd = 0.5 * float(np.median(D)) if kind == "huber" else None
    a = G.minimize_stress(D, q, kind, huber_delta=hd, max_iters=iters, rel_tol=1e-300, Y0=Y0, storage=G.F32)
    monkeypatch.setenv("GMDS_HOST_GD", "1")
    b = G.minimize_stress(D, q, kind, huber_delta=hd, max_iters=iters, rel_tol=1e-300, Y0=Y0, storage=G.F32)
    assert a["iterations"] == b["iterations"] and a["converged"] == b["converged"]
    assert np.array_equal(np.array(a["stress_history"]), np.array(b["stress_history"]))
    assert np.array_equal(a["coords"], b["coords"])
    assert a["passes"] <= b["passes"] + max(3, iters // 20)


@pytest.mark.parametrize("q,iters", [(2, 260), (3, 200)])
def test_device_loop_keeps_decisions_on_device(monkeypatch, q, iters):
    # image-like data above the small-fit size, fp32 storage, seeded N(0, 0.1^2) init: past the
    # step-doubling run the full step hovers at the Armijo threshold, so slot-1 acceptances,
    # further halvings, pending (difference-pass) decisions and tiny-phase rejections all occur.
    # The device-resident loop decides them itself (GdState::fix / rt, merged launches): same
    # history and coordinates, bit for bit, as with the hand-backs to the host loop (whose
    # trajectories test_gpu_large.py pins to the reference's at n = 2600, 5000 and 20000).
    from bench import make_image_like

    n = 2600
    X = make_image_like(n, 784)
    D = G.pairwise_matrix(X, 2.0)
    Y0 = np.random.default_rng(2605).normal(0.0, 0.1, (n, q))
    a = G.minimize_stress(D, q, "kruskal", max_iters=iters, rel_tol=1e-300, Y0=Y0, storage=G.F32)
    monkeypatch.setenv("GMDS_NO_ONDEV", "1")
    monkeypatch.setenv("GMDS_NO_MULTI", "1")
    monkeypatch.setenv("GMDS_NO_SOLO", "1")
    b = G.minimize_stress(D, q, "kruskal", max_iters=iters, rel_tol=1e-300, Y0=Y0, storage=G.F32)
    assert a["iterations"] == b["iterations"] == iters
    assert np.array_equal(np.array(a["stress_history"]), np.array(b["stress_history"]))
    assert np.array_equal(a["coords"], b["coords"])
    assert a["passes"] <= b["passes"] + 3


def test_tune_batched_eigensolver_matches(monkeypatch):
    # tune_nu's classical cells of a fold go through one batched eigensolver call;
    # per-cell dense solves give the same mean stresses
    rng = np.random.default_rng(12)
    X = rng.standard_normal((300, 4))
    grid = list(np.linspace(1.2, 4.0, 7))
    a = G.tune_nu(X, 2, grid, 3)
    monkeypatch.setenv("GMDS_NO_BATCHED_EIG", "1")
    b = G.tune_nu(X, 2, grid, 3)
    assert a["nu_star"] == b["nu_star"]
    assert np.allclose(a["mean_stress"], b["mean_stress"], rtol=1e-9, atol=0)
    r = O.tune_nu(X, 2, grid, 3) if hasattr(O, "tune_nu") else None
    if r is not None:
        assert np.allclose(a["mean_stress"], r.mean_stress, rtol=1e-8)


def test_image_shape_fp32_storage_trajectory_scaled_init():
    # the metric data's shape at moderate n: fp32 storage of D and a seeded init at
    # D's scale (RMS(D)/sqrt(2q)) follow the fp64 reference trajectory within the
    # north-star tolerance over the first iterations
    g = np.random.default_rng(77)
    n, p = 1800, 784
    X = g.integers(0, 256, size=(n, p)).astype(np.float64) / 255.0
    X += g.normal(0.0, 0.1, size=(n, p))
    np.clip(X, 0.0, 1.0, out=X)
    X[g.random((n, p)) < 0.8] = 0.0
    X = X.astype(np.float32)
    D = G.pairwise_matrix(X, 2.0)
    iu = np.triu_indices(n, 1)
    s = float(np.sqrt(np.mean(D[iu] ** 2) / 4.0))
    Y0 = g.normal(0.0, s, (n, 2))
    a = G.minimize_stress(D, 2, "kruskal", max_iters=30, rel_tol=1e-300, Y0=Y0, storage=G.F32)
    o = O.minimize_stress(D, 2, "kruskal", max_iters=30, rel_tol=1e-300, Y0=Y0)
    h, ho = np.array(a["stress_history"]), np.array(o.stress_history)
    m = min(len(h), len(ho))
    assert m >= 20
    assert np.max(np.abs(h[:m] - ho[:m]) / ho[:m]) <= TRAJ


def test_fp32_storage_follows_fp64_through_tiny_steps():
    # Kruskal from N(0, 0.1^2) against Gini distances ~3e4: the reference's first
    # iterations change the loss by ~1e-13 relative, below fp32 storage's resolution;
    # those decisions are re-evaluated (fp64 arithmetic), so the fp32-storage fit
    # follows the fp64-storage trajectory instead of stalling or wandering
    g = np.random.default_rng(78)
    n, p = 2600, 784
    X = g.integers(0, 256, size=(n, p)).astype(np.float64) / 255.0
    X += g.normal(0.0, 0.1, size=(n, p))
    np.clip(X, 0.0, 1.0, out=X)
    X[g.random((n, p)) < 0.8] = 0.0
    X = X.astype(np.float32)
    D = G.pairwise_matrix(X, 2.0)
    Y0 = g.normal(0.0, 0.1, (n, 2))
    a = G.minimize_stress(D, 2, "kruskal", max_iters=60, rel_tol=1e-300, Y0=Y0, storage=G.F32)
    b = G.minimize_stress(D, 2, "kruskal", max_iters=60, rel_tol=1e-300, Y0=Y0, storage=G.F64)
    assert a["iterations"] == b["iterations"] == 60
    h, hb = np.array(a["stress_history"]), np.array(b["stress_history"])
    assert np.max(np.abs(h - hb) / hb) <= 1e-6
    assert hb[-1] < 0.9 * hb[0]  # the fit left the tiny-step phase


@pytest.mark.parametrize("kind", ["sammon", "huber"])
def test_fp32_storage_other_kinds_follow_fp64(kind):
    # the same regime for the other gradient-descent kinds: sub-resolution decisions are
    # handed to the host and re-taken in fp64 arithmetic over the fp32 image
    g = np.random.default_rng(79)
    n, p = 2600, 300  # above the persistent small-fit size: the tiled fp32 passes
    X = g.integers(0, 256, size=(n, p)).astype(np.float64) / 255.0
    X += g.normal(0.0, 0.1, size=(n, p))
    np.clip(X, 0.0, 1.0, out=X)
    X[g.random((n, p)) < 0.8] = 0.0
    X = X.astype(np.float32)
    D = G.pairwise_matrix(X, 2.0)
    Y0 = g.normal(0.0, 0.1, (n, 2))
    hd = 0.5 * float(np.median(D)) if kind == "huber" else None
    a = G.minimize_stress(D, 2, kind, huber_delta=hd, max_iters=40, rel_tol=1e-300, Y0=Y0, storage=G.F32)
    b = G.minimize_stress(D, 2, kind, huber_delta=hd, max_iters=40, rel_tol=1e-300, Y0=Y0, storage=G.F64)
    assert a["iterations"] == b["iterations"]
    h, hb = np.array(a["stress_history"]), np.array(b["stress_history"])
    assert np.max(np.abs(h - hb) / np.abs(hb)) <= 1e-5


def test_metric_shape_fit_properties():
    # BASELINE's metric shape (n = 20000, p = 784, nu = 2, q = 2, Kruskal from a
    # seeded N(0, 0.1^2) init, the bench's fit): the fp32-storage trajectory
    # (difference passes in the tiny-step phase) equals the fp64-storage one to
    # 1e-6 over 100 iterations, the history never increases (Armijo), and the
    # reported stress is the Kruskal stress of the returned coordinates
    torch = pytest.importorskip("torch")
    g = np.random.default_rng(2025)
    n, p = 20000, 784
    X = g.integers(0, 256, size=(n, p)).astype(np.float64) / 255.0
    X += g.normal(0.0, 0.1, size=(n, p))
    np.clip(X, 0.0, 1.0, out=X)
    X[g.random((n, p)) < 0.8] = 0.0
    X = X.astype(np.float32)
    dX = torch.from_numpy(X).cuda()
    D32 = G.dmat_gini_device(dX.data_ptr(), G.F32, n, p, 2.0, G.F32)
    D64 = G.dmat_gini_device(dX.data_ptr(), G.F32, n, p, 2.0, G.F64)
    Y0 = g.normal(0.0, 0.1, (n, 2))
    a = G.minimize_stress(D32, 2, "kruskal", max_iters=100, rel_tol=1e-300, Y0=Y0)
    b = G.minimize_stress(D64, 2, "kruskal", max_iters=100, rel_tol=1e-300, Y0=Y0)
    assert a["iterations"] == b["iterations"] == 100
    h, hb = np.array(a["stress_history"]), np.array(b["stress_history"])
    assert np.max(np.abs(h - hb) / hb) <= 1e-6
    assert np.all(np.diff(hb) <= 0.0) and np.all(np.diff(h) <= 0.0)
    assert hb[-1] < 0.9 * hb[0]
    assert abs(G.kruskal_stress(b["coords"], D64) - b["stress"]) <= 1e-12 * b["stress"]
    assert abs(G.kruskal_stress(a["coords"], D32) - a["stress"]) <= 1e-6 * a["stress"]


def test_tiny_phase_one_pass(monkeypatch):
    # the device loop's sub-resolution phase: one difference + gradient pass per iteration (the
    # gradient at the first trial from the difference pass's own per-pair quantities) instead of the
    # fused pass + a difference pass; same decisions, trajectory to round-off, fewer passes
    g = np.random.default_rng(78)
    n, p = 2600, 784
    X = g.integers(0, 256, size=(n, p)).astype(np.float64) / 255.0
    X += g.normal(0.0, 0.1, size=(n, p))
    np.clip(X, 0.0, 1.0, out=X)
    X[g.random((n, p)) < 0.8] = 0.0
    D = G.pairwise_matrix(X.astype(np.float32), 2.0)
    Y0 = g.normal(0.0, 0.1, (n, 2))
    a = G.minimize_stress(D, 2, "kruskal", max_iters=60, rel_tol=1e-300, Y0=Y0, storage=G.F32)
    monkeypatch.setenv("GMDS_NO_TINY", "1")
    b = G.minimize_stress(D, 2, "kruskal", max_iters=60, rel_tol=1e-300, Y0=Y0, storage=G.F32)
    assert a["iterations"] == b["iterations"] == 60
    h, hb = np.array(a["stress_history"]), np.array(b["stress_history"])
    assert np.max(np.abs(h - hb) / hb) <= 1e-7
    assert a["passes"] < b["passes"] - 10


def test_metric_shape_fp32_gradient_accuracy():
    # the fused passes accumulate each thread's row sums over up to 8 blocks (1024 pairs) in fp32
    # before the fp64 reduction: at the metric shape the Kruskal gradient with fp32 storage stays
    # within 1e-5 (max-normalised) of the fp64-storage gradient (itself oracle-checked)
    torch = pytest.importorskip("torch")
    g = np.random.default_rng(2025)
    n, p = 20000, 784
    X = g.integers(0, 256, size=(n, p)).astype(np.float64) / 255.0
    X += g.normal(0.0, 0.1, size=(n, p))
    np.clip(X, 0.0, 1.0, out=X)
    X[g.random((n, p)) < 0.8] = 0.0
    dX = torch.from_numpy(X.astype(np.float32)).cuda()
    D32 = G.dmat_gini_device(dX.data_ptr(), G.F32, n, p, 2.0, G.F32)
    D64 = G.dmat_gini_device(dX.data_ptr(), G.F32, n, p, 2.0, G.F64)
    Y = g.normal(0.0, 30.0, (n, 2))
    a = G.stress_gradient("kruskal", Y, D32)
    b = G.stress_gradient("kruskal", Y, D64)
    assert np.max(np.abs(a - b)) <= 1e-5 * np.max(np.abs(b))
