"""CPU tests: the oracle restatement against the reference's known-answer
tests, the golden vectors (outputs of the UNMODIFIED reference compiled by
oracle/Makefile) and, when present, the live reference library."""
import math

import numpy as np
import pytest

from oracle import gini_oracle as O
from oracle import ref_lib as R
from _util import unpad

needs_ref = pytest.mark.skipif(R.load() is None, reason="oracle/_ref not built (make -C oracle)")


# --- known-answer tests from the reference suites -------------------------------------------

def test_worked_example_594():
    # test_metrics.cpp:180-182, acceptance_main.cpp:50-59
    assert O.gini_pseudo_distance([10.0, 1200.0], [10.0, 12.0]) == 594.0
    assert abs(O.gen_gini_distance([10.0, 1200.0], [10.0, 12.0], 2.0) - 594.0) <= 1e-10
    assert abs(O.gen_gini_distance([10.0, 1200.0], [10.0, 12.0], 3.0) - 594.0) <= 594.0 * 1e-12


def test_directed_445_742():
    # test_metrics.cpp:245-252
    assert O.gen_gini_directed([10.0, 1200.0], [10.0, 12.0], 2.0) == pytest.approx(594.0, rel=1e-12)
    assert O.gen_gini_directed([10.0, 1200.0], [10.0, 12.0], 3.0) == pytest.approx(445.5, rel=1e-12)
    assert O.gen_gini_directed([10.0, 12.0], [10.0, 1200.0], 3.0) == pytest.approx(742.5, rel=1e-12)


def test_midrank_examples():
    # test_metrics.cpp:94-119
    assert list(O.midrank([3.0, 1.0, 2.0])) == [3.0, 1.0, 2.0]
    assert list(O.midrank([0.0, 0.0, 0.0, 0.0])) == [2.5] * 4
    assert list(O.midrank([1.0, 2.0, 2.0, 4.0])) == [1.0, 2.5, 2.5, 4.0]
    assert list(O.midrank([-0.0, 0.0, 1.0])) == [1.5, 1.5, 3.0]
    for bad in ([1.0, math.nan], [math.inf], []):
        with pytest.raises(O.InvalidInput):
            O.midrank(bad)


def test_gini_norm_and_survival():
    # test_metrics.cpp:151-160, 216-226
    assert O.gini_norm([5.0, 5.0, 5.0]) == 0.0
    assert O.gini_norm([1.0, 2.0, 3.0]) == pytest.approx(2.0, rel=1e-14)
    assert O.gini_norm([-2.0, -4.0, -6.0]) == pytest.approx(4.0, rel=1e-14)
    assert list(O.empirical_survival([0.0, 1188.0])) == [0.75, 0.25]
    assert list(O.empirical_survival([7.0] * 5)) == [0.5] * 5


def test_error_contract():
    # GiniParams (metrics.hpp:35-36), NuGrid (tune.cpp:74-83), pairwise_matrix (metrics.cpp:196-197)
    for nu in (1.0, 0.5, 0.743):
        with pytest.raises(O.InvalidConfig):
            O.gen_gini_distance([1.0], [2.0], nu)
    with pytest.raises(O.InvalidInput):
        O.pairwise_matrix(np.zeros((1, 3)), 2.0)
    with pytest.raises(O.InvalidConfig):
        O.nugrid_from_values([2.0, 2.0])
    with pytest.raises(O.InvalidConfig):
        O.nugrid_linspace(1.1, 5.0, 0)
    with pytest.raises(O.InvalidInput):
        O.from_matrix(np.array([[0.0, 1.0], [2.0, 0.0]]))
    with pytest.raises(O.InvalidInput):
        O.from_matrix(np.array([[1.0, 1.0], [1.0, 0.0]]))
    with pytest.raises(O.InvalidInput):
        O.from_matrix(np.array([[0.0, -1.0], [-1.0, 0.0]]))
    D = np.array([[0, 0, 1], [0, 0, 1], [1, 1, 0.0]])
    with pytest.raises(O.DegenerateInput):
        O.stress_loss("sammon", np.zeros((3, 2)), D)
    with pytest.raises(O.InvalidConfig):
        O.stress_loss("huber", np.zeros((3, 2)), D)


def test_nugrid_linspace():
    g = O.nugrid_linspace()
    assert len(g) == 30 and g[0] == 1.1 and g[-1] == 5.0


# --- restatement vs golden (outputs of the real reference) -----------------------------------

def test_midrank_golden(golden):
    g = golden("midrank")
    for v, r, m in zip(g["values"], g["ranks"], g["lengths"]):
        assert np.array_equal(O.midrank(unpad(v, m)), unpad(r, m))


def test_distance_golden(golden):
    g = golden("distance")
    for x, y, m, nu, fwd, dist in zip(g["x"], g["y"], g["lengths"], g["nu"], g["directed"], g["distance"]):
        x, y = unpad(x, m), unpad(y, m)
        assert O.gen_gini_directed(x, y, nu) == fwd  # bit-exact
        assert O.gen_gini_distance(x, y, nu) == dist


def test_pairwise_golden(golden):
    g = golden("pairwise")
    for name in ("t888", "t321", "c1", "ties"):
        X = g[f"{name}_X"]
        iu = np.triu_indices(X.shape[0], 1)
        for k, nu in enumerate(g[f"{name}_nus"]):
            assert np.array_equal(O.pairwise_matrix(X, float(nu))[iu], g[f"{name}_D{k}"])
        assert np.allclose(O.pairwise_matrix(X, None)[iu], g[f"{name}_E"], rtol=1e-15, atol=0)


def test_stress_golden(golden):
    g = golden("stress")
    n = 200
    D = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    D[iu] = g["c1_D"]
    D = D + D.T
    cm = O.classical_mds(D, 2)
    assert np.allclose(cm.coords, g["cmds_coords"], atol=1e-10)
    assert cm.stress == pytest.approx(float(g["cmds_stress"]), rel=1e-12)
    assert cm.clamped_mass == pytest.approx(float(g["cmds_clamped_mass"]), rel=1e-10)
    for kind in ("kruskal", "sammon", "smacof", "huber"):
        hd = float(g[f"{kind}_huber_delta"]) if kind == "huber" else None
        e = O.minimize_stress(D, 2, kind, huber_delta=hd, max_iters=500, rel_tol=1e-300)
        ref = g[f"{kind}_history"]
        assert len(e.stress_history) == len(ref)
        assert np.allclose(e.stress_history[:51], ref[:51], rtol=1e-10, atol=0)
        assert e.stress == pytest.approx(float(ref[-1]), rel=1e-6)
        if kind != "smacof":
            Y = g["cmds_coords"]
            assert O.stress_loss(kind, Y, D, hd) == pytest.approx(float(g[f"{kind}_loss0"]), rel=1e-12)
            assert np.allclose(O.stress_gradient(kind, Y, D, hd), g[f"{kind}_grad0"], rtol=1e-9, atol=1e-14)
    for kind in ("kruskal", "huber", "sammon", "smacof"):
        e = O.minimize_stress(g[f"rd_{kind}_D"], 2, kind, huber_delta=(0.5 if kind == "huber" else None))
        assert e.iterations == int(g[f"rd_{kind}_iterations"])
        assert e.converged == bool(g[f"rd_{kind}_converged"])
        assert e.stress == pytest.approx(float(g[f"rd_{kind}_stress"]), rel=1e-9)
    e = O.minimize_stress(g["auto_D"], 2, "huber")
    assert e.huber_delta == float(g["auto_huber_delta"])


def test_tune_golden(golden):
    g = golden("tune")
    r = O.tune_nu(g["t_X"], 2, list(g["t_grid"]), 3, "classical", 42)
    assert np.allclose(r.mean_stress, g["t_mean"], rtol=1e-12)  # p=3: all nu tie to round-off
    r = O.tune_nu(g["u_X"], 2, list(g["u_grid"]), 3, "classical", 4)
    assert np.allclose(r.mean_stress, g["u_mean"], rtol=1e-12)
    assert r.nu_star == float(g["u_nu_star"])
    assert np.allclose(r.best_embedding.coords, g["u_coords"], atol=1e-9)
    r = O.tune_nu(g["s_X"], 2, list(g["s_grid"]), 2, "smacof", 11)
    assert np.allclose(r.mean_stress, g["s_mean"], rtol=1e-9)
    a = O.alternating_tune(g["a_X"], 2, 3, list(g["a_grid"]), 17)
    assert a.nu_path == list(g["a_path"])
    assert a.embedding.stress == pytest.approx(float(g["a_stress"]), rel=1e-9)


def test_tune_tie_to_smaller_nu():
    # test_tune.cpp:85-93: constant data -> all zero distances -> first grid value
    X = np.full((12, 3), 4.2)
    r = O.tune_nu(X, 1, O.nugrid_linspace(1.5, 3.5, 4), 3, "classical", 5)
    assert r.nu_star == 1.5 and all(s == 0.0 for s in r.mean_stress)


# --- restatement vs the live reference library (this container / GPU boxes with oracle/_ref) ---

@needs_ref
def test_rng_matches_reference():
    a, b = O.Rng(2024), R.RefRng(2024)
    for _ in range(500):
        assert a.uniform01() == b.uniform01()
        assert a.normal() == b.normal()
        assert a.uniform_below(97) == b.uniform_below(97)
    assert O.mix_seed(9, 4, 2) == R.load().ref_mix_seed(9, 4, 2)


@needs_ref
def test_pairwise_matches_reference_random():
    g = np.random.default_rng(0)
    for n, p in ((17, 1), (40, 33), (25, 64)):
        X = g.standard_normal((n, p))
        X[g.random(X.shape) < 0.3] = 0.0
        for nu in (1.01, 2.0, 4.5):
            assert np.array_equal(O.pairwise_matrix(X, nu), R.pairwise_matrix(X, nu))


@needs_ref
def test_thread_count_bit_identity():
    # test_metrics.cpp:268-277 on the reference itself
    rng = O.Rng(321)
    X = O.random_matrix(rng, 24, 4, 2.0)
    R.set_max_threads(1)
    d1 = R.pairwise_matrix(X, 1.8)
    R.set_max_threads(4)
    d4 = R.pairwise_matrix(X, 1.8)
    R.set_max_threads(0)
    assert np.array_equal(d1, d4)


def test_pairwise_properties():
    # Size-independent properties the GPU tests also check at full size
    # (symmetric, zero diagonal, non-negative, zero on duplicated rows), plus
    # invariance under one permutation of the features applied to every row.
    g = np.random.default_rng(7)
    X = g.standard_normal((12, 9))
    X[g.random(X.shape) < 0.3] = 0.0
    X[5] = X[2]
    perm = g.permutation(X.shape[1])
    for nu in (1.5, 2.0, 3.0):
        D = O.pairwise_matrix(X, nu)
        assert np.array_equal(D, D.T)
        assert np.all(np.diag(D) == 0.0)
        assert np.all(D >= 0.0)
        assert D[2, 5] == 0.0
        Dp = O.pairwise_matrix(X[:, perm], nu)
        np.testing.assert_allclose(Dp, D, rtol=1e-12, atol=1e-12 * D.max())
