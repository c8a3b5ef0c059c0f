"""Fused nu-sweep scorer: Kruskal stress of a fixed embedding
against every grid nu from one distance pass, no D_nu materialised -- vs the
oracle's kruskal_stress(Y, pairwise_matrix(X, nu)) per nu."""
import numpy as np
import pytest

from oracle import gini_oracle as O

pytestmark = pytest.mark.gpu
G = pytest.importorskip("paper_2605_25124_b200.gmds")


def image_like(n, p, seed):
    g = np.random.default_rng(seed)
    X = g.integers(0, 256, size=(n, p)).astype(np.float64) / 255.0 + g.normal(0.0, 0.1, size=(n, p))
    np.clip(X, 0.0, 1.0, out=X)
    X[g.random((n, p)) < 0.8] = 0.0
    return X.astype(np.float32)


@pytest.mark.parametrize("case", ["dense_neg", "sparse_merge", "dense_wide", "tiny"])
def test_sweep_matches_per_nu_kruskal(case):
    rng = np.random.default_rng(3)
    if case == "dense_neg":
        X = rng.standard_normal((150, 12))
    elif case == "sparse_merge":
        X = image_like(120, 300, 4)
    elif case == "dense_wide":
        X = rng.lognormal(0, 1, (60, 600)).astype(np.float32)
    else:
        X = rng.standard_normal((5, 3))
    n = X.shape[0]
    Y = rng.standard_normal((n, 2))
    grid = list(O.nugrid_linspace(1.1, 5.0, 30 if case != "dense_wide" else 9))
    ks = G.nu_sweep_kruskal(X, Y, grid)
    Xd = X.astype(np.float64)
    ref = np.array([O.kruskal_stress(Y, O.pairwise_matrix(Xd, nu)) for nu in grid])
    assert np.max(np.abs(ks - ref) / ref) <= 1e-10
    assert int(np.argmin(ks)) == int(np.argmin(ref))


def test_sweep_errors():
    with pytest.raises(G.InvalidConfig):
        G.nu_sweep_kruskal(np.ones((4, 2)), np.zeros((4, 1)), [1.0, 2.0])
    with pytest.raises(G.DegenerateInput):
        G.nu_sweep_kruskal(np.full((6, 3), 2.0), np.zeros((6, 2)), [1.5, 2.0])
