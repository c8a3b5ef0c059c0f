"""the Euclidean pairwise_matrix branch (metrics.cpp:220-235) on the
tcgen05 tensor cores (euclid_tc.cu: bf16x3 split Gram GEMM accumulated in TMEM,
fp64 norm corrections, near-duplicates recomputed in the reference's arithmetic)
against the exact fp64 kernel (bit-identical to the reference) and the oracle.
Bar: 1e-6 relative, max-normalised (BASELINE north_star); duplicated rows exactly 0."""
import numpy as np
import pytest

from oracle import gini_oracle as O
from oracle import synth as S

torch = pytest.importorskip("torch")
G = pytest.importorskip("paper_2605_25124_b200.gmds")
pytestmark = pytest.mark.gpu


def _euclid_device(X, mode):
    import ctypes

    n, p = X.shape
    dX = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    dD = torch.empty((n, n), dtype=torch.float64, device="cuda")
    xt = G.F32 if X.dtype == np.float32 else G.F64
    G._check(G.lib().gmds_pairwise_euclidean_device(ctypes.c_void_p(dX.data_ptr()), G._i32(xt), G._i64(n), G._i64(p),
                                                    ctypes.c_void_p(dD.data_ptr()), G._i32(mode), ctypes.c_void_p(0)))
    return dD.cpu().numpy()


@pytest.mark.parametrize("shape,kind", [((1500, 128), "lognormal"), ((1030, 784), "image"), ((700, 3), "gauss"),
                                        ((900, 70), "gauss64")])
def test_tc_matches_exact_and_reference(shape, kind):
    n, p = shape
    g = np.random.default_rng(n + p)
    if kind == "lognormal":
        X = np.exp(g.standard_normal((n, p))).astype(np.float32)
        X[g.choice(n, 15, replace=False)] = X[g.choice(n, 15, replace=False)]  # duplicated rows
    elif kind == "image":
        X = S.image_like(n, p, 7)
    elif kind == "gauss":
        X = (g.standard_normal((n, p)) * 100.0 + 5e3).astype(np.float32)  # large offset: centring matters
    else:
        X = g.standard_normal((n, p)) * np.linspace(0.1, 10.0, p)
    tc = _euclid_device(X, 2)
    ex = _euclid_device(X, 1)
    scale = np.max(ex)
    assert np.max(np.abs(tc - ex)) <= 1e-6 * scale
    assert np.array_equal(tc, tc.T) and np.all(np.diag(tc) == 0.0)
    dup = np.all(X[:, None, :] == X[None, :, :], axis=2) if n <= 1500 else None
    if dup is not None:
        assert np.all(tc[dup] == 0.0)
    # the exact kernel is the reference's arithmetic; spot-check it against the oracle
    idx = g.integers(0, n, (2, 200))
    Xd = X.astype(np.float64)
    ref = np.sqrt(np.sum((Xd[idx[0]] - Xd[idx[1]]) ** 2, axis=1))
    assert np.max(np.abs(ex[idx[0], idx[1]] - ref)) <= 1e-12 * scale


def test_host_entry_uses_tc_above_512_and_agrees():
    g = np.random.default_rng(3)
    X = g.standard_normal((600, 40))
    D = G.pairwise_matrix(X, None)  # n >= 512: the tcgen05 path
    R = O.pairwise_matrix(X, None) if hasattr(O, "pairwise_matrix") else None
    ref = np.sqrt(np.maximum(0.0, np.sum((X[:, None, :] - X[None, :, :]) ** 2, axis=2)))
    assert np.max(np.abs(D - ref)) <= 1e-6 * np.max(ref)
    if R is not None:
        assert np.max(np.abs(D - R)) <= 1e-6 * np.max(R)
