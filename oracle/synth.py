"""Seeded synthetic inputs for BASELINE.json's configs (SURVEY 8(d) generators) --
TEST INFRASTRUCTURE, shared by oracle/make_golden_large.py, tests/ and
tools/bench_configs.py so the golden fixtures and the GPU checks see the same
bytes.  numpy PCG64 streams are platform-independent, so a GPU box regenerates
exactly the X the fixtures were made from.  (bench.py keeps its own identical
copy of ``image_like`` so the engine arm does not import oracle/.)

The paper's datasets (MNIST, UCI) are not in the container; these
generators stand in with the configs' shapes and value distributions.
"""
from __future__ import annotations

import numpy as np


def image_like(n, p, seed):
    """C3 / C5 / metric: 80% exact zeros per row, the rest uniform over the 256
    levels k/255 plus N(0, 0.1^2) noise, clipped to [0, 1]; fp32."""
    g = np.random.default_rng(seed)
    X = g.integers(0, 256, size=(n, p)).astype(np.float64) / 255.0
    X += g.normal(0.0, 0.1, size=(n, p))
    np.clip(X, 0.0, 1.0, out=X)
    X[g.random((n, p)) < 0.8] = 0.0
    return X.astype(np.float32)


def mixture_contaminated(n=1000, p=20, seed=2):
    """C2: 3-component Gaussian mixture (means ~ N(0, 9 I), unit covariance, equal
    weights), 5% of rows multiplied by 10 sigma_j (contaminate, data.cpp:288-295); fp64."""
    rng = np.random.default_rng(seed)
    means = rng.normal(0.0, 3.0, (3, p))
    X = means[rng.integers(0, 3, n)] + rng.standard_normal((n, p))
    rows = rng.choice(n, int(round(0.05 * n)), replace=False)
    X[rows] *= 10.0 * X.std(axis=0)
    return X


def c2_grid():
    """8 nu log-spaced in [1.1, 8] (F5: the reference rejects nu <= 1)."""
    return list(np.exp(np.linspace(np.log(1.1), np.log(8.0), 8)))


def lognormal_dup(n=20000, p=128, seed=4):
    """C4: log-normal(0, 1) fp32 features, 1% of rows overwritten by copies of other rows."""
    g = np.random.default_rng(seed)
    X = np.exp(g.standard_normal((n, p))).astype(np.float32)
    dup = g.choice(n, n // 100, replace=False)
    src = g.choice(n, n // 100, replace=False)
    X[dup] = X[src]
    return X, dup, src


C4_NUS = [1.5, 2.0, 3.0, 5.0]


def sample_pairs(n, m, seed, extra=None):
    """m seeded pairs i < j (plus `extra` pairs, e.g. duplicated rows), int64."""
    g = np.random.default_rng(seed)
    I = g.integers(0, n, 2 * m + 64)
    J = g.integers(0, n, 2 * m + 64)
    keep = I != J
    I, J = I[keep][:m], J[keep][:m]
    I, J = np.minimum(I, J), np.maximum(I, J)
    if extra is not None:
        ei, ej = np.asarray(extra[0]), np.asarray(extra[1])
        ok = ei != ej
        ei, ej = ei[ok], ej[ok]
        I = np.concatenate([I, np.minimum(ei, ej)])
        J = np.concatenate([J, np.maximum(ei, ej)])
    return I.astype(np.int64), J.astype(np.int64)


def rank_weights(p, seed=99):
    """Integer weights for per-pair rank fingerprints: sum_k 2 R_k w_k is exact in int64."""
    return np.random.default_rng(seed).integers(1, 1 << 20, p).astype(np.int64)


def rank_fingerprints(R, w):
    """R: (m, p) midranks (half-integers) -> (m,) int64 sum_k 2 R_k w_k."""
    twoR = np.rint(2.0 * np.asarray(R)).astype(np.int64)
    return twoR @ w
