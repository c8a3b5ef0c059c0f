"""CPU restatement of the reference Gini-MDS hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module, and only as the checker.
The product (paper_2605_25124_b200, libgmds.so) never calls it; there is no
CPU fallback anywhere in the product path.

Every function restates the reference C++ (``/root/reference/proj/core``) and
cites the file:line it follows.  Parity of this restatement is pinned two
ways (see tests/test_oracle.py):

* against the UNMODIFIED reference compiled here from its own sources
  (``oracle/_ref/libginimds_ref.so``, built by ``oracle/Makefile``), on the
  reference tests' own seeded inputs -- midranks and distances bit-exact,
  stress values / trajectories to round-off;
* against the golden vectors in ``tests/golden/`` (generated from that
  library by ``oracle/make_golden.py``) and the reference's known-answer
  tests (594, 445.5 / 742.5, Hazen survival, ...).

Arithmetic is fp64 throughout, as in the reference (metrics.hpp:12-13).
``pow`` goes through ``math.pow`` (the C library's pow, exactly what
``std::pow`` calls) on the 2p-1 possible half-integer midranks -- numpy's
vectorised power is not bit-identical to libm.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# Exceptions (error.hpp:9-53).  ``code`` matches the C-ABI gmds_status values.


class GiniError(Exception):
    code = 5


class InvalidInput(GiniError):
    code = 1


class InvalidConfig(GiniError):
    code = 2


class DegenerateInput(GiniError):
    code = 3


class NumericFailure(GiniError):
    code = 4


KINDS = ("kruskal", "huber", "sammon", "smacof")  # StressKind, embed.hpp:13
METHODS = ("classical", "kruskal", "huber", "sammon", "smacof")  # EmbeddingMethod, embed.hpp:15

# ---------------------------------------------------------------------------
# rng.hpp / rng.cpp: mt19937_64 with 53-bit uniforms, splitmix mixing.

_M64 = (1 << 64) - 1


class Rng:
    """std::mt19937_64 (rng.hpp:20-45) restated in pure Python."""

    _NN, _MM = 312, 156
    _MATRIX_A = 0xB5026F5AA96619E9
    _UM, _LM = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int):
        mt = [0] * self._NN
        mt[0] = seed & _M64
        for i in range(1, self._NN):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self._mt, self._mti = mt, self._NN

    def next_u64(self) -> int:
        NN, MM, mt = self._NN, self._MM, self._mt
        if self._mti >= NN:
            for i in range(NN):
                x = (mt[i] & self._UM) | (mt[(i + 1) % NN] & self._LM)
                xa = x >> 1
                if x & 1:
                    xa ^= self._MATRIX_A
                mt[i] = mt[(i + MM) % NN] ^ xa
            self._mti = 0
        x = mt[self._mti]
        self._mti += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _M64

    def uniform01(self) -> float:  # rng.hpp:27-29
        return (float(self.next_u64() >> 11) + 0.5) * 2.0**-53

    def uniform_below(self, bound: int) -> int:  # rng.cpp:29-37
        if bound <= 1:
            return 0
        limit = (bound * (_M64 // bound)) & _M64
        while True:
            x = self.next_u64()
            if x < limit:
                return x % bound

    def normal(self) -> float:  # rng.cpp:39-43 (Box-Muller)
        u1 = self.uniform01()
        u2 = self.uniform01()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)

    def log_normal(self, sigma: float) -> float:  # rng.cpp:63
        return math.exp(sigma * self.normal())


def _splitmix64(state: int) -> tuple[int, int]:  # rng.cpp:9-15
    state = (state + 0x9E3779B97F4A7C15) & _M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return state, z ^ (z >> 31)


def mix_seed(base: int, a: int, b: int = 0) -> int:  # rng.cpp:20-27
    state, _ = _splitmix64(base & _M64)
    state ^= (a * 0xD1342543DE82EF95) & _M64
    state, _ = _splitmix64(state)
    state ^= (b * 0xAF251AF3B0F025B5) & _M64
    _, out = _splitmix64(state)
    return out


def shuffle_indices(indices: list[int], rng: Rng) -> None:  # rng.cpp:65-70 (Fisher-Yates)
    for i in range(len(indices), 1, -1):
        j = rng.uniform_below(i)
        indices[i - 1], indices[j] = indices[j], indices[i - 1]


# ---------------------------------------------------------------------------
# metrics.cpp


def _check_finite(v: np.ndarray, who: str) -> None:  # metrics.cpp:14-19
    if v.size == 0:
        raise InvalidInput(f"{who}: input vector is empty")
    if not np.all(np.isfinite(v)):
        raise InvalidInput(f"{who}: non-finite input entry")


def _midrank_rows(Z: np.ndarray) -> np.ndarray:
    """midrank_into (metrics.cpp:42-56) applied to every row of Z.

    Sort by '<' (any correct sort gives the same output because tied entries
    share a rank), walk tie groups, group at sorted 0-based positions [a, b)
    gets 0.5*(a+1+b).  -0.0 == +0.0 so signed zeros form one group.
    """
    Z = np.asarray(Z, dtype=np.float64)
    m, d = Z.shape
    order = np.argsort(Z, axis=1, kind="stable")
    s = np.take_along_axis(Z, order, axis=1)
    pos = np.broadcast_to(np.arange(d), (m, d))
    start = np.ones((m, d), dtype=bool)
    start[:, 1:] = s[:, 1:] != s[:, :-1]
    a = np.maximum.accumulate(np.where(start, pos, 0), axis=1)
    # group end b = next start position (or d)
    nxt = np.where(start, pos, d)
    nxt = np.concatenate([nxt[:, 1:], np.full((m, 1), d)], axis=1)
    b = np.minimum.accumulate(nxt[:, ::-1], axis=1)[:, ::-1]
    rank_sorted = 0.5 * (a + 1 + b).astype(np.float64)
    out = np.empty_like(Z)
    np.put_along_axis(out, order, rank_sorted, axis=1)
    return out


def midrank(v) -> np.ndarray:  # metrics.cpp:101-110
    v = np.asarray(v, dtype=np.float64).ravel()
    _check_finite(v, "midrank")
    return _midrank_rows(v[None, :])[0]


def gini_norm(x) -> float:  # metrics.cpp:58-66, 112-115
    x = np.asarray(x, dtype=np.float64).ravel()
    _check_finite(x, "gini_norm")
    r = _midrank_rows(x[None, :])[0]
    center = 0.5 * float(x.size + 1)
    return float(np.cumsum(x * (r - center))[-1])


def gini_pseudo_distance(x, y) -> float:  # metrics.cpp:119-127
    x = np.asarray(x, dtype=np.float64).ravel()
    y = np.asarray(y, dtype=np.float64).ravel()
    if x.size != y.size:
        raise InvalidInput(f"gini_pseudo_distance: length mismatch ({x.size} vs {y.size})")
    _check_finite(x, "gini_pseudo_distance")
    _check_finite(y, "gini_pseudo_distance")
    z = x - y
    r = _midrank_rows(z[None, :])[0]
    center = 0.5 * float(z.size + 1)
    return float(np.cumsum(z * (r - center))[-1])


def empirical_survival(z) -> np.ndarray:  # metrics.cpp:133-144
    z = np.asarray(z, dtype=np.float64).ravel()
    _check_finite(z, "empirical_survival")
    d = z.size
    inv_d = 1.0 / float(d)
    return 1.0 - (_midrank_rows(z[None, :])[0] - 0.5) * inv_d


def _check_nu(nu: float) -> float:  # GiniParams, metrics.hpp:33-36
    if not (nu > 1.0):
        raise InvalidConfig(f"GiniParams: nu must be > 1, got {nu:f}")
    return float(nu)


def survival_pow_table(d: int, nu: float) -> np.ndarray:
    """pow(S(R), nu-1) - pow(0.5, nu-1) for every half-integer midrank R.

    Index h = 2R - 1 in [1, 2d-1]; the expressions are those of
    gen_gini_directed_impl (metrics.cpp:73-79), evaluated with libm pow.
    """
    exponent = nu - 1.0
    inv_d = 1.0 / float(d)
    c = math.pow(0.5, exponent)
    tab = np.zeros(2 * d, dtype=np.float64)
    for h in range(1, 2 * d):
        rank = 0.5 * (h + 1)
        survival = 1.0 - (rank - 0.5) * inv_d
        tab[h] = math.pow(survival, exponent) - c
    return tab


def _directed_rows(Z: np.ndarray, nu: float, tab: np.ndarray | None = None) -> np.ndarray:
    """gen_gini_directed_impl (metrics.cpp:69-82) for every row of Z, bit-exact:
    per-term factor from libm pow, sequential left-to-right sum, times -d."""
    m, d = Z.shape
    if tab is None:
        tab = survival_pow_table(d, nu)
    R = _midrank_rows(Z)
    h = (2.0 * R - 1.0).astype(np.int64)
    terms = Z * tab[h]
    s = np.cumsum(terms, axis=1)[:, -1]  # sequential sum, as the C++ loop
    return -float(d) * s


def gen_gini_directed(x, y, nu: float) -> float:  # metrics.cpp:84-93, 148-151
    nu = _check_nu(nu)
    x = np.asarray(x, dtype=np.float64).ravel()
    y = np.asarray(y, dtype=np.float64).ravel()
    if x.size != y.size:
        raise InvalidInput(f"gen_gini_directed: length mismatch ({x.size} vs {y.size})")
    _check_finite(x, "gen_gini_directed")
    _check_finite(y, "gen_gini_directed")
    return float(_directed_rows((x - y)[None, :], nu)[0])


def gen_gini_distance(x, y, nu: float) -> float:  # metrics.cpp:157-163
    fwd = gen_gini_directed(x, y, nu)
    bwd = gen_gini_directed(y, x, nu)
    return max(0.0, 0.5 * fwd + 0.5 * bwd)


def gini_pairs(X: np.ndarray, I: np.ndarray, J: np.ndarray, nu: float, tab: np.ndarray | None = None) -> np.ndarray:
    """gen_gini_distance for row pairs (I[k], J[k]) of X (metrics.cpp:157-163)."""
    X = np.asarray(X, dtype=np.float64)
    d = X.shape[1]
    if tab is None:
        tab = survival_pow_table(d, nu)
    Z = X[I] - X[J]
    fwd = _directed_rows(Z, nu, tab)
    bwd = _directed_rows(X[J] - X[I], nu, tab)
    return np.maximum(0.0, 0.5 * fwd + 0.5 * bwd)


def pair_midranks(X: np.ndarray, I: np.ndarray, J: np.ndarray) -> np.ndarray:
    """Midranks of x_i - x_j (the forward ranks inside gen_gini_directed_checked)."""
    X = np.asarray(X, dtype=np.float64)
    return _midrank_rows(X[I] - X[J])


def from_matrix(m: np.ndarray) -> np.ndarray:  # DistanceMatrix::from_matrix, metrics.cpp:169-191
    m = np.array(m, dtype=np.float64, copy=True)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise InvalidInput("DistanceMatrix: matrix is not square")
    n = m.shape[0]
    if n < 1:
        raise InvalidInput("DistanceMatrix: matrix is empty")
    scale = float(np.max(np.abs(m)))  # NaN propagates like Eigen's maxCoeff ordering is irrelevant here
    tol = 1e-12 * max(scale, 1.0)
    diag = np.abs(np.diag(m))
    iu = np.triu_indices(n, 1)
    a = m[iu]
    b = m.T[iu]
    # The reference walks rows in order and throws the first violation it meets.
    for i in range(n):
        if diag[i] > tol:
            raise InvalidInput("DistanceMatrix: nonzero diagonal")
        row_a = m[i, i + 1 :]
        row_b = m[i + 1 :, i]
        bad_f = ~(np.isfinite(row_a) & np.isfinite(row_b))
        bad_s = np.abs(row_a - row_b) > tol
        bad_n = (row_a < -tol) | (row_b < -tol)
        first = np.flatnonzero(bad_f | bad_s | bad_n)
        if first.size:
            k = first[0]
            if bad_f[k]:
                raise InvalidInput("DistanceMatrix: non-finite entry")
            if bad_s[k]:
                raise InvalidInput("DistanceMatrix: asymmetric entries")
            raise InvalidInput("DistanceMatrix: negative entry")
    v = np.maximum(0.0, a)
    out = np.zeros_like(m)
    out[iu] = v
    out.T[iu] = v
    del b
    return out


def pairwise_matrix(X: np.ndarray, nu: float | None, chunk: int = 1 << 16) -> np.ndarray:
    """pairwise_matrix (metrics.cpp:193-237). nu=None selects the Euclidean branch."""
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    if n < 2:
        raise InvalidInput("pairwise_matrix: need at least 2 rows")
    if d < 1:
        raise InvalidInput("pairwise_matrix: need at least 1 column")
    D = np.zeros((n, n))
    iu, ju = np.triu_indices(n, 1)
    if nu is not None:
        nu = _check_nu(nu)
        tab = survival_pow_table(d, nu)
        for s in range(0, iu.size, chunk):
            I, J = iu[s : s + chunk], ju[s : s + chunk]
            if not (np.all(np.isfinite(X[I])) and np.all(np.isfinite(X[J]))):
                raise InvalidInput("gen_gini_directed: non-finite input entry")
            v = gini_pairs(X, I, J, nu, tab)
            D[I, J] = v
            D[J, I] = v
    else:
        for s in range(0, iu.size, chunk):
            I, J = iu[s : s + chunk], ju[s : s + chunk]
            delta = X[I] - X[J]
            sq = np.cumsum(delta * delta, axis=1)[:, -1]  # metrics.cpp:226-229, sequential
            v = np.sqrt(sq)
            D[I, J] = v
            D[J, I] = v
    return from_matrix(D)


# ---------------------------------------------------------------------------
# embed.cpp


@dataclass
class Embedding:  # embed.hpp:32-44
    coords: np.ndarray
    eigenvalues: np.ndarray | None = None
    stress: float = 0.0
    method: str = "classical"
    clamped_count: int = 0
    clamped_mass: float = 0.0
    converged: bool = True
    iterations: int = 0
    huber_delta: float = 0.0
    stress_history: list = field(default_factory=list)


def _triu(D: np.ndarray):
    n = D.shape[0]
    iu, ju = np.triu_indices(n, 1)
    return iu, ju, D[iu, ju]


def _dist(Y: np.ndarray, iu, ju) -> np.ndarray:  # embedded_distance, embed.cpp:32-34
    diff = Y[iu] - Y[ju]
    return np.sqrt(np.cumsum(diff * diff, axis=1)[:, -1])


def double_center(S: np.ndarray) -> np.ndarray:  # embed.cpp:382-413
    S = np.asarray(S, dtype=np.float64)
    n = S.shape[0]
    if n < 1 or S.ndim != 2 or S.shape[1] != n:
        raise InvalidInput("double_center: matrix is not square")
    if not np.all(np.isfinite(S)):
        raise InvalidInput("double_center: non-finite entry")
    scale = max(float(np.max(np.abs(S))), 1.0)
    tol = 1e-9 * scale
    for i in range(n):
        if abs(S[i, i]) > tol:
            raise InvalidInput("double_center: nonzero diagonal")
        if np.any(np.abs(S[i, i + 1 :] - S[i + 1 :, i]) > tol):
            raise InvalidInput("double_center: asymmetric input beyond tolerance")
        if np.any(S[i, i + 1 :] < -tol):
            raise InvalidInput("double_center: negative squared distance")
    r = S.mean(axis=1)
    g = r.mean()
    B = -0.5 * (S - r[:, None] - r[None, :] + g)
    B = np.triu(B) + np.triu(B, 1).T  # mirrored upper triangle (embed.cpp:404-411)
    return B


def kruskal_stress(Y: np.ndarray, D: np.ndarray) -> float:  # embed.cpp:462-475
    Y = np.asarray(Y, dtype=np.float64)
    if Y.shape[0] != D.shape[0]:
        raise InvalidInput(
            f"kruskal_stress: coords rows ({Y.shape[0]}) do not match distance matrix size ({D.shape[0]})")
    if not np.all(np.isfinite(Y)):
        raise InvalidInput("kruskal_stress: non-finite coordinates")
    iu, ju, d = _triu(D)
    e = _dist(Y, iu, ju) - d
    num, den = float(np.sum(e * e)), float(np.sum(d * d))
    if den <= 0.0:
        raise DegenerateInput("kruskal_stress: all-zero distance matrix")
    return math.sqrt(num / den)


def classical_mds(D: np.ndarray, p: int) -> Embedding:  # embed.cpp:415-460
    n = D.shape[0]
    if p < 1 or p > n - 1:
        raise InvalidInput(f"classical_mds: target dimension must satisfy 1 <= p <= n-1, got p={p} with n={n}")
    B = double_center(D * D)
    try:
        lam, V = np.linalg.eigh(B)  # ascending, like SelfAdjointEigenSolver
    except np.linalg.LinAlgError as exc:  # pragma: no cover
        raise NumericFailure("classical_mds: eigensolver failed") from exc
    total = float(np.sum(np.abs(lam)))
    neg = float(np.sum(-lam[lam < 0.0]))
    coords = np.zeros((n, p))
    eig = np.zeros(p)
    clamped = 0
    for c in range(p):
        src = n - 1 - c
        lm = float(lam[src])
        eig[c] = lm
        v = V[:, src].copy()
        arg = int(np.argmax(np.abs(v)))  # first index wins ties (embed.cpp:445-452)
        if v[arg] < 0.0:
            v = -v
        if lm < 0.0:
            clamped += 1
        coords[:, c] = v * math.sqrt(max(lm, 0.0))
    iu, ju, d = _triu(D)
    stress = kruskal_stress(coords, D) if float(np.sum(d * d)) > 0.0 else 0.0
    return Embedding(coords=coords, eigenvalues=eig, stress=stress, method="classical", clamped_count=clamped,
                     clamped_mass=(neg / total if total > 0.0 else 0.0))


@dataclass
class LossParams:  # embed.cpp:48-52
    huber_delta: float = 0.0
    sammon_scale: float = 0.0
    weights: np.ndarray | None = None


def resolve_params(kind: str, D: np.ndarray, huber_delta, weights, who: str) -> LossParams:  # embed.cpp:54-109
    p = LossParams()
    iu, ju, d = _triu(D)
    n = D.shape[0]
    if kind == "kruskal":
        if float(np.sum(d * d)) <= 0.0:
            raise DegenerateInput(f"{who}: all-zero distance matrix")
    elif kind == "huber":
        if huber_delta is None:
            raise InvalidConfig(f"{who}: huber_delta auto mode is resolved by minimize_stress; pass an explicit delta here")
        if not (huber_delta > 0.0):
            raise InvalidConfig(f"{who}: huber_delta must be > 0")
        p.huber_delta = float(huber_delta)
    elif kind == "sammon":
        if np.any(d <= 0.0):
            raise DegenerateInput(f"{who}: Sammon loss requires strictly positive off-diagonal distances (deduplicate points first)")
        p.sammon_scale = 1.0 / float(np.cumsum(d)[-1])
    elif kind == "smacof":
        if weights is not None:
            w = np.asarray(weights, dtype=np.float64)
            if w.shape != (n, n):
                raise InvalidConfig(f"{who}: smacof_weights size mismatch")
            wu, wl = w[iu, ju], w.T[iu, ju]
            if np.any(~(wu >= 0.0)) or np.any(np.abs(wu - wl) > 0.0):
                raise InvalidConfig(f"{who}: smacof_weights must be symmetric and nonnegative")
            p.weights = w
    else:
        raise InvalidConfig(f"unknown stress kind {kind}")
    return p


def loss_value(kind: str, Y: np.ndarray, D: np.ndarray, p: LossParams) -> float:  # embed.cpp:111-159
    iu, ju, d = _triu(D)
    dist = _dist(Y, iu, ju)
    if kind == "kruskal":
        e = dist - d
        return math.sqrt(float(np.sum(e * e)) / float(np.sum(d * d)))
    e = d - dist
    if kind == "huber":
        a = np.abs(e)
        delta = p.huber_delta
        return float(np.sum(np.where(a <= delta, 0.5 * e * e, delta * (a - 0.5 * delta))))
    if kind == "sammon":
        return p.sammon_scale * float(np.sum(e * e / d))
    w = p.weights[iu, ju] if p.weights is not None else 1.0
    return float(np.sum(w * e * e))


def gradient_value(kind: str, Y: np.ndarray, D: np.ndarray, p: LossParams) -> np.ndarray:  # embed.cpp:164-212
    n, q = Y.shape
    grad = np.zeros((n, q))
    iu, ju, d = _triu(D)
    dist = _dist(Y, iu, ju)
    if kind == "kruskal":
        e0 = dist - d
        num, den = float(np.sum(e0 * e0)), float(np.sum(d * d))
        ks = math.sqrt(num / den)
        if ks <= 0.0:
            return grad
        factor = 1.0 / (ks * den)
    keep = dist > 0.0
    iu, ju, d, dist = iu[keep], ju[keep], d[keep], dist[keep]
    e = d - dist
    if kind == "kruskal":
        qv = -factor * e
    elif kind == "huber":
        qv = -np.clip(e, -p.huber_delta, p.huber_delta)
    elif kind == "sammon":
        qv = -2.0 * p.sammon_scale * e / d
    else:
        w = p.weights[iu, ju] if p.weights is not None else 1.0
        qv = -2.0 * w * e
    g = (qv / dist)[:, None] * (Y[iu] - Y[ju])
    for t in range(q):
        grad[:, t] += np.bincount(iu, weights=g[:, t], minlength=n)
        grad[:, t] -= np.bincount(ju, weights=g[:, t], minlength=n)
    return grad


@dataclass
class IterativeResult:  # embed.cpp:214-220
    coords: np.ndarray
    loss: float = 0.0
    converged: bool = True
    iterations: int = 0
    history: list = field(default_factory=list)


_TINY = 1e-300  # embed.cpp:13


def gradient_descent(kind, Y, D, p, max_iters, rel_tol) -> IterativeResult:  # embed.cpp:222-272
    Y = np.array(Y, dtype=np.float64, copy=True)
    f = loss_value(kind, Y, D, p)
    hist = [f]
    step = 1.0
    armijo = 1e-4
    it = 0
    stalled = False
    while it < max_iters:
        g = gradient_value(kind, Y, D, p)
        gsq = float(np.sum(g * g))
        if gsq <= 0.0:
            stalled = True
            break
        accepted = False
        f_new = f
        trial = Y
        for _ in range(60):
            trial = Y - step * g
            f_new = loss_value(kind, trial, D, p)
            if f_new <= f - armijo * step * gsq:
                accepted = True
                break
            step *= 0.5
        if not accepted:
            stalled = True
            break
        Y = trial
        hist.append(f_new)
        decrease = (f - f_new) / max(f, _TINY)
        f = f_new
        step *= 2.0
        if decrease < rel_tol:
            it += 1
            stalled = True
            break
        it += 1
    return IterativeResult(coords=Y, loss=f, converged=stalled or it < max_iters, iterations=it, history=hist)


def guttman_transform(Z, D, weights, v_pinv) -> np.ndarray:  # embed.cpp:276-294
    n = D.shape[0]
    iu, ju, d = _triu(D)
    dist = _dist(Z, iu, ju)
    keep = dist > 0.0
    w = weights[iu, ju] if weights is not None else 1.0
    b = np.where(keep, -w * d / np.where(keep, dist, 1.0), 0.0)
    B = np.zeros((n, n))
    B[iu, ju] = b
    B[ju, iu] = b
    np.fill_diagonal(B, -B.sum(axis=1))
    if v_pinv is not None:
        return v_pinv @ (B @ Z)
    return (B @ Z) / float(n)


def smacof_iterate(Y, D, p, max_iters, rel_tol) -> IterativeResult:  # embed.cpp:296-347
    n = D.shape[0]
    v_pinv = None
    if p.weights is not None:
        W = p.weights.copy()
        np.fill_diagonal(W, 0.0)
        V = -W
        np.fill_diagonal(V, W.sum(axis=1))
        lam, U = np.linalg.eigh(V)
        cutoff = 1e-12 * max(float(np.max(np.abs(lam))), 1.0)
        inv = np.where(lam > cutoff, 1.0 / np.where(lam > cutoff, lam, 1.0), 0.0)
        v_pinv = (U * inv) @ U.T
    Y = np.array(Y, dtype=np.float64, copy=True)
    f = loss_value("smacof", Y, D, p)
    hist = [f]
    it = 0
    reached = False
    while it < max_iters:
        nxt = guttman_transform(Y, D, p.weights, v_pinv)
        f_new = loss_value("smacof", nxt, D, p)
        Y = nxt
        hist.append(f_new)
        decrease = (f - f_new) / max(f, _TINY)
        f = f_new
        it += 1
        if decrease < rel_tol:
            reached = True
            break
    return IterativeResult(coords=Y, loss=f, converged=reached or it < max_iters, iterations=it, history=hist)


def stress_loss(kind, Y, D, huber_delta=None, weights=None) -> float:  # embed.cpp:477-482
    _check_coords(Y, D, "stress_loss")
    return loss_value(kind, np.asarray(Y, float), D, resolve_params(kind, D, huber_delta, weights, "stress_loss"))


def stress_gradient(kind, Y, D, huber_delta=None, weights=None) -> np.ndarray:  # embed.cpp:484-489
    _check_coords(Y, D, "stress_gradient")
    return gradient_value(kind, np.asarray(Y, float), D, resolve_params(kind, D, huber_delta, weights, "stress_gradient"))


def _check_coords(Y, D, who):  # embed.cpp:15-21
    Y = np.asarray(Y)
    if Y.shape[0] != D.shape[0]:
        raise InvalidInput(f"{who}: coords rows ({Y.shape[0]}) do not match distance matrix size ({D.shape[0]})")
    if not np.all(np.isfinite(Y)):
        raise InvalidInput(f"{who}: non-finite coordinates")


def median_offdiag(D) -> float:  # embed.cpp:36-46
    _, _, v = _triu(D)
    v = np.sort(v)
    m = v.size
    return float(v[m // 2]) if m % 2 == 1 else 0.5 * float(v[m // 2 - 1] + v[m // 2])


def minimize_stress(D, p: int, kind: str = "smacof", huber_delta=None, weights=None, max_iters: int = 300,
                    rel_tol: float = 1e-6, Y0=None) -> Embedding:
    """minimize_stress (embed.cpp:491-532).  ``Y0`` injects a start layout in
    place of ``classical_mds(D, p).coords`` (embed.cpp:495) -- the seeded-init
    mode of BASELINE config 1; Y0=None is the reference exactly."""
    if max_iters < 1:
        raise InvalidConfig("minimize_stress: max_iters must be >= 1")
    if not (rel_tol > 0.0):
        raise InvalidConfig("minimize_stress: rel_tol must be > 0")
    init = classical_mds(D, p).coords if Y0 is None else np.array(Y0, dtype=np.float64)
    if kind == "huber" and huber_delta is None:
        med = median_offdiag(D)
        base = med if med > 0.0 else 1.0
        best, best_ks = None, math.inf
        for factor in (0.5, 1.0, 2.0):
            e = minimize_stress(D, p, kind, factor * base, weights, max_iters, rel_tol, Y0)
            ks = kruskal_stress(e.coords, D)
            if ks < best_ks:
                best_ks, best = ks, e
        return best
    params = resolve_params(kind, D, huber_delta, weights, "minimize_stress")
    if kind == "smacof":
        r = smacof_iterate(init, D, params, max_iters, rel_tol)
    else:
        r = gradient_descent(kind, init, D, params, max_iters, rel_tol)
    return Embedding(coords=r.coords, stress=r.loss, method=kind, converged=r.converged, iterations=r.iterations,
                     stress_history=r.history, huber_delta=(huber_delta if kind == "huber" else 0.0))


# ---------------------------------------------------------------------------
# tune.cpp


def nugrid_linspace(lo=1.1, hi=5.0, count=30) -> list[float]:  # tune.cpp:60-72
    if count < 1:
        raise InvalidConfig("NuGrid: count must be >= 1")
    if count == 1:
        vals = [lo]
    else:
        step = (hi - lo) / float(count - 1)
        vals = [lo + step * i for i in range(count)]
        vals[-1] = hi
    return nugrid_from_values(vals)


def nugrid_from_values(vals) -> list[float]:  # tune.cpp:74-83
    vals = [float(v) for v in vals]
    if not vals:
        raise InvalidConfig("NuGrid: empty grid")
    for i, v in enumerate(vals):
        if not (v > 1.0):
            raise InvalidConfig("NuGrid: every value must be > 1")
        if i > 0 and not (v > vals[i - 1]):
            raise InvalidConfig("NuGrid: values must be strictly increasing (no duplicates)")
    return vals


def make_folds(n: int, k: int, seed: int) -> list[list[int]]:  # tune.cpp:39-56
    idx = list(range(n))
    shuffle_indices(idx, Rng(seed))
    base, extra = n // k, n % k
    folds, off = [], 0
    for f in range(k):
        size = base + (1 if f < extra else 0)
        folds.append(sorted(idx[off : off + size]))
        off += size
    return folds


def embed_distances(D, p, method):  # tune.cpp:20-33
    if method == "classical":
        return classical_mds(D, p)
    return minimize_stress(D, p, kind=method)


@dataclass
class TuneReport:  # tune.hpp:27-34
    grid: list
    mean_stress: list
    nu_star: float
    best_embedding: Embedding
    folds: int
    seed: int


def tune_nu(X, p, grid, k_folds, method="classical", seed=0) -> TuneReport:  # tune.cpp:85-135
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    grid = nugrid_from_values(grid)
    if k_folds < 1:
        raise InvalidConfig("tune_nu: k_folds must be >= 1")
    if n < k_folds:
        raise InvalidConfig("tune_nu: more folds than rows")
    folds = make_folds(n, k_folds, seed)
    for fold in folds:
        if len(fold) < p + 1:
            raise InvalidConfig(f"tune_nu: a fold has {len(fold)} points, need at least p + 1 = {p + 1}")
    cell = np.zeros((len(grid), k_folds))
    for g, nu in enumerate(grid):
        for f, fold in enumerate(folds):
            D = pairwise_matrix(X[fold], nu)
            if float(D.max()) <= 0.0:
                cell[g, f] = 0.0
                continue
            e = embed_distances(D, p, method)
            cell[g, f] = kruskal_stress(e.coords, D)
    mean = [float(np.cumsum(cell[g])[-1] / float(k_folds)) for g in range(len(grid))]
    best = 0
    for g in range(1, len(grid)):
        if mean[g] < mean[best]:
            best = g
    nu_star = grid[best]
    full = pairwise_matrix(X, nu_star)
    return TuneReport(grid=grid, mean_stress=mean, nu_star=nu_star, best_embedding=embed_distances(full, p, method),
                      folds=k_folds, seed=seed)


@dataclass
class AlternatingResult:  # tune.hpp:36-40
    embedding: Embedding
    nu_star: float
    nu_path: list


def alternating_tune(X, p, outer_iters, grid, seed=0) -> AlternatingResult:  # tune.cpp:137-167
    if outer_iters < 1:
        raise InvalidConfig("alternating_tune: need at least one outer iteration")
    grid = nugrid_from_values(grid)
    X = np.asarray(X, dtype=np.float64)
    nu = 2.0
    path = []
    emb = None
    for _ in range(outer_iters):
        D = pairwise_matrix(X, nu)
        emb = minimize_stress(D, p, kind="sammon")
        sweep = [kruskal_stress(emb.coords, pairwise_matrix(X, g)) for g in grid]
        best = 0
        for g in range(1, len(grid)):
            if sweep[g] < sweep[best]:
                best = g
        nu = grid[best]
        path.append(nu)
    return AlternatingResult(embedding=emb, nu_star=nu, nu_path=path)


# ---------------------------------------------------------------------------
# The reference tests' input generators (test_util.hpp:15-39), for fixtures.


def random_vector(rng: Rng, d: int, scale: float = 1.0) -> np.ndarray:
    return np.array([scale * (2.0 * rng.uniform01() - 1.0) for _ in range(d)])


def random_vector_with_ties(rng: Rng, d: int) -> np.ndarray:
    scale = math.pow(10.0, float(rng.uniform_below(5)) - 2.0)
    v = random_vector(rng, d, scale)
    if rng.uniform01() < 0.4:
        v = np.array([_cpp_round(x * 4.0 / scale) * scale / 4.0 for x in v])
    return v


def _cpp_round(x: float) -> float:
    """std::round: halves away from zero (numpy rounds halves to even)."""
    if x < 0:
        return -_cpp_round(-x)
    f = math.floor(x)
    return f + 1.0 if x - f >= 0.5 else f


def random_matrix(rng: Rng, rows: int, cols: int, scale: float = 1.0) -> np.ndarray:
    m = np.zeros((rows, cols))
    for i in range(rows):
        for j in range(cols):
            m[i, j] = scale * (2.0 * rng.uniform01() - 1.0)
    return m
