"""ctypes binding of oracle/_ref/libginimds_ref.so -- TEST INFRASTRUCTURE ONLY.

The library is the UNMODIFIED reference core compiled by oracle/Makefile
(see oracle/ref_capi.cpp).  ``load()`` returns None when it has not been
built (e.g. on a box that never had /root/reference); callers skip then.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libginimds_ref.so")

_dp = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64
_lib = None


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        return None
    L = ctypes.CDLL(LIB_PATH)
    L.ref_last_error.restype = ctypes.c_char_p
    L.ref_rng_new.restype = ctypes.c_void_p
    L.ref_rng_new.argtypes = [ctypes.c_uint64]
    L.ref_rng_free.argtypes = [ctypes.c_void_p]
    L.ref_rng_uniform01.restype = ctypes.c_double
    L.ref_rng_uniform01.argtypes = [ctypes.c_void_p]
    L.ref_rng_uniform_below.restype = ctypes.c_uint64
    L.ref_rng_uniform_below.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
    L.ref_rng_normal.restype = ctypes.c_double
    L.ref_rng_normal.argtypes = [ctypes.c_void_p]
    L.ref_rng_log_normal.restype = ctypes.c_double
    L.ref_rng_log_normal.argtypes = [ctypes.c_void_p, ctypes.c_double]
    L.ref_mix_seed.restype = ctypes.c_uint64
    L.ref_mix_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
    L.ref_max_threads.restype = ctypes.c_int
    _lib = L
    return L


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _check(rc: int):
    if rc != 0:
        raise RefError(rc, _lib.ref_last_error().decode())


def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def set_max_threads(n: int):
    load().ref_set_max_threads(ctypes.c_int(n))


def max_threads() -> int:
    return load().ref_max_threads()


def midrank(v):
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.zeros(v.size)
    _check(load().ref_midrank(_p(v), _i64(v.size), _p(out)))
    return out


def _xy(fn, x, y, *extra):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros(1)
    _check(fn(_p(x), _i64(x.size), _p(y), _i64(y.size), *extra, _p(out)))
    return float(out[0])


def gen_gini_distance(x, y, nu):
    return _xy(load().ref_gen_gini_distance, x, y, ctypes.c_double(nu))


def gen_gini_directed(x, y, nu):
    return _xy(load().ref_gen_gini_directed, x, y, ctypes.c_double(nu))


def gini_pseudo_distance(x, y):
    return _xy(load().ref_gini_pseudo_distance, x, y)


def gini_norm(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(1)
    _check(load().ref_gini_norm(_p(x), _i64(x.size), _p(out)))
    return float(out[0])


def empirical_survival(z):
    z = np.ascontiguousarray(z, dtype=np.float64)
    out = np.zeros(z.size)
    _check(load().ref_empirical_survival(_p(z), _i64(z.size), _p(out)))
    return out


def pairwise_matrix(X, nu=None):
    X = _f(X)
    n, p = X.shape
    D = np.zeros((n, n), order="F")
    _check(load().ref_pairwise_matrix(_p(X), _i64(n), _i64(p), ctypes.c_double(nu or 0.0),
                                      ctypes.c_int(1 if nu is None else 0), _p(D)))
    return np.ascontiguousarray(D)


def gini_rows(X, nu, r0, r1):
    """Rows [r0, r1) of the Gini matrix (upper part only), reference per-pair code."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, p = X.shape
    out = np.zeros((r1 - r0, n))
    _check(load().ref_gini_rows(_p(X), _i64(n), _i64(p), ctypes.c_double(nu), _i64(r0), _i64(r1), _p(out)))
    return out


def from_matrix(M):
    M = _f(M)
    out = np.zeros_like(M, order="F")
    _check(load().ref_distance_matrix_validate(_p(M), _i64(M.shape[0]), _p(out)))
    return np.ascontiguousarray(out)


def double_center(S):
    S = _f(S)
    out = np.zeros_like(S, order="F")
    _check(load().ref_double_center(_p(S), _i64(S.shape[0]), _p(out)))
    return np.ascontiguousarray(out)


def classical_mds(D, q):
    D = _f(D)
    n = D.shape[0]
    coords = np.zeros((n, q), order="F")
    ev = np.zeros(q)
    cc = ctypes.c_int()
    cm = ctypes.c_double()
    st = ctypes.c_double()
    _check(load().ref_classical_mds(_p(D), _i64(n), ctypes.c_int(q), _p(coords), _p(ev), ctypes.byref(cc),
                                    ctypes.byref(cm), ctypes.byref(st)))
    return dict(coords=np.ascontiguousarray(coords), eigenvalues=ev, clamped_count=cc.value,
                clamped_mass=cm.value, stress=st.value)


KIND = {"kruskal": 0, "huber": 1, "sammon": 2, "smacof": 3}
METHOD = {"classical": 0, "kruskal": 1, "huber": 2, "sammon": 3, "smacof": 4}


def kruskal_stress(Y, D):
    Y, D = _f(Y), _f(D)
    out = np.zeros(1)
    _check(load().ref_kruskal_stress(_p(Y), _i64(Y.shape[0]), ctypes.c_int(Y.shape[1]), _p(D), _p(out)))
    return float(out[0])


def _w(weights):
    return None if weights is None else _p(_f(weights))


def stress_loss(kind, Y, D, huber_delta=None, weights=None):
    Y, D = _f(Y), _f(D)
    out = np.zeros(1)
    wk = None if weights is None else _f(weights)
    _check(load().ref_stress_loss(ctypes.c_int(KIND[kind]), _p(Y), _i64(Y.shape[0]), ctypes.c_int(Y.shape[1]), _p(D),
                                  ctypes.c_double(math.nan if huber_delta is None else huber_delta),
                                  None if wk is None else _p(wk), _p(out)))
    return float(out[0])


def stress_gradient(kind, Y, D, huber_delta=None, weights=None):
    Y, D = _f(Y), _f(D)
    g = np.zeros_like(Y, order="F")
    wk = None if weights is None else _f(weights)
    _check(load().ref_stress_gradient(ctypes.c_int(KIND[kind]), _p(Y), _i64(Y.shape[0]), ctypes.c_int(Y.shape[1]),
                                      _p(D), ctypes.c_double(math.nan if huber_delta is None else huber_delta),
                                      None if wk is None else _p(wk), _p(g)))
    return np.ascontiguousarray(g)


def minimize_stress(D, q, kind="smacof", huber_delta=None, weights=None, max_iters=300, rel_tol=1e-6):
    D = _f(D)
    n = D.shape[0]
    coords = np.zeros((n, q), order="F")
    cap = max_iters + 2
    hist = np.zeros(cap)
    hl = ctypes.c_int64()
    it = ctypes.c_int()
    conv = ctypes.c_int()
    st = ctypes.c_double()
    hd = ctypes.c_double()
    wk = None if weights is None else _f(weights)
    _check(load().ref_minimize_stress(_p(D), _i64(n), ctypes.c_int(q), ctypes.c_int(KIND[kind]),
                                      ctypes.c_double(math.nan if huber_delta is None else huber_delta),
                                      None if wk is None else _p(wk), ctypes.c_int(max_iters),
                                      ctypes.c_double(rel_tol), _p(coords), _p(hist), _i64(cap), ctypes.byref(hl),
                                      ctypes.byref(it), ctypes.byref(conv), ctypes.byref(st), ctypes.byref(hd)))
    return dict(coords=np.ascontiguousarray(coords), stress_history=list(hist[: hl.value]), iterations=it.value,
                converged=bool(conv.value), stress=st.value, huber_delta=hd.value)


def tune_nu(X, q, grid, k_folds, method="classical", seed=0):
    X = _f(X)
    g = np.ascontiguousarray(grid, dtype=np.float64)
    ms = np.zeros(g.size)
    ns = ctypes.c_double()
    coords = np.zeros((X.shape[0], q), order="F")
    bs = ctypes.c_double()
    _check(load().ref_tune_nu(_p(X), _i64(X.shape[0]), _i64(X.shape[1]), ctypes.c_int(q), _p(g), _i64(g.size),
                              ctypes.c_int(k_folds), ctypes.c_int(METHOD[method]), ctypes.c_uint64(seed), _p(ms),
                              ctypes.byref(ns), _p(coords), ctypes.byref(bs)))
    return dict(mean_stress=list(ms), nu_star=ns.value, coords=np.ascontiguousarray(coords), stress=bs.value)


def alternating_tune(X, q, outer, grid, seed=0):
    X = _f(X)
    g = np.ascontiguousarray(grid, dtype=np.float64)
    path = np.zeros(outer)
    ns = ctypes.c_double()
    coords = np.zeros((X.shape[0], q), order="F")
    st = ctypes.c_double()
    _check(load().ref_alternating_tune(_p(X), _i64(X.shape[0]), _i64(X.shape[1]), ctypes.c_int(q), ctypes.c_int(outer),
                                       _p(g), _i64(g.size), ctypes.c_uint64(seed), _p(path), ctypes.byref(ns),
                                       _p(coords), ctypes.byref(st)))
    return dict(nu_path=list(path), nu_star=ns.value, coords=np.ascontiguousarray(coords), stress=st.value)


class RefRng:
    def __init__(self, seed: int):
        self._h = load().ref_rng_new(ctypes.c_uint64(seed))

    def __del__(self):
        if getattr(self, "_h", None):
            load().ref_rng_free(self._h)

    def uniform01(self):
        return load().ref_rng_uniform01(self._h)

    def uniform_below(self, b):
        return load().ref_rng_uniform_below(self._h, ctypes.c_uint64(b))

    def normal(self):
        return load().ref_rng_normal(self._h)


# ---- seeded-init iterate loops and sampled pairs (oracle/ref_seeded.cpp) ----
SEEDED_PATH = os.path.join(HERE, "_ref", "libginimds_ref_seeded.so")
_seeded = None


def load_seeded():
    """The reference's gradient_descent / smacof_iterate (embed.cpp:222-347) with a
    caller-supplied start, and gen_gini_distance over a pair list.
    None when oracle/_ref was not built."""
    global _seeded
    if _seeded is not None:
        return _seeded
    if not os.path.exists(SEEDED_PATH):
        return None
    L = ctypes.CDLL(SEEDED_PATH)
    L.ref_seeded_last_error.restype = ctypes.c_char_p
    _seeded = L
    return L


def _check_seeded(rc: int):
    if rc != 0:
        raise RefError(rc, _seeded.ref_seeded_last_error().decode())


def seeded_fit(D, Y0, kind="kruskal", huber_delta=None, max_iters=300, rel_tol=1e-6):
    """minimize_stress with Y0 in place of the classical init (embed.cpp:518-522)."""
    L = load_seeded()
    D = _f(D)
    n = D.shape[0]
    Y0 = _f(Y0)
    q = Y0.shape[1]
    coords = np.zeros((n, q), order="F")
    cap = max_iters + 2
    hist = np.zeros(cap)
    hl, it, conv, loss = ctypes.c_int64(), ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    _check_seeded(L.ref_seeded_fit(_p(D), _i64(n), ctypes.c_int(q), ctypes.c_int(KIND[kind]),
                                   ctypes.c_double(math.nan if huber_delta is None else huber_delta),
                                   ctypes.c_int(max_iters), ctypes.c_double(rel_tol), _p(Y0), _p(coords), _p(hist),
                                   _i64(cap), ctypes.byref(hl), ctypes.byref(it), ctypes.byref(conv),
                                   ctypes.byref(loss)))
    return dict(coords=np.ascontiguousarray(coords), stress_history=list(hist[: hl.value]), iterations=it.value,
                converged=bool(conv.value), stress=loss.value)


def gini_pairs(X, I, J, nu):
    """gen_gini_distance(X[I[k]], X[J[k]], nu) for every k (the reference's own per-pair call)."""
    L = load_seeded()
    X = np.ascontiguousarray(X, dtype=np.float64)
    I = np.ascontiguousarray(I, dtype=np.int64)
    J = np.ascontiguousarray(J, dtype=np.int64)
    out = np.zeros(I.size)
    ip = ctypes.POINTER(ctypes.c_int64)
    _check_seeded(L.ref_gini_pairs(_p(X), _i64(X.shape[0]), _i64(X.shape[1]), ctypes.c_double(nu),
                                   I.ctypes.data_as(ip), J.ctypes.data_as(ip), _i64(I.size), _p(out)))
    return out
