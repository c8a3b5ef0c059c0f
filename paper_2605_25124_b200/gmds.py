"""ctypes binding of libgmds.so (the C-ABI declared in include/gmds.h).

This is how tests/ and bench.py reach the CUDA engine: every call below goes
through the same extern "C" entry points a C/C++/Go/... caller would bind.
There is no fallback -- if the shared library is missing or no CUDA device
is visible, calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GMDS_LIB_PATH") or os.path.join(HERE, "lib", "libgmds.so")  # override: experiments

OK, INVALID_INPUT, INVALID_CONFIG, DEGENERATE_INPUT, NUMERIC_FAILURE, ERROR, CUDA_ERROR, NCCL_ERROR = range(8)
F32, F64 = 0, 1
ROW_MAJOR, COL_MAJOR = 0, 1
KIND = {"kruskal": 0, "huber": 1, "sammon": 2, "smacof": 3}
METHOD = {"classical": 0, "kruskal": 1, "huber": 2, "sammon": 3, "smacof": 4}


class GmdsError(Exception):
    """Base class; mirrors ginimds::Error (error.hpp:9-13)."""

    status = ERROR

    def __init__(self, msg: str):
        super().__init__(msg)


class InvalidInput(GmdsError):
    status = INVALID_INPUT


class InvalidConfig(GmdsError):
    status = INVALID_CONFIG


class DegenerateInput(GmdsError):
    status = DEGENERATE_INPUT


class NumericFailure(GmdsError):
    status = NUMERIC_FAILURE


class CudaError(GmdsError):
    status = CUDA_ERROR


class NcclError(GmdsError):
    status = NCCL_ERROR


_ERRORS = {c.status: c for c in (InvalidInput, InvalidConfig, DegenerateInput, NumericFailure, CudaError, NcclError)}

_lib = None
_dp = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


class StressCfg(ctypes.Structure):  # gmds_stress_cfg
    _fields_ = [("kind", ctypes.c_int32), ("huber_delta", ctypes.c_double), ("smacof_weights", _dp),
                ("max_iters", ctypes.c_int32), ("rel_tol", ctypes.c_double), ("seed", ctypes.c_uint64)]


class FitResult(ctypes.Structure):  # gmds_fit_result
    _fields_ = [("coords", _dp), ("history", _dp), ("history_cap", ctypes.c_int64), ("history_len", ctypes.c_int64),
                ("iterations", ctypes.c_int32), ("converged", ctypes.c_int32), ("stress", ctypes.c_double),
                ("huber_delta", ctypes.c_double), ("passes", ctypes.c_int64)]


def lib():
    """Load libgmds.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        L.gmds_last_error.restype = ctypes.c_char_p
        L.gmds_version.restype = ctypes.c_char_p
        L.gmds_launch_count.restype = ctypes.c_int64
        L.gmds_packed_elems.restype = ctypes.c_int64
        L.gmds_packed_elems.argtypes = [ctypes.c_int64]
        L.gmds_dmat_n.restype = ctypes.c_int64
        L.gmds_dmat_n.argtypes = [ctypes.c_void_p]
        L.gmds_dmat_free.argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != OK:
        msg = lib().gmds_last_error().decode()
        raise _ERRORS.get(rc, GmdsError)(msg)


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _vp(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _xarg(X):
    """(contiguous array, dtype code, layout code) for an n x p input."""
    X = np.asarray(X)
    if X.dtype == np.float32:
        xt = F32
    else:
        X = X.astype(np.float64, copy=False)
        xt = F64
    if X.flags.c_contiguous:
        return X, xt, ROW_MAJOR
    if X.flags.f_contiguous:
        return X, xt, COL_MAJOR
    return np.ascontiguousarray(X), xt, ROW_MAJOR


def version() -> str:
    return lib().gmds_version().decode()


def device_count() -> int:
    return lib().gmds_device_count()


def launch_count() -> int:
    return lib().gmds_launch_count()


def packed_elems(n: int) -> int:
    return lib().gmds_packed_elems(n)


# ---- metrics ---------------------------------------------------------------------------------------


def midrank_batch(V) -> np.ndarray:
    V = np.ascontiguousarray(V, dtype=np.float64)
    if V.ndim == 1:
        V = V[None, :]
    m, d = V.shape
    out = np.zeros((m, d))
    _check(lib().gmds_midrank_batch(_p(V), _i64(m), _i64(d), _p(out)))
    return out


def midrank(v) -> np.ndarray:
    """metrics.hpp:71-72."""
    return midrank_batch(np.asarray(v, dtype=np.float64).ravel()[None, :])[0]


def pair_midranks(X, I, J) -> np.ndarray:
    X, xt, lx = _xarg(X)
    n, p = X.shape
    pairs = np.ascontiguousarray(np.stack([np.asarray(I), np.asarray(J)], axis=1).astype(np.int64))
    out = np.zeros((pairs.shape[0], p))
    _check(lib().gmds_pair_midranks(_vp(X), _i32(xt), _i32(lx), _i64(n), _i64(p),
                                    pairs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _i64(pairs.shape[0]),
                                    _p(out)))
    return out


def gen_gini_distance(x, y, nu: float) -> float:
    """metrics.hpp:105-107."""
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    y = np.ascontiguousarray(y, dtype=np.float64).ravel()
    out = np.zeros(1)
    _check(lib().gmds_gen_gini_distance(_p(x), _i64(x.size), _p(y), _i64(y.size), ctypes.c_double(nu), _p(out)))
    return float(out[0])


def pairwise_gini(X, nus, out_dtype=np.float64, out=None) -> np.ndarray:
    """pairwise_matrix(X, gini(nu)) for every nu at once -> (len(nus), n, n).
    `out` may be a caller buffer of that shape (e.g. pinned host memory, which
    the library fills row stripe by row stripe while later tiles compute)."""
    X, xt, lx = _xarg(X)
    n, p = X.shape
    nus = np.ascontiguousarray(np.atleast_1d(np.asarray(nus, dtype=np.float64)))
    ot = F32 if np.dtype(out_dtype) == np.float32 else F64
    shape, dt = (nus.size, n, n), (np.float32 if ot == F32 else np.float64)
    if out is None:
        out = np.zeros(shape, dtype=dt)
    elif out.shape != shape or out.dtype != dt or not out.flags.c_contiguous:
        raise ValueError("pairwise_gini: out must be a C-contiguous %s array of shape %s" % (np.dtype(dt), shape))
    _check(lib().gmds_pairwise_gini(_vp(X), _i32(xt), _i32(lx), _i64(n), _i64(p), _p(nus), _i32(nus.size), _i32(ot),
                                    _vp(out)))
    return out


def pairwise_matrix(X, nu=None) -> np.ndarray:
    """metrics.hpp:112: nu=None selects MetricSpec::euclidean()."""
    if nu is None:
        X, xt, lx = _xarg(X)
        n, p = X.shape
        out = np.zeros((n, n))
        _check(lib().gmds_pairwise_euclidean(_vp(X), _i32(xt), _i32(lx), _i64(n), _i64(p), _p(out)))
        return out
    return pairwise_gini(X, [nu])[0]


def pairwise_gini_device(dX_ptr: int, xt: int, n: int, p: int, nus, out_t: int, packed: bool, dD_ptr: int,
                         shard: int = 0, nshards: int = 1, stream: int = 0):
    """Device-pointer entry (inputs already in HBM); pointers are raw CUDA addresses."""
    nus = np.ascontiguousarray(np.atleast_1d(np.asarray(nus, dtype=np.float64)))
    _check(lib().gmds_pairwise_gini_device(ctypes.c_void_p(dX_ptr), _i32(xt), _i64(n), _i64(p), _p(nus),
                                           _i32(nus.size), _i32(out_t), _i32(1 if packed else 0),
                                           ctypes.c_void_p(dD_ptr), _i32(shard), _i32(nshards),
                                           ctypes.c_void_p(stream)))


# ---- device DistanceMatrix + stress (embed.hpp) ---------------------------------------------------


class DMat:
    """Owning handle of a device-resident DistanceMatrix (packed upper triangle)."""

    def __init__(self, handle: int, n: int):
        self._h = ctypes.c_void_p(handle)
        self.n = n

    @property
    def handle(self):
        return self._h

    def download(self) -> np.ndarray:
        out = np.zeros((self.n, self.n))
        _check(lib().gmds_dmat_download(self._h, _p(out)))
        return out

    def free(self):
        if self._h:
            lib().gmds_dmat_free(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def dmat_from_host(D, storage=F64) -> DMat:
    """DistanceMatrix::from_matrix (metrics.cpp:169-191) + upload."""
    D = np.asfortranarray(np.asarray(D, dtype=np.float64))
    n = D.shape[0]
    if D.ndim != 2 or D.shape[1] != n:
        raise InvalidInput("DistanceMatrix: matrix is not square")
    h = ctypes.c_void_p()
    _check(lib().gmds_dmat_from_host(_p(D), _i64(n), _i32(storage), ctypes.byref(h)))
    return DMat(h.value, n)


def dmat_gini(X, nu: float, storage=F64) -> DMat:
    """pairwise_matrix(X, gini(nu)) kept on the device."""
    X, xt, lx = _xarg(X)
    n, p = X.shape
    h = ctypes.c_void_p()
    _check(lib().gmds_dmat_gini(_vp(X), _i32(xt), _i32(lx), _i64(n), _i64(p), ctypes.c_double(nu), _i32(storage),
                                ctypes.byref(h)))
    return DMat(h.value, n)


def dmat_gini_device(dX_ptr: int, xt: int, n: int, p: int, nu: float, storage=F32) -> DMat:
    h = ctypes.c_void_p()
    _check(lib().gmds_dmat_gini_device(ctypes.c_void_p(dX_ptr), _i32(xt), _i64(n), _i64(p), ctypes.c_double(nu),
                                       _i32(storage), ctypes.byref(h)))
    return DMat(h.value, n)


def _as_dmat(D, storage=F64) -> DMat:
    return D if isinstance(D, DMat) else dmat_from_host(D, storage)


def _coords(Y):
    Y = np.asfortranarray(np.asarray(Y, dtype=np.float64))
    if Y.ndim == 1:
        Y = Y[:, None]
    return Y


def kruskal_stress(Y, D) -> float:
    Dm = _as_dmat(D)
    Y = _coords(Y)
    if Y.shape[0] != Dm.n:
        raise InvalidInput(f"kruskal_stress: coords rows ({Y.shape[0]}) do not match distance matrix size ({Dm.n})")
    out = np.zeros(1)
    _check(lib().gmds_kruskal_stress(Dm.handle, _p(Y), _i32(Y.shape[1]), _p(out)))
    return float(out[0])


def _hd(huber_delta):
    return ctypes.c_double(math.nan if huber_delta is None else float(huber_delta))


def _wp(weights):
    if weights is None:
        return None, None
    W = np.asfortranarray(np.asarray(weights, dtype=np.float64))
    return W, _p(W)


def stress_loss(kind: str, Y, D, huber_delta=None, weights=None) -> float:
    Dm = _as_dmat(D)
    Y = _coords(Y)
    if Y.shape[0] != Dm.n:
        raise InvalidInput(f"stress_loss: coords rows ({Y.shape[0]}) do not match distance matrix size ({Dm.n})")
    W, wp = _wp(weights)
    out = np.zeros(1)
    _check(lib().gmds_stress_loss(_i32(KIND[kind]), Dm.handle, _p(Y), _i32(Y.shape[1]), _hd(huber_delta), wp, _p(out)))
    return float(out[0])


def stress_gradient(kind: str, Y, D, huber_delta=None, weights=None) -> np.ndarray:
    Dm = _as_dmat(D)
    Y = _coords(Y)
    if Y.shape[0] != Dm.n:
        raise InvalidInput(f"stress_gradient: coords rows ({Y.shape[0]}) do not match distance matrix size ({Dm.n})")
    W, wp = _wp(weights)
    g = np.zeros(Y.shape, order="F")
    _check(lib().gmds_stress_gradient(_i32(KIND[kind]), Dm.handle, _p(Y), _i32(Y.shape[1]), _hd(huber_delta), wp,
                                      _p(g)))
    return np.ascontiguousarray(g)


def classical_mds(D, q: int) -> dict:
    Dm = _as_dmat(D)
    coords = np.zeros((Dm.n, q), order="F")
    ev = np.zeros(max(q, 1))
    cc = ctypes.c_int32()
    cm = ctypes.c_double()
    st = ctypes.c_double()
    _check(lib().gmds_classical_mds(Dm.handle, _i32(q), _p(coords), _p(ev), ctypes.byref(cc), ctypes.byref(cm),
                                    ctypes.byref(st)))
    return dict(coords=np.ascontiguousarray(coords), eigenvalues=ev[:q], clamped_count=cc.value,
                clamped_mass=cm.value, stress=st.value)


def classical_mds_topq(D, q: int, tol: float = 1e-10, max_iters: int = 2000) -> dict:
    """Top-q classical MDS by device subspace iteration."""
    Dm = _as_dmat(D)
    coords = np.zeros((Dm.n, q), order="F")
    ev = np.zeros(max(q, 1))
    cc = ctypes.c_int32()
    its = ctypes.c_int32()
    _check(lib().gmds_classical_mds_topq(Dm.handle, _i32(q), ctypes.c_double(tol), _i32(max_iters), _p(coords),
                                         _p(ev), ctypes.byref(cc), ctypes.byref(its)))
    return dict(coords=np.ascontiguousarray(coords), eigenvalues=ev[:q], clamped_count=cc.value,
                iterations=its.value)


def minimize_stress(D, q: int, kind: str = "smacof", huber_delta=None, weights=None, max_iters: int = 300,
                    rel_tol: float = 1e-6, Y0=None, storage=F64) -> dict:
    """minimize_stress (embed.cpp:491-532); Y0 = seeded-init mode."""
    Dm = _as_dmat(D, storage)
    W, wp = _wp(weights)
    cfg = StressCfg(kind=KIND[kind], huber_delta=(math.nan if huber_delta is None else float(huber_delta)),
                    smacof_weights=wp, max_iters=int(max_iters), rel_tol=float(rel_tol), seed=0)
    coords = np.zeros((Dm.n, q), order="F")
    cap = int(max_iters) + 2
    hist = np.zeros(cap)
    res = FitResult(coords=_p(coords), history=_p(hist), history_cap=cap)
    y0 = None
    if Y0 is not None:
        y0 = _coords(Y0)
        if y0.shape != (Dm.n, q):
            raise InvalidInput("minimize_stress: Y0 shape mismatch")
    _check(lib().gmds_minimize_stress(Dm.handle, _i32(q), ctypes.byref(cfg), None if y0 is None else _p(y0),
                                      ctypes.byref(res)))
    return dict(coords=np.ascontiguousarray(coords), stress_history=list(hist[: min(res.history_len, cap)]),
                iterations=res.iterations, converged=bool(res.converged), stress=res.stress,
                huber_delta=res.huber_delta, passes=res.passes)


# ---- tune (tune.hpp) --------------------------------------------------------------------------------


def tune_nu(X, q: int, grid, k_folds: int, method: str = "classical", seed: int = 0) -> dict:
    """tune_nu (tune.cpp:85-135)."""
    X, xt, lx = _xarg(X)
    n, p = X.shape
    g = np.ascontiguousarray(np.asarray(grid, dtype=np.float64))
    ms = np.zeros(max(g.size, 1))
    ns = ctypes.c_double()
    st = ctypes.c_double()
    coords = np.zeros((n, q), order="F")
    _check(lib().gmds_tune_nu(_vp(X), _i32(xt), _i32(lx), _i64(n), _i64(p), _i32(q), _p(g), _i32(g.size),
                              _i32(k_folds), _i32(METHOD[method]), ctypes.c_uint64(seed), _p(ms), ctypes.byref(ns),
                              _p(coords), ctypes.byref(st)))
    return dict(mean_stress=list(ms[: g.size]), nu_star=ns.value, coords=np.ascontiguousarray(coords), stress=st.value)


def alternating_tune(X, q: int, outer_iters: int, grid, seed: int = 0) -> dict:
    """alternating_tune (tune.cpp:137-167)."""
    X, xt, lx = _xarg(X)
    n, p = X.shape
    g = np.ascontiguousarray(np.asarray(grid, dtype=np.float64))
    path = np.zeros(max(outer_iters, 1))
    ns = ctypes.c_double()
    st = ctypes.c_double()
    coords = np.zeros((n, q), order="F")
    _check(lib().gmds_alternating_tune(_vp(X), _i32(xt), _i32(lx), _i64(n), _i64(p), _i32(q), _i32(outer_iters),
                                       _p(g), _i32(g.size), ctypes.c_uint64(seed), _p(path), ctypes.byref(ns),
                                       _p(coords), ctypes.byref(st)))
    return dict(nu_path=list(path[:outer_iters]), nu_star=ns.value, coords=np.ascontiguousarray(coords),
                stress=st.value)


# ---- remaining metrics / embed entry points -------------------------------------------------------


def gen_gini_directed(x, y, nu: float) -> float:
    """metrics.hpp:95-97."""
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    y = np.ascontiguousarray(y, dtype=np.float64).ravel()
    out = np.zeros(1)
    _check(lib().gmds_gen_gini_directed(_p(x), _i64(x.size), _p(y), _i64(y.size), ctypes.c_double(nu), _p(out)))
    return float(out[0])


def gini_norm(x) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    out = np.zeros(1)
    _check(lib().gmds_gini_norm(_p(x), _i64(x.size), _p(out)))
    return float(out[0])


def gini_pseudo_distance(x, y) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    y = np.ascontiguousarray(y, dtype=np.float64).ravel()
    out = np.zeros(1)
    _check(lib().gmds_gini_pseudo_distance(_p(x), _i64(x.size), _p(y), _i64(y.size), _p(out)))
    return float(out[0])


def empirical_survival(z) -> np.ndarray:
    z = np.ascontiguousarray(z, dtype=np.float64).ravel()
    out = np.zeros(z.size)
    _check(lib().gmds_empirical_survival(_p(z), _i64(z.size), _p(out)))
    return out


def double_center(S) -> np.ndarray:
    S = np.asfortranarray(np.asarray(S, dtype=np.float64))
    if S.ndim != 2 or S.shape[0] != S.shape[1] or S.shape[0] < 1:
        raise InvalidInput("double_center: matrix is not square")
    out = np.zeros_like(S, order="F")
    _check(lib().gmds_double_center(_p(S), _i64(S.shape[0]), _p(out)))
    return np.ascontiguousarray(out)


def nu_sweep_kruskal(X, Y, grid) -> np.ndarray:
    """kruskal_stress(Y, pairwise_matrix(X, gini(nu))) for every grid nu, one distance pass."""
    X, xt, lx = _xarg(X)
    n, p = X.shape
    Y = _coords(Y)
    g = np.ascontiguousarray(np.asarray(grid, dtype=np.float64))
    out = np.zeros(g.size)
    _check(lib().gmds_nu_sweep_kruskal(_vp(X), _i32(xt), _i32(lx), _i64(n), _i64(p), _p(Y), _i32(Y.shape[1]), _p(g),
                                       _i32(g.size), _p(out)))
    return out


# ---- multi-GPU: collectives + row-sharded D / fit, sharded nu sweep -----------------


class Comm:
    """One rank's collective handle (gmds_comm)."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)

    @property
    def handle(self):
        return self._h

    @property
    def rank(self) -> int:
        return lib().gmds_comm_rank(self._h)

    @property
    def size(self) -> int:
        return lib().gmds_comm_size(self._h)

    def allreduce_device(self, dptr: int, count: int, op: int = 0, stream: int = 0):
        _check(lib().gmds_comm_allreduce_device(self._h, ctypes.c_void_p(dptr), _i64(count), _i32(op),
                                                ctypes.c_void_p(stream)))

    def free(self):
        if self._h:
            lib().gmds_comm_free(self._h)
            self._h = ctypes.c_void_p(0)


def comm_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(lib().gmds_comm_unique_id(buf))
    return bytes(buf)


def comm_init_nccl(uid: bytes, nranks: int, rank: int) -> Comm:
    """NCCL rank on the current device (gmds_set_device first); uid from rank 0's comm_unique_id."""
    buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
    h = ctypes.c_void_p()
    _check(lib().gmds_comm_init_nccl(buf, _i32(nranks), _i32(rank), ctypes.byref(h)))
    return Comm(h.value)


def comm_init_local(nranks: int) -> list:
    """nranks ranks in this process on the current device (drive each from its own thread)."""
    hs = (ctypes.c_void_p * nranks)()
    _check(lib().gmds_comm_init_local(_i32(nranks), hs))
    return [Comm(h) for h in hs]


def dmat_gini_sharded(comm: Comm, dX_ptr: int, xt: int, n: int, p: int, nu: float, storage=F32) -> DMat:
    """This rank's contiguous share of the packed blocks of pairwise_matrix(X, gini(nu))."""
    h = ctypes.c_void_p()
    _check(lib().gmds_dmat_gini_sharded(comm.handle, ctypes.c_void_p(dX_ptr), _i32(xt), _i64(n), _i64(p),
                                        ctypes.c_double(nu), _i32(storage), ctypes.byref(h)))
    return DMat(h.value, n)


def minimize_stress_sharded(comm: Comm, D: DMat, Y0, kind: str = "kruskal", huber_delta=None, max_iters: int = 300,
                            rel_tol: float = 1e-6) -> dict:
    y0 = _coords(Y0)
    q = y0.shape[1]
    cfg = StressCfg(kind=KIND[kind], huber_delta=(math.nan if huber_delta is None else float(huber_delta)),
                    smacof_weights=None, max_iters=int(max_iters), rel_tol=float(rel_tol), seed=0)
    coords = np.zeros((D.n, q), order="F")
    cap = int(max_iters) + 2
    hist = np.zeros(cap)
    res = FitResult(coords=_p(coords), history=_p(hist), history_cap=cap)
    _check(lib().gmds_minimize_stress_sharded(comm.handle, D.handle, _i32(q), ctypes.byref(cfg), _p(y0),
                                              ctypes.byref(res)))
    return dict(coords=np.ascontiguousarray(coords), stress_history=list(hist[: min(res.history_len, cap)]),
                iterations=res.iterations, converged=bool(res.converged), stress=res.stress, passes=res.passes)


def nu_sweep_kruskal_sharded(comm: Comm, X, Y, grid) -> np.ndarray:
    X, xt, lx = _xarg(X)
    n, p = X.shape
    Y = _coords(Y)
    g = np.ascontiguousarray(grid, dtype=np.float64)
    ks = np.zeros(g.size)
    _check(lib().gmds_nu_sweep_kruskal_sharded(comm.handle, _vp(X), _i32(xt), _i32(lx), _i64(n), _i64(p), _p(Y),
                                               _i32(Y.shape[1]), _p(g), _i32(g.size), _p(ks)))
    return ks
