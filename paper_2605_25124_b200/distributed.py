"""Multi-GPU drivers: one process per GPU, torch.distributed
for the plumbing, libgmds kernels for the work.

* ``tile_range`` / ``pair_tiles`` -- the distance matrix's work units (upper-
  triangle tiles) split into contiguous, equal-count shards; a rank computes
  only its tiles (``gmds_pairwise_gini_device(..., shard, nshards)``), no
  collective on the data path (the north star's "rows sharded").
* ``nu_sweep`` -- the nu grid split across ranks (replicas: each rank builds
  its own D_nu and scores it); one all-gather of the per-nu scores, then the
  reference's argmin with ties to the smaller nu (tune.cpp:126-130).
* ``minimize_stress_sharded`` -- one single-nu fit over tile-sharded D: every
  rank runs ``gmds_stress_partial`` on its tiles, the raw [loss | gradient]
  sums are all-reduced, and every rank takes the identical Armijo / SMACOF
  decision (embed.cpp:222-272, 296-347), so all ranks hold the same Y.

The collective is injected (``allreduce_sum`` / ``allgather``), so the same
drivers run under NCCL on GPUs and under gloo on CPU in the tests.
"""
from __future__ import annotations

import math
from typing import Callable, Sequence

import numpy as np

_TINY = 1e-300  # embed.cpp:13


def tile_range(units: int, shard: int, nshards: int) -> tuple[int, int]:
    """[begin, end) of shard `shard` -- same split as run_gini (gini_plan.cu)."""
    if nshards < 1 or not (0 <= shard < nshards):
        raise ValueError("bad shard")
    return units * shard // nshards, units * (shard + 1) // nshards


def pair_tiles(n: int, tile: int):
    """Row-major upper-triangle tiles (I <= J) of an n x n matrix with edge `tile`."""
    nbt = -(-n // tile)
    return [(I, J) for I in range(nbt) for J in range(I, nbt)]


def shard_pairs(n: int, tile: int, shard: int, nshards: int):
    """(i, j), i < j, of one shard's tiles."""
    tiles = pair_tiles(n, tile)
    b, e = tile_range(len(tiles), shard, nshards)
    out = []
    for I, J in tiles[b:e]:
        for i in range(I * tile, min(n, I * tile + tile)):
            for j in range(max(i + 1, J * tile), min(n, J * tile + tile)):
                out.append((i, j))
    return out


def nu_shard(grid: Sequence[float], rank: int, world: int) -> list[int]:
    """Indices of the grid values owned by `rank` (contiguous blocks)."""
    b, e = tile_range(len(grid), rank, world)
    return list(range(b, e))


def argmin_smaller_nu(scores: Sequence[float]) -> int:
    """tune.cpp:126-130: strict '<' keeps the first (smaller nu) on ties."""
    best = 0
    for g in range(1, len(scores)):
        if scores[g] < scores[best]:
            best = g
    return best


def nu_sweep(grid: Sequence[float], score: Callable[[float], float], rank: int, world: int,
             allgather: Callable[[object], list]) -> tuple[float, list[float]]:
    """Score every grid value (this rank: its own block), gather, argmin."""
    mine = {g: float(score(grid[g])) for g in nu_shard(grid, rank, world)}
    merged: dict[int, float] = {}
    for part in allgather(mine):
        merged.update(part)
    scores = [merged[g] for g in range(len(grid))]
    return grid[argmin_smaller_nu(scores)], scores


# ---------------------------------------------------------------------------------------------------
# sharded single-nu fit


KIND_SCALE = {"kruskal", "sammon"}


def minimize_stress_sharded(partial: Callable[[str, np.ndarray], tuple[float, np.ndarray]],
                            allreduce_sum: Callable[[np.ndarray], np.ndarray], Y0: np.ndarray, kind: str,
                            stats: Sequence[float], n: int, huber_delta=None, max_iters: int = 300,
                            rel_tol: float = 1e-6) -> dict:
    """Reference control flow over all-reduced partial passes.

    partial(kind, Y[, huber_delta]) -> (raw_loss, raw_grad) over this rank's tiles (kind
    "guttman" for the SMACOF transform); allreduce_sum sums a flat float64
    vector across ranks.  stats = (sum D^2, sum D, min D, max D).
    """
    sum_sq, sum_d = float(stats[0]), float(stats[1])
    if kind == "huber" and huber_delta is None:
        # the reference's auto mode (embed.cpp:499-515) fits three deltas from the median and keeps the
        # lowest Kruskal stress; the sharded driver takes an explicit delta (resolved by the caller)
        raise ValueError("minimize_stress_sharded: huber needs an explicit huber_delta (auto mode is "
                         "minimize_stress's)")
    if kind == "huber" and not (huber_delta > 0.0):
        raise ValueError("minimize_stress_sharded: huber_delta must be > 0")
    Y = np.array(Y0, dtype=np.float64, copy=True)

    def full(kd, Yc):
        raw, g = partial(kd, Yc, huber_delta) if kd == "huber" else partial(kd, Yc)
        v = allreduce_sum(np.concatenate([[raw], np.asarray(g, dtype=np.float64).ravel()]))
        return float(v[0]), v[1:].reshape(Yc.shape)

    def loss_of(kd, raw):
        if kd == "kruskal":
            return math.sqrt(raw / sum_sq)
        if kd == "sammon":
            return (1.0 / sum_d) * raw
        return raw

    hist = []
    if kind == "smacof":
        raw, g = full("guttman", Y)
        f = raw
        hist.append(f)
        nxt = g / float(n)
        it, reached = 0, False
        while it < max_iters:
            Y = nxt
            raw, g = full("guttman", Y)
            f_new = raw
            hist.append(f_new)
            dec = (f - f_new) / max(f, _TINY)
            f = f_new
            it += 1
            if dec < rel_tol:
                reached = True
                break
            nxt = g / float(n)
        return dict(coords=Y, stress=f, iterations=it, converged=reached or it < max_iters, stress_history=hist)

    raw, _ = full(kind, Y)
    f = loss_of(kind, raw)
    hist.append(f)
    step, armijo = 1.0, 1e-4
    it, stalled = 0, False
    while it < max_iters:
        raw, g = full(kind, Y)
        if kind == "kruskal":
            ks = math.sqrt(raw / sum_sq)
            g = g * (0.0 if ks <= 0.0 else 1.0 / (ks * sum_sq))
        elif kind == "sammon":
            g = g * (2.0 * (1.0 / sum_d))
        gsq = float(np.sum(g * g))
        if gsq <= 0.0:
            stalled = True
            break
        accepted, f_new, trial = False, f, Y
        for _ in range(60):
            trial = Y - step * g
            raw_t, _ = full(kind, trial)  # (the trial's gradient is discarded, as in the reference)
            f_new = loss_of(kind, raw_t)
            if f_new <= f - armijo * step * gsq:
                accepted = True
                break
            step *= 0.5
        if not accepted:
            stalled = True
            break
        Y = trial
        hist.append(f_new)
        dec = (f - f_new) / max(f, _TINY)
        f = f_new
        step *= 2.0
        it += 1
        if dec < rel_tol:
            stalled = True
            break
    return dict(coords=Y, stress=f, iterations=it, converged=stalled or it < max_iters, stress_history=hist)


def gpu_partial(dmat, rank: int, world: int, huber_delta=None):
    """partial() for minimize_stress_sharded on a device DistanceMatrix (C-ABI gmds_stress_partial)."""
    import ctypes

    from . import gmds as G

    codes = {"kruskal": 0, "huber": 1, "sammon": 2, "smacof": 3, "guttman": 4}

    def partial(kind, Y, delta=None):
        Yf = np.asfortranarray(Y, dtype=np.float64)
        g = np.zeros_like(Yf, order="F")
        raw = ctypes.c_double()
        delta = huber_delta if delta is None else delta
        hd = ctypes.c_double(math.nan if delta is None else float(delta))
        G._check(G.lib().gmds_stress_partial(G._i32(codes[kind]), dmat.handle, G._p(Yf), G._i32(Yf.shape[1]), hd,
                                             G._i32(rank), G._i32(world), ctypes.byref(raw), G._p(g)))
        return raw.value, np.ascontiguousarray(g)

    return partial


def dmat_stats(dmat) -> list[float]:
    from . import gmds as G

    out = np.zeros(4)
    G._check(G.lib().gmds_dmat_stats(dmat.handle, G._p(out)))
    return list(out)


def torch_collectives(group=None):
    """(allreduce_sum, allgather) over an initialised torch.distributed group (gloo or nccl)."""
    import torch
    import torch.distributed as dist

    def allreduce_sum(v: np.ndarray) -> np.ndarray:
        backend = dist.get_backend(group)
        t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
        if backend == "nccl":
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t.cpu().numpy()

    def allgather(obj) -> list:
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, obj, group=group)
        return out

    return allreduce_sum, allgather
