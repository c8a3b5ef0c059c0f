"""Multi-GPU host logic on CPU with the gloo backend, world size
2: tile shards cover the matrix exactly once, the sharded nu sweep picks the
same nu as the single-process sweep, and the all-reduced sharded fit follows
the single-process reference trajectory.  The per-rank partial pass here is a
numpy restatement over the rank's pairs; on GPUs it is gmds_stress_partial
(tests/test_gpu_distributed.py)."""
import math
import os
import socket
import tempfile

import numpy as np
import pytest

from oracle import gini_oracle as O
from paper_2605_25124_b200 import distributed as MD


def numpy_partial(D, pairs):
    """raw loss / raw row sums of c_ij (y_i - y_j) over `pairs` (the C-ABI's conventions)."""
    I = np.array([p[0] for p in pairs], dtype=np.int64)
    J = np.array([p[1] for p in pairs], dtype=np.int64)
    d = D[I, J]

    def partial(kind, Y):
        dy = Y[I] - Y[J]
        dist = np.sqrt(np.sum(dy * dy, axis=1))
        e = d - dist
        inv = np.where(dist > 0, 1.0 / np.where(dist > 0, dist, 1.0), 0.0)
        if kind == "kruskal":
            term, c = e * e, -e * inv
        elif kind == "sammon":
            term, c = e * e / d, -e / d * inv
        elif kind == "smacof":
            term, c = e * e, -2.0 * e * inv
        else:  # guttman
            term, c = e * e, d * inv
        g = np.zeros_like(Y)
        for t in range(Y.shape[1]):
            g[:, t] += np.bincount(I, weights=c * dy[:, t], minlength=Y.shape[0])
            g[:, t] -= np.bincount(J, weights=c * dy[:, t], minlength=Y.shape[0])
        return float(np.sum(term)), g

    return partial


def test_tile_shards_cover_once():
    for n, tile, world in ((37, 8, 3), (100, 16, 4), (5, 32, 2)):
        seen = []
        for r in range(world):
            seen += MD.shard_pairs(n, tile, r, world)
        assert sorted(seen) == [(i, j) for i in range(n) for j in range(i + 1, n)]


def test_argmin_ties_to_smaller():
    assert MD.argmin_smaller_nu([0.3, 0.2, 0.2, 0.5]) == 1
    assert MD.nu_shard(list(range(10)), 0, 3) == [0, 1, 2] and MD.nu_shard(list(range(10)), 2, 3) == [6, 7, 8, 9]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    allreduce_sum, allgather = MD.torch_collectives()
    rng = np.random.default_rng(0)
    X = rng.standard_normal((40, 6))
    # nu sweep: score = Kruskal stress of the classical embedding (tune_nu's classical cell, one fold)
    grid = [1.2, 1.7, 2.5, 4.0, 6.0]

    def score(nu):
        D = O.pairwise_matrix(X, nu)
        return O.kruskal_stress(O.classical_mds(D, 2).coords, D)

    nu_star, scores = MD.nu_sweep(grid, score, rank, world, allgather)
    # sharded fit at nu = 2
    D = O.pairwise_matrix(X, 2.0)
    iu = np.triu_indices(40, 1)
    stats = [float(np.sum(D[iu] ** 2)), float(np.sum(D[iu])), float(D[iu].min()), float(D[iu].max())]
    Y0 = O.classical_mds(D, 2).coords
    res = {}
    for kind in ("kruskal", "sammon", "smacof"):
        part = numpy_partial(D, MD.shard_pairs(40, 8, rank, world))
        r = MD.minimize_stress_sharded(part, allreduce_sum, Y0, kind, stats, 40, max_iters=40, rel_tol=1e-300)
        res[kind] = np.array(r["stress_history"])
    if rank == 0:
        np.savez(os.path.join(out_dir, "res.npz"), nu_star=nu_star, scores=np.array(scores), **res)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sweep_and_sharded_fit():
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        r = np.load(os.path.join(d, "res.npz"))
        rng = np.random.default_rng(0)
        X = rng.standard_normal((40, 6))
        grid = [1.2, 1.7, 2.5, 4.0, 6.0]
        scores = []
        for nu in grid:
            D = O.pairwise_matrix(X, nu)
            scores.append(O.kruskal_stress(O.classical_mds(D, 2).coords, D))
        assert np.allclose(r["scores"], scores, rtol=1e-12)
        assert float(r["nu_star"]) == grid[MD.argmin_smaller_nu(scores)]
        D = O.pairwise_matrix(X, 2.0)
        for kind in ("kruskal", "sammon", "smacof"):
            ref = O.minimize_stress(D, 2, kind, max_iters=40, rel_tol=1e-300).stress_history
            h = r[kind]
            assert len(h) == len(ref)
            assert np.max(np.abs(h - ref) / ref[0]) <= 1e-9
