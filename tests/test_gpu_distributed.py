"""The sharded stress pass on the device: shards of gmds_stress_partial sum to
the full pass, and a sharded fit (ranks emulated in-process, their partial
passes run one after another on the single GPU; the all-reduce is a sum over
them) follows the single-GPU trajectory; and the libgmds multi-GPU path
(gmds_comm + row-sharded D + the device-resident sharded fit) with ranks as
a local group on the one GPU, and a one-rank NCCL communicator."""
import os

import numpy as np
import pytest

from oracle import gini_oracle as O

pytestmark = pytest.mark.gpu
G = pytest.importorskip("paper_2605_25124_b200.gmds")
from paper_2605_25124_b200 import distributed as MD  # noqa: E402


@pytest.mark.parametrize("chunk", [None, "8"])
def test_partials_sum_to_full_pass(monkeypatch, chunk):
    # chunk "8": shards made of multi-block chunks (the large-n default), fp32 storage at n = 2600
    n = 700 if chunk is None else 2600
    if chunk:
        monkeypatch.setenv("GMDS_STRESS_CHUNK", chunk)
    rng = np.random.default_rng(4)
    X = rng.random((n, 30))
    Dm = G.dmat_gini(X, 2.0, storage=G.F64 if chunk is None else G.F32)
    Y = rng.standard_normal((n, 2))
    for world in (1, 2, 3, 5):
        tot_l, tot_g = 0.0, np.zeros((n, 2))
        for r in range(world):
            l, g = MD.gpu_partial(Dm, r, world)("smacof", Y)
            tot_l += l
            tot_g += g
        assert tot_l == pytest.approx(G.stress_loss("smacof", Y, Dm), rel=1e-12 if chunk is None else 1e-6)
        ref = G.stress_gradient("smacof", Y, Dm)
        assert np.max(np.abs(tot_g - ref)) <= (1e-10 if chunk is None else 1e-5) * np.max(np.abs(ref))


@pytest.mark.parametrize("kind", ["kruskal", "sammon", "smacof"])
def test_sharded_fit_matches_single_gpu(kind):
    rng = np.random.default_rng(5)
    X = rng.random((600, 20))
    Dm = G.dmat_gini(X, 2.0)
    Y0 = rng.normal(0, 0.1, (600, 2))
    world = 3
    parts = [MD.gpu_partial(Dm, r, world) for r in range(world)]

    def partial_all(kd, Y):  # what the all-reduce of the 3 ranks' partials returns
        outs = [p(kd, Y) for p in parts]
        return sum(o[0] for o in outs), sum(o[1] for o in outs)

    r = MD.minimize_stress_sharded(partial_all, lambda v: v, Y0, kind, MD.dmat_stats(Dm), 600, max_iters=30,
                                   rel_tol=1e-300)
    e = G.minimize_stress(Dm, 2, kind, max_iters=30, rel_tol=1e-300, Y0=Y0)
    h, he = np.array(r["stress_history"]), np.array(e["stress_history"])
    assert len(h) == len(he)
    assert np.max(np.abs(h - he) / he) <= 1e-9


# ---- the libgmds multi-GPU path: gmds_comm + row-sharded D + device-resident sharded fit ----------

from concurrent.futures import ThreadPoolExecutor  # noqa: E402

from oracle import synth as S  # noqa: E402


def _ranks(world, fn):
    """Run fn(rank, comm) for every rank of a local group, one host thread per rank (the
    library's collectives order the ranks' streams with events; no kernel waits on another)."""
    comms = G.comm_init_local(world)
    try:
        with ThreadPoolExecutor(max_workers=world) as ex:
            futs = [ex.submit(fn, r, comms[r]) for r in range(world)]
            return [f.result() for f in futs]
    finally:
        for c in comms:
            c.free()


def _image(n, p, seed):
    torch = pytest.importorskip("torch")
    X = S.image_like(n, p, seed)
    return X, torch.from_numpy(X).cuda()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_fit_device_loop_matches_single_gpu(world):
    # image-like data above the small-fit size, Kruskal from N(0, 0.1^2), fp32 storage: the
    # bench path (TMA passes, difference passes, device gd_step loop) with D row-sharded over
    # `world` ranks and one all-reduce of [gradient | loss sums] per pass
    n, p = 2600, 784
    X, dX = _image(n, p, 78)
    Y0 = np.random.default_rng(78).normal(0.0, 0.1, (n, 2))
    single = G.minimize_stress(G.dmat_gini_device(dX.data_ptr(), G.F32, n, p, 2.0, G.F32), 2, "kruskal",
                               max_iters=60, rel_tol=1e-300, Y0=Y0)

    def rank(r, comm):
        G.lib().gmds_set_device(0)
        D = G.dmat_gini_sharded(comm, dX.data_ptr(), G.F32, n, p, 2.0, G.F32)
        stats = MD.dmat_stats(D)
        e = G.minimize_stress_sharded(comm, D, Y0, "kruskal", max_iters=60, rel_tol=1e-300)
        D.free()
        return e, stats

    outs = _ranks(world, rank)
    full_stats = MD.dmat_stats(G.dmat_gini_device(dX.data_ptr(), G.F32, n, p, 2.0, G.F32))
    for e, stats in outs:  # every rank holds the same result, bit for bit
        assert np.array_equal(e["coords"], outs[0][0]["coords"])
        assert e["stress_history"] == outs[0][0]["stress_history"]
        assert np.allclose(stats, full_stats, rtol=1e-12)
    h, hs = np.array(outs[0][0]["stress_history"]), np.array(single["stress_history"])
    assert outs[0][0]["iterations"] == single["iterations"] == 60
    assert np.max(np.abs(h - hs) / hs) <= 1e-7
    # against the reference's own loop (golden fixture, n = 2600)
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "large_img2600.npz"))
    ref = g["fit_history"]
    assert np.max(np.abs(h[:51] - ref[:51]) / ref[:51]) <= 1e-4


@pytest.mark.parametrize("kind", ["sammon", "smacof", "huber"])
def test_sharded_fit_other_kinds(kind):
    rng = np.random.default_rng(6)
    n = 2300
    X = rng.random((n, 12)).astype(np.float32)
    torch = pytest.importorskip("torch")
    dX = torch.from_numpy(X).cuda()
    Y0 = rng.normal(0, 0.1, (n, 2))
    Dfull = G.dmat_gini_device(dX.data_ptr(), G.F32, n, 12, 2.0, G.F32)
    hd = 0.5 * MD.dmat_stats(Dfull)[1] / (n * (n - 1) / 2) if kind == "huber" else None
    single = G.minimize_stress(Dfull, 2, kind, huber_delta=hd, max_iters=40, rel_tol=1e-300, Y0=Y0)

    def rank(r, comm):
        D = G.dmat_gini_sharded(comm, dX.data_ptr(), G.F32, n, 12, 2.0, G.F32)
        return G.minimize_stress_sharded(comm, D, Y0, kind, huber_delta=hd, max_iters=40, rel_tol=1e-300)

    outs = _ranks(2, rank)
    assert outs[0]["stress_history"] == outs[1]["stress_history"]
    h, hs = np.array(outs[0]["stress_history"]), np.array(single["stress_history"])
    assert len(h) == len(hs)
    assert np.max(np.abs(h - hs) / np.abs(hs)) <= 1e-6


def test_sharded_entry_errors():
    torch = pytest.importorskip("torch")
    X = np.random.default_rng(1).random((300, 8)).astype(np.float32)
    dX = torch.from_numpy(X).cuda()
    (c,) = G.comm_init_local(1)
    try:
        D = G.dmat_gini_sharded(c, dX.data_ptr(), G.F32, 300, 8, 2.0, G.F32)
        Y0 = np.zeros((300, 2))
        with pytest.raises(G.InvalidConfig):  # Huber auto mode needs all of D
            G.minimize_stress_sharded(c, D, Y0, "huber")
        with pytest.raises(G.InvalidInput):  # a sharded D is refused by the single-GPU entries
            G.kruskal_stress(Y0, D)
        with pytest.raises(G.InvalidConfig):
            G.dmat_gini_sharded(c, dX.data_ptr(), G.F32, 300, 8, 1.0, G.F32)
        D.free()
    finally:
        c.free()


def test_nccl_single_rank_comm():
    # a real NCCL communicator of one rank: the same trajectory as the unsharded fit
    torch = pytest.importorskip("torch")
    n, p = 2200, 64
    X = S.image_like(n, p, 5)
    dX = torch.from_numpy(X).cuda()
    Y0 = np.random.default_rng(5).normal(0.0, 0.1, (n, 2))
    c = G.comm_init_nccl(G.comm_unique_id(), 1, 0)
    try:
        D = G.dmat_gini_sharded(c, dX.data_ptr(), G.F32, n, p, 2.0, G.F32)
        e = G.minimize_stress_sharded(c, D, Y0, "kruskal", max_iters=30, rel_tol=1e-300)
        s = G.minimize_stress(G.dmat_gini_device(dX.data_ptr(), G.F32, n, p, 2.0, G.F32), 2, "kruskal", max_iters=30,
                              rel_tol=1e-300, Y0=Y0)
        assert e["iterations"] == s["iterations"]
        assert np.max(np.abs(np.array(e["stress_history"]) - s["stress_history"]) / s["stress_history"]) <= 1e-9
        D.free()
    finally:
        c.free()


def test_sharded_nu_sweep_matches_single():
    rng = np.random.default_rng(8)
    X = rng.random((500, 16)).astype(np.float32)
    X[rng.random(X.shape) < 0.6] = 0.0
    Y = rng.standard_normal((500, 2))
    grid = list(np.exp(np.linspace(np.log(1.1), np.log(8.0), 7)))
    ref = G.nu_sweep_kruskal(X, Y, grid)
    for world in (2, 3):
        outs = _ranks(world, lambda r, c: G.nu_sweep_kruskal_sharded(c, X, Y, grid))
        for o in outs:
            assert np.allclose(o, ref, rtol=1e-12, atol=0)
