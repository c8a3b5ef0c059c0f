"""The sharded stress pass on the device: shards of gmds_stress_partial sum to
the full pass, and a sharded fit (ranks emulated in-process, their partial
passes run one after another on the single GPU; the all-reduce is a sum over
them) follows the single-GPU trajectory."""
import numpy as np
import pytest

from oracle import gini_oracle as O

pytestmark = pytest.mark.gpu
G = pytest.importorskip("paper_2605_25124_b200.gmds")
from paper_2605_25124_b200 import distributed as MD  # noqa: E402


def test_partials_sum_to_full_pass():
    rng = np.random.default_rng(4)
    X = rng.random((700, 30))
    Dm = G.dmat_gini(X, 2.0)
    Y = rng.standard_normal((700, 2))
    for world in (1, 2, 3, 5):
        tot_l, tot_g = 0.0, np.zeros((700, 2))
        for r in range(world):
            l, g = MD.gpu_partial(Dm, r, world)("smacof", Y)
            tot_l += l
            tot_g += g
        assert tot_l == pytest.approx(G.stress_loss("smacof", Y, Dm), rel=1e-12)
        assert np.allclose(tot_g, G.stress_gradient("smacof", Y, Dm), rtol=1e-10, atol=1e-10)


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
