"""GPU parity: rank + distance kernels (through the C-ABI) vs the oracle and
the reference's golden vectors.  Ranks bit-exact; distances within the
north-star 1e-6 max-normalised tolerance (observed ~1e-15)."""
import numpy as np
import pytest

from oracle import gini_oracle as O
from _util import unpad

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_2605_25124_b200.gmds")

TOL = 1e-6  # north_star: distance matrix within 1e-6 relative, max-normalised


def maxnorm_err(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    scale = max(np.max(np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b)) / scale) if a.size else 0.0


def test_device_visible():
    assert G.device_count() >= 1


def test_midrank_golden_bitexact(golden):
    g = golden("midrank")
    for v, r, m in zip(g["values"], g["ranks"], g["lengths"]):
        assert np.array_equal(G.midrank(unpad(v, m)), unpad(r, m))


@pytest.mark.parametrize("d", [1, 2, 31, 32, 33, 100, 511, 1024, 1025, 3000, 20000])
def test_midrank_batch_vs_oracle(d):
    rng = np.random.default_rng(d)
    V = rng.integers(-5, 6, size=(7, d)).astype(np.float64) * 0.25
    V[:, ::3] = rng.standard_normal(V[:, ::3].shape)
    V[V == 0.0] = -0.0
    got = G.midrank_batch(V)
    for k in range(V.shape[0]):
        assert np.array_equal(got[k], O.midrank(V[k]))


def test_midrank_errors():
    with pytest.raises(G.InvalidInput):
        G.midrank([1.0, np.nan])
    with pytest.raises(G.InvalidInput):
        G.midrank([np.inf])


@pytest.mark.parametrize("p,dtype", [(8, np.float64), (20, np.float64), (128, np.float32), (784, np.float32),
                                     (784, np.float64), (1025, np.float32)])
def test_pair_midranks_bitexact(p, dtype):
    rng = np.random.default_rng(p)
    n = 40
    X = rng.random((n, p))
    X[rng.random((n, p)) < 0.8] = 0.0  # heavy exact-zero ties (config 3 shape)
    X[3] = X[5]                        # duplicated row: all-tied z
    X = X.astype(dtype)
    I = np.array([0, 3, 1, 7, 39, 12])
    J = np.array([1, 5, 2, 8, 0, 30])
    got = G.pair_midranks(X, I, J)
    ref = O.pair_midranks(X.astype(np.float64), I, J)
    assert np.array_equal(got, ref)


def test_known_answers():
    x, y = [10.0, 1200.0], [10.0, 12.0]
    assert G.gen_gini_distance(x, y, 2.0) == 594.0
    assert G.gen_gini_distance(x, y, 3.0) == 594.0
    assert G.gen_gini_distance(x, x, 3.5) == 0.0
    ones = np.ones(5)
    for nu in (1.5, 2.0, 3.0, 5.0):
        assert G.gen_gini_distance(2.0 * ones, -6.0 * ones, nu) == 0.0  # egalitarian null
    D = G.pairwise_matrix(np.array([[10.0, 1200.0], [10.0, 12.0]]), 2.0)
    assert D[0, 1] == 594.0 and D[1, 0] == 594.0 and D[0, 0] == 0.0
    D = G.pairwise_matrix(np.array([[1.0, 2.0, 3.0], [1.0, 2.0, 3.0]]), 2.5)
    assert D[0, 1] == 0.0


def test_distance_golden(golden):
    g = golden("distance")
    for x, y, m, nu, dist in zip(g["x"], g["y"], g["lengths"], g["nu"], g["distance"]):
        got = G.gen_gini_distance(unpad(x, m), unpad(y, m), float(nu))
        assert abs(got - dist) <= 1e-12 * max(1.0, abs(dist))


def test_pairwise_golden(golden):
    g = golden("pairwise")
    for name in ("t888", "t321", "c1", "ties"):
        X = g[f"{name}_X"]
        iu = np.triu_indices(X.shape[0], 1)
        nus = list(g[f"{name}_nus"])
        Ds = G.pairwise_gini(X, nus)
        for k in range(len(nus)):
            assert maxnorm_err(Ds[k][iu], g[f"{name}_D{k}"]) <= 1e-13
            assert np.array_equal(Ds[k], Ds[k].T) and np.all(np.diag(Ds[k]) == 0.0)
        E = G.pairwise_matrix(X, None)
        assert np.array_equal(E[iu], g[f"{name}_E"])  # Euclidean branch is bit-exact


@pytest.mark.parametrize("n,p,dtype,nus", [(64, 1, np.float64, [2.0]), (50, 33, np.float64, [1.1, 2.0, 8.0]),
                                           (97, 128, np.float32, [1.5, 2.0, 3.0, 5.0]),
                                           (40, 784, np.float32, [2.0]), (33, 784, np.float64, [1.3, 4.0]),
                                           (20, 1100, np.float32, [2.0, 3.0])])
def test_pairwise_vs_oracle(n, p, dtype, nus):
    rng = np.random.default_rng(n * p)
    X = rng.lognormal(0.0, 1.0, (n, p))
    X[rng.random((n, p)) < 0.5] = 0.0
    X[4] = X[9]
    X = X.astype(dtype)
    Ds = G.pairwise_gini(X, nus)
    for k, nu in enumerate(nus):
        ref = O.pairwise_matrix(X.astype(np.float64), nu)
        assert maxnorm_err(Ds[k], ref) <= TOL
        assert Ds[k][4, 9] == 0.0


def test_pairwise_fp32_output():
    rng = np.random.default_rng(7)
    X = rng.standard_normal((70, 20))
    D32 = G.pairwise_gini(X, [2.0], out_dtype=np.float32)[0]
    ref = O.pairwise_matrix(X, 2.0)
    assert D32.dtype == np.float32 and maxnorm_err(D32, ref) <= 1e-6


def test_pairwise_colmajor_input():
    rng = np.random.default_rng(8)
    X = np.asfortranarray(rng.standard_normal((45, 12)))
    assert maxnorm_err(G.pairwise_matrix(X, 1.7), O.pairwise_matrix(np.ascontiguousarray(X), 1.7)) <= 1e-13


def test_pairwise_errors():
    with pytest.raises(G.InvalidConfig):
        G.pairwise_matrix(np.zeros((3, 2)), 1.0)
    with pytest.raises(G.InvalidConfig):
        G.pairwise_matrix(np.zeros((3, 2)), 0.5)
    with pytest.raises(G.InvalidInput):
        G.pairwise_matrix(np.zeros((1, 2)), 2.0)
    with pytest.raises(G.InvalidInput):
        G.pairwise_matrix(np.zeros((3, 0)), 2.0)
    X = np.zeros((3, 2))
    X[1, 1] = np.nan
    with pytest.raises(G.InvalidInput):
        G.pairwise_matrix(X, 2.0)
    with pytest.raises(G.InvalidInput):
        G.gen_gini_distance([1.0, 2.0], [1.0], 2.0)


def test_device_entry_sharded_matches_full():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(9)
    X = rng.random((300, 64)).astype(np.float32)
    dX = torch.from_numpy(X).cuda()
    full = torch.zeros((2, 300, 300), dtype=torch.float64, device="cuda")
    G.pairwise_gini_device(dX.data_ptr(), G.F32, 300, 64, [2.0, 3.0], G.F64, False, full.data_ptr())
    sh = torch.zeros_like(full)
    for s in range(3):
        G.pairwise_gini_device(dX.data_ptr(), G.F32, 300, 64, [2.0, 3.0], G.F64, False, sh.data_ptr(), s, 3)
    torch.cuda.synchronize()
    assert torch.equal(full, sh)
    ref = O.pairwise_matrix(X.astype(np.float64), 3.0)
    assert maxnorm_err(full[1].cpu().numpy(), ref) <= 1e-12


def image_like(n, p, seed, zero_frac=0.8):
    g = np.random.default_rng(seed)
    X = g.integers(0, 256, size=(n, p)).astype(np.float64) / 255.0
    X += g.normal(0.0, 0.1, size=(n, p))
    np.clip(X, 0.0, 1.0, out=X)
    X[g.random((n, p)) < zero_frac] = 0.0
    return X.astype(np.float32)


@pytest.mark.parametrize("p", [200, 300, 784, 1000])
def test_sparse_split_path_vs_oracle(p):
    # config-3 shaped data: bitmask-sparse panels, zero compaction, sign-split sorts
    X = image_like(90, p, p)
    X[11] = X[12]  # duplicate row -> D == 0
    nus = [1.1, 2.0, 3.0, 5.0, 8.0]
    Ds = G.pairwise_gini(X, nus)
    Xd = X.astype(np.float64)
    for k, nu in enumerate(nus):
        assert maxnorm_err(Ds[k], O.pairwise_matrix(Xd, nu)) <= TOL
    assert Ds[0][11, 12] == 0.0


def test_overflow_list_path():
    # p = 784 with a few dense rows: dense-dense pairs have > 512 nonzeros and
    # take the overflow list; everything else the split kernel
    X = image_like(70, 784, 5)
    X[:6] = np.random.default_rng(6).lognormal(0.0, 1.0, (6, 784)).astype(np.float32)
    D = G.pairwise_gini(X, [2.0, 4.0])
    Xd = X.astype(np.float64)
    assert maxnorm_err(D[0], O.pairwise_matrix(Xd, 2.0)) <= TOL
    assert maxnorm_err(D[1], O.pairwise_matrix(Xd, 4.0)) <= TOL


@pytest.mark.parametrize("p", [300, 600])
def test_dense_mid_p(p):
    X = np.random.default_rng(p).lognormal(0.0, 1.0, (50, p)).astype(np.float32)
    assert maxnorm_err(G.pairwise_matrix(X, 2.5), O.pairwise_matrix(X.astype(np.float64), 2.5)) <= TOL


def test_all_zero_rows_and_constant_shift():
    X = np.zeros((20, 784), dtype=np.float32)
    X[5, 3] = 1.0
    X[7] = 0.25  # constant row: z = const - 0 on most features
    D = G.pairwise_matrix(X, 2.0)
    assert maxnorm_err(D, O.pairwise_matrix(X.astype(np.float64), 2.0)) <= TOL
    assert D[0, 1] == 0.0


def test_directed_norm_survival_golden(golden):
    g = golden("distance")
    for x, y, m, nu, fwd in zip(g["x"], g["y"], g["lengths"], g["nu"], g["directed"]):
        x, y = unpad(x, m), unpad(y, m)
        assert abs(G.gen_gini_directed(x, y, float(nu)) - fwd) <= 1e-12 * max(1.0, abs(fwd))
    assert G.gen_gini_directed([10.0, 1200.0], [10.0, 12.0], 3.0) == pytest.approx(445.5, rel=1e-12)
    assert G.gen_gini_directed([10.0, 12.0], [10.0, 1200.0], 3.0) == pytest.approx(742.5, rel=1e-12)
    assert G.gini_pseudo_distance([10.0, 1200.0], [10.0, 12.0]) == 594.0
    assert G.gini_norm([1.0, 2.0, 3.0]) == pytest.approx(2.0, rel=1e-14)
    assert G.gini_norm([5.0, 5.0, 5.0]) == 0.0
    assert list(G.empirical_survival([0.0, 1188.0])) == [0.75, 0.25]
    rng = np.random.default_rng(3)
    for d in (1, 7, 40, 300):
        v = np.round(rng.standard_normal(d), 1)
        assert np.array_equal(G.empirical_survival(v), O.empirical_survival(v))
        assert G.gini_norm(v) == pytest.approx(O.gini_norm(v), rel=1e-12, abs=1e-12)
    with pytest.raises(G.InvalidConfig):
        G.gen_gini_directed([1.0], [2.0], 1.0)


def test_double_center():
    S = np.array([[0.0, 4.0], [4.0, 0.0]])
    assert np.allclose(G.double_center(S), [[1.0, -1.0], [-1.0, 1.0]], rtol=1e-14)
    rng = np.random.default_rng(1)
    P = rng.standard_normal((30, 3))
    D = O.pairwise_matrix(P, None)
    B = G.double_center(D * D)
    assert np.allclose(B, O.double_center(D * D), rtol=1e-10, atol=1e-12)
    assert np.array_equal(B, B.T)
    with pytest.raises(G.InvalidInput):
        G.double_center(np.array([[0.0, 1.0], [3.0, 0.0]]))


def test_merge_path_exact_keys_adversarial():
    # The merge path orders each sign half by 32-bit keys (fp32 magnitude rounded
    # toward zero + an "inexact" bit).  Craft sparse non-negative fp32 rows where
    # (a) two different differences fall in the same fp32 interval (key collision
    # -> exact fp64 fallback), (b) a difference ties EXACTLY with a plain value of
    # the other row, (c) magnitudes span 1e-30 .. 1e30 (inexact differences).
    p = 96
    rng = np.random.default_rng(17)
    X = np.zeros((48, p), dtype=np.float32)
    for i in range(48):
        idx = rng.choice(p, 20, replace=False)
        X[i, idx] = rng.choice(np.float32([1.0, 0.5, 0.25, 0.75, 2.0 ** -30, 2.0 ** -29, 1e-30, 1e30, 3.0,
                                           1.0 + 2.0 ** -23]), 20)
    X[0, :4] = [1.0, 1.0, 0.0, 0.25]
    X[1, :4] = [2.0 ** -30, 2.0 ** -29, 0.25, 0.0]  # z = 1-2^-30, 1-2^-29 (same fp32 interval), -0.25, 0.25
    X[2, :3] = [0.5, 0.25, 0.0]
    X[3, :3] = [0.25, 0.0, 0.25]                   # z = 0.25 (S_ab) ties with 0.25 (S_a)
    Xd = X.astype(np.float64)
    for nu in (1.3, 2.0, 4.0):
        D = G.pairwise_matrix(X, nu)
        ref = O.pairwise_matrix(Xd, nu)
        assert maxnorm_err(D, ref) <= 1e-12
        # and pair by pair relative to the pair's own value (ties change D at ~1e-8 relative)
        iu = np.triu_indices(48, 1)
        big = ref[iu] > 1e-6 * ref.max()
        assert np.max(np.abs(D[iu][big] - ref[iu][big]) / ref[iu][big]) <= 1e-9


@pytest.mark.parametrize("case", ["merge", "split", "full"])
def test_pairwise_pinned_output_pipelined(case):
    # a pinned destination is filled stripe by stripe during the computation
    # (copy stream); the result must equal the copy-after path bit for bit
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    if case == "merge":  # sparse non-negative fp32, p > 32
        X = (rng.random((700, 300)) * (rng.random((700, 300)) < 0.2)).astype(np.float32)
        nus = [2.0, 3.5]
    elif case == "split":  # dense, small p
        X = rng.standard_normal((650, 40))
        nus = [1.5]
    else:  # dense fp32, p > 512: the all-keys kernel
        X = rng.standard_normal((300, 600)).astype(np.float32)
        nus = [2.0]
    ref = G.pairwise_gini(X, nus)
    pinned = torch.zeros((len(nus),) + ref.shape[1:], dtype=torch.float64).pin_memory().numpy()
    got = G.pairwise_gini(X, nus, out=pinned)
    assert np.array_equal(got, ref)
    sub = X[:60].astype(np.float64)
    assert np.max(np.abs(ref[0][:60, :60] - O.pairwise_matrix(sub, nus[0]))) <= 1e-9 * max(1.0, np.max(ref[0]))


def test_pairwise_nonfinite_input_device_check():
    X = np.ones((50, 10))
    X[7, 3] = np.nan
    with pytest.raises(G.InvalidInput, match="non-finite input"):
        G.pairwise_gini(X, [2.0])
    X[7, 3] = np.inf
    with pytest.raises(G.InvalidInput, match="non-finite input"):
        G.pairwise_gini(X, [2.0])


@pytest.mark.parametrize("kind", ["image", "levels", "dense_overlap"])
def test_merge_fast_path_vs_oracle(kind, monkeypatch):
    # rank-by-counting fast path of the merge kernel (nnu <= 4): ranks from
    # counts on the pre-sorted rows; row-internal tie groups (clipped 1.0s,
    # quantised levels), duplicate rows, and |S_ab| above the fast cap (the
    # pair falls back to the merge path inside the same kernel)
    rng = np.random.default_rng({"image": 1, "levels": 2, "dense_overlap": 3}[kind])
    if kind == "image":
        X = image_like(160, 784, 11)
        nus = [2.0]
    elif kind == "levels":  # heavy ties inside rows and across S_a / S_b
        X = rng.choice(np.float32([0.25, 0.5, 1.0, 2.0]), size=(150, 300)).astype(np.float32)
        X[rng.random(X.shape) < 0.75] = 0.0
        nus = [1.5, 2.0, 3.0, 5.0]
    else:  # ~45% density: many pairs with |S_ab+| or |S_ab-| > 64
        X = (rng.random((120, 400)) * (rng.random((120, 400)) < 0.45)).astype(np.float32)
        nus = [1.2, 4.0]
    X[7] = X[8]
    monkeypatch.setenv("GMDS_MERGE_FAST", "1")
    Ds = G.pairwise_gini(X, nus)
    Xd = X.astype(np.float64)
    for k, nu in enumerate(nus):
        ref = O.pairwise_matrix(Xd, nu)
        assert maxnorm_err(Ds[k], ref) <= 1e-12
    assert Ds[0][7, 8] == 0.0


def test_merge_fast_path_matches_merge_path(monkeypatch):
    # the same matrix with and without the counting path (GMDS_MERGE_FAST): equal
    # to round-off (different summation order), both equal to the oracle
    X = image_like(200, 784, 23)
    b = G.pairwise_matrix(X, 2.5)
    monkeypatch.setenv("GMDS_MERGE_FAST", "1")
    a = G.pairwise_matrix(X, 2.5)
    assert np.max(np.abs(a - b)) <= 1e-12 * np.max(b)
    assert maxnorm_err(a, O.pairwise_matrix(X.astype(np.float64), 2.5)) <= 1e-12


@pytest.mark.parametrize("kind", ["image", "levels", "overlap", "wide"])
def test_linear_weight_path_vs_oracle(kind, monkeypatch):
    # nu = 2 and nu = 3: G(R) is affine in R, the merge kernel assembles D from
    # per-row prefix sums and the features nonzero in both rows (gmd_pair);
    # checked against the oracle and against the general paths
    rng = np.random.default_rng({"image": 4, "levels": 5, "overlap": 6, "wide": 7}[kind])
    if kind == "image":
        X = image_like(180, 784, 31)
    elif kind == "levels":  # ties everywhere: within rows, across rows, S_ab values equal to row values
        X = rng.choice(np.float32([0.25, 0.5, 0.75, 1.0]), size=(150, 200)).astype(np.float32)
        X[rng.random(X.shape) < 0.7] = 0.0
    elif kind == "overlap":  # ~45% density: many pairs with more than 64 shared features (fallback)
        X = (rng.random((120, 300)) * (rng.random((120, 300)) < 0.45)).astype(np.float32)
    else:  # p = 1000 (W = 32 mask words), a few rows with > 256 nonzeros (fallback)
        X = image_like(100, 1000, 8)
        X[:3] = rng.random((3, 1000)).astype(np.float32) * (rng.random((3, 1000)) < 0.4)
    X[5] = X[9]
    Xd = X.astype(np.float64)
    D = G.pairwise_gini(X, [2.0, 3.0])
    for k, nu in enumerate((2.0, 3.0)):
        assert maxnorm_err(D[k], O.pairwise_matrix(Xd, nu)) <= 1e-12
    assert D[0][5, 9] == 0.0
    monkeypatch.setenv("GMDS_NO_LINEAR", "1")
    Dg = G.pairwise_gini(X, [2.0])
    assert np.max(np.abs(D[0] - Dg[0])) <= 1e-12 * np.max(Dg[0])


@pytest.mark.parametrize("nshards", [2, 3, 7])
def test_linear_weight_kernel_sharded_matches_full(nshards):
    # tile shards of the linear-weight kernel (multi-GPU split of the distance
    # step): the union of the shards' writes is the full matrix, bit for bit
    torch = pytest.importorskip("torch")
    X = image_like(333, 300, 41)
    dX = torch.from_numpy(X).cuda()
    pe = G.packed_elems(333)
    full = torch.zeros(pe, dtype=torch.float32, device="cuda")
    G.pairwise_gini_device(dX.data_ptr(), G.F32, 333, 300, [2.0], G.F32, True, full.data_ptr())
    sh = torch.zeros_like(full)
    for s in range(nshards):
        G.pairwise_gini_device(dX.data_ptr(), G.F32, 333, 300, [2.0], G.F32, True, sh.data_ptr(), s, nshards)
    torch.cuda.synchronize()
    assert torch.equal(full, sh)
    D = G.pairwise_matrix(X, 2.0)
    assert maxnorm_err(D, O.pairwise_matrix(X.astype(np.float64), 2.0)) <= 1e-12


def test_linear_weight_kernel_dense_rows_overflow():
    # a few dense rows (600 of 784 features) would make the panels too large for
    # shared memory: the kernel caps its panel stride and sends those rows' pairs
    # to the exact overflow list instead of leaving the linear-weight path
    X = image_like(140, 784, 51)
    rng = np.random.default_rng(52)
    for r in (3, 77):
        X[r] = (rng.random(784) * (rng.random(784) < 0.77)).astype(np.float32)
    D = G.pairwise_matrix(X, 2.0)
    assert maxnorm_err(D, O.pairwise_matrix(X.astype(np.float64), 2.0)) <= 1e-12


@pytest.mark.parametrize("kind", ["image", "heavy_tail", "edge_counts", "clipped", "tiny_values"])
def test_batched_bucket_kernels_match_round1_kernels_and_oracle(kind, monkeypatch):
    # gini_gmd2_kernel / gini_gen2_kernel (F lists built 8 pairs at a time, bucket-table lower
    # bounds, sorted-value panel) against the round-1 kernels (GMDS_GMD_V1 / GMDS_GEN_V1) and
    # the oracle, on data that stresses the bucket tables: heavy tails (most values in
    # bucket 0), rows of exactly 255 / 256 / 257 nonzeros (the u8 counters' limit: 256+ overflow),
    # many values equal to the row maximum (the last bucket), denormal-range values
    rng = np.random.default_rng({"image": 71, "heavy_tail": 72, "edge_counts": 73, "clipped": 74, "tiny_values": 75}[kind])
    if kind == "image":
        X = image_like(260, 784, 76)
    elif kind == "heavy_tail":
        X = (rng.lognormal(0.0, 3.0, size=(200, 300)) * (rng.random((200, 300)) < 0.3)).astype(np.float32)
    elif kind == "edge_counts":
        X = image_like(150, 784, 77)
        for r, c in ((2, 255), (40, 256), (41, 257), (90, 255)):
            X[r] = 0.0
            X[r, rng.choice(784, size=c, replace=False)] = rng.random(c).astype(np.float32) + 0.01
    elif kind == "clipped":
        X = image_like(180, 400, 78)
        X[(X > 0.6)] = 1.0  # a third of the nonzeros sit on the row maximum
    else:
        X = (rng.random((160, 200)) * (rng.random((160, 200)) < 0.35)).astype(np.float32)
        X[::3] *= np.float32(1e-38)  # rows in the denormal range next to rows of order 1
        X[1::3] *= np.float32(1e-30)
    X[5] = X[9]
    Xd = X.astype(np.float64)
    nus = [2.0, 3.0]
    D = G.pairwise_gini(X, nus)
    for k, nu in enumerate(nus):
        assert maxnorm_err(D[k], O.pairwise_matrix(Xd, nu)) <= 1e-12
    assert D[0][5, 9] == 0.0
    gn = [1.5, 2.5, 4.0]
    Dg = G.pairwise_gini(X, gn)
    for k, nu in enumerate(gn):
        assert maxnorm_err(Dg[k], O.pairwise_matrix(Xd, nu)) <= 1e-12
    monkeypatch.setenv("GMDS_GMD_V1", "1")
    monkeypatch.setenv("GMDS_GEN_V1", "1")
    # the same terms, added in list order instead of feature order: equal to round-off
    D1, Dg1 = G.pairwise_gini(X, nus), G.pairwise_gini(X, gn)
    assert np.max(np.abs(D - D1)) <= 1e-13 * np.max(np.abs(D1))
    assert np.max(np.abs(Dg - Dg1)) <= 1e-13 * np.max(np.abs(Dg1))


@pytest.mark.parametrize("kind", ["image", "levels", "mixed", "wide"])
def test_general_counting_kernel_vs_oracle(kind, monkeypatch):
    # other nu (<= 4 per launch) on sparse non-negative fp32 data: midranks counted
    # from the shared-feature structures (gini_gen_kernel), ties in rows handled,
    # ties between S_ab values and row values sent to the exact overflow kernel;
    # checked against the oracle and against the merge kernel (GMDS_NO_GEN)
    rng = np.random.default_rng({"image": 61, "levels": 62, "mixed": 63, "wide": 64}[kind])
    if kind == "image":
        X = image_like(170, 784, 65)
        nus = [2.5]
    elif kind == "levels":  # quantised values: many S_ab values equal row values (overflow path)
        X = rng.choice(np.float32([0.25, 0.5, 0.75, 1.0]), size=(150, 200)).astype(np.float32)
        X[rng.random(X.shape) < 0.7] = 0.0
        nus = [1.3, 4.0]
    elif kind == "mixed":
        X = image_like(160, 300, 66)
        X[::7] = np.round(X[::7] * 4) / 4  # some quantised rows
        nus = [1.1, 1.7, 5.0, 8.0]
    else:
        X = image_like(100, 1000, 67)
        X[:2] = rng.random((2, 1000)).astype(np.float32) * (rng.random((2, 1000)) < 0.4)
        nus = [6.0]
    X[5] = X[9]
    Xd = X.astype(np.float64)
    D = G.pairwise_gini(X, nus)
    for k, nu in enumerate(nus):
        assert maxnorm_err(D[k], O.pairwise_matrix(Xd, nu)) <= 1e-12
    assert D[0][5, 9] == 0.0
    monkeypatch.setenv("GMDS_NO_GEN", "1")
    Dm = G.pairwise_gini(X, nus)
    assert np.max(np.abs(D - Dm)) <= 1e-12 * np.max(np.abs(Dm))


@pytest.mark.parametrize("nu", [2.0, 2.5])
def test_metric_shape_full_size_properties(nu):
    # BASELINE's metric shape (n = 20000, p = 784, image-like): the whole matrix
    # on the device (fp32, full layout), then size-independent checks --
    # finite, non-negative, zero diagonal, symmetric, bit-identical on a repeat
    # and across a 2-way tile sharding -- and 400 random pairs plus the
    # duplicated-row pair against the oracle (fp32 output: 1e-6 max-normalised)
    torch = pytest.importorskip("torch")
    n, p = 20000, 784
    X = image_like(n, p, 2024)
    X[17] = X[19011]
    dX = torch.from_numpy(X).cuda()
    D = torch.empty(n * n, dtype=torch.float32, device="cuda")
    G.pairwise_gini_device(dX.data_ptr(), G.F32, n, p, [nu], G.F32, False, D.data_ptr())
    torch.cuda.synchronize()
    M = D.view(n, n)
    assert bool(torch.isfinite(M).all()) and float(M.min()) >= 0.0
    assert float(M.diagonal().abs().max()) == 0.0
    scale = float(M.max())
    rng = np.random.default_rng(int(nu * 10))
    I = rng.integers(0, n, 400)
    J = rng.integers(0, n, 400)
    I, J = np.minimum(I, J), np.maximum(I, J)
    keep = I < J
    I, J = np.append(I[keep], 17), np.append(J[keep], 19011)
    ti, tj = torch.from_numpy(I).cuda(), torch.from_numpy(J).cuda()
    got = M[ti, tj].double().cpu().numpy()
    assert np.array_equal(got, M[tj, ti].double().cpu().numpy())
    ref = O.gini_pairs(X.astype(np.float64), I, J, nu)
    assert np.max(np.abs(got - ref)) <= 1e-6 * scale
    assert got[-1] == 0.0
    R = torch.empty_like(D)
    G.pairwise_gini_device(dX.data_ptr(), G.F32, n, p, [nu], G.F32, False, R.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(D, R)
    del R
    pe = G.packed_elems(n)
    full = torch.zeros(pe, dtype=torch.float32, device="cuda")
    G.pairwise_gini_device(dX.data_ptr(), G.F32, n, p, [nu], G.F32, True, full.data_ptr())
    sh = torch.zeros_like(full)
    for s in range(2):
        G.pairwise_gini_device(dX.data_ptr(), G.F32, n, p, [nu], G.F32, True, sh.data_ptr(), s, 2)
    torch.cuda.synchronize()
    assert torch.equal(full, sh)


def test_metric_shape_pinned_drop_in_matches_device():
    # the bench's e2e call at the metric shape: host fp32 X -> pinned fp64 n x n,
    # filled stripe by stripe while later tiles compute (launches capped at
    # nbt/24 block rows); every entry written (NaN-prefilled destination) and
    # equal bit for bit to the device-resident entry's full fp64 matrix
    torch = pytest.importorskip("torch")
    n, p = 20000, 784
    X = image_like(n, p, 2026)
    pinned = torch.full((1, n, n), float("nan"), dtype=torch.float64).pin_memory()
    got = G.pairwise_gini(X, [2.0], out=pinned.numpy())
    assert not bool(torch.isnan(pinned).any())
    dX = torch.from_numpy(X).cuda()
    D = torch.empty(n * n, dtype=torch.float64, device="cuda")
    G.pairwise_gini_device(dX.data_ptr(), G.F32, n, p, [2.0], G.F64, False, D.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(pinned.view(-1).cuda(), D)
    assert got[0][123, 123] == 0.0 and got[0][5, 19000] == got[0][19000, 5]
