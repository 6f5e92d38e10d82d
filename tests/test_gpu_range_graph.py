"""GPU parity for the §8f-4 consumers of the kd-trees: ball range search and the
k-NN graph, through the C ABI against the oracle.

Rows are bit-exact: ids, the per-query row order (d2, id) and the squared
distances (same no-FMA canonical arithmetic on both sides; RTOL kept as the
north-star bound)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL = 1e-12


def _same(a, b, what):
    for x, y, name in zip(a, b, ("offsets", "ids", "d2")):
        assert x.shape == y.shape, f"{what}: {name} shape {x.shape} vs {y.shape}"
        if name == "d2":
            fin = np.isfinite(y)
            assert np.array_equal(np.isfinite(x), fin), what
            rel = np.abs(x[fin] - y[fin]) / np.maximum(np.abs(y[fin]), 1e-300)
            assert (rel <= RTOL).all(), f"{what}: max rel {rel.max()}"
        else:
            bad = np.nonzero(x != y)[0]
            assert len(bad) == 0, f"{what}: {name} differs at {bad[:5]}"


def _pair(gk, oracle, d, X=1024, leaf=16, heur=0):
    return gk.BDLTree(d, X=X, leaf_size=leaf, heuristic=heur), oracle.BDLTree(d, X=X, leaf=leaf, heuristic=heur)


@pytest.mark.parametrize("d", [2, 3, 5, 7, 8])
def test_range_parity(gk, oracle, d):
    rng = np.random.default_rng(100 + d)
    g, o = _pair(gk, oracle, d, X=256, leaf=8)
    P = rng.random((20_000, d))
    P[15_000:15_500] = P[:500]  # duplicates
    for part in np.array_split(P, 3):
        g.insert(part); o.insert(part)
    E = P[rng.choice(len(P), 2_000, replace=False)]
    assert g.erase(E) == o.erase(E)
    Q = np.concatenate([rng.random((3_000, d)), P[:500]])
    # r2 giving ~ 0.5, ~ 20 and ~ 40 points per query (below / around / above the 32 slots per query), then exact
    # duplicates only
    vol = {2: np.pi, 3: 4.18879, 5: 5.26379, 7: 4.72477, 8: 4.05871}[d]
    for mean in (0.5, 20.0, 40.0):  # 40: most queries above the 32 slots (second traversal + segmented sort)
        r2 = float((mean / len(P) / vol) ** (2.0 / d))
        _same(g.range(Q, r2), o.range(Q, r2), f"d={d} r2={r2}")
        assert np.array_equal(g.range_count(Q, r2), np.diff(o.range(Q, r2)[0]))
    _same(g.range(Q, 0.0), o.range(Q, 0.0), f"d={d} r2=0")


@pytest.mark.parametrize("d", [2, 3, 7])
def test_range_per_query_radii(gk, oracle, d):
    """one squared radius per query (gk_bdl_range_radii*): each query's rows equal the oracle's
    single-radius range search of that query with its own radius (0, +inf and duplicates included)"""
    rng = np.random.default_rng(300 + d)
    g, o = _pair(gk, oracle, d, X=256, leaf=8)
    P = rng.random((8_000, d))
    P[7_000:7_200] = P[:200]
    for part in np.array_split(P, 3):
        g.insert(part); o.insert(part)
    E = P[rng.choice(len(P), 800, replace=False)]
    assert g.erase(E) == o.erase(E)
    Q = np.concatenate([rng.random((400, d)), P[:100]])
    r2 = (rng.random(len(Q)) * 40.0 / len(P)) ** (2.0 / d)
    r2[::37] = 0.0
    r2[5] = np.inf
    parts = [o.range(Q[i:i + 1], float(r2[i])) for i in range(len(Q))]
    want_counts = np.array([int(p[0][-1]) for p in parts], np.uint64)
    want = (np.concatenate([[0], np.cumsum(want_counts)]).astype(np.uint64),
            np.concatenate([p[1] for p in parts]), np.concatenate([p[2] for p in parts]))
    assert np.array_equal(g.range_count(Q, r2), want_counts)
    _same(g.range(Q, r2), want, f"d={d} per-query r2")
    with pytest.raises(ValueError):
        g.range(Q, np.full(len(Q), -1.0))
    with pytest.raises(ValueError):
        g.range_count(Q, np.full(len(Q), np.nan))
    with pytest.raises(ValueError):
        g.range(Q, r2[:-1])


def test_range_per_query_radii_device(gk, oracle):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(31)
    g, o = _pair(gk, oracle, 3)
    P = rng.random((30_000, 3))
    g.insert(P); o.insert(P)
    Q = rng.random((2_000, 3))
    r2 = rng.random(len(Q)) * 2e-3
    want = g.range(Q, r2)  # host per-query path (checked against the oracle above)
    ref = [o.range(Q[i:i + 1], float(r2[i])) for i in range(0, len(Q), 97)]
    for j, i in enumerate(range(0, len(Q), 97)):  # sampled rows straight against the oracle
        a, b = int(want[0][i]), int(want[0][i + 1])
        assert np.array_equal(want[1][a:b], ref[j][1]) and np.array_equal(want[2][a:b], ref[j][2])
    total = int(want[0][-1])
    qd, rd = torch.from_numpy(Q).cuda(), torch.from_numpy(r2).cuda()
    offs = torch.zeros(len(Q) + 1, dtype=torch.int64, device="cuda")
    ids = torch.zeros(total, dtype=torch.int32, device="cuda")
    d2 = torch.zeros(total, dtype=torch.float64, device="cuda")
    assert g.range_device(qd, rd, offs, ids, d2, total) == total
    got = (offs.cpu().numpy().view(np.uint64), ids.cpu().numpy().view(np.uint32), d2.cpu().numpy())
    _same(got, want, "device per-query r2")
    rd[7] = -1.0
    with pytest.raises(ValueError):
        g.range_device(qd, rd, offs, ids, d2, total)
    rd[7] = float("nan")
    with pytest.raises(ValueError):
        g.range_device(qd, rd, offs, ids, d2, total)


def test_range_edges(gk, oracle):
    g, o = _pair(gk, oracle, 3)
    Q = np.random.default_rng(1).random((50, 3))
    offs, ids, d2 = g.range(Q, 1.0)  # empty structure
    assert not offs.any() and len(ids) == 0
    offs, ids, d2 = g.range(Q, np.full(len(Q), 1.0))  # empty structure, per-query radii
    assert not offs.any() and len(ids) == 0
    offs, ids, d2 = g.range(Q[:0], np.zeros(0))  # no queries, per-query radii
    assert offs.tolist() == [0] and len(ids) == 0
    P = np.random.default_rng(2).random((3_000, 3))
    g.insert(P); o.insert(P)
    _same(g.range(Q, np.inf), o.range(Q, np.inf), "r2=inf")  # every live point, sorted
    offs, ids, d2 = g.range(Q[:0], 1.0)
    assert offs.tolist() == [0]
    with pytest.raises(ValueError):
        g.range(Q, -1.0)
    with pytest.raises(ValueError):
        g.range(Q, float("nan"))
    # a too-small capacity fails after writing the offsets
    import ctypes as C
    lib = gk.lib()
    offs = np.zeros(len(Q) + 1, np.uint64)
    ids = np.zeros(4, np.uint32); d2 = np.zeros(4, np.float64)
    rc = lib.gk_bdl_range(g._h, Q.ctypes.data_as(C.c_void_p), len(Q), 0.05, offs.ctypes.data_as(C.c_void_p),
                          ids.ctypes.data_as(C.c_void_p), d2.ctypes.data_as(C.c_void_p), 4)
    assert rc == 5 and int(offs[-1]) == int(o.range(Q, 0.05)[0][-1]) > 4  # GK_ERR_CAPACITY
    # an invalid radius fails before anything is computed and leaves the offsets alone
    offs[:] = 7
    rc = lib.gk_bdl_range(g._h, Q.ctypes.data_as(C.c_void_p), len(Q), float("nan"), offs.ctypes.data_as(C.c_void_p),
                          ids.ctypes.data_as(C.c_void_p), d2.ctypes.data_as(C.c_void_p), 4)
    assert rc == 1 and (offs == 7).all()


def test_range_device(gk, oracle):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(7)
    g, o = _pair(gk, oracle, 3)
    P = rng.random((50_000, 3))
    g.insert(P); o.insert(P)
    Q = rng.random((10_000, 3))
    r2 = 1e-3
    want = o.range(Q, r2)
    total = int(want[0][-1])
    qd = torch.from_numpy(Q).cuda()
    offs = torch.zeros(len(Q) + 1, dtype=torch.int64, device="cuda")
    ids = torch.zeros(total, dtype=torch.int32, device="cuda")
    d2 = torch.zeros(total, dtype=torch.float64, device="cuda")
    assert g.range_device(qd, r2, offs, ids, d2, total) == total
    got = (offs.cpu().numpy().view(np.uint64), ids.cpu().numpy().view(np.uint32), d2.cpu().numpy())
    _same(got, want, "device")


@pytest.mark.parametrize("d,k", [(2, 1), (3, 10), (7, 16), (3, 255), (3, 300)])
def test_knn_graph_parity(gk, oracle, d, k):
    rng = np.random.default_rng(200 + d + k)
    g, o = _pair(gk, oracle, d, X=128, leaf=16)
    n = 2_000 if k >= 255 else 12_000
    P = rng.random((n, d))
    P[n - 300:] = P[:300]  # duplicates at distance 0 with other ids
    for part in np.array_split(P, 4):
        g.insert(part); o.insert(part)
    E = P[rng.choice(n, n // 10, replace=False)]
    assert g.erase(E) == o.erase(E)
    gr, gi, gd = g.knn_graph(k)
    orr, oi, od = o.knn_graph(k)
    assert np.array_equal(gr, orr)
    assert np.array_equal(gi, oi), f"{np.nonzero((gi != oi).any(1))[0][:5]}"
    assert np.array_equal(np.isfinite(gd), np.isfinite(od))
    fin = np.isfinite(od)
    assert (np.abs(gd[fin] - od[fin]) <= RTOL * np.maximum(od[fin], 1e-300)).all()
    assert not (gi == gr[:, None]).any(), "a row lists its own point"


def test_knn_graph_edges(gk, oracle):
    g, o = _pair(gk, oracle, 3)
    rows, ids, d2 = g.knn_graph(3)  # empty
    assert rows.shape == (0,) and ids.shape == (0, 3)
    g.insert(np.array([[0.5, 0.5, 0.5]])); o.insert(np.array([[0.5, 0.5, 0.5]]))
    rows, ids, d2 = g.knn_graph(3)  # one point: all padding
    assert rows.tolist() == [0] and (ids == 0xFFFFFFFF).all() and np.isinf(d2).all()
    with pytest.raises(NotImplementedError):
        g.knn_graph(gk.MAX_K)
    with pytest.raises(ValueError):
        g.knn_graph(0)


def test_knn_graph_device(gk, oracle):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(9)
    g, o = _pair(gk, oracle, 3)
    P = rng.random((30_000, 3))
    g.insert(P); o.insert(P)
    n, k = len(P), 8
    rows = torch.zeros(n, dtype=torch.int32, device="cuda")
    ids = torch.zeros((n, k), dtype=torch.int32, device="cuda")
    d2 = torch.zeros((n, k), dtype=torch.float64, device="cuda")
    g.knn_graph_device(k, rows, ids, d2)
    orr, oi, od = o.knn_graph(k)
    assert np.array_equal(rows.cpu().numpy().view(np.uint32), orr)
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), oi)
    assert np.array_equal(d2.cpu().numpy(), od)


@pytest.mark.slow
def test_full_c2_range_sampled(gk, oracle):
    """BASELINE config 2 structure (10M points): 2M ball queries with ~10 points each; every row
    sorted by (d2, id) with d2 <= r2 recomputed from the coordinates, and exact oracle parity on
    5k sampled queries."""
    from paper_2207_01834_b200.configs import make_inputs
    d, script = make_inputs(2)
    P, Q = script[0][1], script[1][1][:2_000_000]
    r2 = float((10.0 / len(P) / (4.0 / 3.0 * np.pi)) ** (2.0 / 3.0))
    g = gk.BDLTree(3)
    g.insert(P)
    offs, ids, d2 = g.range(Q, r2)
    assert offs[-1] == len(ids) and 5 < len(ids) / len(Q) < 15
    q_of = np.repeat(np.arange(len(Q)), np.diff(offs).astype(np.int64))
    t = Q[q_of] - P[ids]
    rec = t[:, 0] * t[:, 0] + t[:, 1] * t[:, 1] + t[:, 2] * t[:, 2]
    assert np.array_equal(rec, d2) and (d2 <= r2).all()
    same_q = q_of[1:] == q_of[:-1]
    assert ((d2[1:] > d2[:-1]) | ((d2[1:] == d2[:-1]) & (ids[1:] > ids[:-1])) | ~same_q).all()
    o = oracle.BDLTree(3)
    o.insert(P)
    rows = np.random.default_rng(3).choice(len(Q), 5_000, replace=False)
    oo, oi, od = o.range(Q[rows], r2)
    assert np.array_equal(np.diff(offs)[rows], np.diff(oo))
    got_i = np.concatenate([ids[offs[r]:offs[r + 1]] for r in rows])
    got_d = np.concatenate([d2[offs[r]:offs[r + 1]] for r in rows])
    assert np.array_equal(got_i, oi) and np.array_equal(got_d, od)


@pytest.mark.slow
def test_full_c5_knn_graph_sampled(gk, oracle):
    """BASELINE config 5 (10M random-walk points, three 10 % Erase_L batches): the k-NN graph over the
    surviving points; oracle parity (kNN_L with k + 1, self dropped) on 20k sampled rows."""
    from paper_2207_01834_b200.configs import make_inputs
    d, script = make_inputs(5)
    g = gk.BDLTree(2)
    o = oracle.BDLTree(2)
    for op in script:
        if op[0] == "insert":
            g.insert(op[1]); o.insert(op[1])
        elif op[0] == "erase":
            assert g.erase(op[1]) == o.erase(op[1])
    k = 10
    rows, ids, d2 = g.knn_graph(k)
    lid, lpts = o.live()
    assert np.array_equal(rows, lid)
    assert not (ids == rows[:, None]).any()
    smp = np.random.default_rng(5).choice(len(rows), 20_000, replace=False)
    oi, od = o.knn(lpts[smp], k + 1)
    for j, r in enumerate(smp):
        keep = oi[j] != rows[r]
        want_i, want_d = oi[j][keep][:k], od[j][keep][:k]
        assert np.array_equal(ids[r], want_i) and np.array_equal(d2[r], want_d), r


@pytest.mark.parametrize("d", [2, 3, 7])
def test_range_box_parity(gk, oracle, d):
    rng = np.random.default_rng(300 + d)
    g, o = _pair(gk, oracle, d, X=256, leaf=8)
    P = rng.random((20_000, d))
    P[15_000:15_500] = P[:500]
    for part in np.array_split(P, 3):
        g.insert(part); o.insert(part)
    E = P[rng.choice(len(P), 2_000, replace=False)]
    assert g.erase(E) == o.erase(E)
    c = np.concatenate([rng.random((3_000, d)), P[:500]])
    for half in (0.0, 0.02, 0.15):
        lo, hi = c - half, c + half * rng.random((len(c), d))  # asymmetric boxes
        go, gi = g.range_box(lo, hi)
        oo, oi = o.range_box(lo, hi)
        assert np.array_equal(go, oo) and np.array_equal(gi, oi), (d, half)
        assert np.array_equal(g.range_box_count(lo, hi), np.diff(oo))
    go, gi = g.range_box(c + 0.1, c - 0.1)  # empty boxes
    assert not go.any() and len(gi) == 0


def test_range_box_device(gk, oracle):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(17)
    g, o = _pair(gk, oracle, 3)
    P = rng.random((50_000, 3))
    g.insert(P); o.insert(P)
    c = rng.random((10_000, 3))
    lo, hi = c - 0.01, c + 0.01
    oo, oi = o.range_box(lo, hi)
    total = int(oo[-1])
    offs = torch.zeros(len(c) + 1, dtype=torch.int64, device="cuda")
    ids = torch.zeros(max(total, 1), dtype=torch.int32, device="cuda")
    t = g.range_box_device(torch.from_numpy(lo).cuda(), torch.from_numpy(hi).cuda(), offs, ids, total)
    assert t == total
    assert np.array_equal(offs.cpu().numpy().view(np.uint64), oo)
    assert np.array_equal(ids.cpu().numpy().view(np.uint32)[:total], oi)


@pytest.mark.slow
def test_knn_batch_beyond_2_31_queries(gk, oracle):
    """Maximum batch size: one kNN_L call with 2^31 + 2^20 queries (the K2 sort takes 64-bit item
    counts past 2^31); sampled rows exact against the oracle."""
    torch = pytest.importorskip("torch")
    free, _ = torch.cuda.mem_get_info()
    nq = (1 << 31) + (1 << 20)
    if free < nq * (16 + 8 + 4 + 8) * 1.3:
        pytest.skip("needs ~100 GB of free HBM")
    rng = np.random.default_rng(77)
    P = rng.random((200_000, 2))
    g = gk.BDLTree(2)
    g.insert(P)
    gen = torch.Generator(device="cuda").manual_seed(5)
    Q = torch.rand((nq, 2), dtype=torch.float64, device="cuda", generator=gen)
    ids = torch.empty((nq, 1), dtype=torch.int32, device="cuda")
    d2 = torch.empty((nq, 1), dtype=torch.float64, device="cuda")
    g.knn_device(Q, 1, ids, d2)
    rows = torch.from_numpy(np.concatenate([rng.integers(0, nq, 3000), [0, nq - 1, (1 << 31) - 1, 1 << 31]])).cuda()
    q = Q[rows].cpu().numpy()
    o = oracle.BDLTree(2)
    o.insert(P)
    oi, od = o.knn(q, 1)
    assert np.array_equal(ids[rows].cpu().numpy().view(np.uint32), oi)
    assert np.array_equal(d2[rows].cpu().numpy(), od)


def test_pinned_host_knn_default_plans(gk):
    """gk_bdl_knn from pinned buffers with the default chunk plan in its three regimes (one chunk for a
    compute-bound 7D batch, two for a small 3D batch, 7,7,5,3,2 for a large one): rows identical to
    the device API's."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(21)
    for d, n, nq, k in ((7, 200_000, 300_000, 10), (3, 300_000, 1_000_000, 8), (3, 300_000, 4_300_000, 4)):
        g = gk.BDLTree(d)
        g.insert(rng.random((n, d)))
        Q = rng.random((nq, d))
        qd = torch.from_numpy(Q).cuda()
        ids0 = torch.empty((nq, k), dtype=torch.int32, device="cuda")
        d20 = torch.empty((nq, k), dtype=torch.float64, device="cuda")
        for _ in range(2):  # the second call plans from the first one's measured cost per query
            Qp = torch.from_numpy(Q).pin_memory().numpy()
            ids = torch.empty((nq, k), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
            d2 = torch.empty((nq, k), dtype=torch.float64).pin_memory().numpy()
            assert gk.lib().gk_bdl_knn(g._h, Qp.ctypes.data, nq, k, ids.ctypes.data, d2.ctypes.data) == 0
            g.knn_device(qd, k, ids0, d20)
            assert np.array_equal(ids, ids0.cpu().numpy().view(np.uint32)), (d, nq)
            assert np.array_equal(d2, d20.cpu().numpy()), (d, nq)
        g.close()
