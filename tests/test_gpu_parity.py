"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact: neighbour ids, the built trees' point permutation, canonical node
records (vEB slots, splits, boxes), the log structure's F / buffer / live
counts.  Squared distances: within 1e-12 relative (north star); they come out
bit-identical because both sides use the same no-FMA operation order.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL = 1e-12
FIELDS = ("kind", "dim", "mode", "depth", "split", "left", "right", "start", "count", "lo", "hi")


def assert_knn_equal(a, b, what=""):
    ia, da = a
    ib, db = b
    assert ia.shape == ib.shape, what
    bad = np.nonzero((ia != ib).any(1))[0]
    assert len(bad) == 0, f"{what}: {len(bad)} rows differ, first {bad[:5]}: {ia[bad[:1]]} vs {ib[bad[:1]]}"
    fin = np.isfinite(db)
    assert np.array_equal(np.isfinite(da), fin), what
    rel = np.abs(da[fin] - db[fin]) / np.maximum(np.abs(db[fin]), 1e-300)
    assert (rel <= RTOL).all(), f"{what}: max rel {rel.max()}"


def assert_tree_equal(g, o, i):
    gn, gi, gp = g.tree_export(i)
    on, oi, op = o.tree_export(i)
    assert np.array_equal(gi, oi), f"tree {i}: permutation differs"
    dead = o.tree_dead(i)  # the device tombstone is a NaN in coordinate 0
    assert np.array_equal(np.isnan(gp[:, 0]), dead), f"tree {i}: tombstones differ"
    np.testing.assert_array_equal(gp[~dead], op[~dead])
    np.testing.assert_array_equal(gp[dead, 1:], op[dead, 1:])
    assert len(gn) == len(on), f"tree {i}: {len(gn)} vs {len(on)} nodes"
    # the buffer tree (i = -1) is rebuilt rather than collapsed: its root is slot 0
    groot = int(g.info()["root_per_tree"][i]) if i >= 0 else (0 if len(gn) else -1)
    oroot = o.tree_root(i)
    assert groot == oroot, f"tree {i}: root slot {groot} vs {oroot}"
    # nodes reachable from the root (Erase_S collapses splice nodes out; unreachable records are stale)
    reach, stack = [], [groot] if groot >= 0 else []
    while stack:
        v = stack.pop()
        reach.append(v)
        if on[v]["kind"] == 0:
            stack += [int(on[v]["right"]), int(on[v]["left"])]
    reach = np.array(reach, np.int64)
    if not dead.any():
        assert len(reach) == len(on)
    for f in FIELDS:
        assert np.array_equal(gn[f][reach], on[f][reach]), f"tree {i}: node field {f} differs"


def assert_struct_equal(g, o, trees=True):
    gi, oi = g.info(), o.stats()
    assert gi["F"] == oi["F"] and gi["buffer"] == oi["buffer"]
    assert np.array_equal(gi["build_size"], oi["build_size"])
    assert np.array_equal(gi["live_per_tree"], oi["live"])
    if trees:
        for i in range(64):
            if gi["F"] >> i & 1:
                assert_tree_equal(g, o, i)
        if gi["buffer"]:
            assert_tree_equal(g, o, -1)  # Build_S of the buffer (a-7): permutation + nodes bit-exact


def run_script(gk, oracle, d, script, X=1024, leaf=16, heur=0, trees=True):
    g = gk.BDLTree(d, X=X, leaf_size=leaf, heuristic=heur)
    o = oracle.BDLTree(d, X=X, leaf=leaf, heuristic=heur)
    for step, op in enumerate(script):
        if op[0] == "insert":
            g.insert(op[1]); o.insert(op[1])
            assert_struct_equal(g, o, trees)
        elif op[0] == "erase":
            kg, ko = g.erase(op[1]), o.erase(op[1])
            assert kg == ko, f"step {step}: erased {kg} vs {ko}"
            assert_struct_equal(g, o, trees)
        else:
            assert_knn_equal(g.knn(op[1], op[2]), o.knn(op[1], op[2]), f"step {step} knn k={op[2]}")
    return g, o


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_baseline_configs_reduced(gk, oracle, cfg):
    from paper_2207_01834_b200.configs import make_inputs
    d, script = make_inputs(cfg, scale=0.01)
    run_script(gk, oracle, d, script)


def test_golden_fixture(gk):
    import os
    g0 = np.load(os.path.join(os.path.dirname(__file__), "golden", "oracle_small.npz"))
    g = gk.BDLTree(3)
    g.insert(g0["P"])
    ids, d2 = g.knn(g0["Q"], 10)
    assert np.array_equal(ids, g0["ids"]) and np.array_equal(d2, g0["d2"])
    nodes, tids, tpts = g.tree_export(1)
    assert nodes.view(np.uint8).tobytes() == g0["tree1_nodes"].tobytes()
    assert np.array_equal(tids, g0["tree1_ids"]) and np.array_equal(tpts, g0["tree1_pts"])


def test_golden_veb_layout(gk, oracle):  # SPEC.md:476 / Fig. vebconstruct, through BuildvEB_S on the GPU
    P = np.array([(0, 0), (1, 0), (0, 1), (1, 1), (2, 0), (3, 0), (2, 1), (3, 1)], float)
    g = gk.BDLTree(2, X=8, leaf_size=1)
    g.insert(P)
    nodes, _, _ = g.tree_export(0)
    assert [nodes[1]["left"], nodes[1]["right"], nodes[2]["left"], nodes[2]["right"]] == [3, 6, 9, 12]
    on, _, _ = oracle.Tree(P, leaf=1).export()
    assert nodes.tobytes() == on.tobytes()


@pytest.mark.parametrize("d", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("k", [1, 3, 10, 11, 12, 16, 32, 33, 100, 256])
def test_dims_and_k(gk, oracle, d, k):
    rng = np.random.default_rng(100 * d + k)
    P = rng.random((6000, d))
    Q = rng.random((700, d))
    run_script(gk, oracle, d, [("insert", P), ("knn", Q, k), ("knn", P[:500], k)], X=256)


@pytest.mark.parametrize("d,k", [(2, 257), (3, 600), (7, 300), (3, 5000)])
def test_large_k_global_heap(gk, oracle, d, k):
    """k above the shared-memory k-buffers (k > 256): per-lane heaps in a global scratch buffer;
    k = 5000 > n_live for the second script step exercises the padding rows."""
    rng = np.random.default_rng(7 * d + k)
    P = rng.random((4000, d))
    Q = rng.random((300, d))
    run_script(gk, oracle, d, [("insert", P), ("knn", Q, k), ("knn", P[:200], k)], X=256)


@pytest.mark.parametrize("leaf", [1, 2, 8, 32])
@pytest.mark.parametrize("heur", [0, 1])
def test_leaf_and_heuristic(gk, oracle, leaf, heur):
    rng = np.random.default_rng(leaf + 10 * heur)
    P = rng.random((5000, 3))
    run_script(gk, oracle, 3, [("insert", P), ("knn", rng.random((500, 3)), 7)], X=512, leaf=leaf, heur=heur)


def test_degenerate_duplicates(gk, oracle):
    """heavy duplicates: degenerate spatial splits fall back to the (x_c, id) object median"""
    rng = np.random.default_rng(5)
    P = np.round(rng.random((20000, 2)) * 4) / 4
    P[:3000] = 0.5  # one point repeated 3000 times
    P[3000:3100, 0] = -0.0
    P[3100:3200, 0] = 0.0
    Q = np.concatenate([rng.random((300, 2)), P[:50]])
    g, o = run_script(gk, oracle, 2, [("insert", P), ("knn", Q, 16), ("erase", P[2990:3005]), ("knn", Q, 5)], X=1000)


def test_deep_spatial_tree(gk, oracle):
    """exponentially spaced coordinates drive spatial splits past the depth cap (object median below it)"""
    x = 2.0 ** -np.arange(1, 300, dtype=np.float64)
    P = np.stack([x, np.zeros_like(x)], 1)
    P = np.concatenate([P, np.random.default_rng(1).random((500, 2))])
    run_script(gk, oracle, 2, [("insert", P), ("knn", P, 4)], X=len(P), leaf=2)


def test_empty_and_short(gk, oracle):
    g = gk.BDLTree(3)
    ids, d2 = g.knn(np.zeros((4, 3)), 5)  # empty structure: padded rows
    assert (ids == gk.NO_POINT).all() and np.isinf(d2).all()
    P = np.random.default_rng(2).random((3, 3))
    run_script(gk, oracle, 3, [("insert", P), ("knn", np.random.default_rng(3).random((10, 3)), 8)])


def test_errors(gk):
    g = gk.BDLTree(3)
    with pytest.raises(NotImplementedError):
        g.knn(np.zeros((1, 3)), gk.MAX_K + 1)
    with pytest.raises(ValueError):
        g.knn(np.zeros((1, 3)), 0)
    with pytest.raises(ValueError):
        g.insert(np.array([[0.0, np.nan, 1.0]]))
    with pytest.raises(ValueError):
        g.insert(np.zeros((2, 4)))
    assert g.info()["live"] == 0


def test_insert_figure_X4(gk, oracle):  # SPEC.md:578-580 with X = 4
    rng = np.random.default_rng(4)
    script = [("insert", rng.random((4, 2))), ("insert", rng.random((5, 2))), ("insert", rng.random((5, 2))),
              ("insert", rng.random((3, 2))), ("knn", rng.random((50, 2)), 3)]
    g, o = run_script(gk, oracle, 2, script, X=4)
    assert g.info()["F"] == 4 and g.info()["buffer"] == 1


def test_erase_all_and_absent(gk, oracle):
    rng = np.random.default_rng(6)
    P = rng.random((3000, 2))
    script = [("insert", P), ("erase", rng.random((100, 2))), ("knn", P[:20], 3), ("erase", P),
              ("knn", P[:20], 3), ("insert", P[:1500]), ("knn", P[:40], 4)]
    g, o = run_script(gk, oracle, 2, script, X=128)
    assert g.info()["live"] == 1500


def test_model_scripts(gk, oracle):
    """random insert/erase/kNN scripts with a small coordinate universe (duplicates, absent erases,
    half-capacity rebuilds, tombstoned-pool re-decomposition)"""
    rng = np.random.default_rng(77)
    for s in range(12):
        d = int(rng.integers(2, 5))
        X = int(rng.choice([4, 16, 64]))
        script = []
        for op in range(int(rng.integers(5, 15))):
            r = rng.random()
            if r < 0.5:
                script.append(("insert", np.round(rng.random((int(rng.integers(0, 4 * X)), d)) * 6) / 6))
            elif r < 0.8:
                script.append(("erase", np.round(rng.random((int(rng.integers(0, 2 * X)), d)) * 6) / 6))
            else:
                script.append(("knn", rng.random((64, d)), int(rng.integers(1, 9))))
        run_script(gk, oracle, d, script, X=X)


def test_device_api_matches_host_api(gk):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(9)
    P = rng.random((50000, 3))
    Q = rng.random((20000, 3))
    a = gk.BDLTree(3)
    a.insert(P)
    b = gk.BDLTree(3)
    b.insert_device(torch.from_numpy(P).cuda())
    ids = torch.empty((len(Q), 10), dtype=torch.int32, device="cuda")
    d2 = torch.empty((len(Q), 10), dtype=torch.float64, device="cuda")
    b.knn_device(torch.from_numpy(Q).cuda(), 10, ids, d2)
    torch.cuda.synchronize()
    ra = a.knn(Q, 10)
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), ra[0]) and np.array_equal(d2.cpu().numpy(), ra[1])
    c = b.knn_counted_device(torch.from_numpy(Q).cuda(), 10, ids, d2)
    assert c["nodes"] > 0 and c["leaves"] > 0 and c["dists"] >= 10 * len(Q)
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), ra[0])


def _full_properties(P, Q, ids, d2, k):
    """size-independent checks of a full-size kNN result"""
    assert (ids < len(P)).all()
    assert (np.diff(d2, axis=1) >= 0).all()
    same = np.diff(d2, axis=1) == 0
    assert (np.diff(ids.astype(np.int64), axis=1)[same] > 0).all()  # ties by ascending id
    rows = np.random.default_rng(0).choice(len(Q), 20000, replace=False)  # d2 recomputed on a sample
    diff = Q[rows][:, None, :] - P[ids[rows].astype(np.int64)]
    rec = np.zeros(diff.shape[:2])
    for j in range(P.shape[1]):
        rec = rec + diff[..., j] * diff[..., j]
    assert np.array_equal(rec, d2[rows])
    return rows


@pytest.mark.slow
def test_full_c2_every_row_against_oracle(gk, oracle):
    """BASELINE config 2 at full size (10M points, 10M queries): every one of the 10M kNN rows against the
    oracle BDL-tree over the same points (ids bit-exact, d2 within 1e-12), plus the size-independent
    properties, the structure (F / buffer / live counts), the 8.4M-point tree and the buffer tree."""
    from paper_2207_01834_b200.configs import make_inputs
    d, script = make_inputs(2)
    P, (_, Q, k) = script[0][1], script[1]
    g = gk.BDLTree(3)
    g.insert(P)
    ids, d2 = g.knn(Q, k)
    _full_properties(P, Q, ids, d2, k)
    o = oracle.BDLTree(3)
    o.insert(P)
    assert_struct_equal(g, o, trees=False)
    assert_tree_equal(g, o, 13)  # the 8.4M-point tree: permutation + nodes bit-exact
    assert_tree_equal(g, o, -1)  # the buffer tree (640 points)
    assert_knn_equal((ids, d2), o.knn(Q, k), "C2 full, every row")


@pytest.mark.slow
def test_full_c1_self_queries(gk, oracle):
    from paper_2207_01834_b200.configs import make_inputs
    d, script = make_inputs(1)
    P = script[0][1]
    g = gk.BDLTree(2)
    g.insert(P)
    ids, d2 = g.knn(P, 5)
    assert np.array_equal(ids[:, 0], np.arange(len(P), dtype=np.uint32)) and (d2[:, 0] == 0).all()
    _full_properties(P, P, ids, d2, 5)
    o = oracle.BDLTree(2)
    o.insert(P)
    assert_struct_equal(g, o, trees=True)
    assert_knn_equal((ids, d2), o.knn(P, 5), "C1 full, every row")


def test_host_knn_pipelines(gk):
    """host API: pinned buffers take the chunked copy/compute pipeline, pageable ones the same pipeline
    through the handle's pinned staging ring (blocks of 16 MiB, not a multiple of the row size here);
    both identical to the device-resident kNN_L, for every chunk schedule"""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(12)
    P = rng.random((300000, 3))
    Q = rng.random((2_600_000, 3))
    g = gk.BDLTree(3)
    g.insert(P)
    di = torch.empty((len(Q), 8), dtype=torch.int32, device="cuda")
    dd = torch.empty((len(Q), 8), dtype=torch.float64, device="cuda")
    g.knn_device(torch.from_numpy(Q).cuda(), 8, di, dd)
    ids0, d20 = di.cpu().numpy().view(np.uint32), dd.cpu().numpy()
    Qp = torch.from_numpy(Q).pin_memory().numpy()
    pinned = (torch.empty((len(Q), 8), dtype=torch.int32).pin_memory().numpy().view(np.uint32),
              torch.empty((len(Q), 8), dtype=torch.float64).pin_memory().numpy())
    pageable = (np.empty((len(Q), 8), np.uint32), np.empty((len(Q), 8), np.float64))
    mixed = (pinned[0], pageable[1])
    for qbuf, (ids, d2) in ((Qp, pinned), (Q, pageable), (Q, mixed), (Qp, pageable)):
        for chunks, ratio in ((None, None), ("4", "1"), ("5", "1.5"), ("3", "0.5"), ("40", "1")):  # schedule knobs
            if chunks:
                os.environ["GK_PIPE_CHUNKS"], os.environ["GK_PIPE_RATIO"] = chunks, ratio
            ids.fill(0)
            d2.fill(0)
            try:
                rc = gk.lib().gk_bdl_knn(g._h, qbuf.ctypes.data, len(Q), 8, ids.ctypes.data, d2.ctypes.data)
            finally:
                os.environ.pop("GK_PIPE_CHUNKS", None)
                os.environ.pop("GK_PIPE_RATIO", None)
            assert rc == 0, gk.lib().gk_last_error()
            assert np.array_equal(ids, ids0) and np.array_equal(d2, d20), (chunks, ratio)


def test_bloom_filter(gk):
    """SPEC.md:604-606 / acceptance 10: no false negatives over 1e5 keys, FP <= 2% at 10 bits/key, h = 7"""
    rng = np.random.default_rng(2022)
    P = rng.random((100000, 3))
    g = gk.BDLTree(3, X=100000)
    g.insert(P)
    assert g.info()["F"] == 1
    assert g.bloom_may_contain(0, P).all()                      # no false negatives
    fp = g.bloom_may_contain(0, rng.random((200000, 3))).mean()
    assert fp <= 0.02, fp
    g2 = gk.BDLTree(3, X=4)
    g2.insert(np.array([[0.0, -0.0, 1.0]] * 4))
    assert g2.bloom_may_contain(0, np.array([[-0.0, 0.0, 1.0]])).all()  # -0 == +0 probes the same bits


def _script_parity(gk, oracle, cfg, trees=True):
    """Full-size BASELINE script on both sides: structure (F, buffer, live counts, every static tree's and the
    buffer tree's permutation/tombstones/nodes) bit-exact after every operation, every kNN row exact."""
    from paper_2207_01834_b200.configs import make_inputs
    d, script = make_inputs(cfg)
    g = gk.BDLTree(d)
    o = oracle.BDLTree(d)
    for step, op in enumerate(script):
        if op[0] == "insert":
            g.insert(op[1]); o.insert(op[1])
            assert_struct_equal(g, o, trees)
        elif op[0] == "erase":
            assert g.erase(op[1]) == o.erase(op[1])
            assert_struct_equal(g, o, trees)
        else:
            Q, k = op[1], op[2]
            assert_knn_equal(g.knn(Q, k), o.knn(Q, k), f"config {cfg} step {step}, every row")


@pytest.mark.slow
def test_full_c3_every_row(gk, oracle):
    _script_parity(gk, oracle, 3)


@pytest.mark.slow
def test_full_c4_every_row(gk, oracle):
    _script_parity(gk, oracle, 4)


@pytest.mark.slow
def test_full_c5_every_row(gk, oracle):
    _script_parity(gk, oracle, 5)


@pytest.mark.slow
def test_object_median_at_scale(gk, oracle):
    """object-median heuristic on 1M points: every level runs the device radix select
    (thousands of object nodes per level, batched); permutation + nodes bit-exact"""
    rng = np.random.default_rng(21)
    P = rng.random((1_000_000, 3))
    Q = rng.random((20000, 3))
    run_script(gk, oracle, 3, [("insert", P), ("knn", Q, 10)], X=1_000_000, heur=1)


@pytest.mark.slow
def test_heavy_duplicates_at_scale(gk, oracle):
    """600k points on 2000 distinct sites: degenerate spatial splits everywhere -> large
    object-median fallbacks keyed by (x_c, id); then erase whole sites (all duplicates)"""
    rng = np.random.default_rng(22)
    sites = rng.random((2000, 2))
    P = sites[rng.integers(0, 2000, 600_000)]
    script = [("insert", P), ("knn", sites[:500], 16), ("erase", sites[:300]), ("knn", sites[:500], 16),
              ("insert", P[:5000]), ("knn", rng.random((2000, 2)), 7)]
    run_script(gk, oracle, 2, script, X=4096)


def test_bounded_knn(gk, oracle):
    """radius-bounded kNN_L: row i = the exact kNN row cut at d2 <= r2[i] (inclusive), padded with
    (NO_POINT, +inf); r2 = +inf is plain kNN_L, r2 = 0 keeps only coincident points"""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(31)
    P = np.round(rng.random((40000, 3)) * 200) / 200  # duplicates: ties at the radius
    Q = np.concatenate([rng.random((3000, 3)), P[:500]])
    k = 10
    o = oracle.BDLTree(3)
    o.insert(P)
    ei, ed = o.knn(Q, k)
    r2 = ed[np.arange(len(Q)), rng.integers(0, k, len(Q))].copy()  # a radius through some row entry
    r2[::7] = np.inf
    r2[3::7] = 0.0
    r2[5::7] *= 0.5
    g = gk.BDLTree(3)
    g.insert(P)
    ids = torch.empty((len(Q), k), dtype=torch.int32, device="cuda")
    d2 = torch.empty((len(Q), k), dtype=torch.float64, device="cuda")
    g.knn_bounded_device(torch.from_numpy(Q).cuda(), k, torch.from_numpy(r2).cuda(), ids, d2)
    gi, gd = ids.cpu().numpy().view(np.uint32), d2.cpu().numpy()
    keep = ed <= r2[:, None]
    wi = np.where(keep, ei, gk.NO_POINT).astype(np.uint32)
    wd = np.where(keep, ed, np.inf)
    assert np.array_equal(gi, wi) and np.array_equal(gd, wd)
    bad = torch.from_numpy(r2).cuda()
    bad[1] = -1.0
    with pytest.raises(ValueError):
        g.knn_bounded_device(torch.from_numpy(Q).cuda(), k, bad, ids, d2)


def test_device_tensor_validation(gk):
    """the device API refuses tensors whose raw pointers would be misread: host tensors, wrong dtypes,
    strided views, wrong shapes"""
    torch = pytest.importorskip("torch")
    g = gk.BDLTree(3)
    g.insert(np.random.default_rng(1).random((5000, 3)))
    q = torch.rand((100, 3), dtype=torch.float64, device="cuda")
    ids = torch.empty((100, 4), dtype=torch.int32, device="cuda")
    d2 = torch.empty((100, 4), dtype=torch.float64, device="cuda")
    g.knn_device(q, 4, ids, d2)
    for args in ((q.cpu(), 4, ids, d2), (q, 4, ids.long(), d2), (q, 4, ids, d2.float()), (q.t().contiguous().t(), 4, ids, d2),
                 (q, 5, ids, d2), (q[:, :2], 4, ids, d2), (q.float(), 4, ids, d2), (q, 4, ids[:50], d2)):
        with pytest.raises(ValueError):
            g.knn_device(*args)
    with pytest.raises(ValueError):
        g.insert_device(torch.rand((10, 3), dtype=torch.float64))
    with pytest.raises(ValueError):
        g.range_device(q, 0.01, torch.zeros(101, dtype=torch.int64), None, None, 0)
