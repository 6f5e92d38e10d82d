"""The CPU oracle against every known answer the reference states for this path.

The reference ships no tests or fixtures; its pins are the SPEC
examples and acceptance criteria cited per test.  These run without a GPU.
"""
import numpy as np
import pytest


def test_hyperceiling(oracle):
    assert [oracle.hyperceiling(x) for x in (1, 3, 4)] == [1, 4, 4]
    assert [oracle.hyperceiling(x) for x in (2, 5, 8, 9, 1023, 1025)] == [2, 8, 8, 16, 1024, 2048]


def test_knnbuf_spec_example(oracle):  # SPEC.md:493 k=2, [5,1,3,2] -> {1,2}
    d, i, comp, bound = oracle.knnbuf_run(2, np.array([5, 1, 3, 2.0]), np.arange(4))
    assert list(d) == [1.0, 2.0] and list(i) == [1, 3]


def test_knnbuf_one_compaction(oracle):  # SPEC.md:494 2k then one more -> one compaction, bound = kth
    rng = np.random.default_rng(0)
    for k in (1, 3, 10):
        x = rng.random(2 * k + 1)
        d, i, comp, bound = oracle.knnbuf_run(k, x, np.arange(2 * k + 1))
        assert comp == 1
        assert bound == np.sort(x[: 2 * k])[k - 1]
        assert np.array_equal(d, np.sort(x)[:k])


def test_knnbuf_property(oracle):  # SPEC.md:495, 520 extract == k smallest, any order
    rng = np.random.default_rng(1)
    for trial in range(50):
        k = int(rng.integers(1, 20))
        n = int(rng.integers(0, 300))
        x = rng.integers(0, 50, n).astype(np.float64)  # many ties: broken by id
        ids = rng.permutation(n).astype(np.uint32)
        d, i, _, _ = oracle.knnbuf_run(k, x, ids)
        order = np.lexsort((ids, x))[:k]
        assert np.array_equal(d, x[order]) and np.array_equal(i, ids[order])


def test_veb_golden_layout(oracle):  # SPEC.md:476, 705; PAPER.md Fig. vebconstruct
    P = np.array([(0, 0), (1, 0), (0, 1), (1, 1), (2, 0), (3, 0), (2, 1), (3, 1)], float)
    t = oracle.Tree(P, leaf=1)
    nodes, ids, pts = t.export()
    assert t.info()["height"] == 4 and len(nodes) == 15
    assert (nodes[0]["left"], nodes[0]["right"]) == (1, 2)
    assert [nodes[1]["left"], nodes[1]["right"], nodes[2]["left"], nodes[2]["right"]] == [3, 6, 9, 12]
    for s in (3, 6, 9, 12):
        assert nodes[s]["depth"] == 2 and (nodes[s]["left"], nodes[s]["right"]) == (s + 1, s + 2)
        assert nodes[s + 1]["kind"] == 1 and nodes[s + 2]["kind"] == 1


@pytest.mark.parametrize("l,lt_lb", [(4, (2, 2)), (5, (1, 4)), (8, (4, 4)), (9, (1, 8)), (16, (8, 8)),
                                     (17, (1, 16)), (20, (4, 16))])
def test_level_split_table(oracle, l, lt_lb):  # SURVEY.md §4 table (SPEC.md:523 reading)
    lb = oracle.hyperceiling((l + 1) // 2)
    assert (l - lb, lb) == lt_lb


def test_small_trees(oracle):  # SPEC.md:477 (1..16 points -> one leaf), 502, 504
    P = np.random.default_rng(2).random((16, 3))
    t = oracle.Tree(P)
    nodes, _, _ = t.export()
    assert len(nodes) == 1 and nodes[0]["kind"] == 1
    t1 = oracle.Tree(np.array([[0.25, 0.75]]))
    ids, d2 = t1.knn(np.array([[1.0, 1.0]]), 1)
    assert ids[0, 0] == 0 and d2[0, 0] == 0.75 ** 2 + 0.25 ** 2
    P = np.random.default_rng(3).random((500, 2))
    ids, d2 = oracle.Tree(P).knn(P, 1)
    assert np.array_equal(ids[:, 0], np.arange(500)) and np.all(d2[:, 0] == 0)


def _check_kd_order(nodes, pts, d):
    """kd-order invariant: every internal node's children partition
    its range, boxes are tight, spatial splits put x_c < s left and >= s right."""
    for nd in nodes:
        s, c = nd["start"], nd["count"]
        sub = pts[s:s + c]
        assert np.array_equal(nd["lo"][:d], sub.min(0)) and np.array_equal(nd["hi"][:d], sub.max(0))
        if nd["kind"] == 0:
            L, R = nodes[nd["left"]], nodes[nd["right"]]
            assert L["start"] == s and L["count"] + R["count"] == c and R["start"] == s + L["count"]
            if nd["mode"] == 0:
                cd = nd["dim"]
                assert np.all(pts[L["start"]:L["start"] + L["count"], cd] < nd["split"])
                assert np.all(pts[R["start"]:R["start"] + R["count"], cd] >= nd["split"])
                assert nd["split"] == (nd["lo"][cd] + nd["hi"][cd]) / 2


@pytest.mark.parametrize("heur", [0, 1])
def test_kd_invariants_and_knn(oracle, heur):  # SPEC.md:503, 511, 518-519 (reduced script count)
    rng = np.random.default_rng(4 + heur)
    for trial in range(6):
        n = int(rng.integers(1, 4000))
        d = int(rng.integers(2, 6))
        P = rng.random((n, d))
        if trial % 2:
            P = np.round(P * 8) / 8  # heavy duplicates / degenerate spatial splits
        t = oracle.Tree(P, heuristic=heur)
        nodes, ids, pts = t.export()
        assert np.array_equal(np.sort(ids), np.arange(n))
        assert np.array_equal(pts, P[ids])
        _check_kd_order(nodes, pts, d)
        Q = rng.random((200, d))
        k = int(rng.integers(1, 12))
        a = t.knn(Q, k)
        b = oracle.brute_knn(P, Q, k)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        # erase a random subset: surviving set seen by kNN
        er = P[rng.choice(n, n // 3, replace=False)] if n > 3 else P[:0]
        t.erase(er)
        alive = ~(P[:, None, :] == er[None, :, :]).all(-1).any(1) if len(er) else np.ones(n, bool)
        a = t.knn(Q, k)
        b = oracle.brute_knn(P[alive], Q, k, np.arange(n, dtype=np.uint32)[alive])
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_bdl_bitmask_arithmetic(oracle):
    for n, F, buf in ((0, 0, 0), (1024, 1, 0), (3 * 1024 + 1, 3, 1)):
        b = oracle.BDLTree(2)
        if n:
            b.insert(np.random.default_rng(n).random((n, 2)))
        s = b.stats()
        assert (s["F"], s["buffer"]) == (F, buf)


@pytest.mark.parametrize("X", [1024, 4])
def test_bdl_insert_figure(oracle, X):  # SPEC.md:578-580, 707, Fig. bdl-insert
    rng = np.random.default_rng(X)
    b = oracle.BDLTree(2, X=X)
    b.insert(rng.random((X, 2)))
    got = [(b.stats()["F"], b.stats()["buffer"])]
    for m in (X + 1, X + 1, X - 1):
        b.insert(rng.random((m, 2)))
        got.append((b.stats()["F"], b.stats()["buffer"]))
    assert got == [(1, 0), (2, 1), (3, 2), (4, 1)]
    s = b.stats()
    assert s["build_size"][2] == 4 * X and s["live"][2] == 4 * X


def test_bdl_model_scripts(oracle):  # SPEC.md:589, 611, 708 (reduced: 25 scripts)
    rng = np.random.default_rng(7)
    for script in range(25):
        d = int(rng.integers(2, 4))
        X = int(rng.choice([4, 16, 64]))
        b = oracle.BDLTree(d, X=X)
        model_ids, model_pts = [], []
        next_id = 0
        for op in range(int(rng.integers(5, 20))):
            r = rng.random()
            if r < 0.5 or not model_ids:
                m = int(rng.integers(0, 4 * X))
                P = np.round(rng.random((m, d)) * 6) / 6  # small universe: duplicates
                b.insert(P)
                model_ids += list(range(next_id, next_id + m)); model_pts += list(P); next_id += m
            elif r < 0.8:
                m = int(rng.integers(0, 2 * X))
                E = np.round(rng.random((m, d)) * 6) / 6
                killed = b.erase(E)
                es = {tuple(e) for e in E}
                keep = [i for i, p in enumerate(model_pts) if tuple(p) not in es]
                assert killed == len(model_ids) - len(keep)
                model_ids = [model_ids[i] for i in keep]; model_pts = [model_pts[i] for i in keep]
                s = b.stats()
                for i in range(64):  # half-capacity invariant
                    if s["F"] >> i & 1:
                        assert 2 * s["live"][i] >= s["build_size"][i]
            else:
                Q = rng.random((50, d))
                k = int(rng.integers(1, 8))
                a = b.knn(Q, k)
                if model_ids:
                    e = oracle.brute_knn(np.array(model_pts), Q, k, np.array(model_ids, np.uint32))
                else:
                    e = (np.full((50, k), 0xFFFFFFFF, np.uint32), np.full((50, k), np.inf))
                assert np.array_equal(a[0], e[0]) and np.array_equal(a[1], e[1])
            lid, lp = b.live()
            assert np.array_equal(lid, np.array(sorted(model_ids), np.uint32).reshape(-1))


def test_bdl_batching_invariance(oracle):
    rng = np.random.default_rng(8)
    P = rng.random((5000, 3))
    Q = rng.random((300, 3))
    a = oracle.BDLTree(3, X=64); a.insert(P)
    b = oracle.BDLTree(3, X=64)
    for chunk in np.array_split(P, 7):
        b.insert(chunk)
    ra, rb = a.knn(Q, 6), b.knn(Q, 6)
    assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])


def test_determinism_across_threads(oracle):
    P = oracle.gen_uniform(20000, 3, 11)
    Q = oracle.gen_uniform(2000, 3, 12)
    res = []
    for t in (1, 2, oracle.max_threads()):
        oracle.set_threads(t)
        b = oracle.BDLTree(3); b.insert(P)
        res.append(b.knn(Q, 5))
        nodes, ids, pts = b.tree_export(4)
        res.append((nodes.tobytes(), ids))
    oracle.set_threads(oracle.max_threads())
    for r in res[2::2]:
        assert np.array_equal(r[0], res[0][0]) and np.array_equal(r[1], res[0][1])
    for r in res[3::2]:
        assert r[0] == res[1][0] and np.array_equal(r[1], res[1][1])


# --------------------------------------------------- §8f-4: range search, kNN graph
def _brute_d2(P, q):
    """canonical d2 (sum_j (q_j - p_j)^2, left to right, no FMA) of every row of P"""
    t = q[0] - P[:, 0]
    s = t * t
    for j in range(1, P.shape[1]):
        t = q[j] - P[:, j]
        s = s + t * t
    return s


def _small_structure(oracle, d, seed):
    rng = np.random.default_rng(seed)
    o = oracle.BDLTree(d, X=64, leaf=4)
    P = rng.random((700, d))
    P[500:540] = P[:40]  # exact duplicates (distinct ids)
    o.insert(P[:300])
    o.insert(P[300:])
    o.erase(P[rng.choice(700, 90, replace=False)])  # tombstones, collapses, reinsertions
    return o, rng


@pytest.mark.parametrize("d", [2, 3, 7])
def test_range_oracle_vs_brute(oracle, d):  # PAPER.md:188-190, 204 (kd-tree range search)
    o, rng = _small_structure(oracle, d, 11 + d)
    ids_live, P = o.live()
    Q = np.concatenate([rng.random((60, d)), P[:20]])
    for r2 in (0.0, 0.01, 0.2, np.inf):
        offs, ids, d2 = o.range(Q, r2)
        for i, q in enumerate(Q):
            dd = _brute_d2(P, q)
            m = dd <= r2
            order = np.lexsort((ids_live[m], dd[m]))
            a, b = int(offs[i]), int(offs[i + 1])
            assert np.array_equal(ids[a:b], ids_live[m][order]), (r2, i)
            assert np.array_equal(d2[a:b], dd[m][order]), (r2, i)


@pytest.mark.parametrize("k", [1, 5, 17])
def test_knn_graph_oracle_vs_brute(oracle, k):  # PAPER.md:202-203 (k-NN graph generator)
    o, _ = _small_structure(oracle, 3, 5 + k)
    ids_live, P = o.live()
    rows, ids, d2 = o.knn_graph(k)
    assert np.array_equal(rows, ids_live)
    for r in range(len(rows)):
        dd = _brute_d2(P, P[r])
        keep = np.arange(len(P)) != r
        order = np.lexsort((ids_live[keep], dd[keep]))[:k]
        want_i = ids_live[keep][order]
        want_d = dd[keep][order]
        assert np.array_equal(ids[r, :len(want_i)], want_i), r
        assert np.array_equal(d2[r, :len(want_d)], want_d), r


@pytest.mark.parametrize("d", [2, 3, 6])
def test_range_box_oracle_vs_brute(oracle, d):  # orthogonal kd-tree range search
    o, rng = _small_structure(oracle, d, 31 + d)
    ids_live, P = o.live()
    c = np.concatenate([rng.random((50, d)), P[:10]])
    for half in (0.0, 0.05, 0.3, 2.0):
        lo, hi = c - half, c + half
        offs, ids = o.range_box(lo, hi)
        for i in range(len(c)):
            m = ((P >= lo[i]) & (P <= hi[i])).all(1)
            assert np.array_equal(ids[offs[i]:offs[i + 1]], np.sort(ids_live[m])), (half, i)
    offs, ids = o.range_box(c + 0.1, c - 0.1)  # empty boxes
    assert len(ids) == 0
