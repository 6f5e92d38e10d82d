"""Pins the oracle's restatements of the reference's Rng (geokit/core/rng.hpp)
and KnnBuffer (geokit/kdtree/knn_buffer.hpp) against the reference itself:
against committed fixtures generated from the reference headers
(tests/golden/make_golden.py), and live against oracle/_ref when it was built."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def unit_double(u):
    return (np.asarray(u, np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def test_rng_matches_reference_fixture(oracle):
    g = np.load(os.path.join(GOLD, "ref_rng.npz"))
    for i, s in enumerate(g["seeds"]):
        assert np.array_equal(oracle.rng_u64(int(s), 16), g["u64"][i])
        for j, st in enumerate(g["streams"]):
            assert np.array_equal(unit_double(oracle.rng_u64(int(s), 4, stream=int(st))), g["split_dbl"][i, j])
        out = np.zeros(16, np.uint64)
        oracle.lib().gko_rng_below(int(s), 1000003, 16, out.ctypes.data)
        assert np.array_equal(out, g["below"][i])
    for key in g.files:
        if key.startswith("perm_"):
            _, n, s = key.split("_")
            assert np.array_equal(oracle.random_permutation(int(n), int(s)), g[key])
    assert list(g["perm_8_7"]) == [2, 5, 7, 3, 0, 1, 6, 4]  # SURVEY.md §0.6 (reference run)
    assert [int(oracle.lib().gko_mix64(int(x))) for x in (0, 1, 2**64 - 1)] == [int(v) for v in g["mix"]]


def test_rng_first_double_matches_survey(oracle):  # Rng(1).next_double() = 0.69351213901022923
    assert unit_double(oracle.rng_u64(1, 1))[0] == 0.69351213901022923


def test_knnbuf_matches_reference_fixture(oracle):
    g = np.load(os.path.join(GOLD, "ref_knnbuf.npz"))
    for i in range(int(g["n"][0])):
        k = int(g[f"k{i}"][0])
        od, oi, comp, bound = oracle.knnbuf_run(k, g[f"d2{i}"], g[f"ids{i}"])
        assert np.array_equal(od, g[f"od{i}"]) and np.array_equal(oi, g[f"oi{i}"])
        assert comp == int(g[f"comp{i}"][0]) and bound == float(g[f"bound{i}"][0])


def test_knnbuf_matches_reference_live(oracle):
    if oracle.ref_lib() is None:
        pytest.skip("oracle/_ref not built (no /root/reference on this host)")
    rng = np.random.default_rng(99)
    for t in range(300):
        k = int(rng.integers(1, 33))
        n = int(rng.integers(0, 8 * k + 5))
        d2 = rng.integers(0, 20, n).astype(np.float64) * rng.choice([1.0, 0.5])
        ids = rng.permutation(n).astype(np.uint32)
        a = oracle.knnbuf_run(k, d2, ids)
        b = oracle.knnbuf_run(k, d2, ids, use_ref=True)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2:] == b[2:]


def test_rng_matches_reference_live(oracle):
    R = oracle.ref_lib()
    if R is None:
        pytest.skip("oracle/_ref not built (no /root/reference on this host)")
    for seed in (5, 6, 123456789):
        ref = np.zeros(64, np.uint64)
        R.gkref_rng_u64(seed, 77, 1, 64, ref.ctypes.data)
        assert np.array_equal(oracle.rng_u64(seed, 64, stream=77), ref)
        p = np.zeros(1000, np.uint32)
        R.gkref_random_permutation(1000, seed, p.ctypes.data)
        assert np.array_equal(oracle.random_permutation(1000, seed), p)
