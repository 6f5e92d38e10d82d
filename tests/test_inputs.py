"""The product's input generators (libgkbdl.so, host code) agree bit for bit
with the oracle's independent restatement (and so, via test_oracle_pins, with
the reference's rng.hpp).  No GPU needed: the generators are host functions."""
import numpy as np
import pytest


def test_uniform(oracle, gk):
    for n, d, s in ((1, 2, 1), (1000, 3, 2), (777, 7, 4)):
        assert np.array_equal(gk.gen_uniform(n, d, s), oracle.gen_uniform(n, d, s))
    a = gk.gen_uniform(100, 3, 9)
    assert a.min() >= 0 and a.max() < 1


def test_uniform_matches_reference_stream(oracle, gk):
    """point i = Rng(seed).split(i).next_double() x d  (generators.hpp:60-63, side 1)"""
    R = oracle.ref_lib()
    if R is None:
        pytest.skip("oracle/_ref not built")
    pts = gk.gen_uniform(50, 3, 2)
    for i in range(50):
        ref = np.zeros(3, np.float64)
        R.gkref_rng_double(2, i, 1, 3, ref.ctypes.data)
        assert np.array_equal(pts[i], ref)


def test_mixture_walk_sampling(oracle, gk):
    assert np.array_equal(gk.gen_mixture(5000, 7, 4), oracle.gen_mixture(5000, 7, 4))
    m = gk.gen_mixture(5000, 7, 4)
    assert m.min() >= 0 and m.max() <= 1
    assert np.array_equal(gk.gen_walk(20, 300, 5), oracle.gen_walk(20, 300, 5))
    assert np.array_equal(gk.sample_without_replacement(10000, 1000, 6),
                          oracle.sample_without_replacement(10000, 1000, 6))
    s = gk.sample_without_replacement(1000, 1000, 3)
    assert np.array_equal(np.sort(s), np.arange(1000))
    # partial Fisher-Yates == tail of the reference's random_permutation
    assert np.array_equal(oracle.sample_without_replacement(100, 100, 11)[::-1], oracle.random_permutation(100, 11))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_configs_same_inputs(oracle, gk, cfg):
    from paper_2207_01834_b200.configs import make_inputs
    d1, s1 = make_inputs(cfg, scale=0.002)
    d2, s2 = make_inputs(cfg, scale=0.002, gen=oracle)
    assert d1 == d2 and len(s1) == len(s2)
    for a, b in zip(s1, s2):
        assert a[0] == b[0] and np.array_equal(a[1], b[1]) and a[2:] == b[2:]
