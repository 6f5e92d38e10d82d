"""Regenerates tests/golden/*.npz.  Run HERE (needs /root/reference):

    python tests/golden/make_golden.py

ref_rng.npz / ref_knnbuf.npz come from the REFERENCE's own headers
(geokit/core/rng.hpp, geokit/kdtree/knn_buffer.hpp) compiled into
oracle/_ref/libgkref.so — they pin the oracle's restatements.
oracle_small.npz holds small oracle outputs (tree exports, kNN rows) used as
regression fixtures; they are self-generated, not reference pins.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def ref_rng():
    R = O.ref_lib()
    assert R is not None, "build oracle/_ref first (needs /root/reference)"
    seeds = np.array([0, 1, 2, 3, 7, 42, 2**63 + 5], np.uint64)
    streams = np.array([0, 1, 5, 1000, 2**40 + 3], np.uint64)
    u64 = np.zeros((len(seeds), 16), np.uint64)
    split_dbl = np.zeros((len(seeds), len(streams), 4), np.float64)
    below = np.zeros((len(seeds), 16), np.uint64)
    for i, s in enumerate(seeds):
        R.gkref_rng_u64(int(s), 0, 0, 16, u64[i].ctypes.data)
        R.gkref_rng_below(int(s), 1000003, 16, below[i].ctypes.data)
        for j, st in enumerate(streams):
            R.gkref_rng_double(int(s), int(st), 1, 4, split_dbl[i, j].ctypes.data)
    perms = {}
    for n, s in ((8, 7), (1, 3), (0, 3), (100, 11)):
        p = np.zeros(n, np.uint32)
        R.gkref_random_permutation(n, s, p.ctypes.data if n else None)
        perms[f"perm_{n}_{s}"] = p
    mix = np.array([R.gkref_mix64(int(x)) for x in (0, 1, 2**64 - 1)], np.uint64)
    np.savez(os.path.join(OUT, "ref_rng.npz"), seeds=seeds, streams=streams, u64=u64, split_dbl=split_dbl,
             below=below, mix=mix, **perms)


def ref_knnbuf():
    rng = np.random.default_rng(2207)
    cases = []
    for t in range(40):
        k = int(rng.integers(1, 17))
        n = int(rng.integers(0, 6 * k + 10))
        d2 = rng.integers(0, 12, n).astype(np.float64)  # heavy ties -> id tie-break
        ids = rng.permutation(n).astype(np.uint32)
        od, oi, comp, bound = O.knnbuf_run(k, d2, ids, use_ref=True)
        cases.append((k, d2, ids, od, oi, comp, bound))
    arrs = {}
    for i, (k, d2, ids, od, oi, comp, bound) in enumerate(cases):
        arrs[f"k{i}"] = np.array([k]); arrs[f"d2{i}"] = d2; arrs[f"ids{i}"] = ids
        arrs[f"od{i}"] = od; arrs[f"oi{i}"] = oi; arrs[f"comp{i}"] = np.array([comp]); arrs[f"bound{i}"] = np.array([bound])
    np.savez(os.path.join(OUT, "ref_knnbuf.npz"), n=np.array([len(cases)]), **arrs)


def oracle_small():
    P = O.gen_uniform(3000, 3, 2)
    Q = O.gen_uniform(400, 3, 3)
    b = O.BDLTree(3)
    b.insert(P)
    ids, d2 = b.knn(Q, 10)
    nodes, tids, tpts = b.tree_export(1)
    t = O.Tree(np.array([(0, 0), (1, 0), (0, 1), (1, 1), (2, 0), (3, 0), (2, 1), (3, 1)], float), leaf=1)
    gn, _, _ = t.export()
    np.savez(os.path.join(OUT, "oracle_small.npz"), P=P, Q=Q, ids=ids, d2=d2, tree1_nodes=nodes.view(np.uint8),
             tree1_ids=tids, tree1_pts=tpts, golden8=gn.view(np.uint8))


if __name__ == "__main__":
    O.build(ref=True)
    ref_rng()
    ref_knnbuf()
    oracle_small()
    print("wrote", sorted(f for f in os.listdir(OUT) if f.endswith(".npz")))
