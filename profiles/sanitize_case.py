"""Small end-to-end case for compute-sanitizer runs (one tool per run):
   compute-sanitizer --tool memcheck  python profiles/sanitize_case.py
   compute-sanitizer --tool racecheck python profiles/sanitize_case.py
Exercises Insert_L (concurrent cooperative builds), kNN_L (K = 5/10/32, D = 2/3/7,
pair mode), Erase_L (bloom, collapse, half-capacity reinsertion) and the pinned path."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_01834_b200 as gk  # noqa: E402

rng = np.random.default_rng(0)
for d, k in ((3, 10), (2, 5), (7, 32)):
    g = gk.BDLTree(d, X=64)
    P = rng.random((5000, d))
    g.insert(P)
    g.insert(rng.random((777, d)))
    ids, d2 = g.knn(rng.random((3000, d)), k)
    assert (np.diff(d2, axis=1) >= 0).all()
    g.erase(P[:3000])
    g.knn(P[3000:3500], k)
    g.close()
print("sanitize case ok")
