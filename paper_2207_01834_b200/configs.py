"""BASELINE.json's five configurations as seeded operation scripts.

Inputs are synthetic and generated on the host by the repo's own generators
(gk_gen.cpp, restating geokit/core/rng.hpp + generators.hpp with side 1); the
paper's VisualVar 2D-V-10M set is external and absent, so config 5 uses the
random-walk recipe BASELINE.json states.  `scale` < 1 shrinks every size for
parity tests (the recipes and seeds are unchanged).
"""
from __future__ import annotations

import numpy as np

from . import bdltree as B

CONFIGS = {
    1: dict(name="C1 2D-U-1M self-kNN k=5", d=2),
    2: dict(name="C2 3D-U-10M, 10M uniform queries, k=10", d=3),
    3: dict(name="C3 7D Gaussian mixture 2M self-kNN k=10", d=7),
    4: dict(name="C4 3D dynamic: 10 x (Insert_L 1M + kNN_L 1M, k=10)", d=3),
    5: dict(name="C5 2D random walks 10M, 3 x Erase_L 10%, kNN_L 5M k=1 and k=16", d=2),
}
C5_QUERY_SEED = 9  # not given by BASELINE.json; chosen and recorded here


def make_inputs(cfg: int, scale: float = 1.0, gen=None):
    """Returns (d, script) with script a list of ("insert", P) / ("erase", P) / ("knn", Q, k).

    `gen` may supply an alternative generator module with the same functions
    (the tests pass the oracle's to prove the two restatements agree)."""
    g = gen or B

    def n_(x):
        return max(1, int(round(x * scale)))

    if cfg == 1:
        P = g.gen_uniform(n_(1_000_000), 2, 1)
        return 2, [("insert", P), ("knn", P, 5)]
    if cfg == 2:
        P = g.gen_uniform(n_(10_000_000), 3, 2)
        Q = g.gen_uniform(n_(10_000_000), 3, 3)
        return 3, [("insert", P), ("knn", Q, 10)]
    if cfg == 3:
        P = g.gen_mixture(n_(2_000_000), 7, 4, 32, 0.02)
        return 7, [("insert", P), ("knn", P, 10)]
    if cfg == 4:
        script = []
        for b in range(10):
            script.append(("insert", g.gen_uniform(n_(1_000_000), 3, 10 + b)))
            script.append(("knn", g.gen_uniform(n_(1_000_000), 3, 20 + b), 10))
        return 3, script
    if cfg == 5:
        clusters = max(1, int(round(1000 * scale ** 0.5)))
        steps = max(1, int(round(10_000 * scale ** 0.5)))
        P = g.gen_walk(clusters, steps, 5)
        surv = np.arange(len(P), dtype=np.int64)  # survivors, ascending id
        script = [("insert", P)]
        for seed in (6, 7, 8):
            m = len(surv) // 10
            pick = g.sample_without_replacement(len(surv), m, seed).astype(np.int64)
            script.append(("erase", P[surv[pick]]))
            keep = np.ones(len(surv), bool)
            keep[pick] = False
            surv = surv[keep]
        nq = min(len(surv), n_(5_000_000))
        Q = P[surv[g.sample_without_replacement(len(surv), nq, C5_QUERY_SEED).astype(np.int64)]]
        script.append(("knn", Q, 1))
        script.append(("knn", Q, 16))
        return 2, script
    raise ValueError(f"unknown config {cfg}")
