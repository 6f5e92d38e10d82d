"""Randomised model scripts against the oracle, beyond the fixed seeds of tests/: random dimension, leaf size,
X, heuristic and data shapes (uniform, clustered, duplicate-heavy, +-0), sizes that reach multi-block builds
and the bottom phase; structure + every tree compared after every operation.  Diagnostics (GPU box):
  python profiles/stress_model.py [seconds] [seed] [big]     # big: batches of up to 1.5M points"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2207_01834_b200 as gk  # noqa: E402
from oracle import oracle  # noqa: E402
from tests.test_gpu_parity import run_script  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 12345
big = len(sys.argv) > 3
rng = np.random.default_rng(seed)
oracle.build()


def points(n, d, kind):
    if kind == 0:
        return rng.random((n, d))
    if kind == 1:  # clustered
        c = rng.random((max(1, n // 500 + 1), d))
        return np.clip(c[rng.integers(0, len(c), n)] + 0.01 * rng.standard_normal((n, d)), 0, 1)
    if kind == 2:  # small universe: duplicates, ties, degenerate splits
        return np.round(rng.random((n, d)) * 5) / 5
    p = rng.random((n, d)) - 0.5  # +-0 and a constant coordinate
    p[rng.random(n) < 0.2] *= 0.0
    p[:, d - 1] = -0.0
    return p


t0, runs = time.time(), 0
while time.time() - t0 < budget:
    d = int(rng.integers(2, 9))
    leaf = int(rng.choice([1, 2, 4, 8, 16, 16, 16, 32]))
    X = int(rng.choice([4, 16, 64, 256, 1024]))
    heur = int(rng.random() < 0.25)
    scale = int(rng.choice([200000, 600000, 1500000])) if big else int(rng.choice([X, 8 * X, 40 * X, 30000]))
    kind = int(rng.integers(0, 4))
    script, pool = [], []
    for _ in range(int(rng.integers(3, 6 if big else 9))):
        r = rng.random()
        if r < 0.5 or not pool:
            P = points(int(rng.integers(1, max(2, scale if big else min(scale, 60000)))), d, kind)
            pool.append(P)
            script.append(("insert", P))
        elif r < 0.8:
            src = pool[int(rng.integers(0, len(pool)))]
            m = int(rng.integers(0, len(src) + 1))
            E = src[rng.permutation(len(src))[:m]]
            if rng.random() < 0.3:
                E = np.vstack([E, points(int(rng.integers(1, 50)), d, kind)])  # absent points too
            script.append(("erase", E))
        else:
            script.append(("knn", points(int(rng.integers(1, 400)), d, kind), int(rng.integers(1, 40))))
    try:
        run_script(gk, oracle, d, script, X=X, leaf=leaf, heur=heur)
    except Exception:
        print(f"FAILED: seed {seed} run {runs}: d={d} leaf={leaf} X={X} heur={heur} kind={kind} "
              f"ops={[(o[0], len(o[1])) for o in script]}", flush=True)
        raise
    runs += 1
print(f"stress ok: {runs} random scripts in {time.time() - t0:.0f} s (seed {seed})")
