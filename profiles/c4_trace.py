"""C4 Insert_L trace: per-batch Insert_L wall time and (GK_TRACE=1) host phase stamps; diagnostics only.
  python profiles/c4_trace.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_01834_b200 as gk  # noqa: E402
from paper_2207_01834_b200 import configs  # noqa: E402

d, script = configs.make_inputs(4, 1.0)
ins = [torch.from_numpy(op[1]).cuda() for op in script if op[0] == "insert"]
qs = [torch.from_numpy(op[1]).cuda() for op in script if op[0] == "knn"]
with_knn = os.environ.get("KNN") == "1"  # interleave the config's kNN_L batches (as bench.py replays it)
reps = int(os.environ.get("REPS", "2"))
for rep in range(reps):
    g = gk.BDLTree(d)
    tot = 0.0
    for b, P in enumerate(ins):
        F0 = g.info()["F"]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g.insert_device(P)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tot += dt
        if with_knn:
            ids = torch.empty((qs[b].shape[0], 10), dtype=torch.int32, device="cuda")
            d2 = torch.empty((qs[b].shape[0], 10), dtype=torch.float64, device="cuda")
            g.knn_device(qs[b], 10, ids, d2)
        F1 = g.info()["F"]
        built = [i for i in range(64) if (F1 >> i & 1) and not (F0 >> i & 1)]
        if rep or os.environ.get("ALL"):
            print(f"batch {b}: {1e3 * dt:.3f} ms, build {g.last_build_ms()}, new trees {built}", file=sys.stderr, flush=True)
    print(f"rep {rep}: all inserts {1e3 * tot:.2f} ms", file=sys.stderr, flush=True)
    g.close()
