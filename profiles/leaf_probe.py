"""kNN_L throughput against the structure's leaf size (C1/C2/C3 inputs): how much the traversal would gain
from fatter traversal leaves.  python profiles/leaf_probe.py <cfg> [leaf sizes...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_01834_b200 as gk  # noqa: E402
from paper_2207_01834_b200.configs import make_inputs  # noqa: E402

cfg = int(sys.argv[1])
leaves = [int(x) for x in sys.argv[2:]] or [8, 12, 16, 24, 32]
d, script = make_inputs(cfg, 1.0)
P = torch.from_numpy(script[0][1]).cuda()
qop = [op for op in script if op[0] == "knn"][0]
Q = torch.from_numpy(qop[1]).cuda()
k = qop[2]
ids = torch.empty((Q.shape[0], k), dtype=torch.int32, device="cuda")
d2 = torch.empty((Q.shape[0], k), dtype=torch.float64, device="cuda")
for leaf in leaves:
    g = gk.BDLTree(d, leaf_size=leaf)
    g.insert_device(P)
    best = 1e9
    for _ in range(4):
        g.knn_device(Q, k, ids, d2)
        best = min(best, g.last_knn_ms()[1])
    c = g.knn_counted_device(Q, k, ids, d2)
    print(f"cfg {cfg} leaf {leaf}: kNN_L {best:.3f} ms  {Q.shape[0] / best / 1e3:.1f} M q/s  warp_nodes {c.get('warp_nodes')} warp_leaves {c.get('warp_leaves')} "
          f"warp_leaf_points {c.get('warp_leaf_points')} inserts {c.get('inserts')} warp_inserts {c.get('warp_inserts')}", flush=True)
    g.close()
