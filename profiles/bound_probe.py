"""Upper bound of what a per-query initial radius can buy K1: kNN_L seeded with
r2 = s2 * (true k-th d2) (an oracle seed, taken from a first exact run), K1 device
time vs the unseeded kernel; rows must equal the exact ones for s2 >= 1.
  python profiles/bound_probe.py [config]"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2207_01834_b200 as gk
from paper_2207_01834_b200.configs import make_inputs

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
d, script = make_inputs(cfg, 1.0)
P = [op[1] for op in script if op[0] == "insert"][0]
Q, k = [(op[1], op[2]) for op in script if op[0] == "knn"][0]
g = gk.BDLTree(d)
g.insert(P)
qd = torch.from_numpy(Q).cuda()
ids = torch.empty((len(Q), k), dtype=torch.int32, device="cuda")
d2 = torch.empty((len(Q), k), dtype=torch.float64, device="cuda")
base = []
for _ in range(5):
    g.knn_device(qd, k, ids, d2)
    base.append(g.last_knn_ms()[0])
ids0, d20 = ids.clone(), d2.clone()
kth = d20[:, k - 1].contiguous()
print(f"cfg {cfg}: unseeded K1 {min(base):.3f} ms")
for s2 in (1.0, 1.1, 1.25, 1.5, 2.0, 4.0):
    r2 = (kth * s2).contiguous()
    t = []
    for _ in range(5):
        g.knn_bounded_device(qd, k, r2, ids, d2)
        t.append(g.last_knn_ms()[0])
    same = bool(torch.equal(ids, ids0) and torch.equal(d2, d20))
    print(f"  s2={s2:4.2f}  K1 {min(t):.3f} ms  ({min(base)/min(t):.2f}x)  rows exact: {same}")
