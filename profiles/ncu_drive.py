"""Small driver for per-kernel ncu captures (profiles/capture_all.sh): one pass of each BASELINE
path, so `ncu -k regex:<kernel> -c 1` lands on a representative full-size launch.
  python profiles/ncu_drive.py c2   # C2: Insert_L of 10M 3D points, kNN_L of 10M queries, ball range of 2M
  python profiles/ncu_drive.py c5   # C5: Insert_L of 10M 2D random-walk points, 3 Erase_L, kNN_L k=1 / k=16
  python profiles/ncu_drive.py c3   # C3: Insert_L of 2M 7D points, kNN_L self-queries"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_01834_b200 as gk  # noqa: E402
from paper_2207_01834_b200.configs import make_inputs  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = {"c2": 2, "c5": 5, "c3": 3, "c1": 1}[what]
d, script = make_inputs(cfg, 1.0)
g = gk.BDLTree(d)
for op in script:
    x = torch.from_numpy(op[1]).cuda()
    if op[0] == "insert":
        g.insert_device(x)
    elif op[0] == "erase":
        g.erase_device(x)
    else:
        k = op[2]
        ids = torch.empty((x.shape[0], k), dtype=torch.int32, device="cuda")
        d2 = torch.empty((x.shape[0], k), dtype=torch.float64, device="cuda")
        g.knn_device(x, k, ids, d2)
        if what == "c2":
            nr = 2_000_000
            r2 = float(d2[:nr, k - 1].median().item())
            offs = torch.zeros(nr + 1, dtype=torch.int64, device="cuda")
            cap = g.range_device(x[:nr], r2, offs, None, None, 0)
            rid = torch.empty(cap, dtype=torch.int32, device="cuda")
            rd2 = torch.empty(cap, dtype=torch.float64, device="cuda")
            g.range_device(x[:nr], r2, offs, rid, rd2, cap)
torch.cuda.synchronize()
print("drive done", what)
