"""Insert_L phase trace (GK_TRACE=1 host timestamps) for a BASELINE config; diagnostics only.
  python profiles/insert_trace.py [config]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["GK_TRACE"] = "1"
import paper_2207_01834_b200 as gk  # noqa: E402
from paper_2207_01834_b200 import configs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
d, script = configs.make_inputs(cfg, 1.0)
P = [op[1] for op in script if op[0] == "insert"][0]
P_dev = torch.from_numpy(P).cuda()
for rep in range(3):
    g = gk.BDLTree(d)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.insert_device(P_dev)
    print(f"rep {rep}: insert wall {1e3 * (time.perf_counter() - t0):.3f} ms, build {g.last_build_ms()}", file=sys.stderr,
          flush=True)
    g.close()
