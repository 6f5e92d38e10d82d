"""Build timeline of ONE static tree (n = X * 2^i points, so Insert_L builds exactly one tree): run with a
-DGK_BUILD_TIMELINE=1 build (profiles/mkvariant.sh tl "-DGK_BUILD_TIMELINE=1"; GK_LIB=ab/tl/libgkbdl.so).
  python profiles/one_tree_trace.py <dim> <log2 n>"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_01834_b200 as gk  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 19)
P = torch.from_numpy(gk.gen_uniform(n, d, 1)).cuda()
for rep in range(3):
    g = gk.BDLTree(d)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.insert_device(P)
    torch.cuda.synchronize()
    print(f"rep {rep}: insert wall {1e3 * (time.perf_counter() - t0):.3f} ms, build {g.last_build_ms()}", file=sys.stderr, flush=True)
    g.close()
