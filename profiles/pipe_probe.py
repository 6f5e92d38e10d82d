"""e2e pipeline-depth sweep for the pinned host kNN_L path (C2) plus the PCIe transfer floor.
Run on a GPU box: python profiles/pipe_probe.py"""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2207_01834_b200 as gk
from paper_2207_01834_b200.configs import make_inputs
d, script = make_inputs(2)
P, Q, k = script[0][1], script[1][1], script[1][2]
g = gk.BDLTree(3); g.insert(P)
nq = len(Q)
Qh = torch.from_numpy(Q).pin_memory().numpy()
ids = torch.empty((nq, k), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
d2 = torch.empty((nq, k), dtype=torch.float64).pin_memory().numpy()
# transfer floor: H2D of queries and D2H of results, concurrently on 2 streams
dq = torch.empty((nq, 3), dtype=torch.float64, device="cuda"); di = torch.empty((nq, k), dtype=torch.int32, device="cuda"); dd = torch.empty((nq, k), dtype=torch.float64, device="cuda")
Qt = torch.from_numpy(Qh); It = torch.from_numpy(ids.view(np.int32)); Dt = torch.from_numpy(d2)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with torch.cuda.stream(s1): dq.copy_(Qt, non_blocking=True)
    with torch.cuda.stream(s2): It.copy_(di, non_blocking=True); Dt.copy_(dd, non_blocking=True)
    torch.cuda.synchronize(); tf = time.perf_counter() - t0
print("transfer floor ms", tf * 1000, "GB/s d2h", 1.2e9 / tf / 1e9)
for ch in [1, 2, 3, 4, 6, 8, 12, 16]:
    os.environ["GK_PIPE_CHUNKS"] = str(ch)
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        rc = gk.lib().gk_bdl_knn(g._h, Qh.ctypes.data, nq, k, ids.ctypes.data, d2.ctypes.data)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    print("chunks", ch, "ms", best * 1000, "Mq/s", nq / best / 1e6)
