import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2207_01834_b200 as gk
for n in (640, 1000, 2000):
    P = torch.from_numpy(gk.gen_uniform(n, 2, 1)).cuda()
    g = gk.BDLTree(2, X=4096)
    ts = []
    for rep in range(30):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        g.insert_device(P[: n // 30 + 1])
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(n, "buffer rebuild insert: median ms", sorted(ts)[len(ts)//2] * 1e3, "buf", g.info().get("buffer"))
    g.close()
