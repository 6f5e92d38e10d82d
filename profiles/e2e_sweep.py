"""e2e experiment (C2): PCIe copy rates and gk_bdl_knn pipeline depth sweep.

Run on the GPU box:  python profiles/e2e_sweep.py
Prints one line per measurement; not part of the bench contract.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_01834_b200 as gk  # noqa: E402
from paper_2207_01834_b200 import configs  # noqa: E402


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    d, script = configs.make_inputs(int(os.environ.get("CONFIG", "2")), 1.0)
    P = [op[1] for op in script if op[0] == "insert"][0]
    Q, k = [op for op in script if op[0] == "knn"][0][1:]
    nq = len(Q)
    dev = torch.device("cuda", 0)
    out_bytes = nq * k * 12
    in_bytes = nq * d * 8
    h_out = torch.empty(out_bytes, dtype=torch.uint8).pin_memory()
    h_in = torch.empty(in_bytes, dtype=torch.uint8).pin_memory()
    d_out = torch.empty(out_bytes, dtype=torch.uint8, device=dev)
    d_in = torch.empty(in_bytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    t = timeit(lambda: h_out.copy_(d_out, non_blocking=True))
    print(f"D2H {out_bytes/1e9:.2f} GB: {t*1e3:.2f} ms = {out_bytes/t/1e9:.1f} GB/s")
    t = timeit(lambda: d_in.copy_(h_in, non_blocking=True))
    print(f"H2D {in_bytes/1e9:.2f} GB: {t*1e3:.2f} ms = {in_bytes/t/1e9:.1f} GB/s")

    def both():
        with torch.cuda.stream(s1):
            h_out.copy_(d_out, non_blocking=True)
        with torch.cuda.stream(s2):
            d_in.copy_(h_in, non_blocking=True)
    t = timeit(both)
    print(f"D2H+H2D concurrent: {t*1e3:.2f} ms")
    del h_out, h_in, d_out, d_in

    g = gk.BDLTree(d, device=0)
    g.insert(P)
    Qh = torch.from_numpy(Q).pin_memory().numpy()
    ids_h = torch.empty((nq, k), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
    d2_h = torch.empty((nq, k), dtype=torch.float64).pin_memory().numpy()
    Q_dev = torch.from_numpy(Q).to(dev)
    ids_dev = torch.empty((nq, k), dtype=torch.int32, device=dev)
    d2_dev = torch.empty((nq, k), dtype=torch.float64, device=dev)
    t = timeit(lambda: g.knn_device(Q_dev, k, ids_dev, d2_dev))
    print(f"device kNN: {t*1e3:.2f} ms")
    for frac in (2, 4, 8, 16):
        m = nq // frac
        t = timeit(lambda: g.knn_device(Q_dev[:m], k, ids_dev[:m], d2_dev[:m]))
        print(f"device kNN of the first nq/{frac}: {t*1e3:.2f} ms  (x{frac} = {t*frac*1e3:.2f} ms)")
    ref_ids = None
    for spec in os.environ.get("SWEEP", "1 2 3 4 6 8").split():
        nc, _, r = spec.partition(":")
        if nc == "f":  # explicit chunk weights, e.g. f:1,8,7,4,4
            os.environ["GK_PIPE_FRACS"] = r
        else:
            os.environ.pop("GK_PIPE_FRACS", None)
            os.environ["GK_PIPE_CHUNKS"] = nc
            os.environ["GK_PIPE_RATIO"] = r or "1"
        t = timeit(lambda: gk.lib().gk_bdl_knn(g._h, Qh.ctypes.data, nq, k, ids_h.ctypes.data, d2_h.ctypes.data))
        if ref_ids is None:
            ref_ids = ids_h.copy()
        ok = np.array_equal(ref_ids, ids_h)
        print(f"e2e chunks={spec}: {t*1e3:.2f} ms = {nq/t/1e6:.1f} M q/s same={ok}")


if __name__ == "__main__":
    main()
