"""N > 1 host logic on CPU: world_size-2 gloo process group (the GPU bench runs
the same functions over NCCL, one replica per GPU)."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2207_01834_b200.replicas import max_over_ranks, shard_range, whole_job_rate
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    t = max_over_ranks(1.5 + rank)  # per-rank elapsed seconds
    lo, hi = shard_range(10, rank, world)
    q.put((rank, t, lo, hi, whole_job_rate(100, world, t)))
    dist.destroy_process_group()


def test_gloo_world2_max_over_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert [r[1] for r in res] == [2.5, 2.5]          # both ranks agree on the slowest time
    assert [(r[2], r[3]) for r in res] == [(0, 5), (5, 10)]
    assert res[0][4] == pytest.approx(200 / 2.5)      # whole-job units / max time


def test_shard_range_covers():
    from paper_2207_01834_b200.replicas import shard_range
    for n in (0, 1, 7, 1000):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))


def test_reference_arm_under_torchrun_world2():
    """bench.py --impl reference launched like the driver (torchrun, N=2): rank 0 prints one line, rank 1 exits 0"""
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "1", "--scale", "0.002",
                        "--cpu-seconds", "0.5"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["value"] > 0 and j["n_gpus"] == 2 and j["e2e"]["h2d_bytes_per_step"] == 0
