"""The CLI harness: text point files, bdl-script ops and BenchRecord rows,
checked against the library API and the CLI's own --check linear scan."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2207_01834_b200", "_lib", "gk_bdl_cli")


def _write(path, pts, header=True):
    with open(path, "w") as f:
        if header:
            f.write(f"pargeo {pts.shape[1]}\n")
        for p in pts:
            f.write(" ".join(repr(float(x)) for x in p) + "\n")


def test_bdl_script_matches_api(gk, tmp_path):
    rng = np.random.default_rng(3)
    A = np.round(rng.random((6000, 3)), 6)
    B = np.round(rng.random((2500, 3)), 6)
    Q = np.round(rng.random((700, 3)), 6)
    _write(tmp_path / "a.txt", A)
    _write(tmp_path / "b.txt", B, header=False)
    _write(tmp_path / "e.txt", A[:2000])
    _write(tmp_path / "q.txt", Q)
    (tmp_path / "s.txt").write_text("insert a.txt\nknn q.txt 5\ninsert b.txt\nerase e.txt\n# comment\nknn q.txt 12\n")
    r = subprocess.run([EXE, "bdl-script", str(tmp_path / "s.txt"), "-o", str(tmp_path / "out.txt"), "--check",
                        "-X", "256"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rows = [l.split(",") for l in r.stdout.strip().splitlines()]
    assert rows[0] == ["algorithm", "dataset", "n", "d", "threads", "seconds", "summary"]
    assert [x[0] for x in rows[1:]] == ["bdl-insert", "bdl-knn", "bdl-insert", "bdl-erase", "bdl-knn"]
    assert rows[4][6] == "erased=2000"
    g = gk.BDLTree(3, X=256)
    g.insert(A)
    i1, _ = g.knn(Q, 5)
    g.insert(B)
    g.erase(A[:2000])
    i2, _ = g.knn(Q, 12)
    out = (tmp_path / "out.txt").read_text().strip().splitlines()
    got1 = np.array([[int(v) for v in l.split()] for l in out[:700]])
    got2 = np.array([[int(v) for v in l.split()] for l in out[700:]])
    assert np.array_equal(got1, i1.astype(np.int64)) and np.array_equal(got2, i2.astype(np.int64))


def test_knn_task_and_exit_codes(gk, tmp_path):
    rng = np.random.default_rng(4)
    P = rng.random((3000, 2))
    _write(tmp_path / "p.txt", P)
    r = subprocess.run([EXE, "knn", str(tmp_path / "p.txt"), str(tmp_path / "p.txt"), "-k", "3", "--check"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip().splitlines()[-1].startswith("bdl-knn,p.txt,3000,2,1,")
    assert subprocess.run([EXE, "knn", str(tmp_path / "missing.txt"), str(tmp_path / "p.txt"), "-k", "3"],
                          capture_output=True).returncode == 3
    (tmp_path / "bad.txt").write_text("pargeo 2\n1 2\n3 x\n")
    assert subprocess.run([EXE, "knn", str(tmp_path / "bad.txt"), str(tmp_path / "p.txt"), "-k", "3"],
                          capture_output=True).returncode == 3


def _fnv1a(ids):
    h = 1469598103934665603
    for x in np.asarray(ids, np.uint32).ravel().tolist():
        for b in range(4):
            h ^= (x >> (8 * b)) & 0xFF
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def test_bdl_script_replayed_on_the_oracle(gk, oracle, tmp_path):
    """the same bdl-script (inserts with duplicates, an erase of present + absent +
    duplicated points, a reinsertion-triggering erase, kNN with k above the live count) replayed through
    the CLI (GPU) and through the oracle BDL-tree: every result row identical, and every BenchRecord
    summary (live=, erased=, FNV-1a-64 of the result ids) equal to the one the oracle's results give"""
    rng = np.random.default_rng(11)
    A = np.round(rng.random((5000, 2)), 3)           # a 1000 x 1000 grid: many duplicates
    B = np.concatenate([A[:700], np.round(rng.random((1300, 2)), 3)])
    E1 = np.concatenate([A[100:1600], np.round(rng.random((200, 2)), 3) + 2.0, A[100:110]])  # absent + repeats
    E2 = np.concatenate([A[1600:4900], B[700:1900]])  # drops trees below half: survivors reinserted
    Q = np.concatenate([np.round(rng.random((400, 2)), 3), A[:100]])
    for name, arr in (("a", A), ("b", B), ("e1", E1), ("e2", E2), ("q", Q)):
        _write(tmp_path / f"{name}.txt", arr)
    script = ["insert a.txt", "knn q.txt 7", "insert b.txt", "erase e1.txt", "knn q.txt 16", "erase e2.txt",
              "knn q.txt 3", "insert a.txt", "knn q.txt 9000"]
    (tmp_path / "s.txt").write_text("\n".join(script) + "\n")
    r = subprocess.run([EXE, "bdl-script", str(tmp_path / "s.txt"), "-o", str(tmp_path / "out.txt"), "-X", "128"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rows = [l.split(",") for l in r.stdout.strip().splitlines()[1:]]
    out = (tmp_path / "out.txt").read_text().strip().splitlines()
    o = oracle.BDLTree(2, X=128)
    line = 0
    files = {"a.txt": A, "b.txt": B, "e1.txt": E1, "e2.txt": E2, "q.txt": Q}
    for op, rec in zip(script, rows):
        parts = op.split()
        pts = files[parts[1]]
        if parts[0] == "insert":
            o.insert(pts)
            assert rec[0] == "bdl-insert" and rec[6] == f"live={len(o.live()[0])}", (op, rec)
        elif parts[0] == "erase":
            assert rec[0] == "bdl-erase" and rec[6] == f"erased={o.erase(pts)}", (op, rec)
        else:
            k = int(parts[2])
            oi, _ = o.knn(pts, k)
            got = np.array([[int(v) for v in l.split()] for l in out[line:line + len(pts)]], np.int64)
            line += len(pts)
            want = np.where(oi == gk.NO_POINT, -1, oi.astype(np.int64))
            assert np.array_equal(got, want), op
            assert rec[0] == "bdl-knn" and rec[6] == _fnv1a(oi), (op, rec)
    assert line == len(out)
