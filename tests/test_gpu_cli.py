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
