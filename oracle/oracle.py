"""ctypes front-end of the CPU oracle (oracle/gk_oracle.cpp) and of the
reference pins (oracle/_ref/libgkref.so, compiled from /root/reference's own
headers).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package never
imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libgk_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libgkref.so")
REF_INCLUDE = "/root/reference/proj/include"

# mirror of gko::Node / gk_canon_node (168 bytes)
CANON_NODE = np.dtype([
    ("kind", "<i4"), ("dim", "<i4"), ("mode", "<i4"), ("depth", "<i4"),
    ("split", "<f8"), ("left", "<i4"), ("right", "<i4"),
    ("start", "<u4"), ("count", "<u4"),
    ("lo", "<f8", (8,)), ("hi", "<f8", (8,)),
])
assert CANON_NODE.itemsize == 168

_P = C.c_void_p
_u64 = C.c_uint64


def build(ref: bool | None = None) -> None:
    """Compile the oracle (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_INCLUDE)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_P)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build(ref=False)
        L = C.CDLL(LIB_PATH)
        L.gko_hyperceiling.restype = _u64
        L.gko_hyperceiling.argtypes = [_u64]
        L.gko_mix64.restype = _u64
        L.gko_mix64.argtypes = [_u64]
        L.gko_max_threads.restype = C.c_int
        L.gko_node_size.restype = C.c_int
        L.gko_rng_u64.argtypes = [_u64, _u64, C.c_int, _u64, _P]
        L.gko_rng_below.argtypes = [_u64, _u64, _u64, _P]
        L.gko_random_permutation.argtypes = [_u64, _u64, _P]
        L.gko_gen_uniform.argtypes = [_u64, C.c_int, _u64, _P]
        L.gko_gen_mixture.argtypes = [_u64, C.c_int, _u64, C.c_int, C.c_double, _P]
        L.gko_gen_walk.argtypes = [_u64, _u64, _u64, _P]
        L.gko_sample_without_replacement.argtypes = [_u64, _u64, _u64, _P]
        L.gko_knnbuf_run.restype = C.c_int
        L.gko_knnbuf_run.argtypes = [C.c_int, _P, _P, _u64, _P, _P, _P, _P]
        L.gko_tree_build.restype = _P
        L.gko_tree_build.argtypes = [C.c_int, _P, _P, _u64, C.c_int, C.c_int]
        L.gko_tree_free.argtypes = [_P]
        L.gko_tree_info.argtypes = [_P, _P, _P, _P, _P]
        L.gko_tree_export.argtypes = [_P, _P, _P, _P]
        L.gko_tree_dead.argtypes = [_P, _P]
        L.gko_tree_erase.restype = _u64
        L.gko_tree_erase.argtypes = [_P, _P, _u64]
        L.gko_tree_knn.argtypes = [_P, _P, _u64, C.c_int, _P, _P]
        L.gko_bdl_create.restype = _P
        L.gko_bdl_create.argtypes = [C.c_int, _u64, C.c_int, C.c_int]
        L.gko_bdl_free.argtypes = [_P]
        L.gko_bdl_insert.argtypes = [_P, _P, _u64]
        L.gko_bdl_erase.restype = _u64
        L.gko_bdl_erase.argtypes = [_P, _P, _u64]
        L.gko_bdl_knn.argtypes = [_P, _P, _u64, C.c_int, _P, _P, _P]
        L.gko_bdl_stats.argtypes = [_P, _P, _P, _P, _P]
        L.gko_bdl_tree.restype = _P
        L.gko_bdl_tree.argtypes = [_P, C.c_int]
        L.gko_bdl_live.restype = _u64
        L.gko_bdl_live.argtypes = [_P, _P, _P]
        L.gko_bdl_range.restype = _u64
        L.gko_bdl_range.argtypes = [_P, _P, _u64, C.c_double, _P, _P, _P]
        L.gko_bdl_range_box.restype = _u64
        L.gko_bdl_range_box.argtypes = [_P, _P, _P, _u64, _P, _P]
        L.gko_bdl_knn_graph.restype = _u64
        L.gko_bdl_knn_graph.argtypes = [_P, C.c_int, _P, _P, _P]
        L.gko_brute_knn.argtypes = [C.c_int, _P, _P, _u64, _P, _u64, C.c_int, _P, _P]
        L.gko_set_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def ref_lib():
    """The reference's own Rng/KnnBuffer (None when oracle/_ref was not built)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            return None
        R = C.CDLL(REF_PATH)
        R.gkref_mix64.restype = _u64
        R.gkref_mix64.argtypes = [_u64]
        R.gkref_rng_u64.argtypes = [_u64, _u64, C.c_int, _u64, _P]
        R.gkref_rng_double.argtypes = [_u64, _u64, C.c_int, _u64, _P]
        R.gkref_rng_below.argtypes = [_u64, _u64, _u64, _P]
        R.gkref_random_permutation.argtypes = [_u64, _u64, _P]
        R.gkref_knnbuf_run.restype = C.c_int
        R.gkref_knnbuf_run.argtypes = [C.c_int, _P, _P, _u64, _P, _P, _P, _P]
        _ref = R
    return _ref


def set_threads(t: int) -> None:
    lib().gko_set_threads(int(t))


def max_threads() -> int:
    return int(lib().gko_max_threads())


# ------------------------------------------------------------------ inputs --
def gen_uniform(n: int, d: int, seed: int) -> np.ndarray:
    out = np.empty((n, d), np.float64)
    lib().gko_gen_uniform(n, d, seed, _ptr(out))
    return out


def gen_mixture(n: int, d: int, seed: int, nc: int = 32, sigma: float = 0.02) -> np.ndarray:
    out = np.empty((n, d), np.float64)
    lib().gko_gen_mixture(n, d, seed, nc, sigma, _ptr(out))
    return out


def gen_walk(clusters: int, steps: int, seed: int) -> np.ndarray:
    out = np.empty((clusters * steps, 2), np.float64)
    lib().gko_gen_walk(clusters, steps, seed, _ptr(out))
    return out


def sample_without_replacement(n: int, m: int, seed: int) -> np.ndarray:
    out = np.empty(m, np.uint32)
    lib().gko_sample_without_replacement(n, m, seed, _ptr(out))
    return out


def random_permutation(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.uint32)
    lib().gko_random_permutation(n, seed, _ptr(out))
    return out


def rng_u64(seed: int, n: int, stream: int | None = None) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().gko_rng_u64(seed, 0 if stream is None else stream, 0 if stream is None else 1, n, _ptr(out))
    return out


def hyperceiling(x: int) -> int:
    return int(lib().gko_hyperceiling(x))


def knnbuf_run(k: int, d2: np.ndarray, ids: np.ndarray, use_ref: bool = False):
    d2 = np.ascontiguousarray(d2, np.float64)
    ids = np.ascontiguousarray(ids, np.uint32)
    od = np.empty(max(k, 1) * 2 + len(d2), np.float64)
    oi = np.empty_like(od, dtype=np.uint32)
    comp = np.zeros(1, np.uint64)
    bound = np.zeros(1, np.float64)
    L = ref_lib() if use_ref else lib()
    fn = L.gkref_knnbuf_run if use_ref else L.gko_knnbuf_run
    m = fn(k, _ptr(d2), _ptr(ids), len(d2), _ptr(od), _ptr(oi), _ptr(comp), _ptr(bound))
    return od[:m].copy(), oi[:m].copy(), int(comp[0]), float(bound[0])


# -------------------------------------------------------------- one tree ---
class Tree:
    """BuildvEB_S over (pts, ids) in the given order (oracle)."""

    def __init__(self, pts: np.ndarray, ids: np.ndarray | None = None, leaf: int = 16, heuristic: int = 0):
        pts = np.ascontiguousarray(pts, np.float64)
        n, d = pts.shape
        if ids is None:
            ids = np.arange(n, dtype=np.uint32)
        ids = np.ascontiguousarray(ids, np.uint32)
        self.d = d
        self.h = lib().gko_tree_build(d, _ptr(pts), _ptr(ids), n, leaf, heuristic)
        self.n = n

    def __del__(self):
        if getattr(self, "h", None):
            lib().gko_tree_free(self.h)
            self.h = None

    def info(self):
        nn = np.zeros(1, np.uint64); h = np.zeros(1, np.int32); r = np.zeros(1, np.int32); lv = np.zeros(1, np.uint64)
        lib().gko_tree_info(self.h, _ptr(nn), _ptr(h), _ptr(r), _ptr(lv))
        return dict(n_nodes=int(nn[0]), height=int(h[0]), root=int(r[0]), live=int(lv[0]))

    def export(self):
        info = self.info()
        nodes = np.zeros(info["n_nodes"], CANON_NODE)
        ids = np.zeros(self.n, np.uint32)
        pts = np.zeros((self.n, self.d), np.float64)
        lib().gko_tree_export(self.h, _ptr(nodes), _ptr(ids), _ptr(pts))
        return nodes, ids, pts

    def erase(self, pts: np.ndarray) -> int:
        pts = np.ascontiguousarray(pts, np.float64)
        return int(lib().gko_tree_erase(self.h, _ptr(pts), len(pts)))

    def knn(self, q: np.ndarray, k: int):
        q = np.ascontiguousarray(q, np.float64)
        ids = np.empty((len(q), k), np.uint32); d2 = np.empty((len(q), k), np.float64)
        lib().gko_tree_knn(self.h, _ptr(q), len(q), k, _ptr(ids), _ptr(d2))
        return ids, d2


# ------------------------------------------------------------------- BDL ---
class BDLTree:
    """Oracle BDL-tree: Insert_L / Erase_L / kNN_L (PAPER Alg. 3-4)."""

    def __init__(self, d: int, X: int = 1024, leaf: int = 16, heuristic: int = 0):
        self.d = d
        self.X = X
        self.h = lib().gko_bdl_create(d, X, leaf, heuristic)

    def __del__(self):
        if getattr(self, "h", None):
            lib().gko_bdl_free(self.h)
            self.h = None

    def insert(self, pts: np.ndarray) -> None:
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, self.d)
        lib().gko_bdl_insert(self.h, _ptr(pts), len(pts))

    def erase(self, pts: np.ndarray) -> int:
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, self.d)
        return int(lib().gko_bdl_erase(self.h, _ptr(pts), len(pts)))

    def knn(self, q: np.ndarray, k: int, stats: bool = False):
        q = np.ascontiguousarray(q, np.float64).reshape(-1, self.d)
        ids = np.empty((len(q), k), np.uint32); d2 = np.empty((len(q), k), np.float64)
        st = np.zeros(3, np.uint64) if stats else None
        lib().gko_bdl_knn(self.h, _ptr(q), len(q), k, _ptr(ids), _ptr(d2), _ptr(st))
        if stats:
            return ids, d2, dict(nodes=int(st[0]), leaves=int(st[1]), dists=int(st[2]))
        return ids, d2

    def stats(self):
        F = np.zeros(1, np.uint64); b = np.zeros(1, np.uint64)
        bs = np.zeros(64, np.uint64); lv = np.zeros(64, np.uint64)
        lib().gko_bdl_stats(self.h, _ptr(F), _ptr(b), _ptr(bs), _ptr(lv))
        return dict(F=int(F[0]), buffer=int(b[0]), build_size=bs.astype(np.int64), live=lv.astype(np.int64))

    def tree_export(self, i: int):
        """(nodes, ids, pts) of static tree i, or of the buffer tree for i = -1."""
        h = lib().gko_bdl_tree(self.h, i)
        nn = np.zeros(1, np.uint64); ht = np.zeros(1, np.int32); r = np.zeros(1, np.int32); lv = np.zeros(1, np.uint64)
        lib().gko_tree_info(h, _ptr(nn), _ptr(ht), _ptr(r), _ptr(lv))
        st = self.stats()
        n = int(st["build_size"][i]) if i >= 0 else int(st["buffer"])
        nodes = np.zeros(int(nn[0]), CANON_NODE)
        ids = np.zeros(n, np.uint32)
        pts = np.zeros((n, self.d), np.float64)
        lib().gko_tree_export(h, _ptr(nodes), _ptr(ids), _ptr(pts))
        return nodes, ids, pts

    def tree_root(self, i: int) -> int:
        h = lib().gko_bdl_tree(self.h, i)
        nn = np.zeros(1, np.uint64); ht = np.zeros(1, np.int32); r = np.zeros(1, np.int32); lv = np.zeros(1, np.uint64)
        lib().gko_tree_info(h, _ptr(nn), _ptr(ht), _ptr(r), _ptr(lv))
        return int(r[0])

    def tree_dead(self, i: int) -> np.ndarray:
        """tombstone flags of static tree i (leaf order)"""
        h = lib().gko_bdl_tree(self.h, i)
        n = int(self.stats()["build_size"][i]) if i >= 0 else int(self.stats()["buffer"])
        out = np.zeros(n, np.uint8)
        lib().gko_tree_dead(h, _ptr(out))
        return out.astype(bool)

    def range(self, q: np.ndarray, r2: float):
        """ball range search: (offsets (n+1,), ids, d2), rows sorted by (d2, id)"""
        q = np.ascontiguousarray(q, np.float64).reshape(-1, self.d)
        cnt = np.zeros(len(q), np.uint64)
        tot = int(lib().gko_bdl_range(self.h, _ptr(q), len(q), float(r2), _ptr(cnt), None, None))
        ids = np.zeros(max(tot, 1), np.uint32); d2 = np.zeros(max(tot, 1), np.float64)
        lib().gko_bdl_range(self.h, _ptr(q), len(q), float(r2), _ptr(cnt), _ptr(ids), _ptr(d2))
        offs = np.zeros(len(q) + 1, np.uint64)
        offs[1:] = np.cumsum(cnt)
        return offs, ids[:tot], d2[:tot]

    def range_box(self, lo: np.ndarray, hi: np.ndarray):
        """orthogonal range search: (offsets (n+1,), ids ascending per query)"""
        lo = np.ascontiguousarray(lo, np.float64).reshape(-1, self.d)
        hi = np.ascontiguousarray(hi, np.float64).reshape(-1, self.d)
        cnt = np.zeros(len(lo), np.uint64)
        tot = int(lib().gko_bdl_range_box(self.h, _ptr(lo), _ptr(hi), len(lo), _ptr(cnt), None))
        ids = np.zeros(max(tot, 1), np.uint32)
        lib().gko_bdl_range_box(self.h, _ptr(lo), _ptr(hi), len(lo), _ptr(cnt), _ptr(ids))
        offs = np.zeros(len(lo) + 1, np.uint64)
        offs[1:] = np.cumsum(cnt)
        return offs, ids[:tot]

    def knn_graph(self, k: int):
        n = int(lib().gko_bdl_live(self.h, None, None))
        rows = np.zeros(n, np.uint32); ids = np.zeros((n, k), np.uint32); d2 = np.zeros((n, k), np.float64)
        lib().gko_bdl_knn_graph(self.h, k, _ptr(rows), _ptr(ids), _ptr(d2))
        return rows, ids, d2

    def live(self):
        n = int(lib().gko_bdl_live(self.h, None, None))
        ids = np.zeros(n, np.uint32); pts = np.zeros((n, self.d), np.float64)
        lib().gko_bdl_live(self.h, _ptr(ids), _ptr(pts))
        return ids, pts


def brute_knn(P: np.ndarray, Q: np.ndarray, k: int, ids: np.ndarray | None = None):
    P = np.ascontiguousarray(P, np.float64); Q = np.ascontiguousarray(Q, np.float64)
    n, d = P.shape
    if ids is None:
        ids = np.arange(n, dtype=np.uint32)
    ids = np.ascontiguousarray(ids, np.uint32)
    oi = np.empty((len(Q), k), np.uint32); od = np.empty((len(Q), k), np.float64)
    lib().gko_brute_knn(d, _ptr(P), _ptr(ids), n, _ptr(Q), len(Q), k, _ptr(oi), _ptr(od))
    return oi, od
