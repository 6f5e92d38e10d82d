"""Python host mirror of the reference's BDL-tree batch interface over the C ABI.

The reference (arxiv 2207.01834, /root/reference) specifies the operations
bdl_build / bdl_insert / bdl_erase / bdl_knn over
PointSet<D> inputs (geokit/core/point.hpp:11-19) and reports errors as
std::invalid_argument / std::logic_error.  This module binds include/gk_bdl.h
with ctypes and keeps those names, argument meanings and error behaviour:
invalid arguments raise ValueError, logic errors RuntimeError, CUDA failures
GpuError.  There is no CPU fallback: if the CUDA library cannot be loaded every
call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# GK_LIB overrides the library path (A/B experiments between two builds of the same ABI)
LIB_PATH = os.environ.get("GK_LIB") or os.path.join(HERE, "_lib", "libgkbdl.so")

NO_POINT = 0xFFFFFFFF  # geokit::core::kNoPoint
MAX_K = 65536  # GK_MAX_K
SPATIAL_MEDIAN, OBJECT_MEDIAN = 0, 1

CANON_NODE = np.dtype([
    ("kind", "<i4"), ("dim", "<i4"), ("mode", "<i4"), ("depth", "<i4"),
    ("split", "<f8"), ("left", "<i4"), ("right", "<i4"),
    ("start", "<u4"), ("count", "<u4"),
    ("lo", "<f8", (8,)), ("hi", "<f8", (8,)),
])


class GpuError(RuntimeError):
    pass


class CapacityError(ValueError):
    """range search: more rows than the caller's capacity (GK_ERR_CAPACITY); offsets were written"""


class _Info(C.Structure):
    _fields_ = [("F", C.c_uint64), ("buffer", C.c_uint64), ("live", C.c_uint64), ("next_id", C.c_uint64),
                ("build_size", C.c_uint64 * 64), ("live_per_tree", C.c_uint64 * 64),
                ("nodes_per_tree", C.c_uint64 * 64), ("height_per_tree", C.c_int32 * 64),
                ("root_per_tree", C.c_int32 * 64)]


class KnnCounters(C.Structure):
    _fields_ = [("node_bytes", C.c_uint64), ("leaf_bytes", C.c_uint64), ("nodes", C.c_uint64),
                ("leaves", C.c_uint64), ("dists", C.c_uint64), ("warp_nodes", C.c_uint64),
                ("warp_leaves", C.c_uint64), ("inserts", C.c_uint64), ("warp_leaf_points", C.c_uint64),
                ("warp_inserts", C.c_uint64)]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


_P = C.c_void_p
_u64 = C.c_uint64
_lib = None


def _bind(L, name, argtypes):
    """argtypes of one C-ABI entry point; a missing symbol is an error unless GK_LIB points at another
    build (A/B experiments against older builds that predate an entry point)"""
    try:
        getattr(L, name).argtypes = argtypes
    except AttributeError:
        if not os.environ.get("GK_LIB"):
            raise


def lib():
    """Load libgkbdl.so (build it first if it is missing and nvcc is present)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from . import build as _b
            _b.build()
        L = C.CDLL(LIB_PATH)
        L.gk_last_error.restype = C.c_char_p
        L.gk_version.restype = C.c_char_p
        _bind(L, "gk_bdl_create", [C.c_int, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.POINTER(_P)])
        _bind(L, "gk_bdl_destroy", [_P])
        _bind(L, "gk_bdl_insert", [_P, _P, _u64])
        _bind(L, "gk_bdl_insert_device", [_P, _P, _u64])
        _bind(L, "gk_bdl_erase", [_P, _P, _u64, C.POINTER(_u64)])
        _bind(L, "gk_bdl_erase_device", [_P, _P, _u64, C.POINTER(_u64)])
        _bind(L, "gk_bdl_knn", [_P, _P, _u64, C.c_int, _P, _P])
        _bind(L, "gk_bdl_knn_device", [_P, _P, _u64, C.c_int, _P, _P])
        _bind(L, "gk_bdl_knn_bounded_device", [_P, _P, _u64, C.c_int, _P, _P, _P])
        _bind(L, "gk_bdl_knn_counted_device", [_P, _P, _u64, C.c_int, _P, _P, C.POINTER(KnnCounters)])
        _bind(L, "gk_bdl_range_count", [_P, _P, _u64, C.c_double, _P])
        _bind(L, "gk_bdl_range", [_P, _P, _u64, C.c_double, _P, _P, _P, _u64])
        _bind(L, "gk_bdl_range_device", [_P, _P, _u64, C.c_double, _P, _P, _P, _u64, C.POINTER(_u64)])
        _bind(L, "gk_bdl_range_radii_count", [_P, _P, _u64, _P, _P])
        _bind(L, "gk_bdl_range_radii", [_P, _P, _u64, _P, _P, _P, _P, _u64])
        _bind(L, "gk_bdl_range_radii_device", [_P, _P, _u64, _P, _P, _P, _P, _u64, C.POINTER(_u64)])
        _bind(L, "gk_bdl_range_box_count", [_P, _P, _P, _u64, _P])
        _bind(L, "gk_bdl_range_box", [_P, _P, _P, _u64, _P, _P, _u64])
        _bind(L, "gk_bdl_range_box_device", [_P, _P, _P, _u64, _P, _P, _u64, C.POINTER(_u64)])
        _bind(L, "gk_bdl_knn_graph", [_P, C.c_int, _P, _P, _P])
        _bind(L, "gk_bdl_knn_graph_device", [_P, C.c_int, _P, _P, _P])
        _bind(L, "gk_bdl_info_get", [_P, C.POINTER(_Info)])
        _bind(L, "gk_bdl_tree_export", [_P, C.c_int, _P, _P, _P, C.POINTER(_u64), C.POINTER(_u64)])
        _bind(L, "gk_bdl_bloom_query", [_P, C.c_int, _P, _u64, _P])
        L.gk_bdl_stream.restype = _P
        _bind(L, "gk_bdl_stream", [_P])
        _bind(L, "gk_bdl_sync", [_P])
        _bind(L, "gk_bdl_last_knn_ms", [_P, C.POINTER(C.c_float), C.POINTER(C.c_float)])
        _bind(L, "gk_bdl_last_build_ms", [_P, C.POINTER(C.c_float), C.POINTER(_u64)])
        _bind(L, "gk_diag_l2_read_gbs", [C.c_int, _u64, C.POINTER(C.c_double)])
        _bind(L, "gk_gen_uniform", [_u64, C.c_int, _u64, _P])
        _bind(L, "gk_gen_mixture", [_u64, C.c_int, _u64, C.c_int, C.c_double, _P])
        _bind(L, "gk_gen_walk", [_u64, _u64, _u64, _P])
        _bind(L, "gk_sample_without_replacement", [_u64, _u64, _u64, _P])
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().gk_last_error().decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise GpuError(msg)
    if rc == 3:
        raise NotImplementedError(msg)
    if rc == 5:
        raise CapacityError(msg)
    raise RuntimeError(msg)


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(_P)
    return _P(int(a.data_ptr()))  # torch CUDA tensor


def _rows(pts, d: int) -> np.ndarray:
    a = np.ascontiguousarray(pts, dtype=np.float64)
    if a.ndim == 1 and a.size % d == 0:
        a = a.reshape(-1, d)
    if a.ndim != 2 or a.shape[1] != d:
        raise ValueError(f"expected an (n, {d}) point array, got shape {a.shape}")
    return a


class BDLTree:
    """Batch-dynamic kd-tree (BDL-tree), device resident on one B200.

    BDLTree(dim, X=1024, leaf_size=16, heuristic=SPATIAL_MEDIAN, device=0)
      insert(P)        Insert_L  (bdl_insert; bdl_build on an empty tree)
      erase(P) -> int  Erase_L   (bdl_erase), returns #points tombstoned
      knn(S, k)        kNN_L     (bdl_knn) -> (ids uint32 (n,k), sqdist float64 (n,k))
      range(S, r2)     range search (ball; r2 scalar or one per query) -> (offsets uint64 (n+1,), ids, sqdist)
                       rows sorted by (d2, id)
      range_count(S, r2) -> counts uint64 (n,)
      range_box(lo, hi) orthogonal range search -> (offsets uint64 (n+1,), ids ascending)
      knn_graph(k)     k-NN graph -> (row ids (m,), ids (m,k), sqdist (m,k)), one row per live point
    Device variants take torch CUDA tensors and keep everything in HBM.
    """

    def __init__(self, dim: int, X: int = 1024, leaf_size: int = 16, heuristic: int = SPATIAL_MEDIAN,
                 device: int = 0):
        self.d = int(dim)
        self.X = int(X)
        self.leaf_size = int(leaf_size)
        self.device = int(device)
        h = _P()
        _check(lib().gk_bdl_create(self.d, self.X, self.leaf_size, int(heuristic), self.device, C.byref(h)))
        self._h = h

    def _dev(self, t, dtype: str, shape: tuple, name: str, optional: bool = False):
        """Checks a device-API tensor before its raw pointer crosses the C ABI: a CUDA tensor on this
        handle's device, contiguous, of `dtype`, with `shape` (None entries match any size).  A CPU
        tensor, a wrong dtype or a strided view would otherwise be read or written as raw memory."""
        if t is None:
            if optional:
                return None
            raise ValueError(f"{name}: a CUDA tensor is required")
        if not hasattr(t, "data_ptr") or not getattr(t, "is_cuda", False):
            raise ValueError(f"{name}: expected a CUDA torch tensor, got {type(t).__name__}"
                             f"{'' if not hasattr(t, 'device') else ' on ' + str(t.device)}")
        if t.device.index != self.device:
            raise ValueError(f"{name}: tensor is on {t.device}, the handle is on cuda:{self.device}")
        if not str(t.dtype).endswith(dtype):
            raise ValueError(f"{name}: expected dtype {dtype}, got {t.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name}: tensor must be contiguous")
        ts = tuple(int(x) for x in t.shape)
        if len(ts) != len(shape) or any(w is not None and w != g for w, g in zip(shape, ts)):
            want = "(" + ", ".join("n" if w is None else str(w) for w in shape) + ")"
            raise ValueError(f"{name}: expected shape {want}, got {ts}")
        return t

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().gk_bdl_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # --------------------------------------------------------------- host API
    def insert(self, pts) -> None:
        a = _rows(pts, self.d)
        _check(lib().gk_bdl_insert(self._h, _ptr(a), a.shape[0]))

    build = insert  # bdl_build(P) == bdl_insert(P) on an empty structure

    def erase(self, pts) -> int:
        a = _rows(pts, self.d)
        n = _u64(0)
        _check(lib().gk_bdl_erase(self._h, _ptr(a), a.shape[0], C.byref(n)))
        return int(n.value)

    def knn(self, queries, k: int):
        q = _rows(queries, self.d)
        ids = np.empty((q.shape[0], k), np.uint32)
        d2 = np.empty((q.shape[0], k), np.float64)
        _check(lib().gk_bdl_knn(self._h, _ptr(q), q.shape[0], int(k), _ptr(ids), _ptr(d2)))
        return ids, d2

    @staticmethod
    def _radii(r2, n):
        """None for one scalar squared radius, else the per-query radii as a contiguous float64 (n,) array"""
        if np.ndim(r2) == 0:
            return None
        r = np.ascontiguousarray(r2, dtype=np.float64)
        if r.shape != (n,):
            raise ValueError(f"per-query r2 must have shape ({n},), got {r.shape}")
        return r

    def range_count(self, queries, r2) -> np.ndarray:
        """r2: one squared radius, or one per query (gk_bdl_range_radii_count)"""
        q = _rows(queries, self.d)
        out = np.empty(q.shape[0], np.uint64)
        rq = self._radii(r2, q.shape[0])
        if rq is None:
            _check(lib().gk_bdl_range_count(self._h, _ptr(q), q.shape[0], float(r2), _ptr(out)))
        else:
            _check(lib().gk_bdl_range_radii_count(self._h, _ptr(q), q.shape[0], _ptr(rq), _ptr(out)))
        return out

    def range(self, queries, r2):
        """Ball range search: every live point with d2 <= r2 (one squared radius, or one per query),
        per query sorted by (d2, id)."""
        q = _rows(queries, self.d)
        offs = np.zeros(q.shape[0] + 1, np.uint64)
        cap = int(self.range_count(q, r2).sum()) if q.shape[0] else 0
        ids = np.empty(max(cap, 1), np.uint32)
        d2 = np.empty(max(cap, 1), np.float64)
        rq = self._radii(r2, q.shape[0])
        if rq is None:
            _check(lib().gk_bdl_range(self._h, _ptr(q), q.shape[0], float(r2), _ptr(offs), _ptr(ids), _ptr(d2), cap))
        else:
            _check(lib().gk_bdl_range_radii(self._h, _ptr(q), q.shape[0], _ptr(rq), _ptr(offs), _ptr(ids), _ptr(d2),
                                            cap))
        return offs, ids[:cap], d2[:cap]

    def range_box_count(self, lo, hi) -> np.ndarray:
        lo, hi = _rows(lo, self.d), _rows(hi, self.d)
        if lo.shape != hi.shape:
            raise ValueError("lo and hi must have the same shape")
        out = np.empty(lo.shape[0], np.uint64)
        _check(lib().gk_bdl_range_box_count(self._h, _ptr(lo), _ptr(hi), lo.shape[0], _ptr(out)))
        return out

    def range_box(self, lo, hi):
        """Orthogonal range search: ids of the live points in each closed box [lo, hi], ascending."""
        lo, hi = _rows(lo, self.d), _rows(hi, self.d)
        cap = int(self.range_box_count(lo, hi).sum()) if lo.shape[0] else 0
        offs = np.zeros(lo.shape[0] + 1, np.uint64)
        ids = np.empty(max(cap, 1), np.uint32)
        _check(lib().gk_bdl_range_box(self._h, _ptr(lo), _ptr(hi), lo.shape[0], _ptr(offs), _ptr(ids), cap))
        return offs, ids[:cap]

    def knn_graph(self, k: int):
        n = self.info()["live"]
        rows = np.empty(n, np.uint32)
        ids = np.empty((n, k), np.uint32)
        d2 = np.empty((n, k), np.float64)
        _check(lib().gk_bdl_knn_graph(self._h, int(k), _ptr(rows), _ptr(ids), _ptr(d2)))
        return rows, ids, d2

    # ------------------------------------------------------------- device API
    def insert_device(self, pts_dev) -> None:
        self._dev(pts_dev, "float64", (None, self.d), "pts_dev")
        _check(lib().gk_bdl_insert_device(self._h, _ptr(pts_dev), int(pts_dev.shape[0])))

    def erase_device(self, pts_dev) -> int:
        self._dev(pts_dev, "float64", (None, self.d), "pts_dev")
        n = _u64(0)
        _check(lib().gk_bdl_erase_device(self._h, _ptr(pts_dev), int(pts_dev.shape[0]), C.byref(n)))
        return int(n.value)

    def _knn_args(self, q_dev, k, ids_dev, d2_dev):
        self._dev(q_dev, "float64", (None, self.d), "q_dev")
        nq = int(q_dev.shape[0])
        self._dev(ids_dev, "int32", (nq, int(k)), "ids_dev")
        self._dev(d2_dev, "float64", (nq, int(k)), "d2_dev")

    def knn_device(self, q_dev, k: int, ids_dev, d2_dev) -> None:
        self._knn_args(q_dev, k, ids_dev, d2_dev)
        _check(lib().gk_bdl_knn_device(self._h, _ptr(q_dev), int(q_dev.shape[0]), int(k), _ptr(ids_dev),
                                       _ptr(d2_dev)))

    def knn_bounded_device(self, q_dev, k: int, r2_dev, ids_dev, d2_dev) -> None:
        """k nearest within squared radius r2_dev[i] (inclusive); unfilled slots are (NO_POINT, +inf)"""
        self._knn_args(q_dev, k, ids_dev, d2_dev)
        self._dev(r2_dev, "float64", (int(q_dev.shape[0]),), "r2_dev")
        _check(lib().gk_bdl_knn_bounded_device(self._h, _ptr(q_dev), int(q_dev.shape[0]), int(k), _ptr(r2_dev),
                                               _ptr(ids_dev), _ptr(d2_dev)))

    def knn_counted_device(self, q_dev, k: int, ids_dev, d2_dev) -> dict:
        self._knn_args(q_dev, k, ids_dev, d2_dev)
        c = KnnCounters()
        _check(lib().gk_bdl_knn_counted_device(self._h, _ptr(q_dev), int(q_dev.shape[0]), int(k), _ptr(ids_dev),
                                               _ptr(d2_dev), C.byref(c)))
        return c.as_dict()

    def range_device(self, q_dev, r2, offs_dev, ids_dev, d2_dev, capacity: int) -> int:
        """r2: one squared radius (float) or a device tensor of one per query"""
        self._dev(q_dev, "float64", (None, self.d), "q_dev")
        nq = int(q_dev.shape[0])
        self._dev(offs_dev, "int64", (nq + 1,), "offs_dev")
        self._dev(ids_dev, "int32", (None,), "ids_dev", optional=capacity == 0)
        self._dev(d2_dev, "float64", (None,), "d2_dev", optional=capacity == 0)
        if ids_dev is not None and (ids_dev.shape[0] < capacity or d2_dev is None or d2_dev.shape[0] < capacity):
            raise ValueError(f"ids_dev / d2_dev must hold capacity={capacity} rows")
        t = _u64(0)
        if np.ndim(r2) == 0 and not hasattr(r2, "data_ptr"):
            _check(lib().gk_bdl_range_device(self._h, _ptr(q_dev), int(q_dev.shape[0]), float(r2), _ptr(offs_dev),
                                             _ptr(ids_dev), _ptr(d2_dev), int(capacity), C.byref(t)))
        else:
            self._dev(r2, "float64", (nq,), "per-query r2")
            _check(lib().gk_bdl_range_radii_device(self._h, _ptr(q_dev), int(q_dev.shape[0]), _ptr(r2), _ptr(offs_dev),
                                                   _ptr(ids_dev), _ptr(d2_dev), int(capacity), C.byref(t)))
        return int(t.value)

    def range_box_device(self, lo_dev, hi_dev, offs_dev, ids_dev, capacity: int) -> int:
        self._dev(lo_dev, "float64", (None, self.d), "lo_dev")
        nq = int(lo_dev.shape[0])
        self._dev(hi_dev, "float64", (nq, self.d), "hi_dev")
        self._dev(offs_dev, "int64", (nq + 1,), "offs_dev")
        self._dev(ids_dev, "int32", (None,), "ids_dev", optional=capacity == 0)
        if ids_dev is not None and ids_dev.shape[0] < capacity:
            raise ValueError(f"ids_dev must hold capacity={capacity} rows")
        t = _u64(0)
        _check(lib().gk_bdl_range_box_device(self._h, _ptr(lo_dev), _ptr(hi_dev), int(lo_dev.shape[0]), _ptr(offs_dev),
                                             _ptr(ids_dev), int(capacity), C.byref(t)))
        return int(t.value)

    def knn_graph_device(self, k: int, rows_dev, ids_dev, d2_dev) -> None:
        n = self.info()["live"]
        self._dev(rows_dev, "int32", (n,), "rows_dev")
        self._dev(ids_dev, "int32", (n, int(k)), "ids_dev")
        self._dev(d2_dev, "float64", (n, int(k)), "d2_dev")
        _check(lib().gk_bdl_knn_graph_device(self._h, int(k), _ptr(rows_dev), _ptr(ids_dev), _ptr(d2_dev)))

    # ------------------------------------------------------------ inspection
    def info(self) -> dict:
        i = _Info()
        _check(lib().gk_bdl_info_get(self._h, C.byref(i)))
        return dict(F=int(i.F), buffer=int(i.buffer), live=int(i.live), next_id=int(i.next_id),
                    build_size=np.array(i.build_size[:], np.int64), live_per_tree=np.array(i.live_per_tree[:], np.int64),
                    nodes_per_tree=np.array(i.nodes_per_tree[:], np.int64),
                    height_per_tree=np.array(i.height_per_tree[:], np.int32),
                    root_per_tree=np.array(i.root_per_tree[:], np.int32))

    def tree_export(self, tree: int):
        """(canonical nodes in vEB order, ids, AoS points) of static tree `tree` or the buffer tree (-1)."""
        nn, npt = _u64(0), _u64(0)
        _check(lib().gk_bdl_tree_export(self._h, int(tree), None, None, None, C.byref(nn), C.byref(npt)))
        nodes = np.zeros(nn.value, CANON_NODE)
        ids = np.zeros(npt.value, np.uint32)
        pts = np.zeros((npt.value, self.d), np.float64)
        _check(lib().gk_bdl_tree_export(self._h, int(tree), _ptr(nodes), _ptr(ids), _ptr(pts), C.byref(nn),
                                        C.byref(npt)))
        return nodes, ids, pts

    def bloom_may_contain(self, tree: int, pts) -> np.ndarray:
        """bloom prefilter of static tree `tree`: False = definitely absent"""
        a = _rows(pts, self.d)
        out = np.zeros(a.shape[0], np.uint8)
        _check(lib().gk_bdl_bloom_query(self._h, int(tree), _ptr(a), a.shape[0], _ptr(out)))
        return out.astype(bool)

    def stream(self) -> int:
        return int(lib().gk_bdl_stream(self._h) or 0)

    def sync(self) -> None:
        _check(lib().gk_bdl_sync(self._h))

    def last_knn_ms(self):
        a, b = C.c_float(), C.c_float()
        _check(lib().gk_bdl_last_knn_ms(self._h, C.byref(a), C.byref(b)))
        return float(a.value), float(b.value)

    def last_build_ms(self):
        a, n = C.c_float(), _u64()
        _check(lib().gk_bdl_last_build_ms(self._h, C.byref(a), C.byref(n)))
        return float(a.value), int(n.value)


def l2_read_gbs(device: int = 0, nbytes: int = 32 << 20) -> float:
    """measured L2 read bandwidth (GB/s) over an L2-resident buffer (gk_diag_l2_read_gbs)"""
    v = C.c_double()
    _check(lib().gk_diag_l2_read_gbs(int(device), int(nbytes), C.byref(v)))
    return float(v.value)


# ---------------------------------------------------------------- inputs ---
def gen_uniform(n: int, d: int, seed: int) -> np.ndarray:
    out = np.empty((n, d), np.float64)
    _check(lib().gk_gen_uniform(n, d, seed, _ptr(out)))
    return out


def gen_mixture(n: int, d: int, seed: int, centres: int = 32, sigma: float = 0.02) -> np.ndarray:
    out = np.empty((n, d), np.float64)
    _check(lib().gk_gen_mixture(n, d, seed, centres, sigma, _ptr(out)))
    return out


def gen_walk(clusters: int, steps: int, seed: int) -> np.ndarray:
    out = np.empty((clusters * steps, 2), np.float64)
    _check(lib().gk_gen_walk(clusters, steps, seed, _ptr(out)))
    return out


def sample_without_replacement(n: int, m: int, seed: int) -> np.ndarray:
    out = np.empty(m, np.uint32)
    _check(lib().gk_sample_without_replacement(n, m, seed, _ptr(out)))
    return out
