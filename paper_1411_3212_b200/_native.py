"""ctypes binding of the native library `libtickjoin_b200.so` (include/tickjoin_b200.h).

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a).
There is no fallback: if the library or a CUDA device is missing, creating a
context raises `DeviceError` loudly.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint8, c_uint32, c_void_p
from typing import Optional

import numpy as np

from . import errors

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
LIB_PATH = os.environ.get("TJ_LIB_PATH") or os.path.join(LIB_DIR, "libtickjoin_b200.so")  # override: experiments

TJ_MEM_HOST = 0
TJ_MEM_DEVICE = 1
TJ_OUT_IDS32 = 0x100  # out_mem flag: result ids as int32 when they all fit
TJ_REBUILD_EVERY_TICK = 0
TJ_REBUILD_ADAPTIVE = 1

_ERRORS = {
    -1: errors.EmptyBatch,
    -2: errors.OutOfBounds,
    -5: errors.TilingGap,
    -6: errors.CountMismatch,
    -7: errors.DuplicateResult,
    -8: errors.BadConfig,
    -20: ValueError,
    -100: errors.DeviceError,
    -101: errors.DeviceError,
    -102: errors.DeviceError,
    -103: errors.DeviceError,
}


class TjConfig(ctypes.Structure):
    _fields_ = [("th_quad", c_int32), ("l_max", c_int32), ("covering_optimization", c_int32),
                ("rebuild", c_int32), ("device", c_int32), ("split_factor", c_int32)]


class TjTickIn(ctypes.Structure):
    _fields_ = [("n_obj", c_int64), ("obj_id", c_void_p), ("obj_x", c_void_p), ("obj_y", c_void_p),
                ("n_q", c_int64), ("q_issuer", c_void_p), ("q_xa", c_void_p), ("q_ya", c_void_p),
                ("q_xb", c_void_p), ("q_yb", c_void_p), ("mem", c_int32), ("out_mem", c_int32)]


class TjTickOut(ctypes.Structure):
    _fields_ = [("n_q", c_int64), ("n_results", c_int64), ("offsets", c_void_p), ("ids", c_void_p),
                ("mem", c_int32), ("id_bytes", c_int32), ("ids32", c_void_p), ("offsets32", c_void_p),
                ("offset_bytes", c_int32), ("reserved", c_int32)]


class TjStats(ctypes.Structure):
    _fields_ = [(k, c_int64) for k in (
        "n_objects", "n_queries", "containment_tests", "decoded_bits", "subq_intersecting",
        "subq_covering", "covering_results", "active_cells", "results_total", "occ_sum", "occ_sumsq",
        "n_leaves", "l_deep", "n_tasks", "bitmap_words", "n_subqueries", "work_units")] + [
        ("rebuilt", c_int32), ("retries", c_int32)] + [
        (k, c_double) for k in ("t_index_ms", "t_filter_ms", "t_decode_ms", "t_merge_ms", "t_total_ms")] + [
        ("mbr", c_double * 4), ("t_join_ms", c_double), ("task_objects", c_int64), ("task_subqueries", c_int64),
        ("kernel_launches", c_int64), ("t_build_ms", c_double), ("t_scatter_ms", c_double), ("t_sort_ms", c_double),
        ("id_order", c_int32), ("reserved2", c_int32), ("t_decode_kernel_ms", c_double)]


class TjIndexInfo(ctypes.Structure):
    _fields_ = [("mbr", c_double * 4), ("th_quad", c_int32), ("l_max", c_int32), ("l_deep", c_int32),
                ("reserved", c_int32), ("n_leaves", c_int64), ("n_cells", c_int64)]


EXPORTED = (
    "tj_abi_version", "tj_device_count", "tj_create", "tj_destroy", "tj_last_error", "tj_tick",
    "tj_get_index", "tj_get_object_cells", "tj_get_subqueries", "tj_get_directory", "tj_get_bitmaps",
    "tj_get_imbalance", "tj_get_occupancy", "tj_get_staging_flushes", "tj_set_shard", "tj_get_stream", "tj_host_alloc", "tj_host_free",
    "tj_nccl_unique_id", "tj_comm_init", "tj_group_create", "tj_group_destroy", "tj_comm_init_local", "tj_tick_sharded",
)

_lib: Optional[ctypes.CDLL] = None


def _prefer_torch_nccl() -> None:
    """Point the library's NCCL loader (TJ_NCCL_LIB) at the NCCL wheel torch links against, so
    both share one libnccl.so.2 in the process whichever loads first (an older system NCCL
    loaded first would be reused by torch and lack symbols it needs)."""
    if os.environ.get("TJ_NCCL_LIB"):
        return
    import importlib.util

    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for d in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["TJ_NCCL_LIB"] = cand
            return


def load_library() -> ctypes.CDLL:
    """Load the in-tree native library (raises DeviceError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise errors.DeviceError(
            f"native library missing: {LIB_PATH} (run __graft_entry__.build()); there is no CPU fallback")
    _prefer_torch_nccl()
    lib = ctypes.CDLL(LIB_PATH)
    i64p = POINTER(c_int64)
    lib.tj_abi_version.restype = c_int
    lib.tj_device_count.argtypes = [POINTER(c_int)]
    lib.tj_create.argtypes = [POINTER(TjConfig), POINTER(c_void_p)]
    lib.tj_destroy.argtypes = [c_void_p]
    lib.tj_last_error.argtypes = [c_void_p]
    lib.tj_last_error.restype = c_char_p
    lib.tj_tick.argtypes = [c_void_p, POINTER(TjTickIn), POINTER(TjTickOut), POINTER(TjStats)]
    lib.tj_get_index.argtypes = [c_void_p, POINTER(TjIndexInfo), c_void_p, c_int64, c_void_p, c_int64]
    lib.tj_get_object_cells.argtypes = [c_void_p, c_void_p, c_int64]
    lib.tj_get_subqueries.argtypes = [c_void_p, i64p, c_void_p, c_void_p, c_void_p, c_int64]
    lib.tj_get_directory.argtypes = [c_void_p, c_void_p, c_int64, c_void_p, i64p, c_void_p, i64p, c_int64]
    lib.tj_get_bitmaps.argtypes = [c_void_p, i64p, i64p] + [c_void_p] * 6 + [c_int64] * 3
    lib.tj_get_imbalance.argtypes = [c_void_p, c_int32, c_int32, POINTER(c_double)]
    lib.tj_get_occupancy.argtypes = [c_void_p, c_void_p, c_int64, POINTER(c_int64)]
    lib.tj_get_staging_flushes.argtypes = [c_void_p, c_int32, POINTER(c_int64)]
    lib.tj_get_stream.argtypes = [c_void_p, POINTER(c_void_p)]
    lib.tj_set_shard.argtypes = [c_void_p, c_int32, c_int32]
    lib.tj_host_alloc.argtypes = [c_int64, POINTER(c_void_p)]
    lib.tj_host_free.argtypes = [c_void_p]
    lib.tj_nccl_unique_id.argtypes = [c_void_p, c_int32]
    lib.tj_comm_init.argtypes = [c_void_p, c_void_p, c_int32, c_int32]
    lib.tj_group_create.argtypes = [c_int32, POINTER(c_void_p)]
    lib.tj_group_destroy.argtypes = [c_void_p]
    lib.tj_comm_init_local.argtypes = [c_void_p, c_void_p, c_int32]
    lib.tj_tick_sharded.argtypes = [c_void_p, POINTER(TjTickIn), POINTER(TjTickOut), POINTER(TjStats)]
    _lib = lib
    return lib


def device_count() -> int:
    n = c_int(0)
    load_library().tj_device_count(ctypes.byref(n))
    return n.value


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for tj_comm_init; rank 0 makes it, the caller shares it."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    rc = lib.tj_nccl_unique_id(buf, 128)
    if rc != 0:
        raise _ERRORS.get(rc, errors.DeviceError)(lib.tj_last_error(None).decode(errors="replace"))
    return buf.raw


class LocalGroup:
    """In-process group of G contexts (one host thread each) for tj_tick_sharded without NCCL."""

    def __init__(self, nranks: int):
        self.lib = load_library()
        self.h = c_void_p()
        if self.lib.tj_group_create(nranks, ctypes.byref(self.h)) != 0:
            raise errors.DeviceError("tj_group_create failed")
        self.nranks = nranks

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.tj_group_destroy(self.h)
            self.h = None


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


class NativeContext:
    """Owns one `tj_ctx` (one CUDA device, one stream)."""

    def __init__(self, th_quad: int, l_max: int, covering: bool, rebuild: int = 0, device: int = 0,
                 split_factor: int = 0):
        """split_factor > 0: the uniform-grid method ("ug") with that many cells per side."""
        self.lib = load_library()
        cfg = TjConfig(th_quad, l_max, 1 if covering else 0, rebuild, device, split_factor)
        h = c_void_p()
        rc = self.lib.tj_create(ctypes.byref(cfg), ctypes.byref(h))
        if rc != 0:
            self._raise(rc, None)
        self.h = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.tj_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    def _raise(self, rc: int, h) -> None:
        msg = self.lib.tj_last_error(h).decode(errors="replace") if self.lib else ""
        cls = _ERRORS.get(rc, errors.DeviceError)
        raise cls(msg or f"native error {rc}")

    def _check(self, rc: int) -> None:
        if rc != 0:
            self._raise(rc, self.h)

    # -- hot path ---------------------------------------------------------
    def tick_host(self, ids, xs, ys, qids, qxa, qya, qxb, qyb, ids32: bool = False):
        """Host arrays in, host CSR out (copied into fresh NumPy arrays).  ids32: ask for the
        compact 32-bit delivery (TJ_OUT_IDS32): ids come back int32 only if every id fit,
        offsets int32 only if the tick has fewer than 2^31 results."""
        arrs = [np.ascontiguousarray(ids, np.int64), np.ascontiguousarray(xs, np.float64),
                np.ascontiguousarray(ys, np.float64), np.ascontiguousarray(qids, np.int64),
                np.ascontiguousarray(qxa, np.float64), np.ascontiguousarray(qya, np.float64),
                np.ascontiguousarray(qxb, np.float64), np.ascontiguousarray(qyb, np.float64)]
        tin = TjTickIn(len(arrs[0]), _ptr(arrs[0]), _ptr(arrs[1]), _ptr(arrs[2]), len(arrs[3]),
                       _ptr(arrs[3]), _ptr(arrs[4]), _ptr(arrs[5]), _ptr(arrs[6]), _ptr(arrs[7]),
                       TJ_MEM_HOST, TJ_MEM_HOST | (TJ_OUT_IDS32 if ids32 else 0))
        tout = TjTickOut()
        st = TjStats()
        self._check(self.lib.tj_tick(self.h, ctypes.byref(tin), ctypes.byref(tout), ctypes.byref(st)))
        m = tout.n_q
        osrc, otyp = (tout.offsets32, c_int32) if tout.offset_bytes == 4 else (tout.offsets, c_int64)
        offs = np.ctypeslib.as_array(ctypes.cast(osrc, POINTER(otyp)), shape=(m + 1,)).copy()
        res = np.zeros(0, np.int32 if tout.id_bytes == 4 else np.int64)
        if tout.n_results:
            src, typ = (tout.ids32, c_int32) if tout.id_bytes == 4 else (tout.ids, c_int64)
            res = np.ctypeslib.as_array(ctypes.cast(src, POINTER(typ)), shape=(tout.n_results,)).copy()
        return offs, res, st

    def tick_ptrs(self, n, ids, xs, ys, m, qids, qxa, qya, qxb, qyb, mem: int, out_mem: int):
        """Raw-pointer tick (device tensors or pinned host buffers); returns (TjTickOut, TjStats)."""
        tin = TjTickIn(n, ids, xs, ys, m, qids, qxa, qya, qxb, qyb, mem, out_mem)
        tout = TjTickOut()
        st = TjStats()
        self._check(self.lib.tj_tick(self.h, ctypes.byref(tin), ctypes.byref(tout), ctypes.byref(st)))
        return tout, st

    def comm_init(self, unique_id: bytes, rank: int, nranks: int) -> None:
        """NCCL communicator for tj_tick_sharded (collective: every rank calls it)."""
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        self._check(self.lib.tj_comm_init(self.h, buf, rank, nranks))

    def comm_init_local(self, group: "LocalGroup", rank: int) -> None:
        self._check(self.lib.tj_comm_init_local(self.h, group.h, rank))

    def tick_sharded_host(self, ids, xs, ys, qxa, qya, qxb, qyb, ids32: bool = False):
        """This rank's slice in (host arrays), the complete CSR of this rank's queries out."""
        arrs = [np.ascontiguousarray(ids, np.int64), np.ascontiguousarray(xs, np.float64),
                np.ascontiguousarray(ys, np.float64), np.ascontiguousarray(qxa, np.float64),
                np.ascontiguousarray(qya, np.float64), np.ascontiguousarray(qxb, np.float64),
                np.ascontiguousarray(qyb, np.float64)]
        tin = TjTickIn(len(arrs[0]), _ptr(arrs[0]), _ptr(arrs[1]), _ptr(arrs[2]), len(arrs[3]), 0,
                       _ptr(arrs[3]), _ptr(arrs[4]), _ptr(arrs[5]), _ptr(arrs[6]),
                       TJ_MEM_HOST, TJ_MEM_HOST | (TJ_OUT_IDS32 if ids32 else 0))
        tout = TjTickOut()
        st = TjStats()
        self._check(self.lib.tj_tick_sharded(self.h, ctypes.byref(tin), ctypes.byref(tout), ctypes.byref(st)))
        m = tout.n_q
        osrc, otyp = (tout.offsets32, c_int32) if tout.offset_bytes == 4 else (tout.offsets, c_int64)
        offs = np.ctypeslib.as_array(ctypes.cast(osrc, POINTER(otyp)), shape=(m + 1,)).copy()
        res = np.zeros(0, np.int32 if tout.id_bytes == 4 else np.int64)
        if tout.n_results:
            src, typ = (tout.ids32, c_int32) if tout.id_bytes == 4 else (tout.ids, c_int64)
            res = np.ctypeslib.as_array(ctypes.cast(src, POINTER(typ)), shape=(tout.n_results,)).copy()
        return offs, res, st

    def tick_sharded_ptrs(self, n, ids, xs, ys, m, qxa, qya, qxb, qyb, mem: int, out_mem: int):
        """Raw-pointer sharded tick (device tensors or pinned host buffers); returns (TjTickOut, TjStats)."""
        tin = TjTickIn(n, ids, xs, ys, m, 0, qxa, qya, qxb, qyb, mem, out_mem)
        tout = TjTickOut()
        st = TjStats()
        self._check(self.lib.tj_tick_sharded(self.h, ctypes.byref(tin), ctypes.byref(tout), ctypes.byref(st)))
        return tout, st

    def set_shard(self, rank: int, nranks: int) -> None:
        """Leaf-range sharding: this context joins only rank's Morton range of leaves."""
        self._check(self.lib.tj_set_shard(self.h, rank, nranks))

    def stream(self) -> int:
        s = c_void_p()
        self._check(self.lib.tj_get_stream(self.h, ctypes.byref(s)))
        return s.value or 0

    # -- introspection (reference order) ----------------------------------
    def index(self):
        info = TjIndexInfo()
        self._check(self.lib.tj_get_index(self.h, ctypes.byref(info), None, 0, None, 0))
        leaves = np.zeros(info.n_leaves, np.int64)
        zmap = np.zeros(info.n_cells, np.int64)
        self._check(self.lib.tj_get_index(self.h, ctypes.byref(info), _ptr(leaves), len(leaves),
                                          _ptr(zmap), len(zmap)))
        return dict(mbr=tuple(info.mbr), l_deep=info.l_deep, leaves=leaves, zmap=zmap)

    def object_cells(self, n: int) -> np.ndarray:
        out = np.zeros(n, np.int64)
        self._check(self.lib.tj_get_object_cells(self.h, _ptr(out), n))
        return out

    def subqueries(self):
        cnt = c_int64(0)
        self._check(self.lib.tj_get_subqueries(self.h, ctypes.byref(cnt), None, None, None, 0))
        S = cnt.value
        q = np.zeros(S, np.int64)
        cell = np.zeros(S, np.int64)
        cov = np.zeros(S, np.uint8)
        self._check(self.lib.tj_get_subqueries(self.h, ctypes.byref(cnt), _ptr(q), _ptr(cell), _ptr(cov), S))
        return q, cell, cov.astype(bool)

    def directory(self, n: int):
        ni, nc = c_int64(0), c_int64(0)
        self._check(self.lib.tj_get_directory(self.h, None, 0, None, ctypes.byref(ni), None,
                                              ctypes.byref(nc), 0))
        rows = np.zeros(n, np.int64)
        isq = np.zeros(ni.value, np.int64)
        cov = np.zeros(nc.value, np.int64)
        cap = max(ni.value, nc.value)
        self._check(self.lib.tj_get_directory(self.h, _ptr(rows), n, _ptr(isq), ctypes.byref(ni), _ptr(cov),
                                              ctypes.byref(nc), cap))
        return rows, isq, cov

    def bitmaps(self):
        nt, nw = c_int64(0), c_int64(0)
        self._check(self.lib.tj_get_bitmaps(self.h, ctypes.byref(nt), ctypes.byref(nw), None, None, None, None,
                                            None, None, 0, 0, 0))
        T, W = nt.value, nw.value
        cell = np.zeros(T, np.int64)
        nobj = np.zeros(T, np.int64)
        nisq = np.zeros(T, np.int64)
        woff = np.zeros(T + 1, np.int64)
        words = np.zeros(W, np.uint32)
        # counts: one per intersecting subquery of a task; bounded by W
        counts = np.zeros(max(W, 1), np.int64)
        self._check(self.lib.tj_get_bitmaps(self.h, ctypes.byref(nt), ctypes.byref(nw), _ptr(cell), _ptr(nobj),
                                            _ptr(nisq), _ptr(woff), _ptr(words), _ptr(counts), T, W,
                                            len(counts)))
        return dict(cell=cell, nobj=nobj, nisq=nisq, woff=woff, words=words,
                    counts=counts[: int(nisq.sum())])

    def staging_flushes(self, staging_capacity: int) -> int:
        """ug_baseline's shared-buffer flushes (= sync_ops) for the last tick."""
        v = c_int64(0)
        self._check(self.lib.tj_get_staging_flushes(self.h, staging_capacity, ctypes.byref(v)))
        return v.value

    def occupancy(self) -> np.ndarray:
        """Object counts of the non-empty leaves, ascending packed cell order (int64)."""
        n = c_int64(0)
        self._check(self.lib.tj_get_occupancy(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, np.int64)
        self._check(self.lib.tj_get_occupancy(self.h, _ptr(out), len(out), ctypes.byref(n)))
        return out

    def imbalance(self, sim_processors: int, heaviest_first: bool) -> float:
        v = c_double(0.0)
        self._check(self.lib.tj_get_imbalance(self.h, sim_processors, 1 if heaviest_first else 0,
                                              ctypes.byref(v)))
        return v.value
