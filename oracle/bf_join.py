"""ctypes wrapper of oracle/bf_join.c — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

The exact brute-force range join of the reference (`oracle.py:17-28` in
/root/reference/pkg/src/tickjoin/) in C with a pruning grid, multithreaded, for
full-size parity checks (10M-50M objects) where the NumPy port is too slow.
Only tests/ and bench.py's CPU legs use it.  Pinned against the NumPy
`quad_oracle.brute_force` and the reference-generated digests in
tests/test_oracle_golden.py.

Per query it returns the result count and `digest = sum(mix64(id)) mod 2^64`
(splitmix64 finaliser, order-independent); `csr_digests` computes the same
function over a CSR, so a device result can be compared query by query.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import c_double, c_int, c_int32, c_int64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "bf_join.c")
LIB = os.path.join(HERE, "_lib", "libbfjoin.so")

_lib = None


def build_library(force: bool = False) -> str:
    """gcc -O3 -shared -fPIC -pthread oracle/bf_join.c -> oracle/_lib/libbfjoin.so"""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.run(["gcc", "-O3", "-shared", "-fPIC", "-pthread", "-fno-fast-math", "-ffp-contract=off", SRC,
                    "-o", LIB], check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
            build_library()
        lib = ctypes.CDLL(LIB)
        lib.bf_build.restype = c_void_p
        lib.bf_build.argtypes = [c_int64, c_void_p, c_void_p, c_void_p, c_double, c_int32]
        lib.bf_free.argtypes = [c_void_p]
        lib.bf_count.restype = c_int
        lib.bf_count.argtypes = [c_void_p, c_int64, c_void_p] + [c_void_p] * 4 + [c_void_p, c_void_p, c_int]
        lib.bf_lists.restype = c_int
        lib.bf_lists.argtypes = [c_void_p, c_int64, c_void_p] + [c_void_p] * 4 + [c_void_p, c_void_p, c_int]
        lib.bf_csr_digests.argtypes = [c_int64, c_void_p, c_void_p, c_void_p]
        lib.bf_mix64.restype = ctypes.c_uint64
        lib.bf_mix64.argtypes = [ctypes.c_uint64]
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data if a is not None else None


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


class BruteForce:
    """Objects bucketed once; any number of query batches answered exactly."""

    def __init__(self, ids, xs, ys, cell: float = 8.0, gmax: int = 8192):
        self._ids = np.ascontiguousarray(ids, np.int64)
        self._xs = np.ascontiguousarray(xs, np.float64)
        self._ys = np.ascontiguousarray(ys, np.float64)
        self._h = load().bf_build(len(self._ids), _p(self._xs), _p(self._ys), _p(self._ids), float(cell), int(gmax))
        if not self._h:
            raise MemoryError("bf_build failed")

    def close(self):
        if self._h:
            load().bf_free(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _q(qxa, qya, qxb, qyb):
        return [np.ascontiguousarray(a, np.float64) for a in (qxa, qya, qxb, qyb)]

    def counts(self, qxa, qya, qxb, qyb, rows=None, threads: int = 0):
        """(counts int64, digests uint64) for every query (or the given rows)."""
        q = self._q(qxa, qya, qxb, qyb)
        rows = None if rows is None else np.ascontiguousarray(rows, np.int64)
        m = len(q[0]) if rows is None else len(rows)
        cnt = np.zeros(m, np.int64)
        dig = np.zeros(m, np.uint64)
        rc = load().bf_count(self._h, m, _p(rows), *(_p(a) for a in q), _p(cnt), _p(dig),
                             threads or default_threads())
        assert rc == 0
        return cnt, dig

    def lists(self, qxa, qya, qxb, qyb, rows=None, threads: int = 0):
        """CSR (offsets, ids) of the sorted result lists of every query (or the given rows)."""
        cnt, _ = self.counts(qxa, qya, qxb, qyb, rows=rows, threads=threads)
        offs = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        out = np.zeros(int(offs[-1]), np.int64)
        q = self._q(qxa, qya, qxb, qyb)
        rows = None if rows is None else np.ascontiguousarray(rows, np.int64)
        rc = load().bf_lists(self._h, len(cnt), _p(rows), *(_p(a) for a in q), _p(offs), _p(out),
                             threads or default_threads())
        assert rc == 0, "bf_lists: counts changed between passes"
        return offs, out


def csr_digests(offsets, ids) -> np.ndarray:
    """Per-query sum(mix64(id)) of a CSR (uint64), the same function as BruteForce.counts."""
    offsets = np.ascontiguousarray(offsets, np.int64)
    ids = np.ascontiguousarray(ids, np.int64)
    out = np.zeros(len(offsets) - 1, np.uint64)
    load().bf_csr_digests(len(out), _p(offsets), _p(ids), _p(out))
    return out


def mix64(v: int) -> int:
    return int(load().bf_mix64(ctypes.c_uint64(v & 0xFFFFFFFFFFFFFFFF)))
