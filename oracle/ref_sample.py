"""The CPU reference arm's bounded sample of one full-size tick — BENCH INFRASTRUCTURE.

Used only by bench.py (`--impl reference` and the `cpu_baseline` leg); never by
the product.  It times the NumPy restatement of the reference QUAD pipeline
(oracle/quad_oracle.py, each function citing /root/reference/pkg/src/tickjoin/
file:line) on the SAME tick the GPU arm runs (config C @5u: 10M objects, 10M
queries), split so that one bench step stays a few seconds:

* the tick's query-independent work — exact MBR (geometry.py:72-77), the
  quadtree build (quadtree.py:74-158), clipping every query (grid.py:115-122),
  mapping every object to its leaf (quadtree.py:161-165) and grouping the
  objects per leaf (directory.py:119-128) — runs once per tick and is timed
  (`t_fixed`);
* the queries are cut into `n_chunks` spatially coherent chunks (ordered by the
  Morton code of their clipped rect's lower corner: a chunk touches a compact
  region, so its per-leaf tasks carry as many subqueries as in the whole tick);
  a chunk runs the rest of the pipeline for its queries — split into
  subqueries (quadtree.py:168-240), subquery directory (directory.py:129-158),
  per-leaf bitmaps (bitmap.py:70-119), decode + covering expansion
  (decode.py:40-99) and the canonical merge (decode.py:102-123);
* a step runs `workers` chunks at once, one per forked process (all the host
  cores the box gives), timed by wall clock; its cost is that wall time plus
  its queries' share of `t_fixed`: throughput = queries / (wall + t_fixed *
  queries / m).

The chunks of one tick add up to the whole tick's work, except that a leaf on a
chunk boundary is joined once per chunk that touches it (a small per-task
overhead, charged to the reference).
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import quad_oracle as qo

_STATE = None  # the sampler of the parent process, inherited by forked workers


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


class TickSampler:
    def __init__(self, tick, n_chunks: int = 64, th_quad: int = 384, l_max: int = qo.L_MAX):
        self.tick = tick
        ids, xs, ys = tick.ids, tick.xs, tick.ys
        self.m = tick.n_queries
        t0 = time.perf_counter()
        mbr = qo.mbr_of(xs, ys)
        idx = qo.build_index(xs, ys, mbr, th_quad, l_max)
        keep, cxa, cya, cxb, cyb = qo.clip_rects(tick.qxa, tick.qya, tick.qxb, tick.qyb, idx.mbr)
        obj_cell = qo.map_objects(xs, ys, idx)
        obj_order = np.argsort(obj_cell, kind="stable")
        oc = obj_cell[obj_order]
        self.t_fixed = time.perf_counter() - t0
        self.idx, self.keep_rows = idx, np.flatnonzero(keep)
        self.c = (cxa, cya, cxb, cyb)
        self.obj_order, self.oc = obj_order, oc
        # sample selection (not part of the pipeline, untimed): spatial order of the clipped queries
        i, j = qo.cell_coords(cxa, cya, idx.mbr, l_max)
        order = np.argsort(qo.morton(i, j), kind="stable")
        self.chunks = np.array_split(order, n_chunks)

    def run_chunk(self, k: int):
        """The per-query part of the tick for chunk k; returns (queries, results, seconds)."""
        rows = self.chunks[k % len(self.chunks)]
        t0 = time.perf_counter()
        cxa, cya, cxb, cyb = (a[rows] for a in self.c)
        sub = qo.split_queries(cxa, cya, cxb, cyb, self.idx)
        # subquery directory (directory.py:129-158): intersecting / covering blocks per cell
        order = np.lexsort((sub.covering, sub.cell))
        isq = order[~sub.covering[order]]
        cov = order[sub.covering[order]]
        ic = sub.cell[isq]
        cells = np.unique(ic)
        i_lo = np.searchsorted(ic, cells, "left")
        i_hi = np.searchsorted(ic, cells, "right")
        o_lo = np.searchsorted(self.oc, cells, "left")
        o_hi = np.searchsorted(self.oc, cells, "right")
        xs, ys, ids = self.tick.xs, self.tick.ys, self.tick.ids
        parts_q, parts_i = [], []
        for r in range(len(cells)):  # per task: Alg. 2 bitmaps, popcounts, Alg. 4 decode
            if o_hi[r] == o_lo[r]:
                continue
            orow = self.obj_order[o_lo[r]:o_hi[r]]
            srow = isq[i_lo[r]:i_hi[r]]
            qr = sub.qrow[srow]
            words = qo.cell_bitmap(xs[orow], ys[orow], cxa[qr], cya[qr], cxb[qr], cyb[qr])
            counts = qo.word_popcounts(words, len(srow))
            nb = len(words) // len(srow)
            bits = np.unpackbits(words.reshape(len(srow), nb).view(np.uint8), axis=1,
                                 bitorder="little")[:, :len(orow)]
            rr, cc = np.nonzero(bits)
            if np.any(np.bincount(rr, minlength=len(srow)) != counts):
                raise qo.OracleError("CountMismatch", "decode disagrees with popcounts")
            parts_q.append(qr[rr])
            parts_i.append(ids[orow[cc]])
        for k2 in cov:  # covering expansion (decode.py:83-99)
            lo = np.searchsorted(self.oc, sub.cell[k2], "left")
            hi = np.searchsorted(self.oc, sub.cell[k2], "right")
            if hi > lo:
                parts_q.append(np.full(hi - lo, sub.qrow[k2], np.int64))
                parts_i.append(ids[self.obj_order[lo:hi]])
        allq = np.concatenate(parts_q) if parts_q else np.zeros(0, np.int64)
        alli = np.concatenate(parts_i) if parts_i else np.zeros(0, np.int64)
        o = np.lexsort((alli, allq))  # canonical merge (decode.py:102-123)
        allq, alli = allq[o], alli[o]
        if len(allq) > 1 and np.any((allq[1:] == allq[:-1]) & (alli[1:] == alli[:-1])):
            raise qo.OracleError("DuplicateResult", "pair produced twice")
        np.bincount(allq, minlength=len(rows))
        return len(rows), len(alli), time.perf_counter() - t0


def _work(k):
    return _STATE.run_chunk(k)


class ReferenceArm:
    """Steps of `workers` chunks at once (forked processes), wall-clock timed."""

    def __init__(self, tick, workers: int = 0, n_chunks: int = 64):
        global _STATE
        self.workers = workers or host_cores()
        n_chunks = max(n_chunks, self.workers)
        self.sampler = TickSampler(tick, n_chunks=n_chunks)
        _STATE = self.sampler
        self.pool = None
        if self.workers > 1:
            import multiprocessing as mp

            self.pool = mp.get_context("fork").Pool(self.workers)
        self.next = 0

    def step(self):
        ks = list(range(self.next, self.next + self.workers))
        self.next += self.workers
        t0 = time.perf_counter()
        res = self.pool.map(_work, ks, chunksize=1) if self.pool else [_work(k) for k in ks]
        wall = time.perf_counter() - t0
        q = sum(r[0] for r in res)
        cost = wall + self.sampler.t_fixed * q / self.sampler.m
        return q, cost, wall, sum(r[1] for r in res)

    def close(self):
        if self.pool:
            self.pool.close()
            self.pool.join()
            self.pool = None

    def describe(self) -> str:
        s = self.sampler
        return (f"oracle/quad_oracle.py (NumPy restatement of the reference QUAD tick) on the bench's own tick "
                f"({s.tick.n_objects:,} objects, {s.m:,} queries): the query-independent part (MBR, quadtree "
                f"build, clip, object->leaf map and grouping) timed once, {s.t_fixed:.2f} s, charged per query; "
                f"the rest in {len(s.chunks)} spatially coherent query chunks of ~{s.m // len(s.chunks):,}, "
                f"{self.workers} chunks per step in parallel forked processes (wall clock); queries/s = "
                f"queries / (wall + t_fixed * queries / m)")
