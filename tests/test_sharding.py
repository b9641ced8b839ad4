"""Leaf-range sharding across ranks.

CPU: ownership math, partial merging, and world_size-2 gloo runs of
ShardedEngine's host protocol (gather of the ranks' objects, queries routed
to the owners of their leaves, per-rank partial lists, back to the queries'
home ranks, merge) with the oracle restricted to the rank's leaves standing in
for the device tick and its routing.
GPU: sharded contexts on one device reproduce the unsharded tick (the native
data plane itself: tests/test_gpu_sharded.py).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from oracle import quad_oracle as qo
from paper_1411_3212_b200.errors import DuplicateResult
from paper_1411_3212_b200.sharding import leaf_owners, leaf_weight, merge_partials


def test_leaf_owners_contiguous_and_balanced():
    rng = np.random.default_rng(0)
    w = rng.integers(0, 1000, 5000)
    for n in (1, 2, 3, 4, 8):
        own = leaf_owners(w, n)
        assert own.min() == 0 and own.max() == n - 1
        assert np.all(np.diff(own) >= 0)  # contiguous Morton ranges
        loads = np.bincount(own, weights=w, minlength=n)
        assert loads.max() <= w.sum() / n + w.max() + 1


def test_merge_partials_union_sorted_and_duplicates():
    a = (np.array([0, 2, 2, 3]), np.array([1, 9, 4]))
    b = (np.array([0, 1, 2, 2]), np.array([5, 0]))
    offs, ids = merge_partials([a, b])
    assert offs.tolist() == [0, 3, 4, 5] and ids.tolist() == [1, 5, 9, 0, 4]
    with pytest.raises(DuplicateResult):
        merge_partials([a, (np.array([0, 1, 1, 1]), np.array([9]))])


def _partial_for_rank(tick, rank, nranks, th=64):
    """Oracle stand-in for one rank's device tick: the results whose object's
    leaf lies in the rank's Morton range of leaves."""
    t = qo.run_tick(tick["ids"], tick["xs"], tick["ys"], tick["qids"], *tick["rects"], th_quad=th)
    idx, d = t.index, t.directory
    lm = idx.l_max
    lev = idx.leaves >> (2 * lm)
    z = idx.leaves & ((1 << (2 * lm)) - 1)
    morton_order = np.argsort(z << (2 * (idx.l_deep - lev)), kind="stable")  # zmap run order
    cells = idx.leaves[morton_order]
    rows = np.searchsorted(d.cells, cells)
    present = (rows < len(d.cells)) & (d.cells[np.minimum(rows, len(d.cells) - 1)] == cells)
    nobj = np.where(present, (d.o_end - d.o_start)[np.minimum(rows, len(d.cells) - 1)], 0)
    nisq = np.where(present, (d.i_end - d.i_start)[np.minimum(rows, len(d.cells) - 1)], 0)
    ncov = np.where(present, (d.c_end - d.c_start)[np.minimum(rows, len(d.cells) - 1)], 0)
    own = leaf_owners(leaf_weight(nobj), nranks)
    mine = set(cells[own == rank].tolist())
    id_to_cell = dict(zip(tick["ids"].tolist(), t.obj_cell.tolist()))
    offs, ids = t.offsets, t.result_ids
    keep = np.array([id_to_cell[int(v)] in mine for v in ids], bool) if len(ids) else np.zeros(0, bool)
    q_of = np.repeat(np.arange(len(offs) - 1), np.diff(offs))
    counts = np.bincount(q_of[keep], minlength=len(offs) - 1)
    return np.concatenate([[0], np.cumsum(counts)]).astype(np.int64), ids[keep], (offs, ids)


def _small_tick(seed=3):
    from paper_1411_3212_b200.workload import WorkloadConfig, iter_ticks

    tk = next(iter_ticks(WorkloadConfig(n_objects=3000, n_ticks=1, distribution="gaussian", n_hotspots=3,
                                        seed=seed, query_side=(20.0, 300.0))))
    return dict(ids=tk.ids, xs=tk.xs, ys=tk.ys, qids=tk.qids, rects=(tk.qxa, tk.qya, tk.qxb, tk.qyb))


def _stub_partial_tick(ids, xs, ys, qxa, qya, qxb, qyb, rank, world):
    """Stubbed device tick: the given queries' lists restricted to the rank's Morton leaf range."""
    tick = dict(ids=ids, xs=xs, ys=ys, qids=np.arange(len(qxa), dtype=np.int64), rects=(qxa, qya, qxb, qyb))
    offs, pids, _ = _partial_for_rank(tick, rank, world)
    return offs, pids


def _stub_route(ids, xs, ys, qxa, qya, qxb, qyb, rank, world):
    """Stubbed k_route: the ranks owning the leaves that hold a query's results (the device routes
    by every leaf the window touches; for the lists, the ranks holding results are what matters)."""
    m = len(qxa)
    mask = np.zeros(m, np.uint64)
    for j in range(world):
        tick = dict(ids=ids, xs=xs, ys=ys, qids=np.arange(m, dtype=np.int64), rects=(qxa, qya, qxb, qyb))
        offs, _, _ = _partial_for_rank(tick, j, world)
        mask |= np.where(np.diff(offs) > 0, np.uint64(1) << np.uint64(j), np.uint64(0))
    return mask


def _gloo_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_1411_3212_b200 import MethodConfig
    from paper_1411_3212_b200.sharding import ShardedEngine

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = _small_tick()
        n, m = len(full["ids"]), len(full["qids"])
        # uneven contiguous slices of the updates and the queries (rank 0 issues more queries)
        ob = [0, n // 3, n] if world == 2 else [r * n // world for r in range(world + 1)]
        qb = [0, 2 * m // 3, m] if world == 2 else [r * m // world for r in range(world + 1)]
        o0, o1, q0, q1 = ob[rank], ob[rank + 1], qb[rank], qb[rank + 1]
        eng = ShardedEngine(MethodConfig(method="quad", th_quad=64), partial_tick=_stub_partial_tick,
                            route=_stub_route)
        (offs, ids), _ = eng.process_shard(full["ids"][o0:o1], full["xs"][o0:o1], full["ys"][o0:o1],
                                           *(r_[q0:q1] for r_ in full["rects"]))
        eng.close()
        # the complete lists of this rank's queries: the unsharded tick's rows q0..q1
        ref = qo.run_tick(full["ids"], full["xs"], full["ys"], full["qids"], *full["rects"], th_quad=64)
        want_off = ref.offsets[q0:q1 + 1] - ref.offsets[q0]
        want_ids = ref.result_ids[ref.offsets[q0]:ref.offsets[q1]]
        ok = np.array_equal(offs, want_off) and np.array_equal(ids, want_ids)
        # the routing really moved lists: some of this rank's results came from the other rank's leaves
        mine = _partial_for_rank(dict(full), rank, world)
        local = np.diff(mine[0])[q0:q1].sum()
        ok = ok and 0 < local < len(want_ids)
        out.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_world2_allgather_shard_merge():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


@pytest.mark.gpu
def test_two_sharded_contexts_reproduce_the_tick():
    from paper_1411_3212_b200 import _native

    tick = _small_tick(seed=9)
    args = (tick["ids"], tick["xs"], tick["ys"], tick["qids"], *tick["rects"])
    full = _native.NativeContext(64, 12, True)
    f_offs, f_ids, f_st = full.tick_host(*args)
    for n in (2, 3, 4):
        parts = []
        for r in range(n):
            ctx = _native.NativeContext(64, 12, True)
            ctx.set_shard(r, n)
            o, i, _ = ctx.tick_host(*args)
            parts.append((o, i))
            ctx.close()
        offs, ids = merge_partials(parts)
        assert np.array_equal(offs, f_offs) and np.array_equal(ids, f_ids), n
        assert sum(len(p[1]) for p in parts) == len(f_ids)
    full.close()


@pytest.mark.gpu
@pytest.mark.parametrize("sf", [7, 256])
def test_two_sharded_ug_contexts_reproduce_the_tick(sf):
    """Leaf-range sharding is index-agnostic: the uniform grid's cells shard the same way."""
    from paper_1411_3212_b200 import _native

    tick = _small_tick(seed=10)
    args = (tick["ids"], tick["xs"], tick["ys"], tick["qids"], *tick["rects"])
    full = _native.NativeContext(1, 12, True, 0, 0, sf)
    f_offs, f_ids, _ = full.tick_host(*args)
    for n in (2, 3):
        parts = []
        for r in range(n):
            ctx = _native.NativeContext(1, 12, True, 0, 0, sf)
            ctx.set_shard(r, n)
            o, i, _ = ctx.tick_host(*args)
            parts.append((o, i))
            ctx.close()
        offs, ids = merge_partials(parts)
        assert np.array_equal(offs, f_offs) and np.array_equal(ids, f_ids), n
    full.close()
