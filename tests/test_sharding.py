"""Leaf-range sharding across ranks.

CPU: ownership math, partial merging, and a world_size-2 gloo run of the
host path (all-gather of per-rank updates, per-rank partial results, gather +
merge) with the oracle standing in for each rank's device tick.
GPU: two sharded contexts on one device reproduce the unsharded tick.
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


def _gloo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from paper_1411_3212_b200.sharding import all_gather_var

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = _small_tick()
        n, m = len(full["ids"]), len(full["qids"])
        # this rank ingests 1/G of the updates and queries (interleaved split)
        osl, qsl = slice(rank, n, world), slice(rank, m, world)
        mine = [full["ids"][osl], full["xs"][osl], full["ys"][osl], full["qids"][qsl],
                *(r[qsl] for r in full["rects"])]
        gathered = [all_gather_var(torch.as_tensor(np.ascontiguousarray(a)))[0].numpy() for a in mine]
        tick = dict(ids=gathered[0], xs=gathered[1], ys=gathered[2], qids=gathered[3], rects=tuple(gathered[4:]))
        # every rank now holds the same (reordered) tick: identical index on all ranks
        offs, ids, (foffs, fids) = _partial_for_rank(tick, rank, world)
        counts, _ = all_gather_var(torch.as_tensor(np.diff(offs)))
        allids, sizes = all_gather_var(torch.as_tensor(ids))
        counts = counts.numpy().reshape(world, -1)
        parts, base = [], 0
        for r in range(world):
            parts.append((np.concatenate([[0], np.cumsum(counts[r])]), allids.numpy()[base:base + sizes[r]]))
            base += sizes[r]
        moffs, mids = merge_partials(parts)
        ok = np.array_equal(moffs, foffs) and np.array_equal(mids, fids)
        ok = ok and all(len(p[1]) > 0 for p in parts)  # both ranks did real work
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
