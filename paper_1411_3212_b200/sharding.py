"""Multi-GPU leaf-range sharding of the QUAD tick.

One process per GPU.  Each rank passes its slice of the tick's position
updates and queries; the ranks' slices are gathered into the full tick on
every rank, every rank builds the bit-identical index (the index build is
integer-exact), then scatters, joins and decodes only the (query, leaf) pairs
of its contiguous Morton range of leaves, balanced by the per-leaf object
count (device side: `k_shard_mark` in csrc/tj_kernels.cuh).  A rank's
per-query lists are the restriction of the full lists to its leaves: disjoint
across ranks and each sorted.  Each query's partial lists go to its home
rank (the rank whose slice issued it) and are merged there, so every rank
ends with the complete lists of its own queries.

The product path is the native library's `tj_tick_sharded` over NCCL
(csrc/tj_shard.cuh: NCCL broadcasts / send-recv on the library stream, merge
on the device).  `ShardedEngine(..., partial_tick=f)` runs the same protocol
with torch.distributed collectives and a caller-supplied partial tick — the
host restatement the CPU tests drive over gloo with a stubbed device tick.

The reference has no distributed path (multi-GPU / distributed
execution is a non-goal); this module is B200-side plumbing only.
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from .errors import DuplicateResult


def leaf_weight(nobj: np.ndarray) -> np.ndarray:
    """Per-leaf work weight — the device's `LeafWeightIn`: objects + 1 (known
    right after the index build, before the query scatter)."""
    return np.asarray(nobj, np.int64) + 1


def leaf_owners(weights: np.ndarray, nranks: int) -> np.ndarray:
    """Owner rank of every leaf (leaves in Morton order): contiguous ranges
    cut at the weight midpoints — the device's `k_shard_mark`, bit for bit."""
    w = np.asarray(weights, np.int64)
    pre = np.concatenate([[0], np.cumsum(w)[:-1]]) if len(w) else w
    total = max(int(w.sum()), 1)
    owner = ((2 * pre + w) * nranks) // (2 * total)
    return np.minimum(owner, nranks - 1)


def merge_partials(parts: Sequence[tuple]) -> tuple:
    """Union of per-rank partial CSRs (offsets[m+1], ids) into the full CSR.

    Partial lists of one query are disjoint and sorted; the union is sorted
    ascending (decode.py:117) and a repeated id raises DuplicateResult
    (decode.py:118-121).
    """
    m = len(parts[0][0]) - 1
    counts = np.zeros(m, np.int64)
    for offs, _ in parts:
        counts += np.diff(np.asarray(offs, np.int64))
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    qs = np.concatenate([np.repeat(np.arange(m, dtype=np.int64), np.diff(np.asarray(o, np.int64)))
                         for o, _ in parts]) if m else np.zeros(0, np.int64)
    vals = np.concatenate([np.asarray(v, np.int64) for _, v in parts]) if parts else np.zeros(0, np.int64)
    order = np.lexsort((vals, qs))
    qs, vals = qs[order], vals[order]
    if len(vals) > 1 and np.any((qs[1:] == qs[:-1]) & (vals[1:] == vals[:-1])):
        raise DuplicateResult("a (query, object) pair came from two ranks")
    return offsets, vals


def all_gather_var(t, group=None):
    """All-gather of 1-D tensors whose length differs per rank (concatenated in rank order)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(sizes) if sizes else 0
    pad = torch.zeros(cap, dtype=t.dtype, device=t.device)
    pad[: t.numel()] = t
    bufs = [torch.zeros(cap, dtype=t.dtype, device=t.device) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)]), sizes


def split_bounds(total: int, world: int) -> np.ndarray:
    """Contiguous 1/G slices: rank r owns [b[r], b[r + 1])."""
    return np.array([r * total // world for r in range(world + 1)], np.int64)


class ShardedEngine:
    """One rank of a G-GPU QUAD tick (torch.distributed process group already initialised).

    partial_tick=None: the native `tj_tick_sharded` over an NCCL communicator the ranks set
    up here (rank 0's unique id broadcast over the process group).  Otherwise the protocol
    runs on the host with torch.distributed (the restatement of csrc/tj_shard.cuh the gloo
    tests exercise) around two caller-supplied device stand-ins:
    route(ids, xs, ys, qxa, qya, qxb, qyb, rank, world) -> per own query a bit mask of the
    ranks owning leaves it touches (`k_route`), and
    partial_tick(ids, xs, ys, qxa, qya, qxb, qyb, rank, world) -> (offsets[m + 1], ids): the
    lists of the given (received) queries restricted to the rank's leaves (what the device
    computes after `k_shard_mark`)."""

    def __init__(self, cfg, device: Optional[int] = None, group=None, partial_tick=None, route=None):
        import torch.distributed as dist

        cfg.validate()
        self.cfg = cfg
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = cfg.device if device is None else device
        self.partial_tick = partial_tick
        self.route = route
        self.ctx = None
        if partial_tick is None:
            from . import _native

            self.ctx = _native.NativeContext(cfg.th_quad, cfg.l_max, cfg.covering_optimization, 0, self.device)
            uid = [_native.nccl_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(uid, src=0, group=group)
            self.ctx.comm_init(uid[0], self.rank, self.world)

    def process_shard(self, ids, xs, ys, qxa, qya, qxb, qyb):
        """This rank's slice of the tick in (host arrays); the complete CSR of this rank's
        queries out: (offsets, ids), stats (None on the host path)."""
        if self.ctx is not None:
            offs, res, st = self.ctx.tick_sharded_host(ids, xs, ys, qxa, qya, qxb, qyb)
            return (offs, res), st
        return self._host_protocol(ids, xs, ys, qxa, qya, qxb, qyb), None

    def _host_protocol(self, ids, xs, ys, qxa, qya, qxb, qyb):
        """The host restatement of csrc/tj_shard.cuh's sharded_tick (G > 1)."""
        import torch
        import torch.distributed as dist

        G, r, grp = self.world, self.rank, self.group
        # 1. every rank's objects gathered into the full set (slices concatenated in rank order)
        objs = [all_gather_var(torch.as_tensor(np.ascontiguousarray(a)), grp)[0].numpy() for a in (ids, xs, ys)]
        own = [np.ascontiguousarray(a, np.float64) for a in (qxa, qya, qxb, qyb)]
        mr = len(own[0])
        # 2. every own query to the ranks owning the leaves it touches (k_route), grouped per destination
        mask = np.asarray(self.route(*objs, *own, r, G), np.uint64) if mr else np.zeros(0, np.uint64)
        dest = [np.flatnonzero((mask >> np.uint64(j)) & np.uint64(1)) for j in range(G)]
        scnt = torch.tensor([len(x) for x in dest], dtype=torch.int64)
        rcnt_q = torch.empty(G, dtype=torch.int64)
        dist.all_to_all_single(rcnt_q, scnt, group=grp)
        recv = []
        for a in own:
            send = torch.as_tensor(np.concatenate([a[x] for x in dest]) if mr else np.zeros(0))
            out = torch.empty(int(rcnt_q.sum()), dtype=torch.float64)
            dist.all_to_all_single(out, send, output_split_sizes=rcnt_q.tolist(), input_split_sizes=scnt.tolist(),
                                   group=grp)
            recv.append(out.numpy())
        # 3. this rank's leaves, for the queries it received
        poffs, pids = self.partial_tick(*objs, *recv, r, G)
        poffs = np.asarray(poffs, np.int64)
        # 4. each received query's partial list back to its home rank: counts, then the id runs
        rq = rcnt_q.tolist()
        rd = np.concatenate([[0], np.cumsum(rq)]).astype(np.int64)
        back = torch.empty(int(scnt.sum()), dtype=torch.int64)
        dist.all_to_all_single(back, torch.as_tensor(np.diff(poffs)), output_split_sizes=scnt.tolist(),
                               input_split_sizes=rq, group=grp)
        bounds = poffs[rd]
        sid = torch.as_tensor(np.diff(bounds))
        rid = torch.empty(G, dtype=torch.int64)
        dist.all_to_all_single(rid, sid, group=grp)
        rids = torch.empty(int(rid.sum()), dtype=torch.int64)
        dist.all_to_all_single(rids, torch.as_tensor(np.asarray(pids, np.int64)[bounds[0]:bounds[-1]]),
                               output_split_sizes=rid.tolist(), input_split_sizes=sid.tolist(), group=grp)
        # 5. merge: own query q's run from destination j is its place in what was sent to j
        back = back.numpy()
        rids = rids.numpy()
        parts, cb, ib = [], 0, 0
        for j in range(G):
            c = back[cb:cb + len(dest[j])]
            cb += len(dest[j])
            counts = np.zeros(mr, np.int64)
            counts[dest[j]] = c
            o = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
            parts.append((o, rids[ib:ib + int(c.sum())]))
            ib += int(c.sum())
        return merge_partials(parts) if mr else (np.zeros(1, np.int64), np.zeros(0, np.int64))

    def close(self):
        if self.ctx is not None:
            self.ctx.close()
