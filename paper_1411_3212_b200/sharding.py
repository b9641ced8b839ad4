"""Multi-GPU leaf-range sharding of the QUAD tick.

One process per GPU.  Each rank ingests 1/G of the tick's position updates
and queries; an all-gather (NCCL over NVLink on GPUs, gloo on CPU) gives every
rank the full tick; every rank builds the bit-identical index (the index
build is integer-exact), then scatters, joins, decodes and assembles only the
(query, leaf) pairs of its contiguous Morton range of leaves, balanced by the
per-leaf object count (device side: `tj_set_shard`, `k_shard_mark` in
csrc/tj_kernels.cuh, run right after the index build).  A rank's per-query lists are the restriction of the
full lists to its leaves: disjoint across ranks and each sorted, so the
per-query union (merge) is the full result.

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


class ShardedEngine:
    """One rank of a G-GPU QUAD tick (torch.distributed process group already initialised)."""

    def __init__(self, cfg, device: Optional[int] = None, group=None):
        import torch.distributed as dist

        from . import _native

        cfg.validate()
        self.cfg = cfg
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = cfg.device if device is None else device
        self.ctx = _native.NativeContext(cfg.th_quad, cfg.l_max, cfg.covering_optimization, 0, self.device)
        if self.world > 1:
            self.ctx.set_shard(self.rank, self.world)

    def process_shard(self, ids, xs, ys, qids, qxa, qya, qxb, qyb):
        """This rank's share of the tick in (host arrays); the full CSR out on every rank."""
        import torch

        dev = torch.device("cuda", self.device) if torch.cuda.is_available() else torch.device("cpu")
        cols = [torch.as_tensor(np.ascontiguousarray(a)).to(dev) for a in (ids, xs, ys, qids, qxa, qya, qxb, qyb)]
        full = [all_gather_var(c, self.group)[0].cpu().numpy() for c in cols]
        offs, res, st = self.ctx.tick_host(*full)
        counts = torch.as_tensor(np.diff(offs)).to(dev)
        all_counts, _ = all_gather_var(counts, self.group)
        all_ids, sizes = all_gather_var(torch.as_tensor(res).to(dev), self.group)
        m = len(full[3])
        all_counts = all_counts.cpu().numpy().reshape(self.world, m)
        all_ids = all_ids.cpu().numpy()
        parts, base = [], 0
        for r in range(self.world):
            o = np.concatenate([[0], np.cumsum(all_counts[r])]).astype(np.int64)
            parts.append((o, all_ids[base:base + sizes[r]]))
            base += sizes[r]
        return merge_partials(parts), st

    def close(self):
        self.ctx.close()
