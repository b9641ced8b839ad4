"""Checks of a result CSR held in torch tensors (device or CPU) — test helpers.

`device_summary` returns every query's result count and its digest
sum(mix64(id)) mod 2^64, the function oracle/bf_join.c computes per query, and
asserts the canonical order (every list strictly ascending, hence
duplicate-free).  Chunked, so a 2e9-result tick fits in device memory.
"""

from __future__ import annotations

import numpy as np

_C1 = 0xBF58476D1CE4E5B9 - (1 << 64)
_C2 = 0x94D049BB133111EB - (1 << 64)


def _lsr(z, s):
    return (z >> s) & ((1 << (64 - s)) - 1)


def mix64_t(z):
    """splitmix64 finaliser on int64 tensors (wrapping arithmetic) = bf_join.c bf_mix64."""
    z = z ^ _lsr(z, 30)
    z = z * _C1
    z = z ^ _lsr(z, 27)
    z = z * _C2
    return z ^ _lsr(z, 31)


def device_summary(torch, off, ids, chunk=1 << 27):
    m = off.numel() - 1
    R = ids.numel()
    dev = off.device
    assert int(off[0]) == 0 and int(off[-1]) == R, "CSR offsets do not span the ids"
    lens = off[1:] - off[:-1]
    assert bool((lens >= 0).all()), "CSR offsets decrease"
    dig = torch.zeros(m, dtype=torch.int64, device=dev)
    for p0 in range(0, R, chunk):
        p1 = min(R, p0 + chunk)
        pos = torch.arange(p0, p1, dtype=torch.int64, device=dev)
        q = torch.searchsorted(off, pos, right=True) - 1
        dig.index_add_(0, q, mix64_t(ids[p0:p1]))
        # strictly ascending inside a list: ids[p] < ids[p+1] unless p+1 starts another list
        e = min(R, p1 + 1)
        k = e - 1 - p0
        if k > 0:
            d = ids[p0 + 1:e] - ids[p0:e - 1]
            qn = torch.searchsorted(off, pos[:k] + 1, right=True) - 1
            same = qn == q[:k]
            assert not bool(((d <= 0) & same).any()), "a list is not strictly ascending (order or duplicate)"
        del pos, q
    return lens.cpu().numpy(), dig.cpu().numpy().view(np.uint64)
