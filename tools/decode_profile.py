#!/usr/bin/env python
"""Distribution of per-query (runs k, results cnt) and the decode merge path each query takes.

  python tools/decode_profile.py B C5 C20      (GPU box; one tick per workload)
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_1411_3212_b200 import _native  # noqa: E402


def path_of(k, cnt):
    p = np.full(len(k), "copy", dtype=object)
    multi = (k > 1) & (cnt > 1)
    p[multi & (k <= 4) & (cnt <= 128)] = "lane"
    p[multi & ~((k <= 4) & (cnt <= 128)) & (cnt <= 256) & (k >= 3)] = "pair"
    p[multi & ~((k <= 4) & (cnt <= 128)) & ~((cnt <= 256) & (k >= 3))] = "rank"
    p[multi & (cnt > 1024) & (k <= 32)] = "rank_global"
    p[multi & (k > 32)] = "big"
    return p


def main():
    for name in sys.argv[1:] or ["C5"]:
        t = bench.gen_ticks(name, 1)[0]
        ctx = _native.NativeContext(384, 12, True, 0, 0)
        offs, res, st = ctx.tick_host(t.ids, t.xs, t.ys, t.qids, t.qxa, t.qya, t.qxb, t.qyb)
        q, cell, cov = ctx.subqueries()
        m = len(offs) - 1
        k = np.bincount(q, minlength=m)
        cnt = np.diff(offs)
        print(f"== {name}: m={m} results={len(res)} mean cnt {cnt.mean():.1f} mean k {k.mean():.2f}")
        kb = [1, 2, 4, 8, 16, 32, 1 << 30]
        cb = [1, 32, 128, 256, 1024, 4096, 1 << 40]
        print("k\\cnt      " + " ".join(f"<={c:<12}" for c in cb))
        lo = 0
        for kh in kb:
            row = []
            sel_k = (k > lo) & (k <= kh)
            clo = -1
            for ch in cb:
                sel = sel_k & (cnt > clo) & (cnt <= ch)
                row.append(f"{sel.sum():>6}/{cnt[sel].sum():<7}")
                clo = ch
            print(f"{lo + 1:>3}-{kh:<6} " + " ".join(row))
            lo = kh
        p = path_of(k, cnt)
        for name_p in ["copy", "lane", "pair", "rank", "rank_global", "big"]:
            sel = p == name_p
            print(f"  {name_p:12s} queries {sel.sum():>9}  results {cnt[sel].sum():>11}  "
                  f"({cnt[sel].sum() / max(len(res), 1):.1%})  mean k {k[sel].mean() if sel.any() else 0:.1f}")
        ctx.close()


if __name__ == "__main__":
    main()
