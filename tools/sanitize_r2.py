"""Small ticks over every round-2 device path, for `compute-sanitizer --tool memcheck`
(and racecheck / synccheck): keyed lists (shuffled ids, two ticks so the key kernels run),
the bulk-copy join on single- and multi-tile leaves, the warp merge of many-run lists, and
the sharded data plane over the in-process transport (3 ranks on one device).

    compute-sanitizer --tool memcheck python tools/sanitize_r2.py
"""
import sys
import threading

import numpy as np

sys.path.insert(0, ".")
from oracle import quad_oracle as qo  # noqa: E402
from paper_1411_3212_b200 import _native  # noqa: E402


def tick(seed, n, m, side, hot=True):
    rng = np.random.default_rng(seed)
    if hot:
        c = rng.uniform(0, 1000, (4, 2))
        pick = rng.integers(0, 4, n)
        xs = np.clip(c[pick, 0] + rng.normal(0, 30, n), 0, 1000)
        ys = np.clip(c[pick, 1] + rng.normal(0, 30, n), 0, 1000)
        xs[: n // 10] = 500.0  # co-located block: a multi-tile leaf at l_max
        ys[: n // 10] = 500.0
    else:
        xs, ys = rng.uniform(0, 1000, n), rng.uniform(0, 1000, n)
    rows = rng.integers(0, n, m)
    h = rng.uniform(side[0], side[1], m) / 2
    return xs, ys, xs[rows] - h, ys[rows] - h, xs[rows] + h, ys[rows] + h


def check(res_offs, res_ids, ids, xs, ys, rect, th):
    ref = qo.run_tick(ids, xs, ys, np.arange(len(rect[0])), *rect, th_quad=th)
    ok = np.array_equal(res_offs, ref.offsets) and np.array_equal(res_ids, ref.result_ids)
    print("match", ok, "results", len(res_ids))
    return ok


def main():
    ok = True
    n, m = 40_000, 3_000
    xs, ys, *rect = tick(1, n, m, (5.0, 120.0))
    rng = np.random.default_rng(2)
    for th in (16, 384):
        ctx = _native.NativeContext(th, 12, True)
        for t in range(2):  # tick 1 runs the keyed-list kernels
            ids = rng.permutation(n).astype(np.int64) * 5 + 3
            offs, res, st = ctx.tick_host(ids, xs, ys, np.arange(m), *rect)
            ok &= check(offs, res, ids, xs, ys, rect, th)
        ctx.close()
    # sharded: 3 ranks, in-process transport
    ids = np.arange(n, dtype=np.int64)
    G = 3
    group = _native.LocalGroup(G)
    ctxs = [_native.NativeContext(64, 12, True) for _ in range(G)]
    for r, cx in enumerate(ctxs):
        cx.comm_init_local(group, r)
    ob = [r * n // G for r in range(G + 1)]
    qb = [r * m // G for r in range(G + 1)]
    outs = [None] * G

    def work(r):
        sl = (ids[ob[r]:ob[r + 1]], xs[ob[r]:ob[r + 1]], ys[ob[r]:ob[r + 1]],
              *(a[qb[r]:qb[r + 1]] for a in rect))
        outs[r] = ctxs[r].tick_sharded_host(*sl)

    ths = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    for t_ in ths:
        t_.start()
    for t_ in ths:
        t_.join()
    offs = [np.zeros(1, np.int64)]
    res = []
    base = 0
    for o, i, _ in outs:
        offs.append(np.asarray(o[1:], np.int64) + base)
        res.append(np.asarray(i, np.int64))
        base += int(o[-1])
    ok &= check(np.concatenate(offs), np.concatenate(res), ids, xs, ys, rect, 64)
    for cx in ctxs:
        cx.close()
    group.close()
    print("ALL OK" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
