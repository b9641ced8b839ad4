"""GPU: the multi-GPU data plane (tj_tick_sharded) end to end.

Every rank passes only its slice of the tick's objects and queries and gets
back the complete result lists of its own queries: gather of the slices,
the tick on the rank's Morton range of leaves, all-to-all of the partial
lists to the queries' home ranks, device merge.  With the in-process
transport (tj_comm_init_local) G contexts on one B200, driven from one
thread each, run the whole protocol; NCCL (tj_comm_init) runs with one rank
(this pool has one GPU per box).  Concatenating the ranks' outputs must give
the unsharded tick's CSR bit for bit.
"""

from __future__ import annotations

import threading

import numpy as np
import pytest

from oracle import quad_oracle as qo

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def native():
    from paper_1411_3212_b200 import _native

    assert _native.device_count() > 0, "no CUDA device: the GPU tests need a B200"
    return _native


def _tick(seed, n=40_000, m=6_000, side=(2.0, 60.0), shuffle_ids=False, hot=True):
    rng = np.random.default_rng(seed)
    if hot:
        c = rng.uniform(0, 1000, (6, 2))
        pick = rng.integers(0, 6, n)
        xs = np.clip(c[pick, 0] + rng.normal(0, 40, n), 0, 1000)
        ys = np.clip(c[pick, 1] + rng.normal(0, 40, n), 0, 1000)
    else:
        xs, ys = rng.uniform(0, 1000, n), rng.uniform(0, 1000, n)
    ids = rng.permutation(n).astype(np.int64) * 3 + 7 if shuffle_ids else np.arange(n, dtype=np.int64)
    rows = rng.integers(0, n, m)
    h = rng.uniform(side[0], side[1], m) / 2
    cx, cy = xs[rows], ys[rows]
    return ids, xs, ys, cx - h, cy - h, cx + h, cy + h


def _cuts(total, G, rng):
    """Uneven slice boundaries (one slice may be empty)."""
    cuts = np.sort(rng.integers(0, total + 1, G - 1))
    return np.concatenate([[0], cuts, [total]]).astype(np.int64)


def _run_local(native, tick, G, th=64, seed=0, ids32=False, device_inputs=False):
    ids, xs, ys, qxa, qya, qxb, qyb = tick
    rng = np.random.default_rng(seed)
    oc, qc = _cuts(len(ids), G, rng), _cuts(len(qxa), G, rng)
    group = native.LocalGroup(G)
    ctxs = [native.NativeContext(th, 12, True) for _ in range(G)]
    for r, cx in enumerate(ctxs):
        cx.comm_init_local(group, r)
    outs, errs = [None] * G, []

    def worker(r):
        try:
            o0, o1, q0, q1 = oc[r], oc[r + 1], qc[r], qc[r + 1]
            sl = (ids[o0:o1], xs[o0:o1], ys[o0:o1], qxa[q0:q1], qya[q0:q1], qxb[q0:q1], qyb[q0:q1])
            if device_inputs:
                import torch

                t = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in sl]
                torch.cuda.synchronize()
                tout, st = ctxs[r].tick_sharded_ptrs(int(o1 - o0), *(x.data_ptr() if x.numel() else 0 for x in t[:3]),
                                                     int(q1 - q0), *(x.data_ptr() if x.numel() else 0 for x in t[3:]),
                                                     native.TJ_MEM_DEVICE, native.TJ_MEM_HOST)
                import ctypes

                mq = tout.n_q
                offs = np.ctypeslib.as_array(ctypes.cast(tout.offsets, ctypes.POINTER(ctypes.c_int64)),
                                             shape=(mq + 1,)).copy()
                res = (np.ctypeslib.as_array(ctypes.cast(tout.ids, ctypes.POINTER(ctypes.c_int64)),
                                             shape=(tout.n_results,)).copy() if tout.n_results else np.zeros(0, np.int64))
                outs[r] = (offs, res, st)
            else:
                outs[r] = ctxs[r].tick_sharded_host(*sl, ids32=ids32)
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append((r, repr(e)))

    th_ = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for t in th_:
        t.start()
    for t in th_:
        t.join(timeout=600)
    for cx in ctxs:
        cx.close()
    group.close()
    assert not errs, errs
    return outs, oc, qc


def _concat(outs):
    offs, ids, base = [np.zeros(1, np.int64)], [], 0
    for o, i, _ in outs:
        offs.append(np.asarray(o[1:], np.int64) + base)
        ids.append(np.asarray(i, np.int64))
        base += int(o[-1])
    return np.concatenate(offs), np.concatenate(ids) if ids else np.zeros(0, np.int64)


@pytest.mark.parametrize("G", [2, 3, 4])
def test_local_group_equals_unsharded_tick(native, G):
    tick = _tick(100 + G)
    full = native.NativeContext(64, 12, True)
    f_offs, f_ids, _ = full.tick_host(tick[0], tick[1], tick[2], np.arange(len(tick[3])), *tick[3:])
    full.close()
    outs, _, qc = _run_local(native, tick, G, seed=G)
    offs, ids = _concat(outs)
    assert np.array_equal(offs, f_offs) and np.array_equal(ids, f_ids)
    # every rank did part of the join (leaf ranges are balanced by object count)
    assert all(int(st.containment_tests) > 0 for _, _, st in outs)


def test_local_group_device_inputs_and_oracle(native):
    tick = _tick(7, n=20_000, m=3_000)
    ref = qo.run_tick(tick[0], tick[1], tick[2], np.arange(len(tick[3])), *tick[3:], th_quad=64)
    outs, _, _ = _run_local(native, tick, 3, seed=11, device_inputs=True)
    offs, ids = _concat(outs)
    assert np.array_equal(offs, ref.offsets) and np.array_equal(ids, ref.result_ids)


def test_local_group_keyed_ids_and_int32_delivery(native):
    """Shuffled ids (keyed lists on the later ticks of each context), int32 delivery."""
    tick = _tick(9, shuffle_ids=True)
    ref = qo.run_tick(tick[0], tick[1], tick[2], np.arange(len(tick[3])), *tick[3:], th_quad=64)
    outs, _, _ = _run_local(native, tick, 2, seed=5, ids32=True)
    offs, ids = _concat(outs)
    assert np.array_equal(offs, ref.offsets) and np.array_equal(ids, ref.result_ids)


def test_local_group_big_windows_many_ranks_per_query(native):
    """Large windows: most queries have partial lists on several ranks (the head merge)."""
    tick = _tick(13, n=30_000, m=1_500, side=(150.0, 400.0), hot=False)
    full = native.NativeContext(32, 12, True)
    f_offs, f_ids, _ = full.tick_host(tick[0], tick[1], tick[2], np.arange(len(tick[3])), *tick[3:])
    full.close()
    outs, _, _ = _run_local(native, tick, 4, th=32, seed=2)
    offs, ids = _concat(outs)
    assert np.array_equal(offs, f_offs) and np.array_equal(ids, f_ids)


def test_local_group_repeated_ticks(native):
    """Several ticks through the same three contexts (graphs replayed, routing per tick, capacity
    replays of single ranks) keep matching the unsharded tick."""
    G = 3
    group = native.LocalGroup(G)
    ctxs = [native.NativeContext(64, 12, True) for _ in range(G)]
    for r, cx in enumerate(ctxs):
        cx.comm_init_local(group, r)
    full = native.NativeContext(64, 12, True)
    for t, side in enumerate([(2.0, 40.0), (2.0, 40.0), (50.0, 250.0), (2.0, 40.0)]):
        tick = _tick(300 + t, n=30_000, m=2_500, side=side)
        ids, xs, ys, qxa, qya, qxb, qyb = tick
        f_offs, f_ids, _ = full.tick_host(ids, xs, ys, np.arange(len(qxa)), qxa, qya, qxb, qyb)
        rng = np.random.default_rng(t)
        oc, qc = _cuts(len(ids), G, rng), _cuts(len(qxa), G, rng)
        outs, errs = [None] * G, []

        def worker(r):
            try:
                o0, o1, q0, q1 = oc[r], oc[r + 1], qc[r], qc[r + 1]
                outs[r] = ctxs[r].tick_sharded_host(ids[o0:o1], xs[o0:o1], ys[o0:o1], qxa[q0:q1], qya[q0:q1],
                                                    qxb[q0:q1], qyb[q0:q1])
            except Exception as e:  # pragma: no cover
                errs.append((r, repr(e)))

        ths = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
        for x in ths:
            x.start()
        for x in ths:
            x.join(timeout=600)
        assert not errs, errs
        offs, res = _concat(outs)
        assert np.array_equal(offs, f_offs) and np.array_equal(res, f_ids), t
    for cx in ctxs:
        cx.close()
    full.close()
    group.close()


def test_nccl_one_rank_equals_tick(native):
    tick = _tick(21)
    full = native.NativeContext(64, 12, True)
    f_offs, f_ids, _ = full.tick_host(tick[0], tick[1], tick[2], np.arange(len(tick[3])), *tick[3:])
    full.close()
    uid = native.nccl_unique_id()
    ctx = native.NativeContext(64, 12, True)
    ctx.comm_init(uid, 0, 1)
    for _ in range(2):
        offs, ids, _ = ctx.tick_sharded_host(*tick)
        assert np.array_equal(offs, f_offs) and np.array_equal(ids, f_ids)
    ctx.close()
