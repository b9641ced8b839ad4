"""GPU parity for object ids that do not increase in input order.

The reference sorts every per-query list by id (decode.py:117, np.sort in
merge_results).  The device has three ways to get there (tj_stats.id_order):
"monotone" (ids are the rows: runs merge by row), "keyed" (a context that saw
ids other than the rows puts every leaf block in id order and merges runs of
32-bit id offsets) and "sorted" (per-list sorts: the first such tick of a
context, duplicate ids, or an id range of 2^28 or more).  Every one of them must give the oracle's lists, and the
reference-order introspection must not see the device's id-ordered blocks.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_small_cases
from oracle import quad_oracle as qo

pytestmark = pytest.mark.gpu

CASES = load_small_cases()


@pytest.fixture(scope="module")
def pkg():
    import paper_1411_3212_b200 as p
    from paper_1411_3212_b200 import _native

    assert _native.device_count() > 0, "no CUDA device: the GPU tests need a B200"
    return p


def _engine(pkg, th=384, l_max=12, covering=True, **kw):
    return pkg.Engine(pkg.MethodConfig(method="quad", th_quad=th, l_max=l_max, covering_optimization=covering,
                                       **kw))


def _tick(rng, n, m, side=(1.0, 110.0), lo=0.0, hi=1000.0):
    xs = rng.uniform(lo, hi, n)
    ys = rng.uniform(lo, hi, n)
    cx = rng.uniform(lo, hi, m)
    cy = rng.uniform(lo, hi, m)
    h = rng.uniform(side[0], side[1], m) / 2
    return xs, ys, cx - h, cy - h, cx + h, cy + h


def _check(res, ref):
    assert np.array_equal(res.offsets, ref.offsets)
    assert np.array_equal(res.ids, ref.result_ids)


@pytest.mark.parametrize("th", [16, 64])
def test_shuffled_ids_keyed_every_list_shape(pkg, th):
    """A permutation of arange(n) over three ticks of one context: the first is
    sorted per list, the later ones keyed; every merge path of the decode
    (lane merge, warp bitonic, rank merge, oversized lists, > 32 runs) sees
    id-ordered runs of offsets."""
    rng = np.random.default_rng(101 + th)
    n, m = 200_000, 4000
    eng = _engine(pkg, th=th)
    orders = []
    for t in range(3):
        xs, ys, a, b, c, d = _tick(rng, n, m)
        ids = rng.permutation(n).astype(np.int64)
        qids = np.arange(m, dtype=np.int64)
        res, st = eng.process_columns(ids, xs, ys, qids, a, b, c, d)
        _check(res, qo.run_tick(ids, xs, ys, qids, a, b, c, d, th_quad=th))
        orders.append(st.id_order)
    assert orders == ["sorted", "keyed", "keyed"]
    eng.close()


def test_id_kinds_switch_within_one_context(pkg):
    """Ids far from zero (range < 2^28) are keyed, arange ids merge by row,
    increasing non-row ids are keyed without block sorts, and a range of 2^28
    or more falls back to per-list sorts — all in one context."""
    rng = np.random.default_rng(7)
    n, m = 50_000, 5000
    eng = _engine(pkg, th=32)
    base = np.int64(-(2**62))
    plan = [("shuffled", "sorted"), ("shuffled", "keyed"), ("arange", "monotone"), ("shuffled", "sorted"),
            ("increasing", "keyed"), ("wide", "sorted"), ("shuffled", "sorted"), ("shuffled", "keyed")]
    for t, (kind, want) in enumerate(plan):
        xs, ys, a, b, c, d = _tick(rng, n, m, side=(5.0, 60.0))
        if kind == "shuffled":
            ids = base + rng.permutation(3 * n)[:n].astype(np.int64) * 1000
        elif kind == "increasing":
            ids = base + np.arange(n, dtype=np.int64) * 7
        elif kind == "wide":
            ids = rng.permutation(n).astype(np.int64) * 6000  # range 3e8 > 2^28
        else:
            ids = np.arange(n, dtype=np.int64)
        qids = rng.permutation(m).astype(np.int64)
        res, st = eng.process_columns(ids, xs, ys, qids, a, b, c, d)
        _check(res, qo.run_tick(ids, xs, ys, qids, a, b, c, d, th_quad=32))
        assert st.id_order == want, (t, kind, st.id_order)
    eng.close()


def test_keyed_big_leaf_blocks(pkg):
    """Co-located objects make leaf blocks of 600, 3000 and 5000 objects at
    l_max: the id order comes from the counting sort before the leaf sort, so
    block size does not matter."""
    rng = np.random.default_rng(19)
    for big, want in ((600, "keyed"), (3000, "keyed"), (5000, "keyed")):
        n = 20_000
        xs = np.concatenate([rng.uniform(0, 1000, n - big), np.full(big, 321.0)])
        ys = np.concatenate([rng.uniform(0, 1000, n - big), np.full(big, 654.0)])
        m = 2000
        cx = np.concatenate([rng.uniform(0, 1000, m - 50), np.full(50, 321.0)])
        cy = np.concatenate([rng.uniform(0, 1000, m - 50), np.full(50, 654.0)])
        h = rng.uniform(1, 20, m) / 2
        qids = np.arange(m, dtype=np.int64)
        eng = _engine(pkg, th=64)
        for t in range(2):
            ids = rng.permutation(n).astype(np.int64) + 5
            res, st = eng.process_columns(ids, xs, ys, qids, cx - h, cy - h, cx + h, cy + h)
            _check(res, qo.run_tick(ids, xs, ys, qids, cx - h, cy - h, cx + h, cy + h, th_quad=64))
            assert st.id_order == ("sorted" if t == 0 else want), (big, t)
        eng.close()


def test_wide_id_range_sorts_per_list(pkg):
    """An id range of 2^28 or more does not fit the keyed offsets: lists are sorted per query."""
    rng = np.random.default_rng(9)
    n, m = 30_000, 3000
    eng = _engine(pkg, th=32)
    for t in range(3):
        xs, ys, a, b, c, d = _tick(rng, n, m, side=(5.0, 80.0))
        ids = rng.choice(np.int64(2**50), n, replace=False).astype(np.int64) - np.int64(2**49)
        qids = np.arange(m, dtype=np.int64)
        res, st = eng.process_columns(ids, xs, ys, qids, a, b, c, d)
        _check(res, qo.run_tick(ids, xs, ys, qids, a, b, c, d, th_quad=32))
        assert st.id_order == "sorted"
    eng.close()


def test_duplicate_ids_raise_in_every_mode(pkg):
    """Two objects with one id inside one query: DuplicateResult (merge_results),
    on the sorted first tick, on the next (keyed lists requested, declined by the
    presence check) and on the one after (keyed lists no longer requested)."""
    from paper_1411_3212_b200.errors import DuplicateResult

    rng = np.random.default_rng(13)
    n = 4000
    eng = _engine(pkg, th=8)
    for t in range(3):
        xs = rng.uniform(0, 100, n)
        ys = rng.uniform(0, 100, n)
        ids = rng.permutation(n).astype(np.int64)
        ids[5] = ids[6]
        xs[6], ys[6] = xs[5] + 1e-3, ys[5]
        qids = np.array([0, 1], dtype=np.int64)
        a = np.array([xs[5] - 0.5, 10.0])
        b = np.array([ys[5] - 0.5, 10.0])
        c = np.array([xs[5] + 0.5, 20.0])
        d = np.array([ys[5] + 0.5, 20.0])
        with pytest.raises(DuplicateResult):
            res, _ = eng.process_columns(ids, xs, ys, qids, a, b, c, d)
            res.to_result_set()
    eng.close()


@pytest.mark.parametrize("case", CASES[:8], ids=[c.name for c in CASES[:8]])
def test_keyed_introspection_in_reference_order(pkg, case):
    """Keyed lists keep each leaf's objects in id order on the device; the
    directory's object rows and the per-task bitmap words still come back in
    the reference's order (directory.py:128, bitmap.py:89-111), and the lists
    equal the fixtures' with the ids mapped."""
    ids0, xs, ys, qids, qxa, qya, qxb, qyb = case.inputs()
    n = len(ids0)
    if n < 2:
        pytest.skip("needs two objects to shuffle")
    rng = np.random.default_rng(n)
    pid = rng.permutation(n).astype(np.int64) * 3 + 11  # object row r gets id pid[r]
    eng = _engine(pkg, case.th_quad, case.l_max, case.covering)
    for t in range(2):  # tick 0 sorts per list, tick 1 is keyed
        res, st = eng.process_columns(pid, xs, ys, qids, qxa, qya, qxb, qyb)
        ctx = eng.native
        rows, isq, covl = ctx.directory(n)
        assert np.array_equal(rows, case.dir_obj_order)
        bm = ctx.bitmaps()
        assert np.array_equal(bm["words"], case.task_words)
        assert np.array_equal(bm["counts"], case.task_counts)
        # fixture lists hold the fixture's ids (ids0[row]); map them to pid and re-sort per list
        row_of = {int(v): r for r, v in enumerate(ids0)}
        want = np.array([pid[row_of[int(v)]] for v in case.res_ids], dtype=np.int64)
        for q in range(len(case.res_off) - 1):
            want[case.res_off[q]:case.res_off[q + 1]].sort()
        assert np.array_equal(res.offsets, case.res_off)
        assert np.array_equal(res.ids, want)
        if t == 1:
            assert st.id_order == "keyed"
    eng.close()
