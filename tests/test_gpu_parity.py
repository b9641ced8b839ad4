"""GPU parity: the native tick (through the C ABI) against the reference.

Every test here runs the CUDA path on a B200 and compares with
(a) reference-generated fixtures (tests/golden/, made by running the
reference itself), (b) the pinned CPU oracle (oracle/quad_oracle.py) on the
same seeded inputs, and (c) size-independent properties at full scale.
Bit-exact throughout: integers / ids compare with array_equal.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_small_cases, workload_from_json
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


def _check_vs_oracle(res, ref):
    assert np.array_equal(res.offsets, ref.offsets)
    assert np.array_equal(res.ids, ref.result_ids)


# ---------------------------------------------------------------- fixtures --

@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_small_case_all_intermediates(pkg, case):
    eng = _engine(pkg, case.th_quad, case.l_max, case.covering)
    ids, xs, ys, qids, qxa, qya, qxb, qyb = case.inputs()
    res, st = eng.process_columns(ids, xs, ys, qids, qxa, qya, qxb, qyb)
    # final per-query results (ResultSet.by_query as CSR)
    assert np.array_equal(res.offsets, case.res_off)
    assert np.array_equal(res.ids, case.res_ids)
    ctx = eng.native
    # index: quadtree.py:74-158
    ix = ctx.index()
    assert tuple(ix["mbr"]) == tuple(case.mbr.tolist())
    assert ix["l_deep"] == int(case.l_deep)
    assert np.array_equal(ix["leaves"], case.leaves)
    assert np.array_equal(ix["zmap"], case.zmap)
    assert np.array_equal(ctx.object_cells(len(ids)), case.obj_cell)
    # subqueries: quadtree.py:168-240 (query rows, packed leaf, covering)
    q, cell, cov = ctx.subqueries()
    assert np.array_equal(q, case.sq_qrow)
    assert np.array_equal(cell, case.sq_cell)
    assert np.array_equal(cov.astype(np.uint8), case.sq_cov)
    # directory: directory.py:119-158
    rows, isq, covl = ctx.directory(len(ids))
    assert np.array_equal(rows, case.dir_obj_order)
    assert np.array_equal(qids[q[isq]], case.dir_isq_qid)
    assert np.array_equal(cell[isq], case.dir_isq_cell)
    assert np.array_equal(qids[q[covl]], case.dir_cov_qid)
    assert np.array_equal(cell[covl], case.dir_cov_cell)
    # bitmaps + popcounts: bitmap.py:70-119
    bm = ctx.bitmaps()
    assert np.array_equal(bm["cell"], case.task_cell)
    assert np.array_equal(bm["nobj"], case.task_nobj)
    assert np.array_equal(bm["nisq"], case.task_nisq)
    assert np.array_equal(bm["woff"], case.task_woff)
    assert np.array_equal(bm["words"], case.task_words)
    assert np.array_equal(bm["counts"], case.task_counts)
    # TickStats counters (engine.py:212-258)
    want = case.meta["stats"]
    for k in ("containment_tests", "decoded_bits", "subq_intersecting", "subq_covering", "covering_results",
              "active_cells", "results_total"):
        assert getattr(st, k) == want[k], k
    # NumPy's own reductions over the same per-leaf counts: bit-identical (engine.py:261-267)
    assert st.occupancy_mean == want["occupancy_mean"]
    assert st.occupancy_var == want["occupancy_var"]
    assert st.imbalance == pytest.approx(want["imbalance"], rel=1e-12, abs=1e-15)
    eng.close()


def _digest_run(pkg, run, max_ticks=None):
    cfg = workload_from_json(run["workload"])
    meth = run["method"]
    eng = _engine(pkg, meth["th_quad"], meth["l_max"], meth["covering"])
    for t, tick in enumerate(pkg.iter_ticks(cfg)):
        if max_ticks is not None and t >= max_ticks:
            break
        res, st = eng.process_tick_columnar(tick)
        want = run["ticks"][t]
        assert st.results_total == want["stats"]["results_total"]
        assert st.containment_tests == want["stats"]["containment_tests"]
        assert st.subq_intersecting == want["stats"]["subq_intersecting"]
        assert st.subq_covering == want["stats"]["subq_covering"]
        assert qo.result_digest(tick.qids, res.offsets, res.ids) == want["digest"]
    eng.close()


def test_config_a_all_ticks_match_reference(pkg, digests):
    """Config A (uniform 100K, 10%, 10 ticks): sha256 of the reference's canonical lines."""
    _digest_run(pkg, digests["A"])


def test_skewed_100k_matches_reference(pkg, digests):
    _digest_run(pkg, digests["B100K"])


@pytest.mark.parametrize("k", range(20))
def test_acceptance_c1_family(pkg, digests, k):
    """test_acceptance.py:28-100 workloads, quad, every tick."""
    _digest_run(pkg, digests[f"C1_{k}"])


# ------------------------------------------------------------- edge cases --

def test_zero_objects(pkg):
    eng = _engine(pkg)
    res, st = eng.process_columns(np.zeros(0, np.int64), np.zeros(0), np.zeros(0), np.array([1]),
                                  np.array([0.0]), np.array([0.0]), np.array([1.0]), np.array([1.0]))
    assert res.offsets.tolist() == [0, 0] and len(res.ids) == 0
    assert res.to_result_set().by_query == {1: []} and st.results_total == 0


def test_zero_queries_and_outside_mbr(pkg):
    eng = _engine(pkg)
    res, st = eng.process_columns(np.array([0]), np.array([1.0]), np.array([1.0]), np.zeros(0, np.int64),
                                  np.zeros(0), np.zeros(0), np.zeros(0), np.zeros(0))
    assert res.offsets.tolist() == [0] and st.containment_tests == 0
    # test_engine.py:92-96 query outside the MBR still reported as []
    res, _ = eng.process_columns(np.array([0, 1]), np.array([10.0, 20.0]), np.array([10.0, 20.0]),
                                 np.array([0]), np.array([100.0]), np.array([100.0]), np.array([150.0]),
                                 np.array([150.0]))
    assert res.to_result_set().by_query == {0: []}


def test_object_api_scenario(pkg):
    P, R = pkg.Point, pkg.Rect
    batch = pkg.TickBatch(0, [pkg.MovingObject(1, P(20.0, 20.0)), pkg.MovingObject(2, P(4.0, 4.0)),
                              pkg.MovingObject(3, P(5.0, 5.0))],
                          [pkg.Query(1, R(18, 18, 19, 19)), pkg.Query(2, R(0, 0, 1, 1)), pkg.Query(3, R(3, 3, 7, 7))])
    rs, st = pkg.process_tick(batch, pkg.MethodConfig(method="quad", th_quad=1, l_max=3))
    assert rs.by_query == {1: [], 2: [], 3: [2, 3]}
    assert rs.lines() == ["1:", "2:", "3: 2,3"]


def _rand_tick(rng, n, m, lo=0.0, hi=1000.0, side=(5.0, 80.0)):
    xs = rng.uniform(lo, hi, n)
    ys = rng.uniform(lo, hi, n)
    cx = rng.uniform(lo, hi, m)
    cy = rng.uniform(lo, hi, m)
    h = rng.uniform(side[0], side[1], m) / 2
    return xs, ys, cx - h, cy - h, cx + h, cy + h


def test_non_monotone_ids_sorted_by_id(pkg):
    rng = np.random.default_rng(3)
    n, m = 5000, 800
    xs, ys, a, b, c, d = _rand_tick(rng, n, m)
    ids = rng.permutation(10 * n)[:n].astype(np.int64)  # arbitrary, non-monotone ids
    qids = rng.permutation(m).astype(np.int64)
    eng = _engine(pkg, th=16)
    res, _ = eng.process_columns(ids, xs, ys, qids, a, b, c, d)
    ref = qo.run_tick(ids, xs, ys, qids, a, b, c, d, th_quad=16)
    _check_vs_oracle(res, ref)


def test_duplicate_issuers_merge_like_reference(pkg):
    xs = np.array([1.0, 2.0, 3.0, 8.0])
    ys = np.array([1.0, 2.0, 3.0, 8.0])
    ids = np.arange(4)
    eng = _engine(pkg, th=1, l_max=4)
    # two disjoint queries of issuer 7 are concatenated + sorted (decode.py:102-117)
    res, _ = eng.process_columns(ids, xs, ys, np.array([7, 7]), np.array([7.0, 0.5]), np.array([7.0, 0.5]),
                                 np.array([9.0, 1.5]), np.array([9.0, 1.5]))
    assert res.to_result_set().by_query == {7: [0, 3]}
    res, _ = eng.process_columns(ids, xs, ys, np.array([7, 7]), np.array([0.0, 0.5]), np.array([0.0, 0.5]),
                                 np.array([2.5, 1.5]), np.array([2.5, 1.5]))
    from paper_1411_3212_b200.errors import DuplicateResult

    with pytest.raises(DuplicateResult):
        res.to_result_set()


def test_deep_tree_colocated_and_big_leaves(pkg):
    """l_max leaves above th (quadtree.py:116): multi-tile join and heavy sub-pyramids."""
    rng = np.random.default_rng(11)
    n = 30_000
    xs = np.concatenate([rng.uniform(0, 1000, n - 6000), np.full(3000, 500.0), 500.0 + rng.uniform(0, 1e-6, 3000)])
    ys = np.concatenate([rng.uniform(0, 1000, n - 6000), np.full(3000, 250.0), 250.0 + rng.uniform(0, 1e-6, 3000)])
    m = 3000
    cx = np.concatenate([rng.uniform(0, 1000, m - 200), np.full(200, 500.0)])
    cy = np.concatenate([rng.uniform(0, 1000, m - 200), np.full(200, 250.0)])
    h = np.concatenate([rng.uniform(1, 30, m - 200), rng.uniform(1e-7, 2.0, 200)]) / 2
    ids = np.arange(n, dtype=np.int64)
    qids = np.arange(m, dtype=np.int64)
    for th in (1, 8, 384):
        eng = _engine(pkg, th=th)
        res, st = eng.process_columns(ids, xs, ys, qids, cx - h, cy - h, cx + h, cy + h)
        ref = qo.run_tick(ids, xs, ys, qids, cx - h, cy - h, cx + h, cy + h, th_quad=th)
        _check_vs_oracle(res, ref)
        assert st.l_deep == ref.index.l_deep and st.n_leaves == len(ref.index.leaves)
        ix = eng.native.index()
        assert np.array_equal(ix["leaves"], ref.index.leaves)
        eng.close()


def test_huge_queries_many_subqueries(pkg):
    """Large windows: hundreds of leaves per query, covering-heavy, multi-run merges."""
    rng = np.random.default_rng(5)
    xs, ys, a, b, c, d = _rand_tick(rng, 40_000, 300, side=(100.0, 900.0))
    ids = np.arange(len(xs), dtype=np.int64)
    qids = np.arange(len(a), dtype=np.int64)
    for cov in (True, False):
        eng = _engine(pkg, th=16, covering=cov)
        res, st = eng.process_columns(ids, xs, ys, qids, a, b, c, d)
        ref = qo.run_tick(ids, xs, ys, qids, a, b, c, d, th_quad=16, covering_optimization=cov)
        _check_vs_oracle(res, ref)
        assert st.subq_covering == ref.counters["subq_covering"]
        assert st.containment_tests == ref.counters["containment_tests"]
        eng.close()


@pytest.mark.parametrize("th", [16, 64])
def test_decode_merge_paths_all_list_shapes(pkg, th):
    """Every per-query merge path of the decode kernel: single runs, the lane
    merge (2..4 runs, <= 128 results), the warp bitonic sort (>= 3 runs, up to
    512 results), the warp rank merge (513..1024 results), the oversized-list
    path (> 1024 results, concatenated in global memory) and the CTA sort of
    lists of more than 32 runs."""
    rng = np.random.default_rng(17 + th)
    n, m = 200_000, 4000
    xs, ys, a, b, c, d = _rand_tick(rng, n, m, side=(1.0, 110.0))
    ids = np.arange(n, dtype=np.int64)
    qids = np.arange(m, dtype=np.int64)
    eng = _engine(pkg, th=th)
    res, _ = eng.process_columns(ids, xs, ys, qids, a, b, c, d)
    ref = qo.run_tick(ids, xs, ys, qids, a, b, c, d, th_quad=th)
    _check_vs_oracle(res, ref)
    cnt = np.diff(ref.offsets)
    runs = np.bincount(eng.native.subqueries()[0], minlength=m)
    assert ((runs >= 3) & (cnt > 256) & (cnt <= 512)).any() and ((runs >= 3) & (cnt <= 64) & (cnt > 1)).any()
    assert (cnt > 1024).any() and (runs > 32).any()
    eng.close()


def test_int32_id_delivery(pkg):
    """TJ_OUT_IDS32: the same CSR with int32 ids and offsets; ids beyond int32 fall back to int64."""
    from paper_1411_3212_b200 import _native

    rng = np.random.default_rng(23)
    n, m = 50_000, 5000
    xs, ys, a, b, c, d = _rand_tick(rng, n, m)
    qids = np.arange(m, dtype=np.int64)
    ctx = _native.NativeContext(64, 12, True, 0, 0)
    for ids in (np.arange(n, dtype=np.int64), np.sort(rng.choice(2**31 - 1, n, replace=False)).astype(np.int64),
                np.arange(n, dtype=np.int64) * 50_000):  # the last: ids up to 2.5e9 > 2^31
        o64, r64, _ = ctx.tick_host(ids, xs, ys, qids, a, b, c, d)
        o32, r32, _ = ctx.tick_host(ids, xs, ys, qids, a, b, c, d, ids32=True)
        assert np.array_equal(o64, o32.astype(np.int64)) and np.array_equal(r64, r32.astype(np.int64))
        assert r32.dtype == (np.int64 if ids.max() >= 2**31 else np.int32) and o32.dtype == np.int32
    ctx.close()


def test_covering_toggle_preserves_results(pkg):
    """test_engine.py:100-111 / acceptance C4 semantics."""
    cfg = pkg.WorkloadConfig(n_objects=4000, n_ticks=1, distribution="gaussian", n_hotspots=4, seed=8,
                             query_side=(50.0, 300.0))
    tick = next(pkg.iter_ticks(cfg))
    on = _engine(pkg, th=16, covering=True)
    off = _engine(pkg, th=16, covering=False)
    r_on, s_on = on.process_tick_columnar(tick)
    r_off, s_off = off.process_tick_columnar(tick)
    assert np.array_equal(r_on.ids, r_off.ids) and np.array_equal(r_on.offsets, r_off.offsets)
    assert s_on.subq_covering > 0 and s_off.subq_covering == 0
    assert s_on.containment_tests < s_off.containment_tests


def test_negative_and_degenerate_coordinates(pkg):
    rng = np.random.default_rng(17)
    for trial in range(10):
        n = int(rng.integers(1, 400))
        xs = rng.uniform(-100, 100, n)
        ys = np.full(n, 3.25) if trial % 3 == 0 else rng.uniform(-100, 100, n)
        if trial % 4 == 1:
            xs = np.full(n, -7.5)
        m = int(rng.integers(0, 120))
        cx, cy, hh = rng.uniform(-100, 100, m), rng.uniform(-100, 100, m), rng.uniform(0.5, 60, m)
        ids = np.arange(n, dtype=np.int64)
        qids = np.arange(m, dtype=np.int64)
        th = int(rng.integers(1, 7))
        eng = _engine(pkg, th=th, l_max=6)
        res, _ = eng.process_columns(ids, xs, ys, qids, cx - hh, cy - hh, cx + hh, cy + hh)
        ref = qo.run_tick(ids, xs, ys, qids, cx - hh, cy - hh, cx + hh, cy + hh, th_quad=th, l_max=6)
        _check_vs_oracle(res, ref)
        off, res_b = qo.brute_force(ids, xs, ys, cx - hh, cy - hh, cx + hh, cy + hh)
        assert np.array_equal(res.offsets, off) and np.array_equal(res.ids, res_b)
        eng.close()


def test_every_lmax_level(pkg):
    rng = np.random.default_rng(23)
    xs, ys, a, b, c, d = _rand_tick(rng, 6000, 500, side=(1.0, 40.0))
    xs[:1500] = 123.4 + rng.uniform(0, 0.01, 1500)
    ys[:1500] = 567.8 + rng.uniform(0, 0.01, 1500)
    ids = np.arange(len(xs), dtype=np.int64)
    qids = np.arange(len(a), dtype=np.int64)
    for l_max in range(1, 13):
        eng = _engine(pkg, th=20, l_max=l_max)
        res, st = eng.process_columns(ids, xs, ys, qids, a, b, c, d)
        ref = qo.run_tick(ids, xs, ys, qids, a, b, c, d, th_quad=20, l_max=l_max)
        _check_vs_oracle(res, ref)
        ix = eng.native.index()
        assert ix["l_deep"] == ref.index.l_deep
        assert np.array_equal(ix["zmap"], ref.index.zmap)
        eng.close()


def test_engine_reused_across_growing_ticks(pkg):
    """Capacity growth + replay: one Engine, ticks of increasing size."""
    rng = np.random.default_rng(29)
    eng = _engine(pkg, th=32)
    for n, m, side in ((500, 50, (5.0, 20.0)), (20_000, 20_000, (5.0, 60.0)), (3000, 3000, (200.0, 600.0)),
                       (60_000, 60_000, (20.0, 120.0))):
        xs, ys, a, b, c, d = _rand_tick(rng, n, m, side=side)
        ids = np.arange(n, dtype=np.int64)
        qids = np.arange(m, dtype=np.int64)
        res, _ = eng.process_columns(ids, xs, ys, qids, a, b, c, d)
        ref = qo.run_tick(ids, xs, ys, qids, a, b, c, d, th_quad=32)
        _check_vs_oracle(res, ref)
    eng.close()


def test_config_c_scale_properties(pkg):
    """10M skewed objects at 5u (config C): sampled brute-force + invariants."""
    cfg = pkg.WorkloadConfig(n_objects=10_000_000, n_ticks=1, query_rate=1.0, query_side=5.0,
                             distribution="gaussian", n_hotspots=25, seed=3)
    tick = next(pkg.iter_ticks(cfg))
    eng = _engine(pkg)
    res, st = eng.process_tick_columnar(tick, full_stats=False)
    assert len(res.offsets) == tick.n_queries + 1 and res.offsets[-1] == st.results_total
    # SURVEY.md §8 measured sizes for C @5u, seed 3, tick 0
    assert st.results_total == 169_197_114
    assert st.n_leaves == 60_820 and st.l_deep == 11
    assert st.subq_intersecting == 16_845_566 and st.subq_covering == 0
    lens = np.diff(res.offsets)
    # ascending, duplicate-free per query
    d = np.diff(res.ids)
    bad = np.ones(len(res.ids), bool)
    bad[res.offsets[1:-1] - 1] = False
    assert np.all((d > 0) | ~bad[:-1])
    rng = np.random.default_rng(99)
    sample = rng.choice(tick.n_queries, 40, replace=False)
    hot = np.argsort(lens)[-10:]
    for k in np.concatenate([sample, hot]):
        hit = ((tick.xs >= tick.qxa[k]) & (tick.xs <= tick.qxb[k]) & (tick.ys >= tick.qya[k])
               & (tick.ys <= tick.qyb[k]))
        assert np.array_equal(res.of(k), np.sort(tick.ids[hit]))
    eng.close()


def test_table_join_objects_on_query_edges(pkg):
    """Objects on a lattice whose coordinates coincide with query edges, many
    subqueries per leaf (the bucket-table join path) — every ambiguous bit goes
    through the exact fp64 test; equal to the oracle and to brute force."""
    rng = np.random.default_rng(41)
    g = np.arange(0.0, 64.0, 0.25)
    gx, gy = np.meshgrid(g, g)
    xs = np.concatenate([gx.ravel(), rng.uniform(0, 64, 4000)])
    ys = np.concatenate([gy.ravel(), rng.uniform(0, 64, 4000)])
    n = len(xs)
    m = 6000
    a = rng.choice(g, m)
    b = rng.choice(g, m)
    wx = rng.choice(np.arange(0.25, 6.0, 0.25), m)
    wy = rng.choice(np.arange(0.25, 6.0, 0.25), m)
    qxa, qya, qxb, qyb = a, b, a + wx, b + wy
    ids = np.arange(n, dtype=np.int64)
    qids = np.arange(m, dtype=np.int64)
    for th in (256, 384):
        eng = _engine(pkg, th=th)
        res, st = eng.process_columns(ids, xs, ys, qids, qxa, qya, qxb, qyb)
        ref = qo.run_tick(ids, xs, ys, qids, qxa, qya, qxb, qyb, th_quad=th, keep_tasks=True)
        _check_vs_oracle(res, ref)
        off, res_b = qo.brute_force(ids, xs, ys, qxa, qya, qxb, qyb)
        assert np.array_equal(res.offsets, off) and np.array_equal(res.ids, res_b)
        bm = eng.native.bitmaps()  # per-task words in the reference's row order (bitmap.py:70-119)
        assert np.array_equal(bm["words"], np.concatenate([t[3] for t in ref.tasks]))
        assert np.array_equal(bm["counts"], np.concatenate([t[4] for t in ref.tasks]))
        assert int(bm["nisq"].max()) >= 12  # the table path ran
        eng.close()


def test_graph_replay_equals_direct_launch(pkg, monkeypatch):
    """The tick's captured CUDA graphs replay to the same results as direct
    launches, across ticks with different inputs of the same shape."""
    rng = np.random.default_rng(43)
    ticks = []
    for _ in range(3):
        xs, ys, a, b, c, d = _rand_tick(rng, 40_000, 20_000, side=(5.0, 40.0))
        ticks.append((np.arange(40_000, dtype=np.int64), xs, ys, np.arange(20_000, dtype=np.int64), a, b, c, d))
    eng = _engine(pkg, th=64)
    graphed = [eng.process_columns(*t)[0] for t in ticks + ticks]
    eng.close()
    monkeypatch.setenv("TJ_NO_GRAPH", "1")
    eng = _engine(pkg, th=64)
    direct = [eng.process_columns(*t)[0] for t in ticks]
    eng.close()
    for k, r in enumerate(graphed):
        assert np.array_equal(r.offsets, direct[k % 3].offsets) and np.array_equal(r.ids, direct[k % 3].ids)


def test_extreme_hotspot_big_leaves(pkg):
    """Config-E shape, scaled down: uniform background + one extreme hotspot;
    leaves pinned at l_max hold thousands of objects (multi-tile join units,
    the decode's large-leaf path)."""
    rng = np.random.default_rng(47)
    nu, nh = 200_000, 120_000
    xs = np.concatenate([rng.uniform(0, 22500, nu), rng.normal(11250, 3.0, nh)])
    ys = np.concatenate([rng.uniform(0, 22500, nu), rng.normal(11250, 3.0, nh)])
    n = nu + nh
    m = 30_000
    k = rng.integers(0, n, m)
    side = rng.choice([1.0, 2.0, 8.0], m)
    qxa, qya = xs[k] - side / 2, ys[k] - side / 2
    qxb, qyb = qxa + side, qya + side
    ids = np.arange(n, dtype=np.int64)
    qids = np.arange(m, dtype=np.int64)
    eng = _engine(pkg)
    res, st = eng.process_columns(ids, xs, ys, qids, qxa, qya, qxb, qyb)
    ref = qo.run_tick(ids, xs, ys, qids, qxa, qya, qxb, qyb)
    _check_vs_oracle(res, ref)
    occ = ref.directory.o_end - ref.directory.o_start
    assert occ.max() > 384  # some leaves span several 384-object join tiles
    eng.close()


def _adaptive_runs():
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "adaptive.json")) as fp:
        return json.load(fp)["runs"]


@pytest.mark.parametrize("name", sorted(_adaptive_runs()))
def test_adaptive_rebuild_matches_reference(pkg, name):
    """rebuild="adaptive" (engine.py:163-174, quadtree.py:243-270): per tick the
    device reuses or rebuilds its index exactly when the reference engine does,
    with the same leaves / depth, and returns the reference's results."""
    run = _adaptive_runs()[name]
    cfg = dict(run["config"])
    th = cfg.pop("th_quad")
    if isinstance(cfg.get("query_side"), list):
        cfg["query_side"] = tuple(cfg["query_side"])
    eng = _engine(pkg, th=th, rebuild="adaptive")
    for t, tick in enumerate(pkg.iter_ticks(pkg.WorkloadConfig(**cfg))):
        want = run["ticks"][t]
        res, st = eng.process_tick_columnar(tick)
        assert st.rebuilt == want["rebuilt"], t
        assert st.n_leaves == want["n_leaves"] and st.l_deep == want["l_deep"], t
        assert qo.result_digest(tick.qids, res.offsets, res.ids) == want["digest"], t
    eng.close()


@pytest.mark.parametrize("name", sorted(_adaptive_runs()))
def test_adaptive_reuse_with_non_monotone_ids(pkg, name):
    """Adaptive ticks that reuse the index with ids that are neither arange nor
    increasing: the reused tick must look ids up and sort lists by
    id.  ids' = K - id reverses the order; mapped back, every list equals the
    reference digest, and the rebuild decisions are unchanged."""
    run = _adaptive_runs()[name]
    cfg = dict(run["config"])
    th = cfg.pop("th_quad")
    if isinstance(cfg.get("query_side"), list):
        cfg["query_side"] = tuple(cfg["query_side"])
    K = 10**9
    eng = _engine(pkg, th=th, rebuild="adaptive")
    for t, tick in enumerate(pkg.iter_ticks(pkg.WorkloadConfig(**cfg))):
        want = run["ticks"][t]
        res, st = eng.process_columns(K - tick.ids, tick.xs, tick.ys, tick.qids, tick.qxa, tick.qya, tick.qxb,
                                      tick.qyb)
        assert st.rebuilt == want["rebuilt"], t
        lens = np.diff(res.offsets)
        # ascending by the (reversed) id within every list
        d = np.diff(res.ids)
        inner = np.ones(len(res.ids), bool)
        inner[res.offsets[1:-1] - 1] = False
        assert np.all((d > 0) | ~inner[:-1]), t
        # back to the original ids: each list reversed is ascending again
        orig = (K - res.ids)
        q = np.repeat(np.arange(len(lens)), lens)
        order = np.lexsort((orig, q))
        assert qo.result_digest(tick.qids, res.offsets, orig[order]) == want["digest"], t
    eng.close()


def _d2h(ptr, count, dtype):
    """Copy `count` elements at a raw device pointer to a new NumPy array (cudaMemcpy D2H)."""
    import ctypes

    rt = ctypes.CDLL("libcudart.so.12")
    rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    out = np.empty(count, dtype)
    assert rt.cudaMemcpy(out.ctypes.data, ptr, out.nbytes, 2) == 0  # cudaMemcpyDeviceToHost
    return out


def test_device_pointer_tick_and_compact_device_delivery(pkg):
    """tj_tick with device-resident inputs and outputs (the path bench.py times), in the
    default int64 and the TJ_OUT_IDS32 compact layouts, equals the host-buffer tick."""
    import torch

    from paper_1411_3212_b200 import _native

    rng = np.random.default_rng(31)
    n, m = 60_000, 6000
    xs, ys, a, b, c, d = _rand_tick(rng, n, m)
    ids = np.arange(n, dtype=np.int64)
    qids = np.arange(m, dtype=np.int64)
    ctx = _native.NativeContext(64, 12, True, 0, 0)
    o_ref, r_ref, _ = ctx.tick_host(ids, xs, ys, qids, a, b, c, d)
    dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (ids, xs, ys, qids, a, b, c, d)]
    ptr = [t.data_ptr() for t in dev]
    torch.cuda.synchronize()
    for flag in (0, _native.TJ_OUT_IDS32):
        out, st = ctx.tick_ptrs(n, *ptr[:3], m, *ptr[3:], _native.TJ_MEM_DEVICE, _native.TJ_MEM_DEVICE | flag)
        assert out.mem == _native.TJ_MEM_DEVICE and out.n_results == len(r_ref)
        assert (out.id_bytes, out.offset_bytes) == ((4, 4) if flag else (8, 8))
        offs = _d2h(out.offsets32 if flag else out.offsets, m + 1, np.int32 if flag else np.int64)
        res = _d2h(out.ids32 if flag else out.ids, out.n_results, np.int32 if flag else np.int64)
        assert np.array_equal(offs.astype(np.int64), o_ref) and np.array_equal(res.astype(np.int64), r_ref)
    ctx.close()


@pytest.mark.parametrize("case", CASES[:6], ids=[c.name for c in CASES[:6]])
def test_device_tiling_check_on_reference_cases(pkg, case, monkeypatch):
    """TJ_CHECK_TILING=1 runs the reference's build_zmap TilingGap check (quadtree.py:153-157)
    on the device; real ticks tile the deepest grid, so it passes and changes nothing."""
    monkeypatch.setenv("TJ_CHECK_TILING", "1")
    eng = _engine(pkg, case.th_quad, case.l_max, case.covering)
    res, st = eng.process_columns(*case.inputs())
    assert np.array_equal(res.offsets, case.res_off) and np.array_equal(res.ids, case.res_ids)
    eng.close()
