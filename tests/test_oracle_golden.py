"""Pin the CPU oracle (oracle/quad_oracle.py) before trusting it.

Two kinds of evidence:
1. the known-answer vectors of the reference's own tests, restated here with
   their file:line in /root/reference/pkg/tests;
2. fixtures produced by running the reference itself (tests/golden/make_golden.py):
   full intermediates for small ticks, and sha256 digests of the canonical
   result lines for config A and the acceptance-C1 workload family.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_small_cases, workload_from_json
from oracle import quad_oracle as qo
from paper_1411_3212_b200.workload import iter_ticks


def pack(level, z, l_max):
    return (level << (2 * l_max)) | z


SEVEN = np.array([(0.5, 0.5), (2.5, 0.5), (3.5, 0.5), (2.5, 1.5), (0.5, 2.5), (1.5, 3.5), (3.5, 3.5)])
MIXED = np.array([(12.0, 12.0), (5.0, 9.0), (7.0, 11.0), (1.0, 1.0), (5.0, 5.0), (9.0, 1.0), (13.0, 5.0)])


# ---- test_morton.py KATs -------------------------------------------------

def test_morton_kats():
    assert int(qo.morton(0, 0)) == 0  # test_morton.py:20-21
    assert int(qo.morton(1, 1)) == 3  # test_morton.py:24-25
    assert int(qo.morton(3, 5)) == 39  # test_morton.py:28-30
    assert int(qo.morton(3, 5)) >> 2 == 9  # truncate one level, test_morton.py:37-38
    i, j = qo.unmorton(np.arange(4096))
    assert np.array_equal(qo.morton(i, j), np.arange(4096))


def test_cell_coords_kats():
    r = (0.0, 0.0, 8.0, 8.0)
    assert [int(v[0]) for v in qo.cell_coords([0.0], [0.0], r, 3)] == [0, 0]  # test_morton.py:50-51
    assert [int(v[0]) for v in qo.cell_coords([8.0], [8.0], r, 3)] == [7, 7]  # :54-55 clamp
    assert [int(v[0]) for v in qo.cell_coords([3.5], [5.1], r, 3)] == [3, 5]  # :58-59 floor
    with pytest.raises(qo.OracleError):
        qo.cell_coords([9.0], [0.0], r, 3)  # :62-63 OutOfBounds


# ---- test_quadtree.py / test_acceptance.py C2 KATs -------------------------

def test_fig6_census_and_trace():
    idx = qo.build_index(SEVEN[:, 0], SEVEN[:, 1], (0.0, 0.0, 4.0, 4.0), 1, 2, record_trace=True)
    lv = idx.leaves >> 4
    assert len(idx.leaves) == 10 and int((lv == 2).sum()) == 8 and idx.l_deep == 2
    assert sorted(idx.leaves[lv == 1].tolist()) == [pack(1, 0, 2), pack(1, 3, 2)]
    # test_quadtree.py:106-126 / test_acceptance.py:103-130
    assert idx.trace == [
        [(1, 0, 0, 1, False), (1, 1, 1, 4, True), (1, 2, 4, 6, True), (1, 3, 6, 7, False)],
        [(2, 4, 1, 2, False), (2, 5, 2, 3, False), (2, 6, 3, 4, False), (2, 7, 4, 4, False),
         (2, 8, 4, 5, False), (2, 9, 5, 5, False), (2, 10, 5, 5, False), (2, 11, 5, 6, False)],
    ]
    # zmap golden, test_quadtree.py:84-92
    want = [pack(1, 0, 2)] * 4 + [pack(2, z, 2) for z in range(4, 12)] + [pack(1, 3, 2)] * 4
    assert idx.zmap.tolist() == want


def test_threshold_empty_colocated():
    idx = qo.build_index(np.array([1.0, 2, 3]), np.array([1.0, 2, 3]), (0, 0, 4, 4), 3, 5)
    assert sorted(idx.leaves.tolist()) == [pack(1, z, 5) for z in range(4)] and idx.l_deep == 1
    idx = qo.build_index(np.full(5, 0.1), np.full(5, 0.1), (0, 0, 8, 8), 1, 3)  # :138-147
    assert idx.l_deep == 3
    cells = qo.map_objects(np.full(5, 0.1), np.full(5, 0.1), idx)
    assert set(cells.tolist()) == {pack(3, 0, 3)}


def test_thirteen_leaf_rank_nine():
    pts = np.array([(9.0, 9.0), (1.0, 9.0), (5.0, 13.0), (1.0, 1.0), (5.0, 5.0), (9.0, 1.0), (13.0, 5.0)])
    idx = qo.build_index(pts[:, 0], pts[:, 1], (0, 0, 16, 16), 1, 2)  # test_quadtree.py:111-121
    assert len(idx.leaves) == 13
    cell = qo.map_objects(pts[:, 0], pts[:, 1], idx)[1]
    assert int(cell) == pack(2, 8, 2) and int(np.searchsorted(idx.leaves, cell)) == 9


def test_seven_subquery_split():
    idx = qo.build_index(MIXED[:, 0], MIXED[:, 1], (0, 0, 16, 16), 1, 3)  # test_quadtree.py:150-161
    assert len(idx.leaves) == 16
    sq = qo.split_queries(np.array([3.5]), np.array([7.5]), np.array([6.5]), np.array([10.5]), idx)
    assert len(sq.cell) == 7 and int(sq.covering.sum()) == 1
    assert int(sq.cell[sq.covering][0]) == pack(3, 36, 3)
    # coarse-leaf dedupe, test_quadtree.py:163-170
    idx7 = qo.build_index(SEVEN[:, 0], SEVEN[:, 1], (0, 0, 4, 4), 1, 2)
    sq = qo.split_queries(np.array([2.2]), np.array([2.2]), np.array([3.8]), np.array([3.8]), idx7)
    assert sq.cell.tolist() == [pack(1, 3, 2)] and not sq.covering[0]


# ---- test_bitmap.py / test_decode.py KATs ---------------------------------

def _words(points, rects):
    p = np.asarray(points, float)
    r = np.asarray(rects, float).reshape(-1, 4)
    return qo.cell_bitmap(p[:, 0], p[:, 1], r[:, 0], r[:, 1], r[:, 2], r[:, 3])


def test_bitmap_kats():
    assert _words([(0.5, 0.5)], [(0, 0, 1, 1)]).tolist() == [1]  # test_bitmap.py:24-26
    assert _words([(0.5, 0.5)] * 33, [(0, 0, 1, 1)]).tolist() == [0xFFFFFFFF, 1]  # :29-31
    lin = _words([(0.5, 0.5)] * 40, [(0, 0, 1, 1), (2, 2, 3, 3)])
    assert qo.interlace(lin, 2).tolist() == [0xFFFFFFFF, 0, 0xFF, 0]  # :34-39
    assert _words([(0.5, 0.5)] * 5, [(0, 0, 1, 1)]).tolist() == [0b11111]  # :52-54
    lin = _words([(0, 0), (1, 1), (2, 2)], [(0, 0, 2, 2), (9, 9, 10, 10), (1, 1, 2, 2)])
    assert qo.word_popcounts(lin, 3).tolist() == [3, 0, 2]  # :93-99
    # transpose formula [A,B,C,D] -> [A,C,B,D], :62-70 (interlace is its inverse)
    assert qo.interlace(np.array([0xA, 0xC, 0xB, 0xD], np.uint32), 2).tolist() == [0xA, 0xB, 0xC, 0xD]


def test_decode_33_in_block_order():
    xs = np.arange(33, dtype=float)  # test_decode.py:58-66
    w = qo.cell_bitmap(xs, np.zeros(33), np.array([0.0]), np.array([0.0]), np.array([40.0]), np.array([0.0]))
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")[:33]
    assert (np.arange(1000, 1033)[np.flatnonzero(bits)]).tolist() == list(range(1000, 1033))


def test_scenario_and_cli_golden():
    # conftest.py:53-67, test_acceptance.py:133-140, test_cli.py:9-22
    ids = np.array([1, 2, 3])
    xs = np.array([20.0, 4.0, 5.0])
    ys = np.array([20.0, 4.0, 5.0])
    qids = np.array([1, 2, 3])
    qa = np.array([[18.0, 18, 19, 19], [0, 0, 1, 1], [3, 3, 7, 7]])
    t = qo.run_tick(ids, xs, ys, qids, *qa.T, th_quad=1, l_max=3)
    assert qo.canonical_lines(qids, t.offsets, t.result_ids) == ["1:", "2:", "3: 2,3"]


# ---- reference-generated fixtures -----------------------------------------

CASES = load_small_cases()


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_oracle_matches_reference_intermediates(case):
    ids, xs, ys, qids, qxa, qya, qxb, qyb = case.inputs()
    t = qo.run_tick(ids, xs, ys, qids, qxa, qya, qxb, qyb, th_quad=case.th_quad, l_max=case.l_max,
                    covering_optimization=case.covering, keep_tasks=True)
    assert tuple(t.index.mbr) == tuple(case.mbr.tolist())
    assert t.index.l_deep == int(case.l_deep)
    assert np.array_equal(t.index.leaves, case.leaves)
    assert np.array_equal(t.index.zmap, case.zmap)
    assert np.array_equal(t.obj_cell, case.obj_cell)
    kept = np.flatnonzero(t.keep)
    assert np.array_equal(kept[t.sub.qrow], case.sq_qrow)
    assert np.array_equal(t.sub.cell, case.sq_cell)
    assert np.array_equal(t.sub.covering.astype(np.uint8), case.sq_cov)
    assert np.array_equal(t.directory.obj_order, case.dir_obj_order)
    assert np.array_equal(qids[kept[t.sub.qrow[t.directory.isq_idx]]], case.dir_isq_qid)
    assert np.array_equal(t.sub.cell[t.directory.isq_idx], case.dir_isq_cell)
    assert np.array_equal(qids[kept[t.sub.qrow[t.directory.cov_idx]]], case.dir_cov_qid)
    # per-task linear bitmaps and popcounts (bitmap.py:70-119)
    assert [tk[0] for tk in t.tasks] == case.task_cell.tolist()
    words = np.concatenate([tk[3] for tk in t.tasks]) if t.tasks else np.zeros(0, np.uint32)
    counts = np.concatenate([tk[4] for tk in t.tasks]) if t.tasks else np.zeros(0, np.int64)
    assert np.array_equal(words, case.task_words)
    assert np.array_equal(counts, case.task_counts)
    # final results, CSR in input-query order
    assert np.array_equal(t.offsets, case.res_off)
    assert np.array_equal(t.result_ids, case.res_ids)
    st = case.meta["stats"]
    for k in ("containment_tests", "decoded_bits", "subq_intersecting", "subq_covering",
              "covering_results", "active_cells", "results_total"):
        assert t.counters[k] == st[k], k
    assert t.counters["occupancy_mean"] == pytest.approx(st["occupancy_mean"], rel=1e-12)
    assert t.counters["occupancy_var"] == pytest.approx(st["occupancy_var"], rel=1e-9, abs=1e-12)


def test_brute_force_equals_pipeline(small_cases):
    for case in small_cases:
        ids, xs, ys, qids, qxa, qya, qxb, qyb = case.inputs()
        offs, res = qo.brute_force(ids, xs, ys, qxa, qya, qxb, qyb)
        assert np.array_equal(offs, case.res_off), case.name
        assert np.array_equal(res, case.res_ids), case.name


def _digest_run(run):
    cfg = workload_from_json(run["workload"])
    meth = run["method"]
    for t, tick in enumerate(iter_ticks(cfg)):
        out = qo.run_tick(tick.ids, tick.xs, tick.ys, tick.qids, tick.qxa, tick.qya, tick.qxb,
                          tick.qyb, th_quad=meth["th_quad"], l_max=meth["l_max"],
                          covering_optimization=meth["covering"])
        want = run["ticks"][t]
        assert out.counters["results_total"] == want["stats"]["results_total"]
        assert out.counters["containment_tests"] == want["stats"]["containment_tests"]
        assert qo.result_digest(tick.qids, out.offsets, out.result_ids) == want["digest"]


def test_oracle_digest_config_a_first_ticks(digests):
    run = dict(digests["A"])
    run["workload"] = dict(run["workload"], n_ticks=3)
    _digest_run(run)


@pytest.mark.parametrize("k", [0, 1, 2, 5, 10, 19])
def test_oracle_digest_c1(digests, k):
    _digest_run(digests[f"C1_{k}"])


# ------------------------------------------------------- adaptive rebuild --

def _adaptive_runs():
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "adaptive.json")) as fp:
        return json.load(fp)["runs"]


@pytest.mark.parametrize("name", sorted(_adaptive_runs()))
def test_oracle_adaptive_rebuild_matches_reference(name):
    """needs_rebuild (quadtree.py:243-270) + index reuse (engine.py:163-174):
    the oracle's per-tick rebuild decisions, index shape and results equal
    the reference engine's (tests/golden/make_adaptive_golden.py)."""
    from paper_1411_3212_b200.workload import WorkloadConfig, iter_ticks

    run = _adaptive_runs()[name]
    cfg = dict(run["config"])
    th = cfg.pop("th_quad")
    if isinstance(cfg.get("query_side"), list):
        cfg["query_side"] = tuple(cfg["query_side"])
    index = None
    for tick, want in zip(iter_ticks(WorkloadConfig(**cfg)), run["ticks"]):
        rebuilt = index is None or qo.needs_rebuild(tick.xs, tick.ys, index)
        if rebuilt:
            index = qo.build_index(tick.xs, tick.ys, qo.mbr_of(tick.xs, tick.ys), th, qo.L_MAX)
        assert rebuilt == want["rebuilt"]
        assert len(index.leaves) == want["n_leaves"] and index.l_deep == want["l_deep"]
        assert list(index.mbr) == want["mbr"]
        t = qo.run_tick(tick.ids, tick.xs, tick.ys, tick.qids, tick.qxa, tick.qya, tick.qxb, tick.qyb, th_quad=th,
                        index=index)
        assert qo.result_digest(tick.qids, t.offsets, t.result_ids) == want["digest"]


# ------------------------------------------------------------ uniform grid --

def _ug_runs():
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "ug.json")) as fp:
        return json.load(fp)


def _ug_ticks(run):
    from paper_1411_3212_b200.workload import WorkloadConfig, iter_ticks

    cfg = dict(run["workload"])
    cfg["query_side"] = tuple(cfg["query_side"])
    return list(iter_ticks(WorkloadConfig(**cfg)))


def _ug_subq_sha(t):
    import hashlib

    qrow = np.flatnonzero(t.keep)[t.sub.qrow].astype(np.int32)
    return hashlib.sha256(qrow.tobytes() + t.sub.cell.astype(np.int32).tobytes()
                          + t.sub.covering.astype(np.uint8).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(_ug_runs()))
def test_oracle_ug_matches_reference(name):
    """UG method (grid.py:35-112 + the shared join/decode): results digest,
    TickStats counters and the subquery list (row-major per query) equal the
    reference engine's (tests/golden/make_ug_golden.py), for power-of-two and
    other split factors."""
    import os

    run = _ug_runs()[name]
    subq = np.load(os.path.join(os.path.dirname(__file__), "golden", "ug_subqueries.npz"))
    for t_idx, (tick, want) in enumerate(zip(_ug_ticks(run), run["ticks"])):
        for sf, w in want["split"].items():
            t = qo.run_tick_ug(tick.ids, tick.xs, tick.ys, tick.qids, tick.qxa, tick.qya, tick.qxb, tick.qyb,
                               split_factor=int(sf))
            assert qo.result_digest(tick.qids, t.offsets, t.result_ids) == w["digest"], (t_idx, sf)
            for k, v in w["stats"].items():
                assert t.counters[k] == v, (t_idx, sf, k)
            if "baseline" in w:  # ug_baseline: same results, no decode, staging-buffer counters
                tb = qo.run_tick_ug(tick.ids, tick.xs, tick.ys, tick.qids, tick.qxa, tick.qya, tick.qxb, tick.qyb,
                                    split_factor=int(sf), keep_tasks=True)
                assert qo.result_digest(tick.qids, tb.offsets, tb.result_ids) == w["baseline"]["digest"]
                assert qo.staging_flushes(tb) == w["baseline"]["flushes"] == w["baseline"]["sync_ops"]
                assert tb.counters["containment_tests"] == w["baseline"]["containment_tests"]
            if "subq_sha256" in w:
                assert _ug_subq_sha(t) == w["subq_sha256"], (t_idx, sf)
                key = f"{name}_t{t_idx}_sf{sf}_cell"
                if key in subq.files:
                    assert np.array_equal(t.sub.cell, subq[key])


@pytest.mark.parametrize("name", sorted(_ug_runs()))
def test_oracle_ug_sweep_matches_reference(name):
    """Split-factor sweep (grid.py:125-165, engine.py:154-156): per-candidate
    cost and the chosen factor on the first tick."""
    run = _ug_runs()[name]
    tick = _ug_ticks(run)[0]
    want = run["ticks"][0]["sweep"]
    cands = [c for c, _ in want["costs"]]
    costs = qo.ug_sweep_costs(tick.xs, tick.ys, tick.qxa, tick.qya, tick.qxb, tick.qyb, cands)
    assert [list(c) for c in costs] == want["costs"]
    assert min(costs, key=lambda c: (c[1], c[0]))[0] == want["chosen"]
