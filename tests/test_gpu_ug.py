"""GPU parity of the uniform-grid method ("ug", grid.py) through the C ABI.

The UG index runs on the same kernels as QUAD with the grid's cells as the
leaves.  Checked against (a) fixtures made by running the reference's UG
engine (tests/golden/make_ug_golden.py: result digests, TickStats counters,
subquery lists in the reference's row-major order, sweep costs and the chosen
split factor) and (b) the pinned oracle (oracle/quad_oracle.run_tick_ug) on
seeded random ticks, including split factors that are not powers of two,
the 4096 maximum, degenerate extents and covering off.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import quad_oracle as qo

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def pkg():
    import paper_1411_3212_b200 as p
    from paper_1411_3212_b200 import _native

    assert _native.device_count() > 0, "no CUDA device: the GPU tests need a B200"
    return p


def _runs():
    with open(os.path.join(GOLDEN, "ug.json")) as fp:
        return json.load(fp)


def _ticks(run):
    from paper_1411_3212_b200.workload import WorkloadConfig, iter_ticks

    cfg = dict(run["workload"])
    cfg["query_side"] = tuple(cfg["query_side"])
    return list(iter_ticks(WorkloadConfig(**cfg)))


def _ug(pkg, sf, covering=True):
    return pkg.Engine(pkg.MethodConfig(method="ug", split_factor=sf, covering_optimization=covering))


@pytest.mark.parametrize("name", sorted(_runs()))
def test_ug_matches_reference_fixtures(pkg, name):
    run = _runs()[name]
    for t_idx, (tick, want) in enumerate(zip(_ticks(run), run["ticks"])):
        for sf, w in want["split"].items():
            eng = _ug(pkg, int(sf))
            res, st = eng.process_tick_columnar(tick)
            assert qo.result_digest(tick.qids, res.offsets, res.ids) == w["digest"], (t_idx, sf)
            for k, v in w["stats"].items():
                assert getattr(st, k) == v, (t_idx, sf, k)
            assert st.split_factor == int(sf)
            if "subq_sha256" in w:
                q, cell, cov = eng.native.subqueries()
                sha = hashlib.sha256(q.astype(np.int32).tobytes() + cell.astype(np.int32).tobytes()
                                     + cov.astype(np.uint8).tobytes()).hexdigest()
                assert sha == w["subq_sha256"], (t_idx, sf)
            eng.close()


@pytest.mark.parametrize("name", sorted(_runs()))
def test_ug_sweep_matches_reference(pkg, name):
    """split_factor=None: the first tick sweeps the candidates (engine.py:152-156)."""
    run = _runs()[name]
    tick = _ticks(run)[0]
    want = run["ticks"][0]["sweep"]
    eng = pkg.Engine(pkg.MethodConfig(method="ug"))
    res, st = eng.process_tick_columnar(tick)
    assert [list(c) for c in eng.sweep_costs] == want["costs"]
    assert eng.split_factor == want["chosen"] and st.split_factor == want["chosen"]
    assert qo.result_digest(tick.qids, res.offsets, res.ids) == want["digest"]
    eng.close()


def _rand(rng, n, m, lo=0.0, hi=1000.0, side=(1.0, 120.0)):
    xs = rng.uniform(lo, hi, n)
    ys = rng.uniform(lo, hi, n)
    cx = rng.uniform(lo - 50, hi + 50, m)
    cy = rng.uniform(lo - 50, hi + 50, m)
    h = rng.uniform(side[0], side[1], m) / 2
    return xs, ys, cx - h, cy - h, cx + h, cy + h


@pytest.mark.parametrize("sf", [1, 2, 3, 100, 257, 1000, 4096])
def test_ug_random_ticks_vs_oracle(pkg, sf):
    rng = np.random.default_rng(sf)
    n, m = (40_000, 3000) if sf <= 257 else (6000, 1500)  # the oracle loops over task cells in Python
    xs, ys, a, b, c, d = _rand(rng, n, m, side=(1.0, 120.0 if sf <= 257 else 12.0))
    ids = np.arange(n, dtype=np.int64)
    qids = np.arange(m, dtype=np.int64)
    for cov in (True, False):
        eng = _ug(pkg, sf, cov)
        res, st = eng.process_columns(ids, xs, ys, qids, a, b, c, d)
        ref = qo.run_tick_ug(ids, xs, ys, qids, a, b, c, d, split_factor=sf, covering_optimization=cov)
        assert np.array_equal(res.offsets, ref.offsets) and np.array_equal(res.ids, ref.result_ids)
        for k in ("containment_tests", "subq_intersecting", "subq_covering", "covering_results", "active_cells",
                  "results_total", "decoded_bits"):
            assert getattr(st, k) == ref.counters[k], (sf, cov, k)
        if sf > 1000:  # (the host-side introspection walks every one of the 16.7M cells)
            eng.close()
            continue
        # intermediates: object cells, subquery list (reference order), directory
        assert np.array_equal(eng.native.object_cells(n), ref.obj_cell)
        q, cell, cv = eng.native.subqueries()
        assert np.array_equal(q, np.flatnonzero(ref.keep)[ref.sub.qrow])
        assert np.array_equal(cell, ref.sub.cell) and np.array_equal(cv, ref.sub.covering)
        rows, isq, covl = eng.native.directory(n)
        assert np.array_equal(rows, ref.directory.obj_order)
        assert np.array_equal(isq, ref.directory.isq_idx) and np.array_equal(covl, ref.directory.cov_idx)
        eng.close()


def test_ug_degenerate_extents_and_non_monotone_ids(pkg):
    rng = np.random.default_rng(9)
    n, m = 5000, 500
    xs = np.full(n, 7.5)  # zero-width MBR: every object in column 0 (grid.py:44-46)
    ys = rng.uniform(0, 100, n)
    cx, cy = rng.uniform(0, 20, m), rng.uniform(0, 100, m)
    h = rng.uniform(1, 30, m) / 2
    ids = rng.permutation(10 * n)[:n].astype(np.int64)
    qids = rng.permutation(m).astype(np.int64)
    for sf in (7, 64):
        eng = _ug(pkg, sf)
        res, _ = eng.process_columns(ids, xs, ys, qids, cx - h, cy - h, cx + h, cy + h)
        ref = qo.run_tick_ug(ids, xs, ys, qids, cx - h, cy - h, cx + h, cy + h, split_factor=sf)
        assert np.array_equal(res.offsets, ref.offsets) and np.array_equal(res.ids, ref.result_ids)
        eng.close()


@pytest.mark.parametrize("name", sorted(_runs()))
def test_ug_baseline_matches_reference_fixtures(pkg, name):
    """method="ug_baseline" (baseline.py): the same results, no decode phase, and the
    reference's staging-buffer contention counters (sync_ops = flushes)."""
    run = _runs()[name]
    tick = _ticks(run)[0]
    for sf, w in run["ticks"][0]["split"].items():
        want = w["baseline"]
        eng = pkg.Engine(pkg.MethodConfig(method="ug_baseline", split_factor=int(sf)))
        res, st = eng.process_tick_columnar(tick)
        assert qo.result_digest(tick.qids, res.offsets, res.ids) == want["digest"]
        assert (st.sync_ops, st.flushes, st.decoded_bits, st.containment_tests) == (
            want["sync_ops"], want["flushes"], want["decoded_bits"], want["containment_tests"])
        eng.close()
