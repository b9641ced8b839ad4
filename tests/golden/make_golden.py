"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (the reference is importable only here):

    python tests/golden/make_golden.py

It imports `tickjoin` from /root/reference/pkg/src (read-only), runs the
reference's own QUAD pipeline functions on small deterministic workloads and
writes:

* `small_cases.npz` + `small_cases.json` — full intermediates per tick
  (index, subqueries, directory, per-task linear bitmaps + popcounts, final
  per-query results, TickStats counters) for small inputs;
* `digests.json` — sha256 of the reference's canonical `ResultSet.lines()`
  (plus counters) for larger runs (config A = uniform 100K / 10% / 10 ticks,
  and the acceptance-C1 workload family), which the GPU tests regenerate with
  the RNG-identical columnar generator and compare against.

The fixtures are committed; nothing at test/bench time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from tickjoin import bitmap as rbitmap  # noqa: E402
from tickjoin.directory import ObjectColumns, sort_by_cell  # noqa: E402
from tickjoin.engine import Engine, MethodConfig  # noqa: E402
from tickjoin.geometry import MovingObject, Point, Query, Rect, TickBatch, compute_mbr  # noqa: E402
from tickjoin import grid as rgrid  # noqa: E402
from tickjoin import quadtree as rquad  # noqa: E402
from tickjoin.workload import WorkloadConfig, generate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def lines_digest(lines):
    h = hashlib.sha256()
    for ln in lines:
        h.update(ln.encode())
        h.update(b"\n")
    return h.hexdigest()


def soa(batch):
    ids = np.array([o.id for o in batch.objects], np.int64)
    xs = np.array([o.position.x for o in batch.objects], np.float64)
    ys = np.array([o.position.y for o in batch.objects], np.float64)
    qids = np.array([q.issuer_id for q in batch.queries], np.int64)
    r = np.array([[q.rect.xa, q.rect.ya, q.rect.xb, q.rect.yb] for q in batch.queries],
                 np.float64).reshape(-1, 4)
    return ids, xs, ys, qids, r


def reference_intermediates(batch, cfg: MethodConfig):
    """Replay engine.py:178-259 (quad branch) through the reference's own
    module functions, keeping every intermediate."""
    cols = ObjectColumns.from_objects(batch.objects)
    mbr = compute_mbr(batch)
    idx = rquad.build_quadtree(cols, cfg.th_quad, cfg.l_max, mbr)
    clipped = rgrid.clip_queries(batch.queries, idx.mbr)
    cell_ids = rquad.map_objects_quad(cols, idx)
    sq = rquad.split_queries_quad(clipped, idx)
    if not cfg.covering_optimization:
        sq.covering = np.zeros(len(sq), bool)
    d = sort_by_cell(cols, cell_ids, sq)
    # clipped query row per subquery: issuer ids are unique per tick
    issuer_row = {q.issuer_id: k for k, q in enumerate(batch.queries)}
    sq_qrow = np.array([issuer_row[int(q)] for q in sq.query_ids], np.int64)
    n_obj = d.o_end - d.o_start
    n_isq = d.i_end - d.i_start
    tasks = np.flatnonzero((n_obj > 0) & (n_isq > 0))
    t_cell, t_nobj, t_nisq, t_woff, words_all, counts_all = [], [], [], [0], [], []
    for r in tasks:
        os_, oe = d.o_start[r], d.o_end[r]
        qs, qe = d.i_start[r], d.i_end[r]
        ib = rbitmap.generate_interlaced(int(d.cell_ids[r]), d.obj_xs[os_:oe], d.obj_ys[os_:oe],
                                         d.isq.xa[qs:qe], d.isq.ya[qs:qe], d.isq.xb[qs:qe],
                                         d.isq.yb[qs:qe])
        lb = rbitmap.linearize(ib)
        rc = rbitmap.count_results(lb)
        t_cell.append(int(d.cell_ids[r]))
        t_nobj.append(int(oe - os_))
        t_nisq.append(int(qe - qs))
        words_all.append(lb.words.astype(np.uint32))
        counts_all.append(rc.counts.astype(np.int64))
        t_woff.append(t_woff[-1] + len(lb.words))
    # the input rows of the directory's objects (ids are input rows in these cases)
    row_of_id = {int(o.id): k for k, o in enumerate(batch.objects)}
    obj_order = np.array([row_of_id[int(i)] for i in d.obj_ids], np.int64)
    return dict(
        mbr=np.array([idx.mbr.xa, idx.mbr.ya, idx.mbr.xb, idx.mbr.yb], np.float64),
        l_deep=np.int64(idx.l_deep),
        leaves=idx.leaves.astype(np.int64),
        zmap=idx.zmap.astype(np.int64),
        obj_cell=np.asarray(cell_ids, np.int64),
        sq_qrow=sq_qrow,
        sq_cell=sq.cell_ids.astype(np.int64),
        sq_cov=sq.covering.astype(np.uint8),
        dir_obj_order=obj_order,
        dir_isq_qid=d.isq.query_ids.astype(np.int64),
        dir_isq_cell=d.isq.cell_ids.astype(np.int64),
        dir_cov_qid=d.cov.query_ids.astype(np.int64),
        dir_cov_cell=d.cov.cell_ids.astype(np.int64),
        task_cell=np.array(t_cell, np.int64),
        task_nobj=np.array(t_nobj, np.int64),
        task_nisq=np.array(t_nisq, np.int64),
        task_woff=np.array(t_woff, np.int64),
        task_words=(np.concatenate(words_all) if words_all else np.zeros(0, np.uint32)),
        task_counts=(np.concatenate(counts_all) if counts_all else np.zeros(0, np.int64)),
    )


def result_csr(rs, qids):
    offs = [0]
    parts = []
    for q in qids:
        v = np.asarray(rs.by_query[int(q)], np.int64)
        parts.append(v)
        offs.append(offs[-1] + len(v))
    return np.asarray(offs, np.int64), (np.concatenate(parts) if parts else np.zeros(0, np.int64))


STAT_KEYS = ("containment_tests", "decoded_bits", "subq_intersecting", "subq_covering",
             "covering_results", "active_cells", "results_total", "occupancy_mean",
             "occupancy_var", "dispersion", "imbalance")


def stats_dict(st):
    return {k: getattr(st, k) for k in STAT_KEYS}


def small_cases():
    cases = []

    def mk(points):
        return [MovingObject(i, Point(float(x), float(y))) for i, (x, y) in enumerate(points)]

    # conftest.py:12-30 seven-point layout (Fig. 6) with a handful of queries
    seven = mk([(0.5, 0.5), (2.5, 0.5), (3.5, 0.5), (2.5, 1.5), (0.5, 2.5), (1.5, 3.5), (3.5, 3.5)])
    qs = [Query(0, Rect(2.2, 2.2, 3.8, 3.8)), Query(1, Rect(0.1, 0.1, 0.2, 0.2)),
          Query(2, Rect(0.0, 0.0, 4.0, 4.0)), Query(3, Rect(1.0, 0.0, 3.0, 2.0)),
          Query(4, Rect(-5.0, -5.0, -1.0, -1.0))]
    cases.append(("fig6", TickBatch(0, seven, qs), MethodConfig(method="quad", th_quad=1, l_max=2)))
    # conftest.py:33-50 mixed-depth layout + the 7-subquery query (test_quadtree.py:150-161)
    mixed = mk([(12.0, 12.0), (5.0, 9.0), (7.0, 11.0), (1.0, 1.0), (5.0, 5.0), (9.0, 1.0), (13.0, 5.0)])
    cases.append(("mixed", TickBatch(0, mixed, [Query(1, Rect(3.5, 7.5, 6.5, 10.5)),
                                                Query(5, Rect(0.0, 0.0, 16.0, 16.0))]),
                  MethodConfig(method="quad", th_quad=1, l_max=3)))
    # conftest.py:53-67 Fig. 1 scenario
    scen = TickBatch(0, [MovingObject(1, Point(20.0, 20.0)), MovingObject(2, Point(4.0, 4.0)),
                         MovingObject(3, Point(5.0, 5.0))],
                     [Query(1, Rect(18.0, 18.0, 19.0, 19.0)), Query(2, Rect(0.0, 0.0, 1.0, 1.0)),
                      Query(3, Rect(3.0, 3.0, 7.0, 7.0))])
    cases.append(("scenario", scen, MethodConfig(method="quad", th_quad=1, l_max=3)))
    # randomized negative-coordinate batches (test_engine.py:174-196 family)
    rng = np.random.default_rng(4242)
    for k in range(4):
        n = int(rng.integers(1, 60))
        pts = rng.uniform(-100, 100, (n, 2))
        nq = int(rng.integers(0, 20))
        qs = []
        for q in range(nq):
            x, y, h = rng.uniform(-100, 100), rng.uniform(-100, 100), rng.uniform(0.5, 60)
            qs.append(Query(q, Rect(x - h, y - h, x + h, y + h)))
        cfg = MethodConfig(method="quad", th_quad=int(rng.integers(1, 7)), l_max=6)
        cases.append((f"neg{k}", TickBatch(0, mk(pts), qs), cfg))
    # coincident points / degenerate MBR (width == 0)
    cases.append(("colocated", TickBatch(0, mk([(3.0, 3.0)] * 40 + [(3.0, 7.0)] * 5),
                                         [Query(0, Rect(2.0, 2.0, 4.0, 4.0)),
                                          Query(1, Rect(3.0, 3.0, 3.0, 7.0))]),
                  MethodConfig(method="quad", th_quad=4, l_max=5)))
    # generated workloads: every distribution, covering on/off, shallow/deep trees
    wl = [
        ("uni_th32", WorkloadConfig(n_objects=1500, n_ticks=2, distribution="uniform", seed=11,
                                    query_rate=0.5), MethodConfig(method="quad", th_quad=32)),
        ("gau_th16", WorkloadConfig(n_objects=2500, n_ticks=2, distribution="gaussian",
                                    n_hotspots=4, seed=12, query_side=(50.0, 200.0)),
         MethodConfig(method="quad", th_quad=16)),
        ("gau_th16_nocov", WorkloadConfig(n_objects=2500, n_ticks=1, distribution="gaussian",
                                          n_hotspots=4, seed=12, query_side=(50.0, 200.0)),
         MethodConfig(method="quad", th_quad=16, covering_optimization=False)),
        ("net_th24", WorkloadConfig(n_objects=2000, n_ticks=2, distribution="network",
                                    grid_degree=12, seed=13), MethodConfig(method="quad", th_quad=24)),
        ("gau_default", WorkloadConfig(n_objects=3000, n_ticks=2, distribution="gaussian",
                                       n_hotspots=2, sigma=60.0, seed=14, query_side=(10.0, 60.0)),
         MethodConfig(method="quad")),
        ("gau_lmax4", WorkloadConfig(n_objects=2000, n_ticks=1, distribution="gaussian",
                                     n_hotspots=1, sigma=30.0, seed=15, query_side=(2.0, 12.0)),
         MethodConfig(method="quad", th_quad=8, l_max=4)),
    ]
    for name, wcfg, mcfg in wl:
        run = generate(wcfg)
        for t, b in enumerate(run.batches):
            cases.append((f"{name}_t{t}", b, mcfg))
    return cases


def main():
    t0 = time.time()
    arrays = {}
    meta = {"generated_by": "tests/golden/make_golden.py", "reference": "tickjoin 0.1.0 (/root/reference/pkg)",
            "cases": {}}
    for name, batch, cfg in small_cases():
        eng = Engine(cfg)
        rs, st = eng.process_tick(batch)
        ids, xs, ys, qids, rects = soa(batch)
        offs, res = result_csr(rs, qids)
        inter = reference_intermediates(batch, cfg)
        assert int(inter["task_counts"].sum()) + st.covering_results == st.results_total
        for k, v in dict(ids=ids, xs=xs, ys=ys, qids=qids, rects=rects, res_off=offs,
                         res_ids=res, **inter).items():
            arrays[f"{name}__{k}"] = v
        meta["cases"][name] = dict(th_quad=cfg.th_quad, l_max=cfg.l_max,
                                   covering=cfg.covering_optimization, stats=stats_dict(st),
                                   digest=lines_digest(rs.lines()))
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)
    with open(os.path.join(HERE, "small_cases.json"), "w") as fp:
        json.dump(meta, fp, indent=1, sort_keys=True)
    print(f"small cases: {len(meta['cases'])} in {time.time() - t0:.1f}s")

    digests = {"generated_by": "tests/golden/make_golden.py", "runs": {}}

    def record(key, wcfg, mcfg):
        t1 = time.time()
        run = generate(wcfg)
        eng = Engine(mcfg)
        ticks = []
        for b in run.batches:
            rs, st = eng.process_tick(b)
            ticks.append(dict(digest=lines_digest(rs.lines()), stats=stats_dict(st),
                              n_queries=len(b.queries)))
        digests["runs"][key] = dict(
            workload={k: (list(v) if isinstance(v, tuple) else v) for k, v in wcfg.__dict__.items()},
            method=dict(th_quad=mcfg.th_quad, l_max=mcfg.l_max,
                        covering=mcfg.covering_optimization),
            ticks=ticks)
        print(f"  {key}: {len(ticks)} ticks in {time.time() - t1:.1f}s")

    # config A: uniform 100K, 10%, sides U[200,800], 10 ticks, seed 1
    record("A", WorkloadConfig(n_objects=100_000, n_ticks=10, query_rate=0.1,
                               query_side=(200.0, 800.0), distribution="uniform", seed=1),
           MethodConfig(method="quad"))
    # skewed 100K / 100% / 50u (a scaled-down config B), 3 ticks
    record("B100K", WorkloadConfig(n_objects=100_000, n_ticks=3, query_rate=1.0, query_side=50.0,
                                   distribution="gaussian", n_hotspots=25, seed=2),
           MethodConfig(method="quad"))
    # acceptance C1 family (test_acceptance.py:28-100): 20 workloads x 5 ticks, quad on/off
    rng = np.random.default_rng(20240229)
    dists = ["uniform", "gaussian", "network"]
    for k in range(20):
        n = int(rng.integers(500, 5001))
        wcfg = WorkloadConfig(n_objects=n, n_ticks=5, region_side=22500.0, max_speed=200.0,
                              query_rate=1.0, query_side=(200.0, 800.0), distribution=dists[k % 3],
                              n_hotspots=10, grid_degree=12, seed=1000 + k)
        record(f"C1_{k}", wcfg, MethodConfig(method="quad"))
    with open(os.path.join(HERE, "digests.json"), "w") as fp:
        json.dump(digests, fp, indent=1, sort_keys=True)
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
