"""Golden fixtures for the uniform-grid (UG) method, made by running the REFERENCE.

    python tests/golden/make_ug_golden.py     (build container only)

For a few generated workloads (RNG-identical columnar generator, so tests can
regenerate the ticks) it records, per tick and split factor, the reference
engine's TickStats counters, its subqueries (grid.split_queries: query row,
Morton cell id, covering flag, in the reference's row-major order) and the
sha256 of the canonical result lines; plus the split-factor sweep costs
(grid.sweep_costs) and the factor the engine picks.  Nothing at test time
reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from tickjoin import grid  # noqa: E402
from tickjoin.engine import Engine, MethodConfig  # noqa: E402
from tickjoin.geometry import compute_mbr  # noqa: E402
from tickjoin.workload import WorkloadConfig, generate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

RUNS = {
    "uniform_3k": dict(n_objects=3000, n_ticks=3, max_speed=40.0, query_rate=0.3, query_side=(20.0, 200.0),
                       distribution="uniform", region_side=2000.0, seed=51, split=[1, 5, 16, 48, 100]),
    "gauss_4k": dict(n_objects=4000, n_ticks=3, max_speed=15.0, query_rate=0.5, query_side=(10.0, 120.0),
                     distribution="gaussian", n_hotspots=4, region_side=2000.0, seed=52, split=[8, 31, 64, 160]),
    "gauss_wide": dict(n_objects=2000, n_ticks=2, max_speed=5.0, query_rate=0.1, query_side=(200.0, 700.0),
                       distribution="gaussian", n_hotspots=2, region_side=2000.0, seed=53, split=[3, 32, 96]),
}
SWEEP = (16, 256, 16)  # engine.py:30 DEFAULT_SWEEP

STAT_KEYS = ("containment_tests", "subq_intersecting", "subq_covering", "covering_results", "active_cells",
             "results_total")


def digest(rs) -> str:
    h = hashlib.sha256()  # as make_adaptive_golden.py / oracle.digest_lines
    for ln in rs.lines():
        h.update(ln.encode())
        h.update(b"\n")
    return h.hexdigest()


def main():
    out, arrays = {}, {}
    for name, kw in RUNS.items():
        kw = dict(kw)
        splits = kw.pop("split")
        wl = WorkloadConfig(**kw)
        run = {"workload": {**kw, "query_side": list(kw["query_side"])}, "ticks": []}
        ticks = list(generate(wl).batches)
        for t, batch in enumerate(ticks):
            rec = {"split": {}}
            for sf in splits:
                eng = Engine(MethodConfig(method="ug", split_factor=sf))
                rs, st = eng.process_tick(batch)
                rec["split"][str(sf)] = {"digest": digest(rs), "stats": {k: getattr(st, k) for k in STAT_KEYS}}
                if t == 0:  # subqueries as the reference splits them (clipped to this tick's MBR)
                    mbr = compute_mbr(batch)
                    sq = grid.split_queries(grid.clip_queries(batch.queries, mbr), grid.build_grid(mbr, sf))
                    row_of = {q.issuer_id: k for k, q in enumerate(batch.queries)}
                    key = f"{name}_t{t}_sf{sf}"
                    qrow = np.array([row_of[int(q)] for q in sq.query_ids], np.int32)
                    cell = np.asarray(sq.cell_ids, np.int32)
                    cov = np.asarray(sq.covering, np.uint8)
                    rec["split"][str(sf)]["subq_sha256"] = hashlib.sha256(
                        qrow.tobytes() + cell.tobytes() + cov.tobytes()).hexdigest()
                    if len(cell) <= 150_000:  # the arrays themselves for the small splits
                        arrays[key + "_qrow"], arrays[key + "_cell"], arrays[key + "_cov"] = qrow, cell, cov
                if t == 0:  # the direct-emission comparison path on the same grid (baseline.py)
                    eng = Engine(MethodConfig(method="ug_baseline", split_factor=sf))
                    rs, st = eng.process_tick(batch)
                    rec["split"][str(sf)]["baseline"] = {
                        "digest": digest(rs), "sync_ops": st.sync_ops, "flushes": st.flushes,
                        "decoded_bits": st.decoded_bits, "containment_tests": st.containment_tests}
            if t == 0:
                costs = grid.sweep_costs(batch, list(range(SWEEP[0], SWEEP[1] + 1, SWEEP[2])))
                eng = Engine(MethodConfig(method="ug", split_factor=None))
                rs, st = eng.process_tick(batch)
                rec["sweep"] = {"costs": [[int(a), int(b)] for a, b in costs], "chosen": int(eng.split_factor),
                                "digest": digest(rs)}
            run["ticks"].append(rec)
        out[name] = run
    with open(os.path.join(HERE, "ug.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "ug_subqueries.npz"), **arrays)
    print("wrote ug.json and ug_subqueries.npz:", sum(len(r["ticks"]) for r in out.values()), "ticks")


if __name__ == "__main__":
    main()
