"""Golden fixtures for rebuild="adaptive", made by running the REFERENCE.

    python tests/golden/make_adaptive_golden.py     (build container only)

For a few moving workloads it records, per tick, whether the reference
engine rebuilt its quadtree (engine._quad replaced; engine.py:163-174,
quadtree.py:243-270), the index it used (leaf count, depth, MBR) and the
sha256 of the canonical result lines.  tests/ regenerate the ticks with the
RNG-identical columnar generator; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from tickjoin.engine import Engine, MethodConfig  # noqa: E402
from tickjoin.workload import WorkloadConfig, generate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

RUNS = {
    # slow drift: the index is reused for a while, then overfull leaves force rebuilds
    "drift_uniform_th16": dict(n_objects=3000, n_ticks=8, max_speed=40.0, query_rate=0.3, query_side=(20.0, 120.0),
                               distribution="uniform", region_side=2000.0, seed=41, th=16),
    "drift_gauss_th8": dict(n_objects=2500, n_ticks=8, max_speed=15.0, query_rate=0.5, query_side=(10.0, 60.0),
                            distribution="gaussian", n_hotspots=4, region_side=2000.0, seed=42, th=8),
    # objects that stay put (queries change): the index is reused on every tick after the first
    "static_gauss_th16": dict(n_objects=3000, n_ticks=5, max_speed=0.0, query_rate=0.5, query_side=(20.0, 150.0),
                              distribution="gaussian", n_hotspots=3, region_side=2000.0, seed=44, th=16),
    # fast movement: objects escape the old MBR, rebuild every few ticks
    "fast_uniform_th32": dict(n_objects=4000, n_ticks=6, max_speed=300.0, query_rate=0.2, query_side=(50.0, 200.0),
                              distribution="uniform", region_side=3000.0, seed=43, th=32),
}


def digest(lines):
    h = hashlib.sha256()
    for ln in lines:
        h.update(ln.encode())
        h.update(b"\n")
    return h.hexdigest()


def main():
    out = {"generated_by": "tests/golden/make_adaptive_golden.py", "runs": {}}
    for name, spec in RUNS.items():
        spec = dict(spec)
        th = spec.pop("th")
        run = generate(WorkloadConfig(**spec))
        eng = Engine(MethodConfig(method="quad", th_quad=th, rebuild="adaptive"))
        ticks = []
        prev = None
        for batch in run.batches:
            rs, st = eng.process_tick(batch)
            q = eng._quad
            ticks.append(dict(rebuilt=q is not prev, n_leaves=int(len(q.leaves)), l_deep=int(q.l_deep),
                              mbr=[q.mbr.xa, q.mbr.ya, q.mbr.xb, q.mbr.yb], results=int(rs.total),
                              digest=digest(rs.lines())))
            prev = q
        out["runs"][name] = dict(config=dict(spec, th_quad=th), ticks=ticks)
        print(name, [t["rebuilt"] for t in ticks])
    with open(os.path.join(HERE, "adaptive.json"), "w") as fp:
        json.dump(out, fp, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
