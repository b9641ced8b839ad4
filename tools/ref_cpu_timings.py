"""Time the REFERENCE engine (tickjoin, unmodified, from baseline/_ref) on the CPU host:
`Engine(MethodConfig("quad", n_workers=w)).run(workload)` on configs A (all 10 ticks) and B
(the first --b-ticks of 20), for n_workers = 1 and os.cpu_count(), plus per-stage timings
(the reference's own durations: index / filter / decode / merge) — SURVEY.md §8(d), BASELINE.md §3.

    python tools/ref_cpu_timings.py [--b-ticks 3] > profiles/r02_reference_cpu.json
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)

from tickjoin import engine as E  # noqa: E402
from tickjoin import workload as W  # noqa: E402

CONFIGS = {
    "A": dict(n_objects=100_000, n_ticks=10, query_rate=0.1, query_side=(200.0, 800.0), distribution="uniform",
              seed=1),
    "B": dict(n_objects=1_000_000, n_ticks=20, query_rate=1.0, query_side=50.0, distribution="gaussian",
              n_hotspots=25, seed=2),
}


def one(name, n_ticks, workers):
    kw = dict(CONFIGS[name])
    kw["n_ticks"] = n_ticks
    t0 = time.perf_counter()
    run = W.generate(W.WorkloadConfig(**kw))
    gen_s = time.perf_counter() - t0
    rep = E.Engine(E.MethodConfig(method="quad", n_workers=workers)).run(run)
    tot = [s.durations["total"] for s in rep.stats]
    stages = {k: statistics.mean(s.durations.get(k, 0.0) for s in rep.stats)
              for k in ("index", "filter", "decode", "merge", "total")}
    return {"config": name, "ticks": n_ticks, "n_workers": workers, "bandwidth_queries_per_s": rep.bandwidth,
            "p50_tick_s": statistics.median(tot), "mean_stage_s": stages,
            "results_per_tick": [s.results_total for s in rep.stats], "generate_s": gen_s}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b-ticks", type=int, default=3)
    args = ap.parse_args()
    cpus = os.cpu_count() or 1
    out = {"host": {"os_cpu_count": cpus, "machine": platform.machine(), "python": platform.python_version(),
                    "processor": platform.processor()},
           "runs": []}
    for name, ticks in (("A", 10), ("B", args.b_ticks)):
        for w in sorted({1, cpus}):
            out["runs"].append(one(name, ticks, w))
            print(json.dumps(out["runs"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
