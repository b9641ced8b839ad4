"""Golden digests for config B at full size, made by running the REFERENCE.

    python tests/golden/make_b_golden.py        (build container only; ~1 min/tick, ~11 GB RSS)

Config B: gaussian 1M objects (25 hotspots, sigma 225u),
100% query rate, 50u squares, seed 2.  For each of the first ticks it runs the
reference engine `Engine(MethodConfig("quad")).process_tick` (engine.py:178-259)
and records the TickStats counters plus two digests of its `ResultSet`:

* `digest`: sha256 of the canonical `ResultSet.lines()` text (decode.py:33-37);
* `csr_sha256`: sha256 of the same lists as a CSR in ascending issuer order —
  int64 offsets (n_q + 1) then int64 ids — which a test recomputes from a
  device result in a second instead of formatting 1.6e8 ids as text.

The GPU tests regenerate the ticks with the RNG-identical columnar generator;
nothing at test time reads /root/reference.
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

from tickjoin.engine import Engine, MethodConfig  # noqa: E402
from tickjoin.workload import WorkloadConfig, generate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
N_TICKS = int(os.environ.get("B_TICKS", "5"))


def lines_digest(lines):
    h = hashlib.sha256()
    for ln in lines:
        h.update(ln.encode())
        h.update(b"\n")
    return h.hexdigest()


def csr_sha256(by_query: dict) -> str:
    qids = sorted(by_query)
    lens = np.fromiter((len(by_query[q]) for q in qids), np.int64, len(qids))
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ids = np.fromiter((v for q in qids for v in by_query[q]), np.int64, int(offs[-1]))
    h = hashlib.sha256()
    h.update(offs.tobytes())
    h.update(ids.tobytes())
    return h.hexdigest()


def main():
    wcfg = WorkloadConfig(n_objects=1_000_000, n_ticks=N_TICKS, query_rate=1.0, query_side=50.0,
                          distribution="gaussian", n_hotspots=25, seed=2)
    t0 = time.time()
    run = generate(wcfg)
    print(f"generated {N_TICKS} ticks in {time.time() - t0:.1f}s", flush=True)
    eng = Engine(MethodConfig(method="quad"))
    ticks = []
    for b in run.batches:
        t1 = time.time()
        rs, st = eng.process_tick(b)
        ticks.append(dict(
            digest=lines_digest(rs.lines()), csr_sha256=csr_sha256(rs.by_query), n_queries=len(b.queries),
            stats={k: int(getattr(st, k)) for k in ("containment_tests", "decoded_bits", "subq_intersecting",
                                                     "subq_covering", "covering_results", "active_cells",
                                                     "results_total")},
            seconds=round(time.time() - t1, 1)))
        print(f"  tick {len(ticks) - 1}: {ticks[-1]}", flush=True)
        del rs
    out = {"generated_by": "tests/golden/make_b_golden.py", "reference": "tickjoin 0.1.0 (/root/reference/pkg)",
           "workload": {k: (list(v) if isinstance(v, tuple) else v) for k, v in wcfg.__dict__.items()},
           "method": dict(th_quad=384, l_max=12, covering=True), "ticks": ticks}
    with open(os.path.join(HERE, "digests_b.json"), "w") as fp:
        json.dump(out, fp, indent=1, sort_keys=True)
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
