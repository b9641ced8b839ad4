"""Small big-list tick for compute-sanitizer runs (memcheck of the decode paths)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1411_3212_b200 import Engine, MethodConfig, WorkloadConfig, iter_ticks
from oracle import quad_oracle as qo

cfg = WorkloadConfig(n_objects=int(sys.argv[1]) if len(sys.argv) > 1 else 100_000, n_ticks=1,
                     query_rate=float(sys.argv[3]) if len(sys.argv) > 3 else 0.2,
                     query_side=float(sys.argv[2]) if len(sys.argv) > 2 else 50.0, distribution="gaussian",
                     n_hotspots=25, seed=2)
t = next(iter_ticks(cfg))
eng = Engine(MethodConfig(method="quad"))
res, st = eng.process_tick_columnar(t)
print("results", st.results_total)
if len(sys.argv) <= 4:
    ref = qo.run_tick(t.ids, t.xs, t.ys, t.qids, t.qxa, t.qya, t.qxb, t.qyb)
    print("match", np.array_equal(res.offsets, ref.offsets) and np.array_equal(res.ids, ref.result_ids))
