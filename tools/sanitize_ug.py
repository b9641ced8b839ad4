"""Small UG / ug_baseline ticks for compute-sanitizer runs (memcheck of the grid paths)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import quad_oracle as qo  # noqa: E402
from paper_1411_3212_b200 import Engine, MethodConfig  # noqa: E402

rng = np.random.default_rng(4)
n, m = 20_000, 2000
xs, ys = rng.uniform(0, 500, n), rng.uniform(0, 500, n)
cx, cy, h = rng.uniform(-20, 520, m), rng.uniform(-20, 520, m), rng.uniform(0.5, 60, m) / 2
ids, qids = np.arange(n), np.arange(m)
ok = True
for method, sf in (("ug", 1), ("ug", 3), ("ug", 100), ("ug", 4096), ("ug_baseline", 37), ("ug", None)):
    eng = Engine(MethodConfig(method=method, split_factor=sf, sweep=(16, 64, 16)))
    res, st = eng.process_columns(ids, xs, ys, qids, cx - h, cy - h, cx + h, cy + h)
    ref = qo.run_tick_ug(ids, xs, ys, qids, cx - h, cy - h, cx + h, cy + h, split_factor=eng.split_factor)
    good = np.array_equal(res.offsets, ref.offsets) and np.array_equal(res.ids, ref.result_ids)
    if method == "ug" and sf is not None and sf <= 100:
        eng.native.subqueries()
        eng.native.directory(n)
        eng.native.bitmaps()
    print(method, sf, eng.split_factor, st.results_total, "match" if good else "MISMATCH")
    ok &= good
    eng.close()
sys.exit(0 if ok else 1)
