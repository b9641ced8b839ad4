"""Brute-force ground truth for `Engine.run(verify=True)` (oracle.py:17-28).

Independent of the index: per query, a vectorised closed-rectangle scan over
all objects.  Used only to *check* the native tick when a caller asks for
verification; it never produces the tick's results.
"""

from __future__ import annotations

import numpy as np

from .geometry import TickBatch, object_arrays
from .results import ResultSet


def brute_force_join(batch: TickBatch) -> ResultSet:
    ids, xs, ys = object_arrays(batch.objects)
    out = {}
    for q in batch.queries:
        r = q.rect
        hit = (xs >= r.xa) & (xs <= r.xb) & (ys >= r.ya) & (ys <= r.yb)
        out[q.issuer_id] = np.sort(ids[hit]).tolist()
    return ResultSet(out)
