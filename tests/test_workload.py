"""The columnar generator reproduces the reference generator draw for draw."""

from __future__ import annotations

import sys

import numpy as np
import pytest

from paper_1411_3212_b200.workload import WorkloadConfig, iter_ticks

REF = "/root/reference/pkg/src"


def _ref_generate():
    try:
        if REF not in sys.path:
            sys.path.append(REF)
        from tickjoin.workload import WorkloadConfig as RC, generate

        return RC, generate
    except Exception:  # pragma: no cover - reference absent (GPU box)
        pytest.skip("reference package not importable here")


@pytest.mark.parametrize("dist", ["uniform", "gaussian", "network"])
def test_matches_reference_generator(dist):
    RC, generate = _ref_generate()
    kw = dict(n_objects=700, n_ticks=4, distribution=dist, seed=31, query_rate=0.4, n_hotspots=5,
              grid_degree=7, query_side=(100.0, 300.0))
    run = generate(RC(**kw))
    for b, t in zip(run.batches, iter_ticks(WorkloadConfig(**kw))):
        assert np.array_equal(t.ids, [o.id for o in b.objects])
        assert np.array_equal(t.xs, [o.position.x for o in b.objects])
        assert np.array_equal(t.ys, [o.position.y for o in b.objects])
        assert np.array_equal(t.qids, [q.issuer_id for q in b.queries])
        for arr, f in ((t.qxa, "xa"), (t.qya, "ya"), (t.qxb, "xb"), (t.qyb, "yb")):
            assert np.array_equal(arr, [getattr(q.rect, f) for q in b.queries])


def test_fixed_side_and_validation():
    from paper_1411_3212_b200.errors import BadConfig

    t = next(iter_ticks(WorkloadConfig(n_objects=50, n_ticks=1, query_side=5.0, seed=1)))
    assert np.allclose(t.qxb - t.qxa, 5.0)
    with pytest.raises(BadConfig):
        WorkloadConfig(n_objects=0).validate()
