"""v1 dataset I/O (reference workload.py:241-291) and the host-side `merge_results`
(reference decode.py:102-123): byte-identical files and identical result sets."""

from __future__ import annotations

import io
import sys

import numpy as np
import pytest

from paper_1411_3212_b200 import errors, merge_results
from paper_1411_3212_b200.workload import (WorkloadConfig, generate, iter_ticks, load, load_columnar, read_columnar,
                                           read_run, save, write_columnar, write_run)

REF = "/root/reference/pkg/src"
KW = dict(n_objects=300, n_ticks=3, distribution="gaussian", seed=5, query_rate=0.3, n_hotspots=4,
          query_side=(100.0, 300.0))


def _ref():
    try:
        if REF not in sys.path:
            sys.path.append(REF)
        import tickjoin.decode as d
        import tickjoin.workload as w

        return w, d
    except Exception:  # pragma: no cover - reference absent
        pytest.skip("reference package not importable here")


def test_columnar_writer_is_byte_identical_to_reference():
    w, _ = _ref()
    ref = io.StringIO()
    w.write_run(w.generate(w.WorkloadConfig(**KW)), ref)
    ours = io.StringIO()
    write_columnar(iter_ticks(WorkloadConfig(**KW)), ours, region_side=22500.0)
    assert ours.getvalue() == ref.getvalue()
    obj = io.StringIO()
    write_run(generate(WorkloadConfig(**KW)), obj)
    assert obj.getvalue() == ref.getvalue()


def test_reader_round_trip_bit_exact(tmp_path):
    ticks = list(iter_ticks(WorkloadConfig(**KW)))
    p = tmp_path / "d.txt"
    save(ticks, str(p))
    back = load_columnar(str(p))
    assert len(back) == len(ticks)
    for a, b in zip(ticks, back):
        for c in ("ids", "xs", "ys", "qids", "qxa", "qya", "qxb", "qyb"):
            x, y = getattr(a, c), getattr(b, c)
            assert x.dtype == y.dtype and np.array_equal(x.view(np.int64) if x.dtype == np.float64 else x,
                                                         y.view(np.int64) if y.dtype == np.float64 else y), c
    run = load(str(p))
    assert run.n_ticks == 3 and run.n_objects == 300
    assert run.batches[1].objects[7].position.x == ticks[1].xs[7]


def test_reader_reads_reference_files():
    w, _ = _ref()
    buf = io.StringIO()
    ref_run = w.generate(w.WorkloadConfig(**KW))
    w.write_run(ref_run, buf)
    run = read_run(io.StringIO(buf.getvalue()))
    for rb, b in zip(ref_run.batches, run.batches):
        assert [(o.id, o.position.x, o.position.y) for o in rb.objects] == \
               [(o.id, o.position.x, o.position.y) for o in b.objects]
        assert [(q.issuer_id, q.rect.xa, q.rect.ya, q.rect.xb, q.rect.yb) for q in rb.queries] == \
               [(q.issuer_id, q.rect.xa, q.rect.ya, q.rect.xb, q.rect.yb) for q in b.queries]
    # and the reference reads ours
    ours = io.StringIO()
    write_columnar(iter_ticks(WorkloadConfig(**KW)), ours)
    back = w.read_run(io.StringIO(ours.getvalue()))
    assert back.n_ticks == 3


@pytest.mark.parametrize("text", ["somethingelse 1 1 10\n", "tickjoin-v1 2 1 10.0\nO 0 1.0 2.0\n",
                                  "tickjoin-v1 1 2 10.0\nO 0 1.0 2.0\nQ 0 0.0 0.0 1.0 1.0\n",
                                  "tickjoin-v1 1 1 10.0\nO 0 1.0 zz\n"])
def test_reader_rejects_malformed(text):
    with pytest.raises(errors.BadConfig):
        read_columnar(io.StringIO(text))


def test_merge_results_matches_reference():
    _, d = _ref()
    rng = np.random.default_rng(1)
    issued = list(range(0, 60, 2))
    chunks = []
    for q in issued:
        pool = rng.permutation(500)[: rng.integers(0, 40)]
        cuts = np.sort(rng.integers(0, len(pool) + 1, 3))
        for part in np.split(pool, cuts):
            chunks.append((q, part.astype(np.int64)))
    a = merge_results(chunks, issued)
    b = d.merge_results(chunks, issued)
    assert a.by_query == b.by_query
    assert a.lines() == b.lines()


def test_merge_results_errors():
    with pytest.raises(errors.DuplicateResult):
        merge_results([(1, np.array([3, 4])), (1, np.array([4]))], [1])
    with pytest.raises(errors.DuplicateResult):
        merge_results([(9, np.array([3]))], [1])
    assert merge_results([], [1, 2]).by_query == {1: [], 2: []}
