"""Pin the C brute-force checker (oracle/bf_join.c) before the GPU tests trust it.

It must equal (a) the NumPy restatement of the reference's brute_force_join
(oracle.py:17-28), (b) the reference engine's results on the reference-generated
small cases, and (c) the reference's canonical-lines digests of config A and
the C1 family (tests/golden/digests.json).  CPU only.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_small_cases, workload_from_json
from oracle import bf_join as bf
from oracle import quad_oracle as qo


def _rand(rng, n, m, lo=-50.0, hi=50.0, side=(0.5, 20.0)):
    xs = rng.uniform(lo, hi, n)
    ys = rng.uniform(lo, hi, n)
    a = rng.uniform(lo - 5, hi + 5, m)
    b = rng.uniform(lo - 5, hi + 5, m)
    w = rng.uniform(*side, m)
    h = rng.uniform(*side, m)
    return xs, ys, a, b, a + w, b + h


@pytest.mark.parametrize("cell,gmax", [(1.0, 8192), (7.0, 16), (100.0, 1), (0.01, 64)])
def test_equals_numpy_brute_force(cell, gmax):
    rng = np.random.default_rng(5)
    xs, ys, a, b, c, d = _rand(rng, 3000, 400)
    # objects exactly on query edges and co-located objects
    xs[:50] = a[:50]
    ys[:50] = b[:50]
    xs[50:80] = 3.0
    ys[50:80] = 3.0
    ids = rng.permutation(10_000)[:3000].astype(np.int64) * 7 - 5000  # non-monotone, negative ids
    offs, res = qo.brute_force(ids, xs, ys, a, b, c, d)
    g = bf.BruteForce(ids, xs, ys, cell=cell, gmax=gmax)
    o2, r2 = g.lists(a, b, c, d, threads=3)
    assert np.array_equal(offs, o2) and np.array_equal(res, r2)
    cnt, dig = g.counts(a, b, c, d, threads=2)
    assert np.array_equal(cnt, np.diff(offs))
    assert np.array_equal(dig, bf.csr_digests(offs, res))
    rows = np.array([5, 0, 399, 5], np.int64)
    o3, r3 = g.lists(a, b, c, d, rows=rows)
    for k, q in enumerate(rows):
        assert np.array_equal(r3[o3[k]:o3[k + 1]], res[offs[q]:offs[q + 1]])
    g.close()


def test_degenerate_extents_and_empty():
    g = bf.BruteForce(np.arange(5), np.full(5, 2.0), np.arange(5.0), cell=1.0)
    o, r = g.lists(np.array([2.0, 0.0, 3.0]), np.array([1.0, 0.0, 0.0]), np.array([2.0, 1.0, 9.0]),
                   np.array([3.0, 9.0, 9.0]))
    assert o.tolist() == [0, 3, 3, 3] and r.tolist() == [1, 2, 3]
    g.close()
    g = bf.BruteForce(np.zeros(0, np.int64), np.zeros(0), np.zeros(0))
    cnt, dig = g.counts(np.array([0.0]), np.array([0.0]), np.array([1.0]), np.array([1.0]))
    assert cnt.tolist() == [0] and dig.tolist() == [0]
    g.close()


def test_mix64_is_splitmix64():
    # splitmix64 finaliser, reference values of the published function
    def ref(z):
        m = (1 << 64) - 1
        z ^= z >> 30
        z = (z * 0xBF58476D1CE4E5B9) & m
        z ^= z >> 27
        z = (z * 0x94D049BB133111EB) & m
        return z ^ (z >> 31)

    for v in (0, 1, 2, 12345, 2**40 + 3, (1 << 64) - 1):
        assert bf.mix64(v) == ref(v)


def test_equals_reference_small_cases():
    for case in load_small_cases():
        ids, xs, ys, qids, qxa, qya, qxb, qyb = case.inputs()
        g = bf.BruteForce(ids, xs, ys, cell=1.0)
        o, r = g.lists(qxa, qya, qxb, qyb)
        assert np.array_equal(o, case.res_off), case.name
        assert np.array_equal(r, case.res_ids), case.name
        g.close()


def _digest_check(run, max_ticks):
    from paper_1411_3212_b200.workload import iter_ticks

    cfg = workload_from_json(run["workload"])
    for t, tick in enumerate(iter_ticks(cfg)):
        if t >= max_ticks:
            break
        g = bf.BruteForce(tick.ids, tick.xs, tick.ys, cell=50.0)
        o, r = g.lists(tick.qxa, tick.qya, tick.qxb, tick.qyb)
        g.close()
        want = run["ticks"][t]
        assert int(o[-1]) == want["stats"]["results_total"]
        assert qo.result_digest(tick.qids, o, r) == want["digest"]


def test_reference_digests_config_a(digests):
    _digest_check(digests["A"], 3)


@pytest.mark.parametrize("k", [0, 1, 2, 7, 13])
def test_reference_digests_c1(digests, k):
    _digest_check(digests[f"C1_{k}"], 5)


def test_torch_csr_summary_equals_checker():
    """tests/csr_check.py (what the full-size GPU tests run on the device) computes
    the checker's counts and digests, and rejects unsorted or duplicated lists."""
    import torch

    from csr_check import device_summary

    rng = np.random.default_rng(9)
    xs, ys, a, b, c, d = _rand(rng, 5000, 700)
    ids = (rng.permutation(5000).astype(np.int64) - 2500) * 1_000_003
    g = bf.BruteForce(ids, xs, ys, cell=3.0)
    offs, res = g.lists(a, b, c, d)
    cnt, dig = g.counts(a, b, c, d)
    g.close()
    lens, dg = device_summary(torch, torch.from_numpy(offs), torch.from_numpy(res), chunk=997)
    assert np.array_equal(lens, cnt) and np.array_equal(dg, dig)
    k = int(np.flatnonzero(np.diff(offs) >= 2)[0])
    bad = res.copy()
    bad[offs[k] + 1] = bad[offs[k]]  # a duplicate inside one list
    with pytest.raises(AssertionError):
        device_summary(torch, torch.from_numpy(offs), torch.from_numpy(bad), chunk=64)
