"""Full-size GPU parity on every single-GPU BASELINE configuration.

Configs A (all ticks) and the small fixtures are checked elsewhere against
reference digests.  Here, at the sizes the bench runs:

* C @5u (the headline, 10M skewed objects): ticks 0 and 1 — the whole CSR
  equals the NumPy QUAD oracle's (`oracle/quad_oracle.run_tick`, the reference
  pipeline restated) together with its counters, and the C brute-force
  checker's; ticks 0..4 — the whole CSR equals the checker's.
* C @2u and C @10u: two ticks each, the whole CSR against the checker.
* C @20u (2.3e9 results per tick) and E (50M: 40M uniform + 10M extreme
  hotspot, 1u): two ticks each, every query's count and id digest against the
  checker.
* B (1M gaussian, 50u): five ticks against the REFERENCE ENGINE's own results
  (sha256 of its CSR, tests/golden/digests_b.json, made by
  tests/golden/make_b_golden.py) and all 20 ticks against the checker.
* On every tick: lists strictly ascending (so duplicate-free), offsets
  consistent, and >= 2,000 stratified queries (longest lists = hotspot cores
  and heaviest leaves, queries on the MBR edges, empty results, random)
  compared list by list.

The checker is `oracle/bf_join.c`, an exact restatement of the reference's
`brute_force_join` (oracle.py:17-28) pinned in tests/test_oracle_bf.py; the
reference's own tests assert engine == brute force (test_acceptance.py C1).
Per-query digests are sum(mix64(id)) mod 2^64 over the list; together with the
count and strict ascending order they pin the list.
"""

from __future__ import annotations

import ctypes
import hashlib
import json
import os

import numpy as np
import pytest

import bench
from oracle import bf_join as bf
from oracle import quad_oracle as qo
from csr_check import device_summary

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    assert torch.cuda.is_available(), "no CUDA device: the GPU tests need a B200"
    return torch


def _rt():
    rt = ctypes.CDLL("libcudart.so.12")
    rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    rt.cudaDeviceSynchronize.argtypes = []
    return rt


def device_tick(torch, ctx, tick):
    """One tick through tj_tick with device-resident inputs and outputs; the CSR is
    copied into torch tensors (int64 offsets m+1, int64 ids R)."""
    from paper_1411_3212_b200 import _native

    dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda()
           for a in (tick.ids, tick.xs, tick.ys, tick.qids, tick.qxa, tick.qya, tick.qxb, tick.qyb)]
    torch.cuda.synchronize()
    out, st = ctx.tick_ptrs(tick.n_objects, *(t.data_ptr() for t in dev[:3]), tick.n_queries,
                            *(t.data_ptr() for t in dev[3:]), _native.TJ_MEM_DEVICE, _native.TJ_MEM_DEVICE)
    assert out.id_bytes == 8 and out.offset_bytes == 8
    m, R = int(out.n_q), int(out.n_results)
    off = torch.empty(m + 1, dtype=torch.int64, device="cuda")
    ids = torch.empty(max(R, 1), dtype=torch.int64, device="cuda")[:R]
    rt = _rt()
    assert rt.cudaDeviceSynchronize() == 0
    assert rt.cudaMemcpy(off.data_ptr(), out.offsets, 8 * (m + 1), 3) == 0  # device to device
    if R:
        assert rt.cudaMemcpy(ids.data_ptr(), out.ids, 8 * R, 3) == 0
    assert rt.cudaDeviceSynchronize() == 0
    del dev
    return off, ids, st


def stratified_rows(tick, lens, k=600, seed=0):
    """Query rows to compare list by list: longest lists (hotspot cores, heaviest
    leaves), the rects nearest to (or across) the objects' MBR edges, empty lists,
    random."""
    rng = np.random.default_rng(seed)
    m = tick.n_queries
    longest = np.argsort(lens, kind="stable")[-k:]
    xa, ya, xb, yb = tick.xs.min(), tick.ys.min(), tick.xs.max(), tick.ys.max()
    gap = np.minimum(np.minimum(tick.qxa - xa, tick.qya - ya), np.minimum(xb - tick.qxb, yb - tick.qyb))
    edge = np.argsort(gap, kind="stable")[:k]  # negative gap: the rect crosses the MBR edge
    empty = rng.permutation(np.flatnonzero(lens == 0))[:k]
    rows = np.unique(np.concatenate([longest, edge, empty]).astype(np.int64))
    want = min(m, max(2000, len(rows) + k))  # top up with random rows: >= 2,000 distinct in all
    while len(rows) < want:
        rows = np.unique(np.concatenate([rows, rng.choice(m, want - len(rows), replace=False)]))
    return rows


def compare_rows(torch, tick, off, ids, g, rows):
    o_ref, r_ref = g.lists(tick.qxa, tick.qya, tick.qxb, tick.qyb, rows=rows)
    rows_t = torch.from_numpy(rows).cuda()
    lo, hi = off[rows_t], off[rows_t + 1]
    lens = (hi - lo)
    assert np.array_equal(lens.cpu().numpy(), np.diff(o_ref))
    if int(lens.sum()):
        idx = torch.repeat_interleave(lo - torch.cumsum(lens, 0) + lens, lens) + torch.arange(
            int(lens.sum()), device="cuda")
        got = ids[idx].cpu().numpy()
        assert np.array_equal(got, r_ref)


def check_tick(torch, ctx, tick, cell, label, full=False):
    off, ids, st = device_tick(torch, ctx, tick)
    assert int(st.results_total) == ids.numel()
    lens, dig = device_summary(torch, off, ids)
    g = bf.BruteForce(tick.ids, tick.xs, tick.ys, cell=cell)
    cnt, dig_ref = g.counts(tick.qxa, tick.qya, tick.qxb, tick.qyb)
    bad = np.flatnonzero((cnt != lens) | (dig_ref != dig))
    assert len(bad) == 0, f"{label}: {len(bad)} queries differ from the brute-force checker, e.g. rows {bad[:5]}"
    rows = stratified_rows(tick, lens, seed=int(st.results_total) & 0xFFFF)
    assert len(rows) >= 2000 or len(rows) >= tick.n_queries // 2
    compare_rows(torch, tick, off, ids, g, rows)
    if full:  # the whole CSR, list for list, against the checker's exact lists
        o_ref, r_ref = g.lists(tick.qxa, tick.qya, tick.qxb, tick.qyb)
        assert np.array_equal(off.cpu().numpy(), o_ref), f"{label}: offsets differ"
        assert np.array_equal(ids.cpu().numpy(), r_ref), f"{label}: ids differ"
        del o_ref, r_ref
    g.close()
    del off, ids
    torch.cuda.empty_cache()
    return st, lens


def _ctx():
    from paper_1411_3212_b200 import _native

    return _native.NativeContext(384, 12, True, 0, 0)


# ---------------------------------------------------------------- the headline --

@pytest.mark.parametrize("t", [0, 1])
def test_c5_whole_csr_equals_quad_oracle(t):
    """Config C @5u ticks 0 and 1: the whole CSR and the TickStats counters equal the
    NumPy restatement of the reference QUAD pipeline (about a minute per tick on the host)."""
    tick = list(bench.iter_workload("C5", t + 1))[t]
    ctx = _ctx()
    offs, res, st = ctx.tick_host(tick.ids, tick.xs, tick.ys, tick.qids, tick.qxa, tick.qya, tick.qxb, tick.qyb)
    ctx.close()
    ref = qo.run_tick(tick.ids, tick.xs, tick.ys, tick.qids, tick.qxa, tick.qya, tick.qxb, tick.qyb)
    assert np.array_equal(offs, ref.offsets)
    assert np.array_equal(res, ref.result_ids)
    for k in ("containment_tests", "decoded_bits", "subq_intersecting", "subq_covering", "covering_results",
              "active_cells", "results_total"):
        assert int(getattr(st, k)) == ref.counters[k], k
    assert int(st.n_leaves) == ref.counters["n_leaves"] and int(st.l_deep) == ref.counters["l_deep"]
    # and the brute-force checker agrees list for list
    g = bf.BruteForce(tick.ids, tick.xs, tick.ys, cell=5.0)
    o2, r2 = g.lists(tick.qxa, tick.qya, tick.qxb, tick.qyb)
    g.close()
    assert np.array_equal(offs, o2) and np.array_equal(res, r2)


# (workload, ticks, checker cell size, whole CSR compared list for list as well)
FULL = [("C5", 5, 5.0, True), ("C2", 2, 4.0, True), ("C10", 2, 10.0, True), ("C20", 2, 20.0, False),
        ("E", 2, 2.0, False)]


@pytest.mark.parametrize("name,ticks,cell,full", FULL, ids=[f[0] for f in FULL])
def test_fullsize_every_query(torch_cuda, name, ticks, cell, full):
    ctx = _ctx()
    try:
        for tick in bench.iter_workload(name, ticks):
            st, lens = check_tick(torch_cuda, ctx, tick, cell, f"{name} tick {tick.tick_index}", full=full)
            if name == "C5" and tick.tick_index == 0:  # SURVEY.md §8 measured sizes (reference, tick 0)
                assert int(st.results_total) == 169_197_114
                assert int(st.n_leaves) == 60_820 and int(st.l_deep) == 11
                assert int(st.subq_intersecting) == 16_845_566 and int(st.subq_covering) == 0
    finally:
        ctx.close()


def _b_golden():
    with open(os.path.join(HERE, "golden", "digests_b.json")) as fp:
        return json.load(fp)


def test_config_b_matches_reference_engine(torch_cuda):
    """Config B (1M gaussian, 50u): the reference engine's own results, per tick."""
    gold = _b_golden()
    from conftest import workload_from_json
    from paper_1411_3212_b200.workload import iter_ticks

    ctx = _ctx()
    for t, tick in enumerate(iter_ticks(workload_from_json(gold["workload"]))):
        want = gold["ticks"][t]
        offs, res, st = ctx.tick_host(tick.ids, tick.xs, tick.ys, tick.qids, tick.qxa, tick.qya, tick.qxb,
                                      tick.qyb)
        for k, v in want["stats"].items():
            assert int(getattr(st, k)) == v, (t, k)
        order = np.argsort(tick.qids, kind="stable")  # CSR in ascending issuer order
        lens = np.diff(offs)[order]
        o2 = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        idx = np.repeat(offs[:-1][order] - o2[:-1], lens) + np.arange(int(o2[-1]))
        h = hashlib.sha256()
        h.update(o2.tobytes())
        h.update(res[idx].astype(np.int64).tobytes())
        assert h.hexdigest() == want["csr_sha256"], t
    ctx.close()


def test_config_b_all_ticks_every_query(torch_cuda):
    ctx = _ctx()
    try:
        for tick in bench.iter_workload("B", 20):
            check_tick(torch_cuda, ctx, tick, 50.0, f"B tick {tick.tick_index}")
    finally:
        ctx.close()
