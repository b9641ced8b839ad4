"""`Engine.run` semantics on the device path (reference engine.py:370-417):
β = Σ queries / Σ durations['total'], verify=True against the brute force
(VerificationFailure on a deviation), keep_results, per-tick qos_pass, and the
module-level `run` / `process_tick` wrappers — with the kept result sets
checked against the reference engine's own digests (tests/golden/digests.json)."""

from __future__ import annotations

import dataclasses

import pytest

from conftest import workload_from_json
from oracle import quad_oracle as qo

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_1411_3212_b200 as p
    from paper_1411_3212_b200 import _native

    assert _native.device_count() > 0, "no CUDA device: the GPU tests need a B200"
    return p


def _config_a(n_ticks):
    from conftest import load_digests

    run = load_digests()["A"]
    cfg = dataclasses.replace(workload_from_json(run["workload"]), n_ticks=n_ticks)
    return cfg, run


def test_run_verify_keep_qos_object_api(pkg):
    cfg, ref = _config_a(3)
    work = pkg.generate(cfg)  # object API: TickBatch lists, like the reference's generate
    qos = pkg.QosParams(delta_t=0.05, lam=0.25, q_max=10_000)
    rep = pkg.run(work, pkg.MethodConfig(method="quad"), qos=qos, verify=True, keep_results=True)
    assert rep.label == "quad" and len(rep.stats) == 3 and len(rep.result_sets) == 3
    tot = sum(s.durations["total"] for s in rep.stats)
    assert rep.bandwidth == sum(s.n_queries for s in rep.stats) / tot  # engine.py:394-395
    for t, (st, rs) in enumerate(zip(rep.stats, rep.result_sets)):
        assert st.qos_pass == pkg.check_latency(st.durations["total"], qos)
        assert st.qos_pass == (qos.delta_t + st.durations["total"] <= qos.lam)
        assert qo.digest_lines(rs.lines()) == ref["ticks"][t]["digest"]  # the reference engine's results
        assert st.results_total == ref["ticks"][t]["stats"]["results_total"]
    assert pkg.min_bandwidth(qos) == qos.q_max / (qos.lam - qos.delta_t)


def test_run_columnar_without_results(pkg):
    cfg, ref = _config_a(2)
    eng = pkg.Engine(pkg.MethodConfig(method="quad"))
    try:
        rep = eng.run(list(pkg.iter_ticks(cfg)))
    finally:
        eng.close()
    assert rep.result_sets is None
    assert all(s.qos_pass is None for s in rep.stats)
    assert [s.results_total for s in rep.stats] == [ref["ticks"][t]["stats"]["results_total"] for t in range(2)]
    assert rep.bandwidth > 0


def test_verify_raises_on_deviation(pkg, monkeypatch):
    """A checker that disagrees makes run(verify=True) raise VerificationFailure."""
    from paper_1411_3212_b200 import engine as eng_mod
    from paper_1411_3212_b200 import errors

    cfg, _ = _config_a(1)
    real = eng_mod.brute_force_join

    def wrong(batch):
        rs = real(batch)
        q = next(iter(rs.by_query))
        rs.by_query[q] = rs.by_query[q] + [10 ** 12]
        return rs

    monkeypatch.setattr(eng_mod, "brute_force_join", wrong)
    with pytest.raises(errors.VerificationFailure):
        pkg.run(pkg.generate(cfg), pkg.MethodConfig(method="quad"), verify=True)


def test_module_process_tick(pkg):
    cfg, ref = _config_a(1)
    batch = pkg.generate(cfg).batches[0]
    rs, st = pkg.process_tick(batch, pkg.MethodConfig(method="quad"))
    assert qo.digest_lines(rs.lines()) == ref["ticks"][0]["digest"]
    assert st.tick == 0 and st.n_queries == len(batch.queries) and st.durations["total"] > 0
