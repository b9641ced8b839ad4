"""The tick API, unchanged from the reference, running on the B200 pipeline.

Same names, fields, defaults and error behaviour as `tickjoin/engine.py`
(`MethodConfig` 57-96, `TickStats` 99-121, `RunReport` 124-134, `Engine`
137-402, module-level `process_tick`/`run` 405-417, QoS helpers 42-54) for
method "quad".  Underneath, one `tj_tick` call (include/tickjoin_b200.h) runs
the whole tick on the GPU.  Method "ug" (the uniform grid, `grid.py`) runs
the same kernels with the grid's cells as the leaves (split factors up to
4096; `split_factor=None` sweeps the candidates on the first tick, each
candidate's cost measured by the device pipeline).  "ug_baseline" (the
reference's direct-emission comparison path, baseline.py) returns the same
results through the same pipeline and reports the reference's contention
counters (`sync_ops`, `flushes`: the staging-buffer flushes, counted on the
device) with no decode phase (`decoded_bits` 0).  There is no CPU or
multi-backend fallback.

Besides the object API, `Engine.process_columns` is the columnar fast path
(NumPy host arrays or CUDA tensors in, CSR out) that avoids building millions
of Python objects (SURVEY.md §7 hard part 6).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Optional, Sequence, Union

import numpy as np

from . import _native
from .errors import BadConfig, BadQos, VerificationFailure
from .geometry import TickBatch, object_arrays, query_arrays
from .results import ColumnarResult, ResultSet
from .verify import brute_force_join
from .workload import ColumnarTick, WorkloadRun

L_MAX = 12
METHODS = ("ug", "ug_baseline", "quad")
BUILT_METHODS = ("quad", "ug", "ug_baseline")
MAX_DEVICE_SPLIT_FACTOR = 4096  # the grid is kept as a dense 2^12 x 2^12 cell map
DEFAULT_SWEEP = (16, 256, 16)  # engine.py:30


@dataclass(frozen=True)
class QosParams:
    delta_t: float
    lam: float
    q_max: int


def check_latency(exec_time: float, qos: QosParams) -> bool:
    """Queueing (one tick) plus execution within lam, inclusive (engine.py:42-47)."""
    return qos.delta_t + exec_time <= qos.lam


def min_bandwidth(qos: QosParams) -> float:
    """Queries per time unit needed to absorb q_max (engine.py:50-54)."""
    if qos.lam <= qos.delta_t:
        raise BadQos(f"latency threshold {qos.lam} must exceed tick duration {qos.delta_t}")
    return qos.q_max / (qos.lam - qos.delta_t)


@dataclass
class MethodConfig:
    method: str = "quad"
    split_factor: Optional[int] = None
    sweep: Optional[tuple] = None
    th_quad: int = 384
    l_max: int = L_MAX
    covering_optimization: bool = True
    schedule: str = "heaviest_first"
    n_workers: int = 1
    chunk_size: int = 64
    rebuild: str = "every_tick"
    sim_processors: int = 8
    staging_capacity: int = 1024
    label: Optional[str] = None
    device: int = 0  # CUDA ordinal (B200 addition)

    def validate(self) -> None:
        if self.method not in METHODS:
            raise BadConfig(f"unknown method {self.method!r}")
        if self.method not in BUILT_METHODS:
            raise BadConfig(f"method {self.method!r} is not part of the B200 build (quad, ug)")
        if self.method == "quad":
            if self.th_quad < 1:
                raise BadConfig("th_quad must be >= 1")
            if not 1 <= self.l_max <= L_MAX:
                raise BadConfig(f"l_max must be in [1, {L_MAX}]")
        elif self.split_factor is not None:
            if self.split_factor < 1:
                raise BadConfig("split_factor must be >= 1")
            if self.split_factor > MAX_DEVICE_SPLIT_FACTOR:
                raise BadConfig(f"split factors above {MAX_DEVICE_SPLIT_FACTOR} are not supported on the B200 path")
        if self.schedule not in ("heaviest_first", "unordered"):
            raise BadConfig(f"unknown schedule {self.schedule!r}")
        if self.n_workers < 1 or self.chunk_size < 1 or self.sim_processors < 1:
            raise BadConfig("n_workers, chunk_size and sim_processors must be >= 1")
        if self.rebuild not in ("every_tick", "adaptive"):
            raise BadConfig(f"unknown rebuild policy {self.rebuild!r}")

    @property
    def name(self) -> str:
        return self.label or self.method

    def sweep_candidates(self) -> list:
        lo, hi, step = self.sweep or DEFAULT_SWEEP  # engine.py:93-95
        return list(range(lo, hi + 1, step))


@dataclass
class TickStats:
    tick: int
    method: str
    n_objects: int = 0
    n_queries: int = 0
    containment_tests: int = 0
    decoded_bits: int = 0
    subq_intersecting: int = 0
    subq_covering: int = 0
    covering_results: int = 0
    covering_result_fraction: float = 0.0
    active_cells: int = 0
    occupancy_mean: float = 0.0
    occupancy_var: float = 0.0
    dispersion: float = 0.0
    imbalance: float = 0.0
    sync_ops: int = 0
    flushes: int = 0
    results_total: int = 0
    split_factor: Optional[int] = None
    durations: dict = field(default_factory=dict)
    qos_pass: Optional[bool] = None
    # B200 additions
    n_leaves: int = 0
    l_deep: int = 0
    rebuilt: bool = True  # rebuild="adaptive": False when the previous tick's index was reused
    device_ms: dict = field(default_factory=dict)
    # how the device put result lists in id order: "monotone" (ids increase with the input row),
    # "keyed" (leaf blocks in id order with 32-bit id offsets), "sorted" (per-list sorts;
    # see tj_stats.id_order)
    id_order: str = "monotone"


@dataclass
class RunReport:
    label: str
    stats: list
    bandwidth: float
    result_sets: Optional[list] = None
    sweep_costs: Optional[list] = None

    @property
    def total_queries(self) -> int:
        return sum(s.n_queries for s in self.stats)


def _fill_stats(stats: TickStats, st: "_native.TjStats") -> None:
    stats.containment_tests = int(st.containment_tests)
    stats.decoded_bits = int(st.decoded_bits)
    stats.subq_intersecting = int(st.subq_intersecting)
    stats.subq_covering = int(st.subq_covering)
    stats.covering_results = int(st.covering_results)
    stats.active_cells = int(st.active_cells)
    stats.results_total = int(st.results_total)
    stats.n_leaves = int(st.n_leaves)
    stats.l_deep = int(st.l_deep)
    stats.rebuilt = bool(st.rebuilt)
    stats.id_order = ("monotone", "keyed", "sorted")[int(st.id_order)]
    if stats.results_total:
        stats.covering_result_fraction = stats.covering_results / stats.results_total
    a = int(st.active_cells)
    if a:
        s1, s2 = int(st.occ_sum), int(st.occ_sumsq)
        stats.occupancy_mean = s1 / a
        stats.occupancy_var = (a * s2 - s1 * s1) / (a * a)  # exact rational, one rounding; the engine
        # replaces mean / var with NumPy's reductions over the per-leaf counts (bit-identical to the
        # reference) unless full_stats is off
        stats.dispersion = stats.occupancy_var / stats.occupancy_mean
    stats.device_ms = dict(index=st.t_index_ms, filter=st.t_filter_ms, decode=st.t_decode_ms,
                           merge=st.t_merge_ms, total=st.t_total_ms)


class Engine:
    """Processes ticks one at a time for a fixed method configuration."""

    def __init__(self, cfg: MethodConfig) -> None:
        cfg.validate()
        self.cfg = cfg
        self._split_factor = cfg.split_factor
        self.sweep_costs = None
        self._ctx = None
        if cfg.method == "quad" or self._split_factor is not None:
            self._ctx = self._make_ctx(self._split_factor)

    def _make_ctx(self, split_factor):
        cfg = self.cfg
        if cfg.method in ("ug", "ug_baseline"):
            return _native.NativeContext(1, L_MAX, cfg.covering_optimization, 0, cfg.device, split_factor)
        rebuild = _native.TJ_REBUILD_ADAPTIVE if cfg.rebuild == "adaptive" else _native.TJ_REBUILD_EVERY_TICK
        return _native.NativeContext(cfg.th_quad, cfg.l_max, cfg.covering_optimization, rebuild, cfg.device)

    def _sweep(self, ids, xs, ys, qids, qxa, qya, qxb, qyb) -> None:
        """Split-factor sweep on the first tick (engine.py:152-156, grid.py:125-165): each
        candidate's cost is tests + decoded bitmap bits, as the device pipeline counts them
        (containment_tests + decoded_bits); the cheapest wins, ties to the smaller factor.
        The sweep ignores covering_optimization, like the reference's."""
        costs = []
        for sf in self.cfg.sweep_candidates():
            if sf < 1 or sf > MAX_DEVICE_SPLIT_FACTOR:
                raise BadConfig(f"sweep candidate {sf} outside [1, {MAX_DEVICE_SPLIT_FACTOR}]")
            ctx = _native.NativeContext(1, L_MAX, True, 0, self.cfg.device, sf)
            try:
                _, _, st = ctx.tick_host(ids, xs, ys, qids, qxa, qya, qxb, qyb)
            finally:
                ctx.close()
            costs.append((sf, int(st.containment_tests) + int(st.decoded_bits)))
        self.sweep_costs = costs
        self._split_factor = min(costs, key=lambda c: (c[1], c[0]))[0]
        self._ctx = self._make_ctx(self._split_factor)

    @property
    def split_factor(self) -> Optional[int]:
        return self._split_factor

    @property
    def native(self) -> "_native.NativeContext":
        """The native context (introspection of the last tick)."""
        return self._ctx

    def close(self) -> None:
        if self._ctx is not None:
            self._ctx.close()

    # -- columnar fast path ----------------------------------------------------
    def process_columns(self, ids, xs, ys, qids, qxa, qya, qxb, qyb, tick_index: int = 0,
                        full_stats: bool = True) -> tuple:
        """SoA host arrays in; (ColumnarResult, TickStats) out."""
        t0 = time.perf_counter()
        if self._ctx is None:  # method "ug" without a split factor: sweep on this (first) tick
            if len(ids) == 0:
                return ColumnarResult(np.asarray(qids, np.int64), np.zeros(len(qids) + 1, np.int64),
                                      np.zeros(0, np.int64)), TickStats(tick=tick_index, method=self.cfg.name,
                                                                         n_queries=len(qids))
            self._sweep(ids, xs, ys, qids, qxa, qya, qxb, qyb)
        offs, res, st = self._ctx.tick_host(ids, xs, ys, qids, qxa, qya, qxb, qyb)
        t1 = time.perf_counter()
        stats = TickStats(tick=tick_index, method=self.cfg.name, n_objects=len(ids), n_queries=len(qids))
        if self.cfg.method in ("ug", "ug_baseline"):
            stats.split_factor = self._split_factor
        if len(ids):
            _fill_stats(stats, st)
            if full_stats and stats.active_cells:  # engine.py:261-267 on the same array, in NumPy
                occ = self._ctx.occupancy()
                stats.occupancy_mean = float(occ.mean())
                stats.occupancy_var = float(occ.var())
                stats.dispersion = stats.occupancy_var / stats.occupancy_mean
            if full_stats and stats.containment_tests:
                stats.imbalance = self._ctx.imbalance(self.cfg.sim_processors,
                                                      self.cfg.schedule == "heaviest_first")
        if self.cfg.method == "ug_baseline" and len(ids):  # engine.py:232-236, baseline.py:26-121
            stats.decoded_bits = 0
            stats.sync_ops = stats.flushes = self._ctx.staging_flushes(self.cfg.staging_capacity)
        d = stats.device_ms
        stats.durations = {k: d.get(k, 0.0) / 1e3 for k in ("index", "filter", "decode", "merge")}
        stats.durations["total"] = t1 - t0
        return ColumnarResult(np.asarray(qids, np.int64), offs, res), stats

    def process_tick_columnar(self, tick: ColumnarTick, full_stats: bool = True) -> tuple:
        return self.process_columns(tick.ids, tick.xs, tick.ys, tick.qids, tick.qxa, tick.qya, tick.qxb,
                                    tick.qyb, tick_index=tick.tick_index, full_stats=full_stats)

    # -- object API (engine.py:178-259) ------------------------------------------
    def process_tick(self, batch: TickBatch) -> tuple:
        t0 = time.perf_counter()
        ids, xs, ys = object_arrays(batch.objects)
        qids, qxa, qya, qxb, qyb = query_arrays(batch.queries)
        res, stats = self.process_columns(ids, xs, ys, qids, qxa, qya, qxb, qyb, tick_index=batch.tick_index)
        rs = res.to_result_set()
        stats.durations["total"] = time.perf_counter() - t0
        return rs, stats

    def run(self, workload: Union[WorkloadRun, Sequence[ColumnarTick]], qos: Optional[QosParams] = None,
            verify: bool = False, keep_results: bool = False) -> RunReport:
        """engine.py:370-402: β = Σ queries / Σ durations['total']."""
        stats_list, kept = [], []
        total = 0.0
        batches = workload.batches if isinstance(workload, WorkloadRun) else list(workload)
        for b in batches:
            if isinstance(b, ColumnarTick):
                res, stats = self.process_tick_columnar(b)
                rs = res.to_result_set() if (verify or keep_results) else None
                if verify:
                    expected = brute_force_join(b.to_batch())
            else:
                rs, stats = self.process_tick(b)
                if verify:
                    expected = brute_force_join(b)
            if verify and rs != expected:
                raise VerificationFailure(f"tick {stats.tick}: {self.cfg.name} deviates from the oracle")
            if qos is not None:
                stats.qos_pass = check_latency(stats.durations["total"], qos)
            total += stats.durations["total"]
            stats_list.append(stats)
            if keep_results:
                kept.append(rs)
        queries = sum(s.n_queries for s in stats_list)
        return RunReport(label=self.cfg.name, stats=stats_list,
                         bandwidth=queries / total if total > 0 else 0.0,
                         result_sets=kept if keep_results else None, sweep_costs=self.sweep_costs)


def process_tick(batch: TickBatch, cfg: MethodConfig) -> tuple:
    eng = Engine(cfg)
    try:
        return eng.process_tick(batch)
    finally:
        eng.close()


def run(workload, cfg: MethodConfig, qos: Optional[QosParams] = None, verify: bool = False,
        keep_results: bool = False) -> RunReport:
    eng = Engine(cfg)
    try:
        return eng.run(workload, qos=qos, verify=verify, keep_results=keep_results)
    finally:
        eng.close()
