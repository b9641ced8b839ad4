#!/usr/bin/env python
"""bench.py — QUAD repeated-range-query tick throughput on B200.

Metric (BASELINE.json): range queries/sec (and p50 tick latency) at 10M
skewed objects.  Workload at N=1: config C of SURVEY.md §8(d) — 10,000,000
Gaussian-hotspot objects (25 hotspots, sigma 225u, region 22500u), 100% query
rate, square 5u queries, seed 3, every tick a full index rebuild.  Inputs are
synthetic, produced by the RNG-identical columnar generator; each tick's
inputs (560 MB) exceed the 126 MB L2, so no flush is needed between steps.

A step = one `tj_tick` (index build -> query scatter -> per-leaf bitmap join
-> decode -> canonical per-query lists) over one tick.

  python bench.py [--gpus N --steps K --warmup W]           # our arm
  python bench.py --impl reference [...]                    # CPU reference arm (tickjoin from baseline/_ref)

Under torchrun (N>1) the same 10M-object tick is split over the ranks: each
rank holds 1/N of the updates and queries, an NCCL all-gather gives every rank
the whole tick, every rank builds the (bit-identical) index and joins and
decodes only its contiguous Morton leaf range.
Strong scaling; rank 0 prints the max-over-ranks device time.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "range queries/sec at 10M skewed objects (p50 tick latency alongside)"
UNIT = "queries/s"

WORKLOADS = {
    # SURVEY.md §8(d) config C at 5u (the BASELINE metric's config)
    "C5": dict(n_objects=10_000_000, query_rate=1.0, query_side=5.0, distribution="gaussian", n_hotspots=25,
               seed=3),
    # config B (1M gaussian, 50u) and A (uniform 100K, 10%) for side runs
    "B": dict(n_objects=1_000_000, query_rate=1.0, query_side=50.0, distribution="gaussian", n_hotspots=25,
              seed=2),
    "A": dict(n_objects=100_000, query_rate=0.1, query_side=(200.0, 800.0), distribution="uniform", seed=1),
    # config C at its other query sides
    "C2": dict(n_objects=10_000_000, query_rate=1.0, query_side=2.0, distribution="gaussian", n_hotspots=25,
               seed=3),
    "C10": dict(n_objects=10_000_000, query_rate=1.0, query_side=10.0, distribution="gaussian", n_hotspots=25,
                seed=3),
    "C20": dict(n_objects=10_000_000, query_rate=1.0, query_side=20.0, distribution="gaussian", n_hotspots=25,
                seed=3),
    # config E: 40M uniform (seed 5) + 10M in one extreme hotspot (sigma 100u, seed 6), ids of the
    # second part offset by 40M, 1u queries at 100% rate, each part moved by its own generator
    "E": [dict(n_objects=40_000_000, query_rate=1.0, query_side=1.0, distribution="uniform", seed=5),
          dict(n_objects=10_000_000, query_rate=1.0, query_side=1.0, distribution="gaussian", n_hotspots=1,
               sigma=100.0, seed=6)],
}
DESCR = {
    "C5": "skewed 10M objects (gaussian, 25 hotspots, sigma 225u), 100% query rate, 5u squares, seed 3",
    "B": "gaussian 1M objects, 100% query rate, 50u squares, seed 2",
    "A": "uniform 100K objects, 10% query rate, sides U[200,800]u, seed 1",
    "C2": "skewed 10M objects (gaussian, 25 hotspots, sigma 225u), 100% query rate, 2u squares, seed 3",
    "C10": "skewed 10M objects (gaussian, 25 hotspots, sigma 225u), 100% query rate, 10u squares, seed 3",
    "C20": "skewed 10M objects (gaussian, 25 hotspots, sigma 225u), 100% query rate, 20u squares, seed 3",
    "E": "50M objects: 40M uniform (seed 5) + 10M extreme hotspot (1 hotspot, sigma 100u, seed 6), 100% rate, 1u",
}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fp:
            return float(json.load(fp)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str):
    """Per-launch dram bytes of `kernel` from the committed ncu summary (profiles/)."""
    import glob

    # the newest round first, its final capture before earlier ones
    paths = glob.glob(os.path.join(ROOT, "profiles", "*ncu_summary*.json"))
    for p in sorted(paths, key=lambda q: (os.path.basename(q)[:3], "final" in q, q), reverse=True):
        try:
            with open(p) as fp:
                d = json.load(fp)
            ks = d.get("kernels", {})
            k = ks.get(kernel) or next((v for name, v in ks.items() if name.startswith(kernel + "<")), None)
            if k and k.get("dram_bytes_per_launch"):
                return float(k["dram_bytes_per_launch"]), os.path.relpath(p, ROOT)
        except Exception:
            continue
    return None, None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up takes driver locks: let it settle before the timed region
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 5.0:
                time.sleep(0.01)
            self.lines.clear()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def iter_workload(name: str, count: int, seed_offset: int = 0):
    """The workload's first `count` ticks, lazily (one tick in memory at a time)."""
    import numpy as np

    from paper_1411_3212_b200.workload import ColumnarTick, WorkloadConfig, iter_ticks

    spec = WORKLOADS[name]
    parts = spec if isinstance(spec, list) else [spec]
    streams = []
    for kw in parts:
        kw = dict(kw)
        kw["seed"] = kw["seed"] + seed_offset
        streams.append(iter_ticks(WorkloadConfig(n_ticks=count, **kw)))
    if len(streams) == 1:
        yield from streams[0]
        return
    for k, ts in enumerate(zip(*streams)):
        off = 0
        cols = {c: [] for c in ("ids", "xs", "ys", "qids", "qxa", "qya", "qxb", "qyb")}
        for t in ts:
            cols["ids"].append(t.ids + off)
            cols["qids"].append(t.qids + off)
            for c in ("xs", "ys", "qxa", "qya", "qxb", "qyb"):
                cols[c].append(getattr(t, c))
            off += t.n_objects
        yield ColumnarTick(k, **{c: np.concatenate(v) for c, v in cols.items()})


def gen_ticks(name: str, count: int, seed_offset: int = 0):
    return list(iter_workload(name, count, seed_offset))


class RefEngineSample:
    """The REFERENCE engine (`tickjoin`, installed unmodified in baseline/_ref) on a bounded
    sample of the bench workload's tick, through its public API
    `Engine(MethodConfig("quad", n_workers=...)).process_tick(TickBatch)` (engine.py:178-259).

    A full C5 tick takes the reference minutes (10M objects, 10M queries), so a step is one
    `process_tick` on ALL the tick's objects with one chunk of its queries: the queries sorted by
    the Morton code of their centres and cut into `k` contiguous chunks of m/k (compact regions,
    so every chunk carries its leaves' whole per-task cost, not a thin slice of it).  D0 = the
    same call with no queries (the index build over all objects; median of the warm-up runs).
    A chunk's tick-time estimate is D0 + k * (D_chunk - D0); the value is m over the mean estimate.
    Object construction (Python objects, untimed by the reference too) happens once, up front.
    """

    def __init__(self, workload: str = "C5", k: int = 100, n_workers: int = 0, tick_index: int = 0):
        import numpy as np

        p = os.path.join(ROOT, "baseline", "_ref")
        if not os.path.isdir(os.path.join(p, "tickjoin")):
            raise FileNotFoundError("baseline/_ref/tickjoin is not installed (see DESIGN.md §6)")
        if p not in sys.path:
            sys.path.insert(0, p)
        from tickjoin import engine as ref_engine
        from tickjoin import geometry as ref_geom

        self.E, self.G = ref_engine, ref_geom
        self.n_workers = n_workers or (os.cpu_count() or 1)
        it = iter_workload(workload, tick_index + 1)
        for tick in it:
            pass
        self.tick = tick
        self.m = int(tick.n_queries)
        self.k = max(1, min(k, self.m))
        G = ref_geom
        t0 = time.perf_counter()
        self.objects = [G.MovingObject(i, G.Point(x, y))
                        for i, x, y in zip(tick.ids.tolist(), tick.xs.tolist(), tick.ys.tolist())]
        self.setup_s = time.perf_counter() - t0
        # Morton order of the query centres (16 bits per axis over the queries' extent)
        cx = (tick.qxa + tick.qxb) * 0.5
        cy = (tick.qya + tick.qyb) * 0.5

        def q16(v):
            lo, hi = float(v.min()), float(v.max())
            s = 65535.0 / (hi - lo) if hi > lo else 0.0
            return np.minimum(((v - lo) * s).astype(np.int64), 65535).astype(np.uint64)

        def spread(v):
            v = (v | (v << np.uint64(16))) & np.uint64(0x0000FFFF0000FFFF)
            v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF00FF00FF)
            v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F0F0F0F0F)
            v = (v | (v << np.uint64(2))) & np.uint64(0x3333333333333333)
            return (v | (v << np.uint64(1))) & np.uint64(0x5555555555555555)

        code = spread(q16(cx)) | (spread(q16(cy)) << np.uint64(1))
        self.order = np.argsort(code, kind="stable")
        self.d0 = []

    def _engine(self):
        return self.E.Engine(self.E.MethodConfig(method="quad", n_workers=self.n_workers))

    def chunk_queries(self, j: int):
        t, G = self.tick, self.G
        lo, hi = (j * self.m) // self.k, ((j + 1) * self.m) // self.k
        rows = self.order[lo:hi]
        return [G.Query(int(q), G.Rect(a, b, c, d)) for q, a, b, c, d in
                zip(t.qids[rows].tolist(), t.qxa[rows].tolist(), t.qya[rows].tolist(), t.qxb[rows].tolist(),
                    t.qyb[rows].tolist())]

    def run_d0(self) -> float:
        _, st = self._engine().process_tick(self.G.TickBatch(self.tick.tick_index, self.objects, []))
        self.d0.append(st.durations["total"])
        return self.d0[-1]

    def run_chunk(self, j: int) -> dict:
        qs = self.chunk_queries(j)
        gc.collect()
        _, st = self._engine().process_tick(self.G.TickBatch(self.tick.tick_index, self.objects, qs))
        d0 = statistics.median(self.d0)
        dur = dict(st.durations)
        est = d0 + self.k * (dur["total"] - d0)
        stages = {"index_objects": d0, "index_queries": self.k * (dur["index"] - d0),
                  "filter": self.k * dur["filter"], "decode": self.k * dur["decode"],
                  "merge": self.k * dur.get("merge", 0.0)}
        return {"chunk": j, "queries": len(qs), "D_s": dur["total"], "est_tick_s": est, "stages_s": stages,
                "results": int(st.results_total)}

    def spread_chunks(self, count: int):
        """`count` chunk indices spread evenly over the k chunks (dense and sparse regions alike)."""
        return [(i * self.k) // count + (self.k // (2 * count)) for i in range(count)]


def reference_sample_text(rs: "RefEngineSample", steps: int) -> str:
    return (f"reference tickjoin Engine(MethodConfig('quad', n_workers={rs.n_workers})).process_tick from "
            f"baseline/_ref on the C5 tick {rs.tick.tick_index}: all {rs.tick.n_objects:,} objects with one "
            f"Morton-contiguous chunk of {rs.m // rs.k:,} of its {rs.m:,} queries per step ({steps} chunk(s) spread "
            f"over the k={rs.k} chunks); tick time = D0 + k*(D_chunk - D0), D0 = the same call with no queries "
            f"(index build over all objects, median {statistics.median(rs.d0):.2f} s); the reference's threads "
            f"share one GIL (effectively one core)")


def cpu_reference_sample(n_objects: int, seed: int = 3):
    """The CPU reference (oracle port, oracle/quad_oracle.py) on one tick of the same
    generator configuration with `n_objects` objects; returns (queries/s, seconds, m)."""
    from oracle import quad_oracle as qo
    from paper_1411_3212_b200.workload import WorkloadConfig, iter_ticks

    kw = dict(WORKLOADS["C5"])
    kw["n_objects"] = n_objects
    kw["seed"] = seed
    tick = next(iter_ticks(WorkloadConfig(n_ticks=1, **kw)))
    t0 = time.perf_counter()
    qo.run_tick(tick.ids, tick.xs, tick.ys, tick.qids, tick.qxa, tick.qya, tick.qxb, tick.qyb)
    dt = time.perf_counter() - t0
    return tick.n_queries / dt, dt, tick.n_queries


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    try:
        rs = RefEngineSample(args.workload, k=args.ref_chunks)
    except FileNotFoundError as e:
        print(f"reference engine unavailable ({e}); timing the NumPy port instead", file=sys.stderr)
        return run_reference_port(args)
    for _ in range(max(1, args.warmup)):  # warm-up: the no-query calls that give D0
        rs.run_d0()
    runs = [rs.run_chunk(j) for j in rs.spread_chunks(args.steps)]
    est = [r["est_tick_s"] for r in runs]
    value = rs.m / statistics.mean(est)
    stages = {k: statistics.mean(r["stages_s"][k] for r in runs) for k in runs[0]["stages_s"]}
    sample = reference_sample_text(rs, args.steps)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(est),
        "p50_tick_ms": 1e3 * statistics.median(est), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (RNG-identical reference generator)",
        "config": ref_config(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                         "sample": sample, "n_workers": rs.n_workers, "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_stage_s_per_tick": stages,
        "reference_runs": [{k: v for k, v in r.items() if k != "stages_s"} for r in runs],
        "object_setup_s": rs.setup_s,
    }
    print(json.dumps(line), flush=True)
    return 0


def ref_config(args):
    """The `config` object of both arms (identical, so the two lines describe the same workload)."""
    return {"workload": args.workload, "description": DESCR[args.workload], "method": "quad", "th_quad": 384,
            "l_max": 12, "rebuild": "every_tick",
            "l2": "inputs (>=560 MB/tick at 10M) exceed the 126 MB L2; no flush"}


def cpu_baseline_line(args):
    """`cpu_baseline` of our arm: the reference engine on one bounded chunk of the same tick
    (RefEngineSample: D0 once + the middle chunk, about 30 s of CPU work); the NumPy port if the
    reference is not installed."""
    try:
        rs = RefEngineSample(args.workload, k=args.ref_chunks)
    except FileNotFoundError:
        qps, dt, m = cpu_reference_sample(args.cpu_sample)
        return {"value": qps, "unit": UNIT, "cores": 1, "kind": "port",
                "sample": (f"oracle/quad_oracle.run_tick (NumPy port of the reference QUAD tick) on one tick of "
                           f"{args.cpu_sample:,} objects / {m:,} queries with the workload's generator config; "
                           f"{dt:.1f} s single-threaded (baseline/_ref not installed)")}
    rs.run_d0()
    r = rs.run_chunk(rs.k // 2)
    return {"value": rs.m / r["est_tick_s"], "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
            "sample": reference_sample_text(rs, 1), "n_workers": rs.n_workers,
            "est_tick_s": r["est_tick_s"], "stages_s": r["stages_s"]}


def run_reference_port(args):
    rank, world, _ = dist_env()
    n_sample = args.ref_sample
    times, qs = [], []
    for s in range(args.warmup + args.steps):
        qps, dt, m = cpu_reference_sample(n_sample, seed=3 + s)
        if s >= args.warmup:
            times.append(dt)
            qs.append(m)
    value = sum(qs) / sum(times)
    sample = (f"oracle/quad_oracle.run_tick (NumPy port of the reference QUAD tick), one tick per step of "
              f"{n_sample:,} objects with the workload's generator config (gaussian, 25 hotspots, 100% rate, "
              f"5u), seeds 3..{3 + args.warmup + args.steps - 1}")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "p50_tick_ms": 1e3 * statistics.median(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (RNG-identical reference generator)",
        "config": ref_config(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class Shard:
    """This rank's slice of one tick: a contiguous 1/G of the objects and of the queries
    (device resident, or pinned host memory for the end-to-end leg).  tj_tick_sharded
    gathers the slices into the full tick on every rank (NCCL), runs the rank's Morton range
    of leaves, routes every query's partial lists to its home rank and merges them there."""

    def __init__(self, tick, rank, world, dev, pinned=False):
        import numpy as np
        import torch

        n, m = int(tick.n_objects), int(tick.n_queries)
        o0, o1 = rank * n // world, (rank + 1) * n // world
        q0, q1 = rank * m // world, (rank + 1) * m // world
        self.n, self.m, self.n_total, self.m_total = o1 - o0, q1 - q0, n, m

        def part(a, lo, hi):
            t = torch.from_numpy(np.ascontiguousarray(a[lo:hi]))
            return t.pin_memory() if pinned else t.to(dev)

        self.cols = [part(a, o0, o1) for a in (tick.ids, tick.xs, tick.ys)] + \
                    [part(a, q0, q1) for a in (tick.qxa, tick.qya, tick.qxb, tick.qyb)]

    def ptrs(self):
        return [x.data_ptr() if x.numel() else 0 for x in self.cols]

    def nbytes(self):
        return sum(x.numel() * x.element_size() for x in self.cols)


def run_ours(args):
    import numpy as np
    import torch

    from paper_1411_3212_b200 import Engine, MethodConfig, _native

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or args.sharded
    if sharded:
        import torch.distributed as dist

        for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29517"), ("RANK", "0"), ("WORLD_SIZE", "1")):
            os.environ.setdefault(k, v)
        dist.init_process_group("nccl", device_id=dev)
    pool = max(1, min(args.pool, args.steps + args.warmup))
    ticks = gen_ticks(args.workload, pool)  # the same ticks on every rank
    if args.shuffle_ids:  # ids not increasing in input order: every tick a fresh permutation of 0..n-1
        from paper_1411_3212_b200.workload import ColumnarTick

        rng_ids = np.random.default_rng(12345)
        ticks = [ColumnarTick(t.tick_index, ids=rng_ids.permutation(t.n_objects).astype(np.int64), xs=t.xs,
                              ys=t.ys, qids=t.qids, qxa=t.qxa, qya=t.qya, qxb=t.qxb, qyb=t.qyb) for t in ticks]
    sf = args.split_factor if args.method == "ug" else 0
    eng = Engine(MethodConfig(method=args.method, split_factor=sf or None, device=local))
    ctx = eng.native

    def new_ctx():
        return _native.NativeContext(384, 12, True, 0, local, sf)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)
    if sharded:  # NCCL communicator inside the library; rank 0's unique id shared over torch.distributed
        import torch.distributed as dist

        uid = [_native.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.comm_init(uid[0], rank, world)
        shards = [Shard(t, rank, world, dev) for t in ticks]
    dticks = [[torch.from_numpy(a).to(dev) for a in (t.ids, t.xs, t.ys, t.qids, t.qxa, t.qya, t.qxb, t.qyb)]
              for t in ticks] if (not sharded or rank == 0) else None

    def tick_dev(k):
        if sharded:  # this rank's slice in, the complete lists of this rank's queries out
            sh = shards[k % pool]
            p = sh.ptrs()
            out, st = ctx.tick_sharded_ptrs(sh.n, *p[:3], sh.m, *p[3:], _native.TJ_MEM_DEVICE,
                                            _native.TJ_MEM_DEVICE)
            return out, st, sh.m_total
        a = dticks[k % pool]
        n, m = a[0].numel(), a[3].numel()
        out, st = ctx.tick_ptrs(n, *(x.data_ptr() for x in a[:3]), m, *(x.data_ptr() for x in a[3:]),
                                _native.TJ_MEM_DEVICE, _native.TJ_MEM_DEVICE)
        return out, st, m

    # the clock sampler starts before the warm-up (its start-up otherwise leaves the GPU idle,
    # clocks ramp down, and the first timed tick pays the ramp); samples are kept from the
    # timed region only
    clocks = ClockSampler(local)
    clocks.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    gc.collect()
    for k in range(args.warmup):
        tick_dev(k)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.lines.clear()
    gc.disable()  # no collector pauses between ticks inside the timed region
    ev[0].record(stream)
    stats = []
    queries = 0
    for k in range(args.steps):
        _, st, mq = tick_dev(args.warmup + k)
        ev[k + 1].record(stream)
        stats.append(st)
        queries += mq  # whole-job queries of the step (every rank's queries, each answered completely)
    torch.cuda.synchronize()
    gc.enable()
    clk = clocks.stop()
    total_ms = ev[0].elapsed_time(ev[-1])
    per_tick = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    if os.environ.get("TJ_BENCH_TICKS"):  # diagnostics: every timed tick's duration
        print("ticks_ms", [round(t, 3) for t in per_tick], file=sys.stderr)
    if world > 1:
        t = torch.tensor([total_ms] + per_tick, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms, per_tick = float(t[0].item()), [float(x) for x in t[1:].tolist()]
    value = queries / (total_ms / 1e3)

    st0 = stats[-1]
    n = int(st0.n_objects)
    mean = lambda key: statistics.mean(getattr(s, key) for s in stats)  # noqa: E731
    peak, peak_src = measured_peak()
    # roofline of the dominant kernel (the per-leaf join, K3): algorithmic bytes per launch =
    # 16*P_a (x, y of the task objects) + 36*S_a (clipped rect 32 + result count 4 per
    # intersecting entry) + 4*W (bitmap words written), DESIGN.md §4.
    join_ms = mean("t_join_ms")
    join_bytes = 16 * st0.task_objects + 36 * st0.task_subqueries + 4 * st0.bitmap_words
    achieved = join_bytes / (join_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic("k_join")
    # the dominant kernel, the per-query decode (K4): 4*W (bitmap words read) + 4*R (leaf position ->
    # input row) + 8*R (result ids written) + 8*(m + 1) (CSR offsets); timed alone between events
    R_ = int(st0.results_total)
    m_q = int(st0.n_queries)
    dec_ms = mean("t_decode_kernel_ms")
    dec_bytes = 4 * int(st0.bitmap_words) + 12 * R_ + 8 * (m_q + 1)
    dec_traffic, dec_traffic_src = ncu_traffic("k_decode_query")
    # the query scatter (K2): 40*m (4 rect doubles + count/base per query) + 8*S (slot) + 8*L
    sc_ms = mean("t_scatter_ms")
    sc_bytes = 40 * m_q + 8 * int(st0.n_subqueries) + 8 * int(st0.n_leaves)
    # index build (K0 + K1) against its compulsory bytes 44n + 4Z + 12L.  In the
    # tick the object sort overlaps the query scatter on a side stream, so K1 alone is timed on a
    # second context with the sort kept on the main stream (TJ_SERIAL_SORT=1), a few ticks
    # (rank 0 alone, on the full tick, when sharded)
    build_ms = None
    if dticks is not None:
        os.environ["TJ_SERIAL_SORT"] = "1"
        sctx = new_ctx()
        os.environ.pop("TJ_SERIAL_SORT")
        sst = []
        for k in range(4):
            a_ = dticks[k % pool]
            _, s_ = sctx.tick_ptrs(a_[0].numel(), *(x.data_ptr() for x in a_[:3]), a_[3].numel(),
                                   *(x.data_ptr() for x in a_[3:]), _native.TJ_MEM_DEVICE, _native.TJ_MEM_DEVICE)
            sst.append(s_)
        sctx.close()
        build_ms = statistics.mean(s_.t_build_ms + s_.t_sort_ms for s_ in sst[1:])
        st_full = sst[-1]
        build_bytes = 44 * n + 4 * (4 ** int(st_full.l_deep)) + 12 * int(st_full.n_leaves)

    # end to end through the C ABI with pinned host buffers: H2D inputs + D2H CSR per step.
    # tj_tick uploads ids, x, y and the four rect columns; issuer ids stay on the host
    # (results are keyed by input query row), so they are not counted.
    def h2d_bytes(cols):
        return sum(x.numel() * x.element_size() for k, x in enumerate(cols) if k != 3)

    e2e = None
    if not args.no_e2e:
        e_steps = max(1, min(args.steps, args.e2e_steps))
        out_flag = 0 if args.e2e_ids64 else _native.TJ_OUT_IDS32
        idb, idbs = 8, set()
        if sharded:
            hsh = [Shard(t, rank, world, dev, pinned=True) for t in ticks]

            def tick_host(k):  # this rank's slice from pinned host memory, its queries' lists back to it
                sh = hsh[k % pool]
                p = sh.ptrs()
                out, st = ctx.tick_sharded_ptrs(sh.n, *p[:3], sh.m, *p[3:], _native.TJ_MEM_HOST,
                                                _native.TJ_MEM_HOST | out_flag)
                st.n_queries = sh.m_total  # whole-job queries of the step
                return (out, st), sh.nbytes()
        else:
            hticks = [[torch.from_numpy(a).pin_memory() for a in (t.ids, t.xs, t.ys, t.qids, t.qxa, t.qya, t.qxb,
                                                                    t.qyb)] for t in ticks]

            def tick_host(k):
                a = hticks[k % pool]
                return ctx.tick_ptrs(a[0].numel(), *(x.data_ptr() for x in a[:3]), a[3].numel(),
                                     *(x.data_ptr() for x in a[3:]), _native.TJ_MEM_HOST, _native.TJ_MEM_HOST | out_flag), \
                    h2d_bytes(a)

        if sharded or args.e2e_contexts <= 1:
            tick_host(0)
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            h2d = d2h = eq = 0
            for k in range(e_steps):
                (out, st), hb = tick_host(k)
                h2d += hb
                d2h += out.offset_bytes * (out.n_q + 1) + out.id_bytes * out.n_results
                idb = out.id_bytes
                eq += int(st.n_queries)
            e1.record(stream)
            torch.cuda.synchronize()
            e_ms = e0.elapsed_time(e1)
        else:
            # P contexts (each its own stream and pinned result buffers), one host thread each,
            # ticks dealt round-robin: one tick's upload, another's compute and a third's result
            # download overlap (PCIe is full duplex).  ctypes releases the GIL during tj_tick.
            import threading

            ctxs = [ctx] + [new_ctx() for _ in range(args.e2e_contexts - 1)]

            def host_tick(cx, k):
                a = hticks[k % pool]
                out, st = cx.tick_ptrs(a[0].numel(), *(x.data_ptr() for x in a[:3]), a[3].numel(),
                                       *(x.data_ptr() for x in a[3:]), _native.TJ_MEM_HOST,
                                       _native.TJ_MEM_HOST | out_flag)
                return out, st, h2d_bytes(a)

            for cx in ctxs:
                host_tick(cx, 0)
            torch.cuda.synchronize()
            acc = [[0, 0, 0] for _ in ctxs]

            def worker(j):
                for k in range(j, e_steps, len(ctxs)):
                    out, st, hb = host_tick(ctxs[j], k)
                    acc[j][0] += hb
                    acc[j][1] += out.offset_bytes * (out.n_q + 1) + out.id_bytes * out.n_results
                    idbs.add(out.id_bytes)
                    acc[j][2] += int(st.n_queries)

            ths = [threading.Thread(target=worker, args=(j,)) for j in range(len(ctxs))]
            t0 = time.perf_counter()
            for th in ths:
                th.start()
            for th in ths:
                th.join()
            torch.cuda.synchronize()
            e_ms = (time.perf_counter() - t0) * 1e3
            h2d, d2h, eq = (sum(a_[i] for a_ in acc) for i in range(3))
            idb = max(idbs) if idbs else 8
            for cx in ctxs[1:]:
                cx.close()
        if world > 1:
            t = torch.tensor([e_ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": eq / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d // e_steps,
               "d2h_bytes_per_step": d2h // e_steps, "steps": e_steps,
               "timing": ("wall clock over all steps" if (not sharded and args.e2e_contexts > 1)
                          else "CUDA events on the library stream"),
               "contexts": 1 if sharded else args.e2e_contexts,
               "id_bytes": idb,
               "api": ("tj_tick (C ABI): pinned host inputs -> device, results CSR -> pinned host"
                       + (" (TJ_OUT_IDS32: int32 ids and offsets, every id and offset < 2^31)" if idb == 4 else " (int64 ids)")
                       + ("; per rank (tj_tick_sharded): H2D of its 1/G slice, NCCL gather, its leaf range, partial lists routed to home ranks and merged, D2H of the complete CSR of its own queries"
                          if sharded else ""))}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "p50_tick_ms": statistics.median(per_tick), "max_tick_ms": max(per_tick), "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (RNG-identical reference generator)",
            "config": ref_config(args),
            "config_detail": {"n_objects": n, "queries_per_tick": int(st0.n_queries),
                              "results_per_tick": int(st0.results_total),
                              **({"method": "ug", "split_factor": sf} if sf else {}),
                              "distinct_ticks_cycled": pool,
                              "object_ids": ("a random permutation of 0..n-1 per tick" if args.shuffle_ids
                                             else "arange(n)"),
                              "id_order": ("monotone", "keyed", "sorted")[int(st0.id_order)],
                              "parallelism": (f"leaf-range sharding over {world} GPUs (tj_tick_sharded): NCCL "
                                              f"gather of the ranks' slices, per-rank join/decode of its Morton "
                                              f"leaf range, partial lists routed to the queries' home ranks "
                                              f"(NCCL send/recv) and merged there on the device; every query's "
                                              f"complete list inside the timed region"
                                              if sharded else "1 GPU")},
            "roofline": {"bound": "hbm", "achieved": dec_bytes / (dec_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": dec_bytes / (dec_ms / 1e3) / 1e9 / peak, "traffic": dec_traffic,
                         "kernel": "tj::k_decode_query", "bytes_per_launch": dec_bytes, "ms_per_launch": dec_ms,
                         "bytes_model": "4W + 12R + 8(m+1)", "peak_source": peak_src,
                         "traffic_source": dec_traffic_src},
            "roofline_join": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                              "frac": achieved / peak, "traffic": traffic, "kernel": "tj::k_join",
                              "bytes_per_launch": join_bytes, "ms_per_launch": join_ms,
                              "bytes_model": "16 P_a + 36 S_a + 4 W", "traffic_source": traffic_src,
                              "tests_per_s": st0.containment_tests / (join_ms / 1e3)},
            "roofline_scatter": {"kernels": "K2 query scatter (k_query_count, scans, k_query_fill, k_leaf_stats; "
                                            "concurrent with the object sort)", "ms": sc_ms,
                                 "compulsory_bytes": sc_bytes, "bytes_model": "40m + 8S + 8L",
                                 "achieved": sc_bytes / (sc_ms / 1e3) / 1e9,
                                 "frac": sc_bytes / (sc_ms / 1e3) / 1e9 / peak},
            "roofline_index": {"kernels": "K0 + K1 index build (MBR .. objects in leaf order), timed alone "
                                          "(object sort on the main stream, TJ_SERIAL_SORT=1)",
                               "ms": build_ms, "compulsory_bytes": build_bytes,
                               "achieved": build_bytes / (build_ms / 1e3) / 1e9,
                               "frac": build_bytes / (build_ms / 1e3) / 1e9 / peak},
            "stage_ms": {"build": mean("t_build_ms"), "sort": mean("t_sort_ms"),
                         "scatter": mean("t_scatter_ms"), "join": join_ms,
                         "bitmaps": mean("t_filter_ms"), "decode": mean("t_decode_ms"),
                         "decode_kernel": dec_ms,
                         "merge": mean("t_merge_ms"), "total": mean("t_total_ms")},
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": int(sum(int(s.kernel_launches) for s in stats)),
        }
        print(json.dumps(line), flush=True)
    torch.cuda.synchronize()
    if sharded:
        # torch's NCCL bookkeeping still references the library stream at interpreter teardown;
        # leave the process without running destructors once the collectives are done
        torch.distributed.destroy_process_group()
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)
    eng.close()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="C5")
    ap.add_argument("--method", choices=("quad", "ug"), default="quad",
                    help="index: the quadtree (headline) or the uniform grid (--split-factor cells per side)")
    ap.add_argument("--split-factor", type=int, default=1024)
    ap.add_argument("--pool", type=int, default=3, help="distinct ticks generated and cycled")
    ap.add_argument("--cpu-sample", type=int, default=1_000_000)
    ap.add_argument("--ref-sample", type=int, default=500_000, help="objects per tick of the port fallback")
    ap.add_argument("--ref-chunks", type=int, default=20,
                    help="reference arm: the tick's queries are cut into this many Morton-contiguous chunks")
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--e2e-contexts", type=int, default=3,
                    help="tj_tick contexts driven from this many host threads in the e2e leg (overlap of "
                         "uploads, compute and downloads across ticks)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-ids64", action="store_true",
                    help="e2e leg downloads int64 result ids instead of asking for int32 (TJ_OUT_IDS32)")
    ap.add_argument("--shuffle-ids", action="store_true",
                    help="object ids a random permutation of 0..n-1 per tick instead of arange (non-monotone ids: "
                         "leaf blocks put in id order on the device: keyed lists)")
    ap.add_argument("--sharded", action="store_true",
                    help="leaf-range sharded path (NCCL all-gather + tj_set_shard) even at N=1")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    return run_reference(args) if args.impl == "reference" else run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
