#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (tracked evidence for bench.py's roofline).

  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
      --out profiles/r01_ncu_summary.json

* --rep: an `ncu --set full` report; per kernel launch: duration, DRAM bytes
  read/written, throughputs, IPC, occupancy, top stall reasons.
* --launches: the `--metrics gpu__time_duration.sum` launch list of one bench
  run (cold-cache, serialised); the last tick's per-kernel time and share.
"""

from __future__ import annotations

import argparse
import collections
import csv
import json
import subprocess


def ncu_csv(rep: str, page: str) -> list:
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def summarize_rep(rep: str) -> dict:
    rows = ncu_csv(rep, "raw")
    hdr = rows[0]
    kernels = {}
    for row in rows[2:]:
        if len(row) != len(hdr):
            continue
        d = dict(zip(hdr, row))
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "").strip()

        def f(k):
            try:
                return float(d.get(k, "nan").replace(",", ""))
            except ValueError:
                return float("nan")

        dur_ns = f("gpu__time_duration.sum")
        rd = f("dram__bytes_read.sum")
        wr = f("dram__bytes_write.sum")
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(k) for k in hdr
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        top = sorted(((v, k) for k, v in stalls.items() if v == v), reverse=True)[:5]
        entry = {
            "duration_us": dur_ns / 1e3 if dur_ns == dur_ns else None,
            "dram_read_bytes": rd, "dram_write_bytes": wr,
            "dram_bytes_per_launch": (rd + wr) if rd == rd and wr == wr else None,
            "dram_throughput_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "sm_throughput_pct": f("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            "ipc": f("sm__inst_executed.avg.per_cycle_active"),
            "achieved_occupancy_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "registers": f("launch__registers_per_thread"),
            "top_stalls": [{"reason": k, "samples": v} for v, k in top],
        }
        # units: ncu raw reports bytes in the unit row (row 1); normalise GB/MB to bytes
        units = dict(zip(hdr, rows[1]))
        for key, metric in (("dram_read_bytes", "dram__bytes_read.sum"), ("dram_write_bytes", "dram__bytes_write.sum")):
            u = units.get(metric, "byte")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                     "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "TB": 1e12}.get(u, 1)
            if entry[key] == entry[key]:
                entry[key] *= scale
        du = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
              "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(
            units.get("gpu__time_duration.sum", "nsecond"), 1e-3)
        entry["duration_us"] = dur_ns * du if dur_ns == dur_ns else None
        if entry["dram_read_bytes"] == entry["dram_read_bytes"]:
            entry["dram_bytes_per_launch"] = entry["dram_read_bytes"] + entry["dram_write_bytes"]
        kernels.setdefault(name, entry)  # first captured launch of each kernel
    return kernels


def summarize_launches(path: str) -> dict:
    """Per-kernel time share of one tick of the bench's timed ticks (tools/launch_table.py)."""
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from launch_table import one_tick

    n, rows = one_tick(path)
    tot = sum(us for _, _, us, _ in rows)
    return {"tick_total_us": tot, "launches": n,
            "kernels": [{"kernel": k, "us": us, "share": us / tot, "launches": c, "dram_mb": mb}
                        for k, c, us, mb in sorted(rows, key=lambda x: -x[2])]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    res = {"note": a.note, "kernels": {}}
    for rep in a.rep:
        for k, v in summarize_rep(rep).items():
            res["kernels"].setdefault(k, v)
    if a.launches:
        res["launch_list"] = summarize_launches(a.launches)
    with open(a.out, "w") as fp:
        json.dump(res, fp, indent=1)
    print(f"wrote {a.out}: {len(res['kernels'])} profiled kernels")


if __name__ == "__main__":
    main()
