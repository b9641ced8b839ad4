#!/usr/bin/env python
"""Per-source-line stall samples and executed instructions of one kernel in an ncu report.

  python tools/ncu_lines.py gpurun_out/prof.ncu-rep k_join [top]
"""
import collections
import csv
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname = "?"
    agg = collections.defaultdict(lambda: [0, 0, ""])
    hdr = None
    last_line = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr[2:], r[2:]))
        line = r[0] or last_line
        last_line = line
        key = (fname, line)
        try:
            agg[key][0] += int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            agg[key][1] += int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            pass
        if r[1]:
            agg[key][2] = r[1].strip()[:90]
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_i = sum(v[1] for v in agg.values()) or 1
    print(f"samples {tot_s}  instructions {tot_i}")
    for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% ins  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
