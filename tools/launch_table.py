"""Per-kernel time and DRAM bytes of one tick from an ncu launch list
(`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv`).

    python tools/launch_table.py gpurun_out/launches.csv [tick_from_end]
"""
import collections
import csv
import sys


def one_tick(path, back=6):
    """[(kernel, launches, us, dram MB)] of the tick that starts at the back-th k_mbr from the end
    (the bench's last launches are the serial-sort context's ticks)."""
    rows = list(csv.reader(ln for ln in open(path) if ln.startswith('"')))
    hdr, rows = rows[0], rows[1:]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.OrderedDict()
    for r in rows:
        per.setdefault(int(r[ii]), {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    launches = list(per.values())
    starts = [i for i, v in enumerate(launches) if v["k"].startswith("k_mbr")]
    a = starts[-back] if len(starts) >= back else starts[0]
    b = starts[-back + 1] if len(starts) >= back and back > 1 else len(launches)
    agg = collections.OrderedDict()
    for v in launches[a:b]:
        k = v["k"].split("(")[0].replace("void ", "")
        e = agg.setdefault(k, [0, 0.0, 0.0])
        e[0] += 1
        e[1] += v.get("gpu__time_duration.sum", 0.0) / 1e3
        e[2] += (v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)) / 1e6
    return b - a, [(k, e[0], e[1], e[2]) for k, e in agg.items()]


def main():
    path = sys.argv[1]
    back = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    n, rows = one_tick(path, back)
    agg = {k: [c, us, mb] for k, c, us, mb in rows}
    tot = sum(e[1] for e in agg.values())
    print(f"one tick: {n} launches, {tot:.1f} us serialised")
    for k, e in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
        print(f"{k[:58]:58s} n={e[0]:2d} {e[1]:8.1f} us {100 * e[1] / tot:5.1f}%  {e[2]:8.1f} MB  {e[2] / e[1] if e[1] else 0:5.2f} TB/s")


if __name__ == "__main__":
    main()
