#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python tools/launch_summary.py launches.csv out.txt "command that was profiled"
"""
import csv
import io
import sys
from collections import OrderedDict


def main():
    src, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
    lines = [l for l in open(src) if not l.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "us":
            ns *= 1e3
        elif r["Metric Unit"] == "ms":
            ns *= 1e6
        k = r["Kernel Name"]
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + ns)
    total = sum(t for _, t in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list (gpu__time_duration.sum, --clock-control none), {cmd}\n")
        f.write("# cold-cache, serialised per launch: compare shares, not absolutes; "
                "the fill kernels are the L2 flush between steps\n")
        f.write(f"total_ns {total:.0f}\n")
        for k, (c, t) in agg.items():
            f.write(f"{c:4d} launches {t:12.0f} ns {100 * t / total:5.1f}%  {k[:80]}\n")
    print(open(out).read())


if __name__ == "__main__":
    main()
