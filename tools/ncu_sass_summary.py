#!/usr/bin/env python
"""Summarise an ncu report's SASS page: executed-instruction mix and stall hot spots.

usage: python tools/ncu_sass_summary.py report.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    recs = []
    for r in rows:
        if len(r) > 2 and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) >= len(hdr) - 1 and r[0].startswith("0x"):
            recs.append(dict(zip(hdr, r)))
    f = lambda x: float(x) if x not in ("", "-") else 0.0
    tot_inst = sum(f(d["Instructions Executed"]) for d in recs)
    tot_stall = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in recs) or 1
    ops = collections.Counter()
    for d in recs:
        op = d["Source"].split()[0] if d["Source"].split() else "?"
        if op.startswith("@"):
            op = d["Source"].split()[1]
        ops[op.split(".")[0]] += f(d["Instructions Executed"])
    print(f"warp-instructions executed: {tot_inst:.4g}")
    for op, c in ops.most_common(30):
        print(f"  {op:10s} {c:12.4g}  {100 * c / tot_inst:5.1f}%")
    print("top stall sites:")
    for i, d in enumerate(sorted(recs, key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))[:top]):
        print(f"  {100 * f(d['Warp Stall Sampling (All Samples)']) / tot_stall:5.1f}%  {d['Address'][-5:]}  "
              f"exec={d['Instructions Executed']:>8s}  {d['Source'].strip()[:80]}")


if __name__ == "__main__":
    main()
