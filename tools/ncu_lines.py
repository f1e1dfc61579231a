#!/usr/bin/env python
"""Attribute an ncu report's per-SASS-address executed instructions and stall
samples to CUDA source lines (via nvdisasm -g line tables of the built .so).

usage: python tools/ncu_lines.py report.ncu-rep kernel_substring [top]
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sass_lines(kernel_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2512_20777_b200", "libexpmb.so")],
                   cwd=tmp, capture_output=True)
    cub = glob.glob(os.path.join(tmp, "*.cubin"))[0]
    out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    cur_fn, cur_line, table = None, None, {}
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn and kernel_sub in cur_fn:
            table[int(m.group(1), 16)] = cur_line
    return table


def main():
    rep, ksub = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    table = sass_lines(ksub)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, recs = None, []
    for r in rows:
        if len(r) > 2 and r[0] == "Address":
            hdr = r
            continue
        if hdr and r and r[0].startswith("0x"):
            recs.append(dict(zip(hdr, r)))
    base = min(int(d["Address"], 16) for d in recs)
    f = lambda x: float(x) if x not in ("", "-") else 0.0
    inst = collections.Counter()
    stall = collections.Counter()
    for d in recs:
        off = int(d["Address"], 16) - base
        line = table.get(off, "?")
        inst[line] += f(d["Instructions Executed"])
        stall[line] += f(d["Warp Stall Sampling (All Samples)"])
    ti = sum(inst.values()) or 1
    ts = sum(stall.values()) or 1
    print(f"{'line':28s} {'inst%':>6s} {'stall%':>6s}")
    for line, c in inst.most_common(top):
        print(f"{line:28s} {100 * c / ti:6.1f} {100 * stall[line] / ts:6.1f}")


if __name__ == "__main__":
    main()
