#!/usr/bin/env python
"""Dump an ncu report's SASS page in address order with executed counts
(per-instruction), for reading where a kernel's dynamic instructions go.

usage: python tools/ncu_sass_dump.py report.ncu-rep > dump.txt
"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
hdr = None
for r in csv.reader(io.StringIO(out)):
    if len(r) > 2 and r[0] == "Address":
        hdr = r
        continue
    if hdr and r and r[0].startswith("0x"):
        d = dict(zip(hdr, r))
        print(f"{d['Address'][-5:]} {d['Instructions Executed']:>9s} {d['Warp Stall Sampling (All Samples)']:>6s}  {d['Source'].strip()}")
