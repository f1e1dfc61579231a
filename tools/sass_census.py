#!/usr/bin/env python
"""Per-kernel census of the tensor-core / TMA / TMEM instructions in the built
libexpmb.so (static SASS from cuobjdump): the evidence that a kernel runs on
tcgen05 (UTC*MMA, UTMALDG, LDTM), the FP64 tensor cores (DMMA), mma.sync
(HMMA) or packed FFMA2.

usage: python tools/sass_census.py [lib.so] > profiles/sass_r02.txt"""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ("UTCIMMA", "UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "LDTM", "STTM", "DMMA", "HMMA", "IMMA", "FFMA2",
       "DFMA", "FFMA", "LDGSTS", "SYNCS")


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2512_20777_b200", "libexpmb.so")
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=td, capture_output=True, check=True)
        cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
        sass = subprocess.run(["cuobjdump", "-sass", os.path.join(td, cub)], capture_output=True, text=True).stdout
        names = subprocess.run(["cu++filt"], input="\n".join(re.findall(r"Function : (\S+)", sass)),
                               capture_output=True, text=True).stdout.splitlines()
    counts = collections.OrderedDict()
    fn = None
    it = iter(names)
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = next(it, m.group(1))
            counts[fn] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m and fn:
            op = m.group(1)
            for o in OPS:
                if op == o or op.startswith(o + "."):
                    counts[fn][o] += 1
    print(f"# static SASS census of {os.path.relpath(lib, ROOT)} (cuobjdump -sass; sm_100a)")
    print("# kernel | " + " ".join(OPS))
    for fn, c in counts.items():
        if not any(c[o] for o in OPS[:10]) and not c["FFMA2"]:
            continue
        cut = fn.find(">(")
        short = (fn[:cut + 1] if cut >= 0 else re.sub(r"\(.*", "", fn)).replace("void ", "")[:150]
        print(f"{short}\n    " + "  ".join(f"{o}={c[o]}" for o in OPS if c[o]))


if __name__ == "__main__":
    main()
