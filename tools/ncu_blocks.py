#!/usr/bin/env python
"""Group an ncu report's executed SASS into basic-block runs (contiguous
instructions with the same execution count) and list the heaviest runs with
their instruction totals and stall shares -- a per-phase cost map when source
line attribution is unreliable (heavily inlined code).

usage: python tools/ncu_blocks.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, recs = None, []
    for r in rows:
        if len(r) > 2 and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) >= len(hdr) - 1 and r[0].startswith("0x"):
            recs.append(dict(zip(hdr, r)))
    f = lambda x: float(x) if x not in ("", "-") else 0.0
    tot = sum(f(d["Instructions Executed"]) for d in recs) or 1
    tst = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in recs) or 1
    runs, cur = [], None
    for d in recs:
        e = f(d["Instructions Executed"])
        if cur and cur["exec"] == e:
            cur["n"] += 1
            cur["stall"] += f(d["Warp Stall Sampling (All Samples)"])
            cur["last"] = d["Address"]
            cur["ops"].append(d["Source"].split()[0] if d["Source"].split() else "?")
        else:
            cur = {"first": d["Address"], "last": d["Address"], "exec": e, "n": 1,
                   "stall": f(d["Warp Stall Sampling (All Samples)"]),
                   "ops": [d["Source"].split()[0] if d["Source"].split() else "?"]}
            runs.append(cur)
    runs.sort(key=lambda r: -(r["exec"] * r["n"]))
    print(f"total warp-instructions {tot:.4g}")
    for r in runs[:top]:
        ops = {}
        for o in r["ops"]:
            o = o.split(".")[0]
            ops[o] = ops.get(o, 0) + 1
        mix = " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:5])
        print(f"{r['first'][-5:]}-{r['last'][-5:]} n={r['n']:4d} exec={r['exec']:9.0f} "
              f"inst={100 * r['exec'] * r['n'] / tot:5.1f}% stall={100 * r['stall'] / tst:5.1f}%  {mix}")


if __name__ == "__main__":
    main()
