"""Fused one-CTA-per-matrix kernel (64 < n <= 128) vs the bucketed GEMM
pipeline at n = 96 and 128: device time per call, same inputs, each path in
its own process (EXPMB_FUSED_TILE is read once per process).

usage: python tools/fused_tile_bench.py [out.json]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, json, torch
sys.path.insert(0, sys.argv[1])
import paper_2512_20777_b200 as X
n, B, dt = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
dtype = torch.float32 if dt == "f32" else torch.float64
g = torch.Generator(device="cuda").manual_seed(n)
W = torch.randn(B, n, n, device="cuda", dtype=torch.float64, generator=g)
W *= (10.0 ** (torch.rand(B, device="cuda", generator=g, dtype=torch.float64) * 3 - 1.5) / W.abs().sum(-2).amax(-1))[:, None, None]
W = W.to(dtype).contiguous()
eps = 2.0 ** -24 if dtype == torch.float32 else 2.0 ** -53
out = torch.empty_like(W)
plan = {"m": torch.empty(B, dtype=torch.int8, device="cuda"), "s": torch.empty(B, dtype=torch.int8, device="cuda")}
for _ in range(3): X.expm_into(W, out, eps, "sastre", plan)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): X.expm_into(W, out, eps, "sastre", plan)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"ms": e0.elapsed_time(e1) / 10, "exps_per_s": B / (e0.elapsed_time(e1) / 10e3)}))
"""


def main():
    rows = []
    for n, B, dt in ((96, 8192, "f32"), (128, 8192, "f32"), (96, 4096, "f64"), (128, 4096, "f64")):
        row = {"n": n, "batch": B, "dtype": dt}
        for path, env in (("fused", {}), ("pipeline", {"EXPMB_FUSED_TILE": "0"})):
            r = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(n), str(B), dt],
                               env=dict(os.environ, **env), capture_output=True, text=True, check=True)
            row[path] = json.loads(r.stdout.strip().splitlines()[-1])
        row["speedup"] = row["pipeline"]["ms"] / row["fused"]["ms"]
        print(json.dumps(row), flush=True)
        rows.append(row)
    if len(sys.argv) > 1:
        json.dump(rows, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
