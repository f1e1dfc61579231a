"""Probe: host<->device copy bandwidth with 1..4 concurrent streams, each
direction alone and both together (pinned host memory, 64 MiB total)."""
import time
import torch

N = 64 << 20
h = torch.empty(N, dtype=torch.uint8).pin_memory()
h2 = torch.empty(N, dtype=torch.uint8).pin_memory()
d = torch.empty(N, dtype=torch.uint8, device="cuda")
d2 = torch.empty(N, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(k)]
    for mode in ("h2d", "d2h", "both"):
        def run():
            part = N // k
            for i, s in enumerate(ss):
                with torch.cuda.stream(s):
                    sl = slice(i * part, (i + 1) * part)
                    if mode in ("h2d", "both"):
                        d[sl].copy_(h[sl], non_blocking=True)
                    if mode in ("d2h", "both"):
                        h2[sl].copy_(d2[sl], non_blocking=True)
            torch.cuda.synchronize()
        run()
        t0 = time.perf_counter()
        for _ in range(10):
            run()
        dt = (time.perf_counter() - t0) / 10
        nbytes = N * (2 if mode == "both" else 1)
        print(f"streams {k} {mode:5s} {nbytes / dt / 1e9:6.1f} GB/s")
