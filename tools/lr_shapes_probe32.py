"""fp32 variant of lr_shapes_probe.py: algorithmic bytes (2 n t + n^2) * 4."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2512_20777_b200 as X
for n, t, B in ((64, 8, 16384), (32, 4, 65536), (128, 16, 4096), (256, 32, 1024), (64, 32, 16384)):
    rng = np.random.default_rng(n)
    A1 = torch.as_tensor(rng.uniform(-1, 1, (B, n, t)) / n ** 0.5, device="cuda", dtype=torch.float32)
    A2 = torch.as_tensor(rng.uniform(-1, 1, (B, t, n)) / n ** 0.5, device="cuda", dtype=torch.float32)
    Xo = torch.empty(B, n, n, dtype=torch.float32, device="cuda")
    X.expm_lowrank_into(A1, A2, Xo, 2.0 ** -24)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        X.expm_lowrank_into(A1, A2, Xo, 2.0 ** -24)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    gb = B * (2 * n * t + n * n) * 4 / (ms * 1e-3) / 1e9
    print(f"fp32 n={n} t={t} B={B}: {ms*1e3:.1f} us  {B/ms/1e3:.1f} M/s  {gb:.0f} GB/s = {gb/6547.5:.2f} of HBM", flush=True)
