"""Crossover of the int8-slice path vs the FFMA GEMM over the order n (fp32)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2512_20777_b200 as X
for n, B in ((256, 1024), (320, 512), (384, 256), (448, 256), (512, 128), (768, 64), (1024, 32), (1536, 16)):
    W = torch.as_tensor((np.random.default_rng(n).standard_normal((B, n, n)) * (8.0 / n ** 0.5)).astype(np.float32), device="cuda")
    res = {}
    for flag in ("0", "1"):
        os.environ["EXPMB_I8"] = flag
        X.expm(W, 2.0 ** -24)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            X.expm(W, 2.0 ** -24)
        torch.cuda.synchronize()
        res[flag] = (time.perf_counter() - t0) / 3
    print(f"n={n} B={B} ffma {1e3*res['0']:.2f} ms  i8 {1e3*res['1']:.2f} ms  ratio {res['0']/res['1']:.2f}", flush=True)
