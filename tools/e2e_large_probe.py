"""Probe: e2e (host buffers) of the large-n configs vs HostPipeline chunk count."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2512_20777_b200 as XP
from paper_2512_20777_b200 import workloads as WL

for key in sys.argv[1:]:
    cfg = WL.CONFIGS[key]
    Wh = torch.from_numpy(WL.generate(key)).pin_memory()
    dt = torch.float32 if cfg.dtype == "f32" else torch.float64
    for chunks in (1, 2, 4, 8):
        pipe = XP.HostPipeline(cfg.batch, cfg.n, dt, chunks=chunks)
        pipe.run(Wh, cfg.eps, "sastre", check_finite=False)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            pipe.run(Wh, cfg.eps, "sastre", check_finite=False)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        print(key, "chunks", chunks, "ms", round(1e3 * min(ts), 1), "exps/s", round(cfg.batch / min(ts), 1), flush=True)
        del pipe
        torch.cuda.empty_cache()
