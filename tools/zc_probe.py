"""Probe: e2e of C2 with the kernel reading W from / writing X to pinned host
memory directly (UVA zero-copy) vs the chunked HostPipeline."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2512_20777_b200 as XP
from paper_2512_20777_b200 import _lib, workloads as WL

B = 65536
Wh = torch.from_numpy(WL.generate("C2", indices=np.arange(B))).pin_memory()
Xh = torch.empty_like(Wh).pin_memory()
plan_h = {k: torch.empty(shape, dtype=dt).pin_memory() for k, shape, dt in (
    ("m", (B,), torch.int8), ("s", (B,), torch.int8), ("e1", (B,), torch.float64), ("e2", (B,), torch.float64),
    ("norms", (B, 2), torch.float64), ("mults", (B,), torch.int32), ("nonfinite", (B,), torch.uint8))}
L = _lib.lib()
ws = torch.empty(256, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def zc():
    rc = L.expmb_expm(Wh.data_ptr(), Xh.data_ptr(), B, 16, 0, 2.0 ** -24, 0,
                      *[plan_h[k].data_ptr() for k in ("m", "s", "e1", "e2", "norms", "mults", "nonfinite")],
                      ws.data_ptr(), 256, st)
    assert rc == 0, rc


pipe = XP.HostPipeline(B, 16, torch.float32, chunks=8)
for name, fn in (("zero-copy", zc), ("pipeline", lambda: pipe.run(Wh, 2.0 ** -24, "sastre", check_finite=False))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(name, "ms", round(1e3 * np.median(ts), 3), "exps/s", round(B / np.median(ts) / 1e6, 2), "M")
zc(); torch.cuda.synchronize()
ref = XP.expm(Wh.cuda(), 2.0 ** -24)
print("zero-copy equal:", torch.equal(Xh, ref.value.cpu()), torch.equal(plan_h["m"], ref.plan.m.cpu()))
