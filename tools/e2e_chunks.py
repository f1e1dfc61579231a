"""Time HostPipeline.run for several chunk counts (C2) and the raw copy rates."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_20777_b200 as X
from paper_2512_20777_b200 import workloads as WL

W = torch.from_numpy(WL.generate("C2")).pin_memory()
B, n = W.shape[0], W.shape[-1]
dev = torch.device("cuda", 0)
Wd = W.to(dev)
out = torch.empty_like(W).pin_memory()
torch.cuda.synchronize()
for name, fn in (("h2d", lambda: Wd.copy_(W, non_blocking=True)), ("d2h", lambda: out.copy_(Wd, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"{name}: {dt*1e3:.3f} ms  {W.numel()*4/dt/1e9:.1f} GB/s")
# both directions concurrently on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
Wd2 = torch.empty_like(Wd)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        Wd.copy_(W, non_blocking=True)
    with torch.cuda.stream(s2):
        out.copy_(Wd2, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"duplex: {dt*1e3:.3f} ms  {2*W.numel()*4/dt/1e9:.1f} GB/s total")
for ch in (1, 2, 4, 8, 16, 32, 64):
    pipe = X.HostPipeline(B, n, torch.float32, chunks=ch, device=dev)
    for _ in range(2):
        pipe.run(W, 2.0 ** -24, check_finite=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        pipe.run(W, 2.0 ** -24, check_finite=False)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"chunks {ch:3d}: {dt*1e3:.3f} ms/step  {B/dt/1e6:.1f} M exps/s")
