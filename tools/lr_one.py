"""One low-rank launch of shape (n, t, B) for ncu captures: python tools/lr_one.py n t B"""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2512_20777_b200 as X
n, t, B = (int(a) for a in sys.argv[1:4])
rng = np.random.default_rng(n)
A1 = torch.as_tensor(rng.uniform(-1, 1, (B, n, t)) / n ** 0.5, device="cuda")
A2 = torch.as_tensor(rng.uniform(-1, 1, (B, t, n)) / n ** 0.5, device="cuda")
Xo = torch.empty(B, n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    X.expm_lowrank_into(A1, A2, Xo, 2.0 ** -53)
torch.cuda.synchronize()
print("ok")
