import os, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2512_20777_b200 as X
from oracle import expm_oracle as O
n = 512
rng = np.random.default_rng(3)
d = 2.0 ** np.linspace(-10, 10, n)
W = np.stack([(d[:, None] * rng.standard_normal((n, n)) / d[None, :]) * (t / n ** 0.5) for t in (0.5, 3.0)]).astype(np.float32)
for flag in ("0", "1"):
    os.environ["EXPMB_I8"] = flag
    r = X.expm(torch.as_tensor(W, device="cuda"), 2.0 ** -24, check_finite=False)
    V = r.value.double().cpu().numpy()
    for b in range(2):
        want = O.expm(W[b].astype(np.float64), 2.0 ** -24, tol_floor=2.0 ** -24)
        e = np.abs(V[b] - want.value).sum(0).max() / np.abs(want.value).sum(0).max()
        print("I8" if flag == "1" else "FFMA", b, "m,s", want.m, want.s, "err %.3e" % e)
