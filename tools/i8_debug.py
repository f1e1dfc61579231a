"""Debug: int8-slice path vs FFMA path vs oracle on C5 matrices (one process; the
path switch EXPMB_I8 is read at every call)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2512_20777_b200 as XP
from paper_2512_20777_b200 import workloads as WL
from oracle import expm_oracle as O
idx = [int(x) for x in (sys.argv[1:] or ["0", "37", "101", "255"])]
W = WL.generate("C5", indices=idx)
out = {}
for flag in ("0", "1"):
    os.environ["EXPMB_I8"] = flag
    r = XP.expm(torch.as_tensor(W, device="cuda"), 2.0 ** -24, check_finite=False)
    out[flag] = (r.value.double().cpu().numpy(), r.plan.m.tolist(), r.plan.s.tolist())
for k in range(len(idx)):
    ref = O.expm(W[k].astype(np.float64), 2.0 ** -24, tol_floor=2.0 ** -24)
    e = {f: np.abs(out[f][0][k] - ref.value).sum(0).max() / np.abs(ref.value).sum(0).max() for f in out}
    print(idx[k], "m,s", out["0"][1][k], out["0"][2][k], "ffma err %.3e" % e["0"], "i8 err %.3e" % e["1"], flush=True)
