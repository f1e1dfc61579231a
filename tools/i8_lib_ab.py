"""A/B helper for int8-slice stage builds (`make variant` + EXPMB_LIB): writes
e^W of fixed fp32 inputs (n = 512, 528, 2048; EXPMB_I8=1) to OUT.npz so two
builds can be compared bit for bit (python tools/i8_lib_ab.py OUT.npz)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("EXPMB_I8", "1")
import paper_2512_20777_b200 as X  # noqa: E402

out = {}
for n, B in ((512, 3), (528, 3), (2048, 2)):
    rng = np.random.default_rng(n + 7)
    W = torch.as_tensor((rng.standard_normal((B, n, n)) * (rng.uniform(0.3, 30, B)[:, None, None] / n ** 0.5))
                        .astype(np.float32), device="cuda")
    r = X.expm(W, 2.0 ** -24)
    out[f"v{n}"] = r.value.cpu().numpy()
    out[f"s{n}"] = r.plan.s.cpu().numpy()
np.savez(sys.argv[1], **out)
print("wrote", sys.argv[1])
