"""Worst fp32 error vs the oracle of the current C2 kernel on skew matrices of
growing norm (run with EXPMB_W16=0 / 1 to compare the two n = 16 kernels)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_20777_b200 as X  # noqa: E402
from oracle import expm_oracle as O  # noqa: E402

rng = np.random.default_rng(0)
for lo, hi in ((-2, 1), (1, 1.5), (1.5, 2), (2, 2.5), (2.5, 3)):
    W = rng.standard_normal((400, 16, 16))
    W = (W - W.transpose(0, 2, 1)) / 2
    W *= (10.0 ** rng.uniform(lo, hi, 400) / np.abs(W).sum(axis=1).max(axis=1))[:, None, None]
    W = W.astype(np.float32)
    r = X.expm(torch.as_tensor(W).cuda(), 2.0 ** -24)
    val, m, s, *_ = O.expm_batch(W.astype(np.float64), 2.0 ** -24)
    got = r.value.cpu().numpy().astype(np.float64)
    err = np.abs(got - val).sum(axis=1).max(axis=1) / np.abs(val).sum(axis=1).max(axis=1)
    print(f"norm 10^[{lo},{hi}]: s max {s.max()}  worst {err.max():.3e}  median {np.median(err):.3e}")
