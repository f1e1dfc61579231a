"""GPU parity of the plan-only selectors select_sastre / select_ps
(select.py:223-234) through expmb_select: the same (m, s, e1, e2) as the
oracle ladder (pinned to the reference), the same plan the full expm
reports, NonFiniteError on a non-finite input or power."""
import numpy as np
import pytest
import torch

import paper_2512_20777_b200 as X
from oracle import expm_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 5, 16, 40, 64, 100, 256, 600])
@pytest.mark.parametrize("scheme", ["sastre", "ps"])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_select_matches_oracle_and_expm(n, scheme, dtype):
    rng = np.random.default_rng(n * 7 + (scheme == "ps"))
    B = 24 if n <= 100 else 6
    W = rng.standard_normal((B, n, n))
    W *= (10.0 ** rng.uniform(-6, 2.5, B) / np.abs(W).sum(axis=1).max(axis=1))[:, None, None]
    if dtype == torch.float32:
        W = W.astype(np.float32)
    eps = 2.0 ** -24 if dtype == torch.float32 else 1e-12
    Wd = torch.as_tensor(W).cuda()
    sel = X.select_ps(Wd, eps) if scheme == "ps" else X.select_sastre(Wd, eps)
    full = X.expm(Wd, eps, scheme)
    torch.cuda.synchronize()
    assert torch.equal(sel.m, full.plan.m) and torch.equal(sel.s, full.plan.s)
    # (the fp64 n > 32 expm runs the DMMA kernel: its column sums add in another order)
    torch.testing.assert_close(sel.norms[:, 0], full.plan.norms[:, 0], rtol=1e-13, atol=0)
    gm, gs = sel.m.cpu().numpy(), sel.s.cpu().numpy()
    for i in range(B):
        p = O.select(np.asarray(W[i], np.float64), eps, scheme)
        if (gm[i], gs[i]) != (p.m, p.s):
            assert O.near_threshold_powers(W[i], eps, scheme), (n, scheme, i)
            continue
        if dtype == torch.float64:
            np.testing.assert_allclose(float(sel.e1[i]), p.e1, rtol=1e-12)


def test_select_nonfinite_and_batch_dims():
    W = torch.randn(3, 4, 20, 20, device="cuda", dtype=torch.float64) / 10
    p = X.select_sastre(W, 1e-10)
    assert p.m.shape == (3, 4) and p.norms.shape == (3, 4, 2)
    Wb = W.clone()
    Wb[1, 2, 0, 0] = float("inf")
    with pytest.raises(X.NonFiniteError):
        X.select_sastre(Wb, 1e-10)
    big = torch.full((2, 80, 80), 1e20, device="cuda")  # W^2 overflows fp32
    with pytest.raises(X.NonFiniteError):
        X.select_sastre(big, 2.0 ** -24)
    with pytest.raises(X.ToleranceError):
        X.select_ps(W, 2.0 ** -60)
