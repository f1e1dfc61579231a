"""The opt-in exact int8-slice tensor-core GEMM path (gemm_i8.cuh, EXPMB_I8=1)
for fp32 n >= 512 against the oracle: dense inputs over three norm scales
(the squaring phase's dominant diagonal included), ragged column tiles, PS,
non-finite input.  Graded matrices (entries ~2^20 apart within a row) are
its known weakness (tools/i8_graded_probe.py: 1.6e-3 vs the FFMA path's
4.5e-5), which is why the path is not the default."""
import os

import numpy as np
import pytest
import torch

import paper_2512_20777_b200 as X
from oracle import expm_oracle as O

pytestmark = pytest.mark.gpu


def _rel1(a, b):
    return np.abs(a - b).sum(axis=-2).max(axis=-1) / np.abs(b).sum(axis=-2).max(axis=-1)


@pytest.fixture
def i8_on(monkeypatch):
    monkeypatch.setenv("EXPMB_I8", "1")   # read by the library at every call
    yield


def _check(W, eps, scheme="sastre", tol=1e-5):
    r = X.expm(torch.as_tensor(W, device="cuda"), eps, scheme, check_finite=False)
    V = r.value.double().cpu().numpy()
    worst = 0.0
    for b in range(W.shape[0]):
        want = O.expm(W[b].astype(np.float64), eps, scheme, tol_floor=2.0 ** -24)
        assert (int(r.plan.m[b]), int(r.plan.s[b])) == (want.m, want.s) or O.near_threshold(
            want.norm1, want.norm2, eps)
        e = float(_rel1(V[b], want.value))
        worst = max(worst, e)
        assert e <= tol, (b, e, want.m, want.s)
    return worst


@pytest.mark.parametrize("n", [512, 528, 1040])
def test_i8_dense_and_ragged(i8_on, n):
    rng = np.random.default_rng(n)
    W = np.stack([rng.standard_normal((n, n)) * (t / n ** 0.5) for t in (0.3, 4.0, 30.0)]).astype(np.float32)
    print(f"n={n} worst {_check(W, 2.0 ** -24):.2e}")


def test_i8_ps_and_nonfinite(i8_on):
    n = 512
    rng = np.random.default_rng(5)
    W = (rng.standard_normal((2, n, n)) * (2.0 / n ** 0.5)).astype(np.float32)
    _check(W, 2.0 ** -24, "ps")
    W[1, 3, 7] = np.nan
    r = X.expm(torch.as_tensor(W, device="cuda"), 2.0 ** -24, check_finite=False)
    assert r.nonfinite.cpu().tolist() == [False, True]
