"""The exact int8-slice tensor-core GEMM path (gemm_i8.cuh; default for fp32
n >= 320, EXPMB_I8=1 from n = 256) against the oracle: dense inputs over
three norm scales (the squaring phase's dominant diagonal included), ragged
column tiles, PS, non-finite input, and the per-product routing: graded
operands (entries ~2^20 apart within a row, where per-row scaling would lose
bits: tools/i8_graded_probe.py) must go to the FFMA GEMM, so the results
equal the FFMA path's bit for bit."""
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


def test_i8_routes_graded_operands_to_ffma(monkeypatch):
    n = 512
    rng = np.random.default_rng(3)
    d = 2.0 ** np.linspace(-10, 10, n)
    W = np.stack([(d[:, None] * rng.standard_normal((n, n)) / d[None, :]) * (t / n ** 0.5) for t in (0.5, 3.0)])
    Wt = torch.as_tensor(W.astype(np.float32), device="cuda")
    monkeypatch.setenv("EXPMB_I8", "0")
    ref = X.expm(Wt, 2.0 ** -24, check_finite=False).value
    monkeypatch.setenv("EXPMB_I8", "1")
    got = X.expm(Wt, 2.0 ** -24, check_finite=False).value
    assert torch.equal(ref, got)


def test_i8_default_from_320(monkeypatch):
    """The default crossover: n = 320 runs on the int8-slice path (a different
    result from the FFMA GEMM in the last places), n = 304 does not."""
    monkeypatch.delenv("EXPMB_I8", raising=False)
    rng = np.random.default_rng(11)
    for n, differs in ((320, True), (304, False)):
        W = (rng.standard_normal((2, n, n)) * (6.0 / n ** 0.5)).astype(np.float32)
        _check(W, 2.0 ** -24)
        Wt = torch.as_tensor(W, device="cuda")
        dflt = X.expm(Wt, 2.0 ** -24).value.clone()
        monkeypatch.setenv("EXPMB_I8", "0")
        ffma = X.expm(Wt, 2.0 ** -24).value.clone()
        monkeypatch.delenv("EXPMB_I8", raising=False)
        assert (not torch.equal(dflt, ffma)) == differs, n


def test_i8_default_on_for_large_dense(monkeypatch):
    """Without EXPMB_I8 the path is on for n >= 320 and matches the oracle."""
    monkeypatch.delenv("EXPMB_I8", raising=False)
    n = 1024
    rng = np.random.default_rng(9)
    W = np.stack([rng.standard_normal((n, n)) * (t / n ** 0.5) for t in (1.0, 20.0)]).astype(np.float32)
    print(f"n=1024 default worst {_check(W, 2.0 ** -24):.2e}")


@pytest.mark.parametrize("n", [512, 528])
def test_i8_variants(i8_on, monkeypatch, n):
    """The 2-CTA multicast form of the one-unit-per-CTA stage computes the same
    integer sums as the one-CTA form: e^W must agree bit for bit (528: an odd
    number of column blocks, so the last cluster has a pad CTA).  The
    persistent stage (the default) rounds the int8 part to fp32 before adding
    the diagonal terms, so it is within a few ulps (normwise) of that form."""
    rng = np.random.default_rng(n + 1)
    W = torch.as_tensor((rng.standard_normal((3, n, n)) * (3.0 / n ** 0.5)).astype(np.float32), device="cuda")
    outs = []
    monkeypatch.setenv("EXPMB_I8_PERSIST", "0")
    for mc in ("1", "0"):
        monkeypatch.setenv("EXPMB_I8_MC", mc)
        outs.append(X.expm(W, 2.0 ** -24).value.clone())
    assert torch.equal(outs[0], outs[1])
    monkeypatch.setenv("EXPMB_I8_PERSIST", "1")
    pers = X.expm(W, 2.0 ** -24).value.clone()
    assert torch.equal(pers, X.expm(W, 2.0 ** -24).value)  # deterministic
    d = _rel1(pers.double().cpu().numpy(), outs[0].double().cpu().numpy())
    print(f"n={n} persistent vs one-unit stage: {d.max():.2e}")
    assert d.max() <= 1e-6


def test_i8_split_and_kept_diagonals(i8_on):
    """Rows / columns whose diagonal entry dominates (identity-like operands:
    the squaring phase; a -0.5 I drift) have it split off and applied in the
    epilogue; elsewhere it stays in the slices.  Both, and a mix of the two in
    one matrix, against the oracle."""
    n = 512
    rng = np.random.default_rng(21)
    G = rng.standard_normal((4, n, n)) / n ** 0.5
    W = np.empty_like(G)
    W[0] = 0.02 * G[0] + np.eye(n) * 0.7               # every diagonal entry split
    W[1] = 2.0 * G[1]                                  # none split
    W[2] = 1.5 * G[2] - 0.5 * np.eye(n)                # drift: split
    d = np.where(np.arange(n) % 3 == 0, 3.0, 0.0)      # a third of the rows / columns split
    W[3] = G[3] + np.diag(d)                           # (entries of G are ~0.04, its row maxima ~0.15)
    print(f"split / kept diagonals worst {_check(W.astype(np.float32), 2.0 ** -24):.2e}")


def test_i8_persistent_many_units(i8_on, monkeypatch):
    """More work units than CTAs (8 matrices x 64 tiles at n = 1024 over 148
    CTAs): every CTA of the persistent stage walks several units, handing the
    TMEM accumulators back and forth between its MMA and epilogue warps."""
    n = 1024
    rng = np.random.default_rng(77)
    W = np.stack([rng.standard_normal((n, n)) * (t / n ** 0.5) for t in (0.2, 1.0, 3.0, 7.0, 12.0, 20.0, 33.0, 50.0)])
    print(f"n=1024 x 8 worst {_check(W.astype(np.float32), 2.0 ** -24):.2e}")
