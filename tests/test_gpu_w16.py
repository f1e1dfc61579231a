"""The warp-batched n = 16 fp32 kernel (csrc/fused_w16.cuh, the C2 path).

A warp takes Q = 4 matrices per batch (phase 1: W^2 and norms, phase 2: one
lane per matrix walks the ladder of select.py:164-220, phase 3: evaluate and
square), so the cases below aim at what that schedule can get wrong: batch
sizes that leave partial batches, plan records written by lanes 0..3, matrices
of one batch with different (m, s), and the per-matrix NonFiniteError flags
(engine.py:119-152, matrix.py:56-57 / 97-98) of a batch that mixes good and
bad matrices.  Reference: the oracle (oracle/expm_oracle.py), computed in
binary64 on the upcast inputs as the reference does.
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import paper_2512_20777_b200 as X
from oracle import expm_oracle as O

from test_gpu_parity import _check_batch

pytestmark = pytest.mark.gpu

EPS = 2.0 ** -24


def _mixed(B, seed):
    """16x16 fp32 matrices whose 1-norms span every rung (m = 1..15, s = 0..3):
    skew-symmetric ones up to ||W||_1 = 31, general ones up to 2.  (Past that
    the fp32 rounding of the inputs and of s squarings alone exceeds the 1e-5
    bar against the binary64 oracle -- tools/w16_check.py: worst 1.2e-5 at
    ||W||_1 ~ 100 for both n = 16 kernels; test_matches_fused_small_bitwise
    covers larger norms.)"""
    rng = np.random.default_rng(seed)
    W = rng.standard_normal((B, 16, 16))
    skew = rng.random(B) < 0.6
    W = np.where(skew[:, None, None], (W - W.transpose(0, 2, 1)) / 2, W)
    target = np.where(skew, 10.0 ** rng.uniform(-9, 1.5, B), 10.0 ** rng.uniform(-9, 0.3, B))
    W *= (target / np.abs(W).sum(axis=1).max(axis=1))[:, None, None]
    return W.astype(np.float32)


@pytest.mark.parametrize("B", [1, 2, 3, 4, 5, 7, 8, 31, 33, 127, 4097])
def test_partial_batches(B):
    W = _mixed(B, 100 + B)
    _check_batch(W, EPS, "sastre", torch.float32, f"B={B}")


def test_every_rung_in_one_batch():
    # consecutive matrices (one warp batch) with m = 0, 1, 2, 4, 8, 15 and s > 0
    rng = np.random.default_rng(7)
    base = rng.standard_normal((16, 16))
    base = (base - base.T) / 2
    base /= np.abs(base).sum(axis=0).max()
    norms = [0.0, 1e-9, 1e-4, 2e-3, 5e-2, 0.6, 3.0, 20.0, 30.0, 1e-6, 8.0, 0.0]
    W = np.stack([base * v for v in norms]).astype(np.float32)
    res = X.expm(torch.as_tensor(W).cuda(), EPS)
    torch.cuda.synchronize()
    ms = {int(v) for v in res.plan.m.cpu()}
    assert {0, 1, 2, 4, 8, 15} <= ms, ms
    _check_batch(W, EPS, "sastre", torch.float32, "rungs")


def test_nonfinite_flags_in_mixed_batch():
    rng = np.random.default_rng(11)
    W = _mixed(12, 3)
    W[1, 3, 4] = np.nan          # non-finite input (matrix.py:56-57)
    W[6, 0, 0] = np.inf
    W[9] = np.float32(1e20)      # W^2 overflows fp32 (matrix.py:97-98)
    res = X.expm(torch.as_tensor(W).cuda(), EPS, check_finite=False)
    torch.cuda.synchronize()
    bad = res.nonfinite.cpu().numpy().astype(bool)
    assert list(np.nonzero(bad)[0]) == [1, 6, 9], np.nonzero(bad)[0]
    ok = ~bad
    val, m, s, *_ = O.expm_batch(W[ok].astype(np.float64), EPS)
    err = (np.abs(res.value.cpu().numpy()[ok] - val).sum(axis=1).max(axis=1) /
           np.abs(val).sum(axis=1).max(axis=1))
    assert err.max() <= 1e-5
    with pytest.raises(X.NonFiniteError):
        X.expm(torch.as_tensor(W).cuda(), EPS)


def test_plan_records_and_norms():
    W = _mixed(203, 5)
    res = X.expm(torch.as_tensor(W).cuda(), EPS)
    torch.cuda.synchronize()
    W64 = W.astype(np.float64)
    n1 = np.abs(W64).sum(axis=1).max(axis=1)
    nr = res.plan.norms.cpu().numpy()
    np.testing.assert_allclose(nr[:, 0], n1, rtol=2e-6)
    m = res.plan.m.cpu().numpy()
    has2 = m >= 2
    n2 = np.array([np.abs(w @ w).sum(axis=0).max() for w in W64])
    np.testing.assert_allclose(nr[has2, 1], n2[has2], rtol=2e-5)
    assert np.all(np.isnan(nr[~has2, 1]))  # W^2 not part of the plan (select.py:186-188)
    mults = res.mults.cpu().numpy()
    budget = {0: 0, 1: 0, 2: 1, 4: 2, 8: 3, 15: 4}
    assert np.array_equal(mults, [budget[int(a)] + int(b) for a, b in zip(m, res.plan.s.cpu().numpy())])


def test_select_plan_only_matches_expm():
    W = torch.as_tensor(_mixed(1001, 9)).cuda()
    full = X.expm(W, EPS)
    plan = X.select_sastre(W, EPS)
    torch.cuda.synchronize()
    assert torch.equal(plan.m.cpu(), full.plan.m.cpu())
    assert torch.equal(plan.s.cpu(), full.plan.s.cpu())
    # the plan-only op runs the fused_small kernel: fp32 column sums in another
    # order, so the bounds agree to a few ulps of the fp32 norms
    np.testing.assert_allclose(plan.e1.cpu().numpy(), full.plan.e1.cpu().numpy(), rtol=1e-5)


def test_deterministic_and_offset_views():
    W = torch.as_tensor(_mixed(4096 + 3, 13)).cuda()
    a = X.expm(W, EPS).value
    b = X.expm(W, EPS).value
    assert torch.equal(a, b)
    # a batch that starts mid-warp-batch (offset view) gives the same matrices
    c = X.expm(W[5:].contiguous(), EPS).value
    assert torch.equal(c, a[5:])


_OLD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2512_20777_b200 as X
W = torch.as_tensor(np.load(sys.argv[2])).cuda()
r = X.expm(W, 2.0 ** -24, check_finite=False)
np.savez(sys.argv[3], X=r.value.cpu().numpy(), m=r.plan.m.cpu().numpy(), s=r.plan.s.cpu().numpy())
"""


def test_matches_fused_small_bitwise(tmp_path):
    """Same inputs through the previous n <= 16 kernel (fused_small.cuh, HM
    variant; EXPMB_W16=0 in a child process): the products, formulas and
    squarings are the same code, so e^W must agree bit for bit wherever the
    plans agree -- including norms up to 1000 (s = 8)."""
    rng = np.random.default_rng(21)
    W = rng.standard_normal((2050, 16, 16))
    W = (W - W.transpose(0, 2, 1)) / 2
    W *= (10.0 ** rng.uniform(-8, 3, 2050) / np.abs(W).sum(axis=1).max(axis=1))[:, None, None]
    W = W.astype(np.float32)
    np.save(tmp_path / "w.npy", W)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, EXPMB_W16="0")
    subprocess.run([sys.executable, "-c", _OLD, root, str(tmp_path / "w.npy"), str(tmp_path / "old.npz")],
                   env=env, check=True, timeout=300)
    old = np.load(tmp_path / "old.npz")
    r = X.expm(torch.as_tensor(W).cuda(), EPS, check_finite=False)
    torch.cuda.synchronize()
    m, s = r.plan.m.cpu().numpy(), r.plan.s.cpu().numpy()
    same = (m == old["m"]) & (s == old["s"])
    assert same.mean() > 0.999, same.mean()
    assert np.array_equal(r.value.cpu().numpy()[same].view(np.uint32), old["X"][same].view(np.uint32))
