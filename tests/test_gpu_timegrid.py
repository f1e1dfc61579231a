"""GPU parity of the time-grid path: e^(t_k A) for one A
and many t_k, against the oracle applied to the materialised t_k A (the
reference computes each time point independently, engine.py:119-152).

Bar: identical (m, s) except near-threshold (the plan here comes from
|t| ||A^p||_1, the reference's from ||fl(t A)^p||_1: they differ in the last
bits), relative 1-norm difference <= 1e-12 (fp64) / 1e-5 (fp32)."""
import numpy as np
import pytest
import torch

import paper_2512_20777_b200 as X
from paper_2512_20777_b200 import workloads as WL
from oracle import expm_oracle as O

pytestmark = pytest.mark.gpu


def _rel1(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b).sum(axis=-2).max(axis=-1) / np.abs(b).sum(axis=-2).max(axis=-1)


def _check(A, t, eps, scheme, dtype, tol):
    r = X.expm_timegrid(torch.as_tensor(A, device="cuda", dtype=dtype), torch.as_tensor(t), eps, scheme)
    torch.cuda.synchronize()
    V = r.value.cpu().numpy()
    ms, ss = r.plan.m.cpu().numpy(), r.plan.s.cpu().numpy()
    exempt, worst = 0, 0.0
    for k, tk in enumerate(np.asarray(t)):
        W = (np.asarray(tk, A.dtype) * A).astype(np.float64)   # fl(t A) in the working dtype, as the bench feeds it
        want = O.expm(W, eps, scheme, tol_floor=2.0 ** -24 if dtype == torch.float32 else 2.0 ** -53)
        if (ms[k], ss[k]) != (want.m, want.s):
            assert O.near_threshold_powers(W, eps, scheme), (k, float(tk), scheme, (ms[k], ss[k]), (want.m, want.s))
            exempt += 1
            continue
        err = float(_rel1(V[k], want.value))
        worst = max(worst, err)
        assert err <= tol, (k, float(tk), err, want.m, want.s)
    assert exempt <= max(1, len(t) // 50)
    return r, worst


def test_timegrid_c3_subset_fp32():
    A, t = WL.c3_factors()
    idx = np.random.default_rng(3).choice(len(t), 48, replace=False)
    tt = np.concatenate([t[idx], np.array([0.0, 4.0], np.float32)])
    r, worst = _check(A, tt, 2.0 ** -24, "sastre", torch.float32, 1e-5)
    print(f"C3 time grid fp32 worst rel err {worst:.3e}")
    m = r.plan.m.cpu().numpy()
    assert m[-2] == 0 and (r.value[-2].cpu() == torch.eye(256)).all()   # t = 0 -> I


@pytest.mark.parametrize("scheme", ["sastre", "ps"])
def test_timegrid_fp64(scheme):
    rng = np.random.default_rng(17)
    n = 100
    A = rng.standard_normal((n, n)) / np.sqrt(n) - 0.3 * np.eye(n)
    t = np.concatenate([rng.uniform(-2.0, 3.0, 24), [1e-9, 7.5]])
    _check(A, t, 1e-12, scheme, torch.float64, 1e-12)


def test_timegrid_small_n_is_the_batched_path():
    rng = np.random.default_rng(2)
    A = rng.standard_normal((16, 16)).astype(np.float32)
    t = rng.uniform(0, 2, 100).astype(np.float32)
    r = X.expm_timegrid(torch.as_tensor(A, device="cuda"), torch.as_tensor(t), 2.0 ** -24)
    W = torch.as_tensor(t[:, None, None] * A[None], device="cuda")
    d = X.expm(W, 2.0 ** -24)
    assert torch.equal(r.value, d.value) and torch.equal(r.plan.s, d.plan.s)


def test_timegrid_errors():
    A = torch.eye(80, device="cuda")
    with pytest.raises(X.ToleranceError):
        X.expm_timegrid(A, torch.ones(3), 2.0 ** -30)
    with pytest.raises(X.MatrixError):
        X.expm_timegrid(torch.ones(3, 4, device="cuda"), torch.ones(3), 1e-6)
    with pytest.raises(X.NonFiniteError):
        X.expm_timegrid(A, torch.tensor([1.0, float("nan")]), 1e-6)
    with pytest.raises(X.NonFiniteError):
        X.expm_timegrid(A * 1e30, torch.tensor([1e10]), 1e-6)
    r = X.expm_timegrid(A, torch.zeros(0), 1e-6)
    assert r.value.shape == (0, 80, 80)


def test_timegrid_negative_times_ps_fp32():
    """Negative times (the inverse flow e^{-tA}) and the PS scheme on the shared-power path."""
    rng = np.random.default_rng(23)
    n = 128
    A = (rng.standard_normal((n, n)) / np.sqrt(n)).astype(np.float32)
    t = np.array([-3.0, -1.25, -0.01, 0.5, 2.75], np.float32)
    _check(A, t, 2.0 ** -24, "ps", torch.float32, 1e-5)


@pytest.mark.parametrize("scale", [2.0 ** 80, 2.0 ** -70])
def test_timegrid_extreme_norm_of_A(scale):
    """The shared powers are formed from A / sigma (sigma a power of two near
    ||A||_1), so ||A|| far from 1 neither overflows A^16 nor underflows it:
    e^(t_k A) for t_k ||A|| of order one matches the oracle on fl(t_k A)."""
    rng = np.random.default_rng(23)
    n = 80
    A = rng.standard_normal((n, n)) / np.sqrt(n) * scale
    t = np.array([0.3, 1.0, 2.5, -1.7]) / scale
    _check(A, t, 1e-12, "sastre", torch.float64, 1e-12)
