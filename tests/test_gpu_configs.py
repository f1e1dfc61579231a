"""Per-matrix plan parity on EVERY matrix of the five BASELINE.json configs,
plus widened value parity (all 64 C4 matrices, 512 C3 time points, 32 C5
matrices spanning s = 0..7).

The expected plans come from the unmodified reference's ``select_sastre``
(select.py:228-234) run on the same seeded inputs in the build container
(tests/golden/make_config_plans.py -> tests/golden/config_plans.npz).  Bar
(BASELINE.json north_star): identical (m, s) per matrix except where the
reference's own norms sit within 1e-4 log2 units of a ladder / scaling
threshold (the fixture's ``near`` flag), mults = budget(m) + s, and relative
1-norm difference <= 1e-12 (fp64) / <= 1e-5 (fp32) against the oracle.
"""
import os

import numpy as np
import pytest
import torch

import paper_2512_20777_b200 as X
from paper_2512_20777_b200 import workloads as WL
from oracle import expm_oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = {"f64": 1e-12, "f32": 1e-5}
BUDGET = {0: 0, 1: 0, 2: 1, 4: 2, 8: 3, 15: 4}


@pytest.fixture(scope="module")
def plans():
    return np.load(os.path.join(ROOT, "tests", "golden", "config_plans.npz"))


def _dtype(cfg):
    return torch.float32 if cfg.dtype == "f32" else torch.float64


def _gpu_plans(key, chunk=None):
    cfg = WL.CONFIGS[key]
    B = cfg.batch
    chunk = chunk or B
    ms, ss, e1s, mults = [], [], [], []
    for lo in range(0, B, chunk):
        W = torch.as_tensor(WL.generate(key, indices=np.arange(lo, min(B, lo + chunk)))).to("cuda", _dtype(cfg))
        r = X.expm(W, cfg.eps)
        ms.append(r.plan.m.cpu().numpy().astype(int))
        ss.append(r.plan.s.cpu().numpy().astype(int))
        e1s.append(r.plan.e1.cpu().numpy())
        mults.append(r.mults.cpu().numpy())
        del W, r
    return np.concatenate(ms), np.concatenate(ss), np.concatenate(e1s), np.concatenate(mults)


@pytest.mark.parametrize("key", ["C1", "C2", "C3", "C4", "C5"])
def test_config_plans_every_matrix(plans, key):
    cfg = WL.CONFIGS[key]
    rm, rs = plans[f"{key}_m"].astype(int), plans[f"{key}_s"].astype(int)
    near = plans[f"{key}_near"]
    assert rm.shape[0] == cfg.batch
    gm, gs, ge1, gmu = _gpu_plans(key, chunk=64 if key == "C5" else None)
    diff = (gm != rm) | (gs != rs)
    bad = np.nonzero(diff & ~near)[0]
    assert bad.size == 0, (key, bad[:8].tolist(), list(zip(gm[bad[:8]], gs[bad[:8]])),
                           list(zip(rm[bad[:8]], rs[bad[:8]])))
    same = ~diff
    want_mults = np.array([BUDGET[int(m)] for m in rm]) + rs
    assert np.array_equal(gmu[same], want_mults[same]), key
    # e1 comes from the same norms: binary64 norms agree to rounding, fp32 norms to fp32 rounding
    re1 = plans[f"{key}_e1"]
    fin = same & np.isfinite(re1) & (re1 > 0)
    rtol = 1e-12 if cfg.dtype == "f64" else 2e-4
    np.testing.assert_allclose(ge1[fin], re1[fin], rtol=rtol)
    print(f"{key}: {cfg.batch} matrices, (m,s) mismatches {int(diff.sum())} (all near-threshold: "
          f"{int(near.sum())} flagged)")


def _values(key, idx):
    cfg = WL.CONFIGS[key]
    Wnp = WL.generate(key, indices=idx)
    r = X.expm(torch.as_tensor(Wnp).to("cuda", _dtype(cfg)), cfg.eps, check_finite=False)
    got = r.value.double().cpu().numpy()
    gm, gs = r.plan.m.cpu().numpy().astype(int), r.plan.s.cpu().numpy().astype(int)
    tol_floor = 2.0 ** -24 if cfg.dtype == "f32" else 2.0 ** -53
    worst, checked = 0.0, 0
    for k in range(len(idx)):
        want = O.expm(np.asarray(Wnp[k], np.float64), cfg.eps, tol_floor=tol_floor)
        if (gm[k], gs[k]) != (want.m, want.s):
            assert O.near_threshold(want.norm1, want.norm2, cfg.eps), (key, int(idx[k]))
            continue
        d = np.abs(got[k] - want.value).sum(axis=0).max() / np.abs(want.value).sum(axis=0).max()
        assert d <= TOL[cfg.dtype], (key, int(idx[k]), float(d), want.m, want.s)
        worst = max(worst, float(d))
        checked += 1
    return worst, checked


def test_config_C4_values_all(plans):
    worst, checked = _values("C4", np.arange(64))
    assert checked == 64
    print(f"C4 all 64: worst rel err {worst:.2e}")


def test_config_C3_values_512():
    idx = np.arange(0, 4096, 8)
    worst, checked = _values("C3", idx)
    assert checked >= 500
    print(f"C3 512 time points: worst rel err {worst:.2e}")


def test_config_C5_values_s_sweep(plans):
    s = plans["C5_s"].astype(int)
    idx = []
    for q in range(int(s.max()) + 1):
        idx += np.nonzero(s == q)[0][:4].tolist()
    idx = np.array(sorted(idx))
    assert len(idx) >= 32 and set(s[idx]) == set(range(8))
    worst = 0.0
    for lo in range(0, len(idx), 8):
        w, c = _values("C5", idx[lo:lo + 8])
        assert c == len(idx[lo:lo + 8])
        worst = max(worst, w)
    print(f"C5 {len(idx)} matrices, s = 0..{int(s.max())}: worst rel err {worst:.2e}")
