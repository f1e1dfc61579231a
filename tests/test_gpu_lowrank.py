"""GPU parity of the low-rank path (engine.py:198-257):
the CUDA kernel through the public op / C ABI vs the oracle restatement and
the reference's own golden outputs.

Bar: identical order m except where ||V||_1 / ||V^2||_1 sit within 1e-4
log2 units of a ladder threshold; relative 1-norm difference <= 1e-12 (fp64)
/ <= 1e-5 (fp32, an extension: the reference is binary64 only).  The path is
unscaled by design (engine.py:208-209), so for V with large negative
eigenvalues the series cancels and ANY two evaluation orders differ by about
u * growth, growth = ||I + |A1| psi(|V|) |A2| ||_1 / ||e^W||_1; the bar is
therefore max(1e-12, 64 u growth) (fp64) and max(1e-5, 64 u growth) (fp32),
which is the stated bar wherever growth < ~140 (fp64) / ~2.6 (fp32)."""
import math

import numpy as np
import pytest
import torch

import paper_2512_20777_b200 as X
from conftest import lowrank_cases
from oracle import expm_oracle as O

pytestmark = pytest.mark.gpu


def _rel1(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b).sum(axis=-2).max(axis=-1) / np.abs(b).sum(axis=-2).max(axis=-1)


def _run(A1, A2, eps, dtype=torch.float64):
    a1 = torch.as_tensor(np.asarray(A1)).to("cuda", dtype)
    a2 = torch.as_tensor(np.asarray(A2)).to("cuda", dtype)
    res = X.expm_lowrank(X.LowRankPair(a1, a2), eps)
    torch.cuda.synchronize()
    return res


def _tol(A1, A2, m, Xref, dtype):
    """The parity bar for one matrix (see the module docstring)."""
    V = np.abs(np.asarray(A2, np.float64)) @ np.abs(np.asarray(A1, np.float64))
    S = np.eye(V.shape[0]); P = np.eye(V.shape[0])
    for k in range(1, max(int(m), 0) + 1):
        P = P @ V / (k + 1)
        S = S + P
    growth = (1.0 + (np.abs(A1) @ S @ np.abs(A2)).sum(0).max()) / np.abs(Xref).sum(0).max()
    u = 2.0 ** -53 if dtype == torch.float64 else 2.0 ** -24
    return max(1e-12 if dtype == torch.float64 else 1e-5, 64 * u * growth)


def _gen(rng, B, n, t, lo, hi):
    """The reference generator's recipe (bench.py:134-142), batched."""
    A1 = rng.uniform(-1, 1, (B, n, t))
    A2 = rng.uniform(-1, 1, (B, t, n))
    vn = np.abs(A2 @ A1).sum(axis=-2).max(axis=-1)
    target = 10.0 ** rng.uniform(np.log10(lo), np.log10(hi), B)
    A2 *= (target / vn)[:, None, None]
    return A1, A2


def test_lowrank_golden_fp64(lowrank_golden):
    g = lowrank_golden
    worst = 0.0
    for i, name, A1, A2, Xg, eps in lowrank_cases(g):
        if g["raised"][i]:
            with pytest.raises(X.LowRankOrderError):
                _run(A1, A2, eps)
            continue
        r = _run(A1, A2, eps)
        m = int(r.plan.m.item())
        nv, nv2 = float(g["norm1"][i]), float(g["norm2"][i])
        if m != g["m"][i]:
            assert O.lowrank_near_threshold(nv, nv2 if not math.isnan(nv2) else nv * nv, eps), name
            continue
        assert int(r.mults.item()) == g["mults"][i] and r.rect_mults == 3, name
        assert int(r.plan.s.item()) == 0 and r.plan.scheme == "lowrank"
        e1 = float(r.plan.e1.item())
        assert e1 == g["e1"][i] or abs(e1 - g["e1"][i]) <= 1e-12 * abs(g["e1"][i]), name
        assert abs(float(r.plan.norms[0].item()) - nv) <= 1e-13 * max(nv, 1e-300), name
        err = float(_rel1(r.value.cpu().numpy(), Xg))
        worst = max(worst, err)
        assert err <= _tol(A1, A2, m, Xg, torch.float64), (name, err)
    print(f"low-rank golden fp64 worst rel err {worst:.3e}")


def test_lowrank_golden_fp32(lowrank_golden):
    g = lowrank_golden
    for i, name, A1, A2, Xg, eps in lowrank_cases(g):
        if g["raised"][i]:
            continue
        eps32 = max(eps, 2.0 ** -24)
        a1, a2 = A1.astype(np.float32), A2.astype(np.float32)
        r = _run(a1, a2, eps32, torch.float32)
        want = O.expm_lowrank(a1, a2, eps32)
        if int(r.plan.m.item()) != want.m:
            assert O.lowrank_near_threshold(want.norm1, want.norm2 if not math.isnan(want.norm2) else 0.0,
                                            eps32, margin=1e-3), name
            continue
        err = float(_rel1(r.value.cpu().numpy(), want.value))
        assert err <= _tol(a1, a2, want.m, want.value, torch.float32), (name, err)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_lowrank_ragged_shapes(dtype):
    rng = np.random.default_rng(7)
    for n, t in ((1, 1), (7, 5), (8, 8), (32, 4), (48, 3), (24, 8), (63, 1), (64, 8), (65, 9), (100, 16), (129, 17), (200, 32), (96, 31)):
        A1, A2 = _gen(rng, 3, n, t, 0.05, 2.0 if dtype == torch.float32 else 6.0)
        eps = 1e-8 if dtype == torch.float64 else 2.0 ** -24
        r = _run(A1, A2, eps, dtype)
        for b in range(3):
            a1 = A1[b].astype(np.float32) if dtype == torch.float32 else A1[b]
            a2 = A2[b].astype(np.float32) if dtype == torch.float32 else A2[b]
            want = O.expm_lowrank(a1, a2, eps)
            assert int(r.plan.m[b].item()) == want.m, (n, t, b)
            assert int(r.mults[b].item()) == want.mults
            err = float(_rel1(r.value[b].cpu().numpy(), want.value))
            assert err <= _tol(a1, a2, want.m, want.value, dtype), (n, t, b, err)


def test_lowrank_flow_batch_fp64():
    """A flow-layer batch (n = 64, t = n/8 as the reference generator) in one launch."""
    rng = np.random.default_rng(2024)
    A1, A2 = _gen(rng, 1024, 64, 8, 0.01, 8.0)
    r = _run(A1, A2, 1e-12)
    Xv = r.value.cpu().numpy()
    ms = r.plan.m.cpu().numpy()
    exempt, worst = 0, 0.0
    for b in range(0, 1024, 3):
        want = O.expm_lowrank(A1[b], A2[b], 1e-12)
        if ms[b] != want.m:
            assert O.lowrank_near_threshold(want.norm1, want.norm2, 1e-12)
            exempt += 1
            continue
        err = float(_rel1(Xv[b], want.value))
        assert err <= _tol(A1[b], A2[b], want.m, want.value, torch.float64), (b, err)
        worst = max(worst, err)
    assert exempt <= 3
    assert len(set(ms.tolist())) >= 5   # many ladder rungs in one batch


def test_lowrank_large_order():
    rng = np.random.default_rng(99)
    A1, A2 = _gen(rng, 2, 1000, 32, 0.5, 3.0)
    r = _run(A1, A2, 1e-10)
    for b in range(2):
        want = O.expm_lowrank(A1[b], A2[b], 1e-10)
        assert int(r.plan.m[b].item()) == want.m
        err = float(_rel1(r.value[b].cpu().numpy(), want.value))
        assert err <= _tol(A1[b], A2[b], want.m, want.value, torch.float64), err


def test_lowrank_matches_dense_expm():
    """e^(A1 A2) two ways on the GPU: factored path vs the dense Sastre path
    (criterion 9 of test_acceptance.py:257-270 uses 1e-7 against the oracle)."""
    rng = np.random.default_rng(5)
    A1, A2 = _gen(rng, 64, 64, 8, 0.5, 5.0)
    r = _run(A1, A2, 1e-8)
    W = torch.as_tensor(A1 @ A2, device="cuda")
    d = X.expm(W, 2.0 ** -53)
    err = _rel1(r.value.cpu().numpy(), d.value.cpu().numpy())
    assert err.max() <= 1e-7, err.max()


def test_lowrank_errors():
    with pytest.raises(X.LowRankOrderError):
        _run(np.eye(4, 2) * 10.0, np.eye(2, 4) * 10.0, 1e-8)      # test_engine.py:297-301
    bad = np.ones((4, 2)); bad[1, 1] = np.nan
    with pytest.raises(X.MatrixError):
        _run(bad, np.ones((2, 4)), 1e-8)                          # engine.py:179-180
    with pytest.raises(X.LowRankOrderError):
        _run(np.ones((40, 33)), np.ones((33, 40)), 1e-8)          # t > 32 path: ||V||_1 = 1320 has no order
    bad = np.ones((40, 33)) * 0.01; bad[3, 7] = np.inf
    with pytest.raises(X.MatrixError):
        _run(bad, np.ones((33, 40)) * 0.01, 1e-8)                 # t > 32 path: non-finite factor
    with pytest.raises(X.ToleranceError):
        _run(np.ones((4, 2)), np.ones((2, 4)), 2.0 ** -54)
    # one bad matrix in a batch raises for the batch; the good ones are computed
    A1 = np.stack([np.eye(4, 2) * 0.1, np.eye(4, 2) * 10.0])
    A2 = np.stack([np.eye(2, 4) * 0.1, np.eye(2, 4) * 10.0])
    with pytest.raises(X.LowRankOrderError, match="batch index 1"):
        _run(A1, A2, 1e-8)


def test_lowrank_named_cases():
    n = 6
    a1 = np.zeros((n, 1)); a1[0, 0] = 1.0
    a2 = np.zeros((1, n)); a2[0, 0] = 1.0
    r = _run(a1, a2, 1e-8)                                        # test_engine.py:241-249
    want = np.eye(n); want[0, 0] = math.e
    assert np.abs(r.value.cpu().numpy() - want).max() <= 1e-8
    r = _run(np.zeros((5, 2)), np.ones((2, 5)), 1e-8)              # test_engine.py:252-255
    assert np.array_equal(r.value.cpu().numpy(), np.eye(5)) and int(r.plan.m) == 0 and int(r.mults) == 0
    r = _run(np.array([[1.5]]), np.array([[1.0]]), 1e-8)           # test_engine.py:313-318
    assert float(r.value[0, 0]) == pytest.approx(1.0 + (math.exp(1.5) - 1.0), rel=1e-9)
    r = _run(np.array([[1.0], [0.0]]), np.array([[0.0, 3.0]]), 1e-8)  # V = 0: e^W = I + W
    assert np.array_equal(r.value.cpu().numpy(), np.array([[1.0, 3.0], [0.0, 1.0]]))


def test_lowrank_misaligned_takes_cta_path():
    """Factors at an 8-byte offset cannot use the 16-byte vector kernels: the
    CTA kernel runs and agrees with the oracle."""
    rng = np.random.default_rng(31)
    A1, A2 = _gen(rng, 5, 64, 8, 0.1, 3.0)
    buf1 = torch.empty(5 * 512 + 1, dtype=torch.float64, device="cuda")
    buf2 = torch.empty(5 * 512 + 1, dtype=torch.float64, device="cuda")
    a1 = buf1[1:].view(5, 64, 8)
    a2 = buf2[1:].view(5, 8, 64)
    a1.copy_(torch.as_tensor(A1))
    a2.copy_(torch.as_tensor(A2))
    assert a1.data_ptr() % 16 == 8
    r = X.expm_lowrank(X.LowRankPair(a1, a2), 1e-10)
    for b in range(5):
        want = O.expm_lowrank(A1[b], A2[b], 1e-10)
        assert int(r.plan.m[b]) == want.m
        assert float(_rel1(r.value[b].cpu().numpy(), want.value)) <= _tol(A1[b], A2[b], want.m, want.value,
                                                                       torch.float64)


_PATH_SCRIPT = r"""
import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2512_20777_b200 as X
from paper_2512_20777_b200 import workloads as WL
A1, A2 = WL.generate_lowrank(np.arange(2048))
r = X.expm_lowrank(X.LowRankPair(torch.as_tensor(A1, device='cuda'), torch.as_tensor(A2, device='cuda')), 2.0 ** -53)
np.save(sys.argv[1], r.value.cpu().numpy())
np.save(sys.argv[1] + '.m.npy', r.plan.m.cpu().numpy())
"""


@pytest.mark.parametrize("env", ["EXPMB_LR_NO_DMMA", "EXPMB_LR_CTA"])
def test_lowrank_kernel_variants_agree(tmp_path, env):
    """The fp64 n=64/t=8 batch through the DMMA kernel (default), the FMA warp
    kernel and the CTA kernel: identical orders, values within the fp64 bar."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for name, extra in (("default", {}), (env, {env: "1"})):
        f = str(tmp_path / f"{name}.npy")
        subprocess.run([sys.executable, "-c", _PATH_SCRIPT, f], cwd=root, check=True,
                       env=dict(os.environ, **extra))
        outs[name] = (np.load(f), np.load(f + ".m.npy"))
    assert np.array_equal(outs["default"][1], outs[env][1])
    err = _rel1(outs["default"][0], outs[env][0])
    assert err.max() <= 1e-12, err.max()


def test_lowrank_leading_batch_dims():
    rng = np.random.default_rng(77)
    A1, A2 = _gen(rng, 6, 40, 5, 0.2, 3.0)
    a1 = torch.as_tensor(A1, device="cuda").reshape(2, 3, 40, 5)
    a2 = torch.as_tensor(A2, device="cuda").reshape(2, 3, 5, 40)
    r = X.expm_lowrank(X.LowRankPair(a1, a2), 1e-10)
    assert r.value.shape == (2, 3, 40, 40) and r.plan.m.shape == (2, 3)
    flat = X.expm_lowrank(X.LowRankPair(a1.reshape(6, 40, 5), a2.reshape(6, 5, 40)), 1e-10)
    assert torch.equal(r.value.reshape(6, 40, 40), flat.value)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_lowrank_large_inner_rank(dtype):
    """t > 32 (t x t operands in the device workspace, lowrank_large.cuh):
    identical order, mults and e1 to the oracle, values within the bar, over
    ragged (n, t) up to the reference generator's t = n/8 at n = 1024
    (bench.py:134-142) and every ladder order."""
    rng = np.random.default_rng(33 + (dtype == torch.float32))
    for (n, t, B, lo, hi) in ((33, 33, 3, 1e-3, 3.0), (64, 40, 4, 1e-6, 4.0), (100, 64, 3, 1e-2, 5.0),
                              (200, 128, 2, 0.3, 5.0), (1024, 128, 2, 0.5, 3.0)):
        A1, A2 = _gen(rng, B, n, t, lo, hi)
        if dtype == torch.float32:
            A1, A2 = A1.astype(np.float32), A2.astype(np.float32)
        eps = 1e-12 if dtype == torch.float64 else 2.0 ** -24
        r = _run(A1, A2, eps, dtype)
        got = r.value.double().cpu().numpy()
        for b in range(B):
            want = O.expm_lowrank(np.asarray(A1[b], np.float64), np.asarray(A2[b], np.float64), eps,
                                  tol_floor=2.0 ** -24 if dtype == torch.float32 else 2.0 ** -53)
            if int(r.plan.m[b]) != want.m:
                assert O.lowrank_near_threshold(want.norm1, want.norm2, eps), (n, t, b)
                continue
            assert int(r.mults[b]) == want.mults, (n, t, b)
            err = float(_rel1(got[b], want.value))
            assert err <= _tol(A1[b], A2[b], want.m, want.value, dtype), (n, t, b, err, want.m)


def test_lowrank_large_inner_rank_graph_capture():
    """The t > 32 path is sync-free: expm_lowrank_into with a workspace captures into a CUDA graph."""
    rng = np.random.default_rng(5)
    A1, A2 = _gen(rng, 3, 96, 48, 0.5, 2.0)
    a1 = torch.as_tensor(A1, device="cuda")
    a2 = torch.as_tensor(A2, device="cuda")
    xo = torch.empty(3, 96, 96, dtype=torch.float64, device="cuda")
    wsb = int(X._lib.lib().expmb_lowrank_workspace_bytes(3, 96, 48, 1))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    X.expm_lowrank_into(a1, a2, xo, 1e-12, workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        X.expm_lowrank_into(a1, a2, xo, 1e-12, workspace=ws)
    a2.mul_(1.7)
    g.replay()
    torch.cuda.synchronize()
    ref = X.expm_lowrank(X.LowRankPair(a1.clone(), a2.clone()), 1e-12)
    assert torch.equal(xo, ref.value)


@pytest.mark.parametrize("n,t", [(2, 1), (64, 8), (40, 20), (80, 40)])
def test_lowrank_overflow_in_assembly_gives_nan_x(n, t):
    """V = A2 A1 = 0 (m = 0) but I + A1 A2 overflows fp32: the matrix is flagged
    non-finite and its X is all NaN (include/expmb.h), on every kernel."""
    A1 = np.zeros((1, n, t), np.float32)
    A2 = np.zeros((1, t, n), np.float32)
    A1[0, 0, 0] = 1e30
    A2[0, 0, n - 1] = 1e30          # A2 A1 = 0 (disjoint supports), A1 A2 has one 1e60 entry
    a1 = torch.as_tensor(A1, device="cuda")
    a2 = torch.as_tensor(A2, device="cuda")
    xo = torch.zeros(1, n, n, device="cuda")
    flags = torch.zeros(1, dtype=torch.uint8, device="cuda")
    X.expm_lowrank_into(a1, a2, xo, 2.0 ** -24, {"flags": flags})
    torch.cuda.synchronize()
    assert int(flags[0]) & 2
    assert torch.isnan(xo).all()
    with pytest.raises(X.NonFiniteError):
        _run(A1[0], A2[0], 2.0 ** -24, torch.float32)
