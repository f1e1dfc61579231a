"""GPU parity: the CUDA path (through the public op / C ABI) vs the CPU oracle.

Bar (BASELINE.json north_star): identical (m, s) per matrix except where the
reference's own norms sit within 1e-4 log2 units of a ladder/scaling
threshold, and relative 1-norm difference <= 1e-12 (fp64) / <= 1e-5 (fp32).
"""
import math

import numpy as np
import pytest
import torch

import paper_2512_20777_b200 as X
from paper_2512_20777_b200 import workloads as WL
from oracle import expm_oracle as O

pytestmark = pytest.mark.gpu

TOL = {torch.float64: 1e-12, torch.float32: 1e-5}


def _rel1(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.abs(a - b).sum(axis=-2).max(axis=-1)
    r = np.abs(b).sum(axis=-2).max(axis=-1)
    return d / r


def _run(Wnp, eps, scheme="sastre", dtype=torch.float64, check_finite=True):
    W = torch.as_tensor(Wnp).to(device="cuda", dtype=dtype)
    if scheme == "baseline":
        res = X.expm_baseline(W, eps, check_finite=check_finite)
    else:
        res = X.expm(W, eps, scheme, check_finite=check_finite)
    torch.cuda.synchronize()
    return res


def _oracle_batch(Wnp, eps, scheme="sastre"):
    if scheme == "baseline":
        Wb = np.asarray(Wnp, np.float64)
        B, n = Wb.shape[0], Wb.shape[-1]
        out = np.full((B, n, n), np.nan)
        m = np.zeros(B, np.int64); s = np.zeros(B, np.int64); e1 = np.zeros(B); e2 = np.zeros(B)
        mults = np.zeros(B, np.int64); bad = np.zeros(B, bool)
        for i in range(B):
            try:
                r = O.expm_baseline(Wb[i], eps)
            except O.NonFiniteError:
                bad[i] = True
                continue
            out[i], m[i], s[i], e1[i], e2[i], mults[i] = r.value, r.m, r.s, r.e1, r.e2, r.mults
        return out, m, s, e1, e2, mults, bad
    return O.expm_batch(np.asarray(Wnp, np.float64), eps, scheme)


def _check_batch(Wnp, eps, scheme, dtype, label=""):
    """Full parity check of one batch; returns (#exempt, worst rel err)."""
    res = _run(Wnp, eps, scheme, dtype, check_finite=False)
    val, m, s, e1, e2, mults, bad = _oracle_batch(Wnp, eps, scheme)
    gm = res.plan.m.cpu().numpy().astype(int)
    gs = res.plan.s.cpu().numpy().astype(int)
    gmu = res.mults.cpu().numpy()
    gbad = res.nonfinite.cpu().numpy()
    assert np.array_equal(gbad, bad), (label, np.nonzero(gbad != bad))
    ok = ~bad
    diff = (gm != m) | (gs != s)
    exempt = 0
    for i in np.nonzero(diff & ok)[0]:
        W64 = np.asarray(Wnp[i], np.float64)
        n1 = O.one_norm(W64)
        n2 = O.one_norm(W64 @ W64)
        assert scheme == "sastre" and O.near_threshold(n1, n2, eps), \
            (label, i, (gm[i], gs[i]), (m[i], s[i]), n1, n2)
        exempt += 1
    same = ok & ~diff
    assert np.array_equal(gmu[same], mults[same]), label
    err = _rel1(res.value.cpu().numpy()[ok], val[ok]) if ok.any() else np.zeros(0)
    worst = float(err.max()) if err.size else 0.0
    assert worst <= TOL[dtype], (label, worst, int(np.argmax(err)))
    # e1/e2 are derived from the same norms: tight for fp64, loose for fp32 norms
    if same.any():
        ge1 = res.plan.e1.cpu().numpy()[same]
        rtol = 1e-12 if dtype == torch.float64 else 1e-4
        fin = np.isfinite(e1[same])
        np.testing.assert_allclose(ge1[fin], e1[same][fin], rtol=rtol)
    return exempt, worst


# ---------------------------------------------------------------------------
# golden vectors of the reference itself (tests/golden)
# ---------------------------------------------------------------------------

def _golden_cases(g):
    offs = g["offsets"]
    for i in range(len(g["names"])):
        n = int(g["n"][i])
        yield (i, str(g["names"][i]), g["W"][offs[i]:offs[i + 1]].reshape(n, n),
               g["X"][offs[i]:offs[i + 1]].reshape(n, n), float(g["eps"][i]), str(g["scheme"][i]))


def test_golden_fp64_vs_reference(golden):
    worst = 0.0
    for i, name, W, Xref, eps, scheme in _golden_cases(golden):
        if golden["raised"][i]:
            with pytest.raises(X.NonFiniteError):
                _run(W[None], eps, scheme)
            continue
        res = _run(W[None], eps, scheme)
        gm, gs = int(res.plan.m[0]), int(res.plan.s[0])
        if (gm, gs) != (golden["m"][i], golden["s"][i]):
            assert scheme == "sastre" and O.near_threshold(O.one_norm(W), O.one_norm(W @ W), eps), (name, scheme)
            continue
        assert int(res.mults[0]) == golden["mults"][i], name
        err = _rel1(res.value[0].cpu().numpy(), Xref)
        worst = max(worst, float(err))
        assert err <= 1e-12, (name, scheme, float(err))
    print(f"golden fp64 worst rel 1-norm diff {worst:.2e}")


def test_golden_fp32_vs_oracle(golden):
    """fp32 inputs (golden matrices rounded to fp32) vs the oracle on the same values."""
    for i, name, W, Xref, eps, scheme in _golden_cases(golden):
        if golden["raised"][i] or eps < 2.0 ** -24:
            continue
        W32 = W.astype(np.float32)
        if not np.isfinite(W32).all() or O.one_norm(W) > 25.0:
            continue  # e^W itself would leave the fp32 range
        _check_batch(W32[None], eps, scheme, torch.float32, name)


@pytest.mark.parametrize("scheme", ["sastre", "ps"])
def test_named_plans(scheme):
    cases = {
        "zero": (np.zeros((4, 4)), (0, 0, 0)),
        "diag1": (np.diag([1.0] * 5), (15, 0, 4) if scheme == "sastre" else (12, 0, 5)),
        "nil": (np.array([[0.0, 1.0], [0.0, 0.0]]), None),
    }
    for name, (W, want) in cases.items():
        res = _run(W[None], 1e-8, scheme)
        got = (int(res.plan.m[0]), int(res.plan.s[0]), int(res.mults[0]))
        if want:
            assert got == want, (name, got)
    res = _run(np.zeros((3, 4, 4)), 1e-8, scheme)
    assert torch.equal(res.value.cpu(), torch.eye(4, dtype=torch.float64).expand(3, 4, 4))
    nil = _run(np.array([[[0.0, 1.0], [0.0, 0.0]]]), 1e-8, scheme).value[0].cpu().numpy()
    assert np.abs(nil - np.array([[1.0, 1.0], [0.0, 1.0]])).max() <= 1e-15


# ---------------------------------------------------------------------------
# ragged orders, both dtypes, both schemes, tolerance sweep
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("scheme", ["sastre", "ps"])
def test_ragged_orders(dtype, scheme):
    rng = np.random.default_rng(101)
    sizes = (1, 2, 3, 5, 8, 15, 16, 17, 31, 32, 33, 47, 63, 64, 65, 100, 129)
    epss = ((1e-12, 1e-8, 1e-4, 2.0 ** -24, 2.0 ** -53) if dtype == torch.float64
            else (1e-6, 1e-4, 2.0 ** -24))
    for n in sizes:
        B = 6 if n <= 64 else 3
        arr = rng.uniform(-1, 1, (B, n, n))
        target = 10.0 ** rng.uniform(-7, 2.3 if dtype == torch.float64 else 1.4, B)
        W = arr * (target / np.abs(arr).sum(axis=1).max(axis=1))[:, None, None]
        if dtype == torch.float32:
            W = W.astype(np.float32)
        for eps in epss:
            _check_batch(W, eps, scheme, dtype, f"n={n} eps={eps}")


def test_generator_kinds_sweep():
    """Structured inputs (reference bench.py:100-143 kinds) at small orders."""
    rng = np.random.default_rng(7)
    for n in (4, 16, 32, 64):
        mats = []
        for kind in range(5):
            for _ in range(4):
                a = rng.uniform(-1, 1, (n, n))
                if kind == 0:
                    a = np.diag(np.diag(a))
                elif kind == 2:
                    a = np.triu(a) * 0.5 ** np.maximum(np.arange(n)[None, :] - np.arange(n)[:, None], 0)
                elif kind == 3:
                    a = np.triu(a, 1) + 1e-8 * rng.uniform(-1, 1, (n, n))
                elif kind == 4:
                    a = np.zeros((n, n))
                    for i in range(n // 2):
                        th = rng.uniform(0.25, 1.0)
                        a[2 * i, 2 * i + 1], a[2 * i + 1, 2 * i] = th, -th
                t = 10.0 ** rng.uniform(-3, 2)
                mats.append(a * t / np.abs(a).sum(axis=0).max())
        W = np.stack(mats)
        for scheme in ("sastre", "ps"):
            for eps in (1e-12, 1e-8, 2.0 ** -53):
                _check_batch(W, eps, scheme, torch.float64, f"kinds n={n}")


# ---------------------------------------------------------------------------
# BASELINE configs
# ---------------------------------------------------------------------------

def test_config_C1_full():
    cfg = WL.CONFIGS["C1"]
    W = WL.generate("C1")
    ex, worst = _check_batch(W, cfg.eps, "sastre", torch.float64, "C1")
    print(f"C1: exempt {ex}, worst {worst:.2e}")


def test_config_C2_full():
    cfg = WL.CONFIGS["C2"]
    W = WL.generate("C2")
    ex, worst = _check_batch(W, cfg.eps, "sastre", torch.float32, "C2")
    assert ex <= 8
    print(f"C2: exempt {ex}, worst {worst:.2e}")


def test_config_C2_orthogonality():
    """exp of a skew-symmetric matrix is orthogonal: a size-independent property."""
    W = torch.as_tensor(WL.generate("C2")).cuda()
    Q = X.expm(W, 2.0 ** -24).value
    I = torch.eye(16, device="cuda")
    dev = (Q @ Q.transpose(-1, -2) - I).abs().amax()
    assert float(dev) < 2e-5


def test_config_C3_subset_and_full_properties():
    cfg = WL.CONFIGS["C3"]
    idx = np.arange(0, 4096, 64)               # 64 of 4096 time points
    W = WL.generate("C3", indices=idx)
    ex, worst = _check_batch(W, cfg.eps, "sastre", torch.float32, "C3")
    print(f"C3 subset: exempt {ex}, worst {worst:.2e}")
    # full batch: finite, and exp(t A) determinant = exp(t tr A)
    Wf = torch.as_tensor(WL.generate("C3")).cuda()
    res = X.expm(Wf, cfg.eps)
    A, t = WL.c3_factors()
    sel = torch.arange(0, 4096, 256, device="cuda")
    ld = torch.linalg.slogdet(res.value[sel].double())[1].cpu().numpy()
    want = t[sel.cpu().numpy()].astype(np.float64) * np.trace(A.astype(np.float64))
    assert np.abs(ld - want).max() <= 1e-3 * np.abs(want).max()


@pytest.mark.slow
def test_config_C4_subset():
    cfg = WL.CONFIGS["C4"]
    W = WL.generate("C4", indices=np.arange(0, 64, 8))
    ex, worst = _check_batch(W, cfg.eps, "sastre", torch.float64, "C4")
    print(f"C4 subset: exempt {ex}, worst {worst:.2e}")


@pytest.mark.slow
def test_config_C5_subset():
    cfg = WL.CONFIGS["C5"]
    W = WL.generate("C5", indices=[0, 37, 101, 255])
    ex, worst = _check_batch(W, cfg.eps, "sastre", torch.float32, "C5")
    print(f"C5 subset: exempt {ex}, worst {worst:.2e}")


@pytest.mark.parametrize("dtype,scheme", [(torch.float64, "sastre"), (torch.float32, "sastre"),
                                          (torch.float64, "ps")])
def test_large_odd_orders(dtype, scheme):
    """Orders that are not multiples of the 128-wide GEMM tiles or of 4 (the
    vector width): ragged tile edges in every stage, both schemes."""
    rng = np.random.default_rng(41)
    for n in (65, 131, 777):
        W = np.stack([rng.standard_normal((n, n)) * (t / n ** 0.5) for t in (0.05, 3.0, 40.0)])
        ex, worst = _check_batch(W.astype(np.float32) if dtype == torch.float32 else W,
                                 2.0 ** -24 if dtype == torch.float32 else 1e-12, scheme, dtype, f"odd n={n}")


# ---------------------------------------------------------------------------
# error behaviour and invariants
# ---------------------------------------------------------------------------

def test_errors():
    W = torch.eye(3, device="cuda", dtype=torch.float64)[None]
    with pytest.raises(X.ToleranceError):
        X.expm(W, 2.0 ** -54)
    with pytest.raises(X.ToleranceError):
        X.expm(W, float("nan"))
    with pytest.raises(X.ToleranceError):
        X.expm(W.float(), 2.0 ** -30)
    X.expm(W, 2.0 ** -53)
    with pytest.raises(X.MatrixError):
        X.expm(W, 1e-8, "pade")
    with pytest.raises(X.MatrixError):
        X.expm(torch.zeros(2, 3, 4, device="cuda"), 1e-8)
    with pytest.raises(RuntimeError):
        X.expm(torch.eye(3, dtype=torch.float64)[None], 1e-8)
    bad = torch.eye(3, device="cuda", dtype=torch.float64)[None].clone()
    bad[0, 1, 1] = float("nan")
    with pytest.raises(X.NonFiniteError):
        X.expm(bad, 1e-8)
    big = torch.diag(torch.tensor([1e300, 1.0], dtype=torch.float64)).cuda()[None]
    with pytest.raises(X.NonFiniteError):
        X.expm(big, 1e-8)
    r = X.expm(torch.zeros(0, 5, 5, device="cuda"), 1e-4)
    assert r.value.shape == (0, 5, 5)


def test_batch_shape_and_determinism():
    rng = np.random.default_rng(3)
    W = torch.as_tensor(rng.uniform(-1, 1, (2, 3, 24, 24))).cuda()
    a = X.expm(W, 1e-10)
    b = X.expm(W, 1e-10)
    assert a.value.shape == (2, 3, 24, 24) and a.plan.m.shape == (2, 3)
    assert torch.equal(a.value, b.value)
    flat = X.expm(W.reshape(6, 24, 24), 1e-10)
    assert torch.equal(flat.value.reshape(2, 3, 24, 24), a.value)


def test_inverse_identity_fp64():
    rng = np.random.default_rng(37)
    for n in (8, 33, 64, 96):
        W = rng.uniform(-1, 1, (4, n, n))
        W *= (rng.uniform(0.1, 2.0, 4) / np.abs(W).sum(axis=1).max(axis=1))[:, None, None]
        Wt = torch.as_tensor(W).cuda()
        F = X.expm(Wt, 1e-12).value
        Bk = X.expm(-Wt, 1e-12).value
        I = torch.eye(n, dtype=torch.float64, device="cuda")
        d = torch.linalg.matrix_norm(F @ Bk - I) / math.sqrt(n)
        assert float(d.max()) <= 1e-10


def test_host_pipeline_matches_device_path():
    """Host-buffer entry (chunked 3-stream pipeline) == device path, bit for bit."""
    W = torch.as_tensor(WL.generate("C2", batch=4100))  # not a multiple of the chunking
    dev = X.expm(W.cuda(), 2.0 ** -24)
    host = X.expm_host(W.pin_memory(), 2.0 ** -24, chunks=7)
    assert host.value.device.type == "cpu"
    assert torch.equal(host.value, dev.value.cpu())
    assert torch.equal(host.plan.m, dev.plan.m.cpu()) and torch.equal(host.mults, dev.mults.cpu())
    W64 = torch.as_tensor(WL.generate("C1", batch=37))
    assert torch.equal(X.expm_host(W64, 2.0 ** -53, chunks=3).value, X.expm(W64.cuda(), 2.0 ** -53).value.cpu())


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_baseline_alg1_vs_oracle(dtype):
    """GPU Alg. 1 (engine.py:90-116) vs the oracle: same (m, s, mults), values within the bar."""
    rng = np.random.default_rng(90)
    for n in (1, 3, 8, 16, 17, 32, 40, 64):
        W = rng.uniform(-1, 1, (5, n, n))
        W *= (10.0 ** rng.uniform(-3, 1.2, 5) / np.abs(W).sum(axis=1).max(axis=1))[:, None, None]
        if dtype == torch.float32:
            W = W.astype(np.float32)
        for eps in ((1e-12, 1e-8, 2.0 ** -53) if dtype == torch.float64 else (1e-6, 2.0 ** -24)):
            _check_batch(W, eps, "baseline", dtype, f"baseline n={n}")


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_baseline_alg1_large_n_vs_oracle(dtype):
    """Alg. 1 for n > 64 on the GEMM pipeline (term stages over device active
    lists, cooperative squaring): same (m, s, mults) as the oracle (pinned to
    engine.py:90-116), values within the bar, including s well above 8."""
    rng = np.random.default_rng(91)
    for n in (65, 100, 256):
        B = 4 if n < 256 else 3
        W = rng.uniform(-1, 1, (B, n, n))
        # fp32: norms up to ~16 (s <= 6), as the n <= 64 test -- every squaring doubles the fp32 error
        top = 2.7 if dtype == torch.float64 else 1.2
        W *= (10.0 ** rng.uniform(-3, top, B) / np.abs(W).sum(axis=1).max(axis=1))[:, None, None]
        if dtype == torch.float32:
            W = W.astype(np.float32)
        for eps in ((1e-12, 2.0 ** -53) if dtype == torch.float64 else (2.0 ** -24,)):
            _check_batch(W, eps, "baseline", dtype, f"baseline n={n}")
    # a batch mixing the fused-kernel size limit's neighbour orders
    Wz = np.zeros((2, 96, 96))
    Wz[1] = np.diag(np.full(96, -30.0))  # s = 7, e^W = e^-30 I
    if dtype == torch.float32:
        Wz = Wz.astype(np.float32)
    _check_batch(Wz, 1e-12 if dtype == torch.float64 else 2.0 ** -24, "baseline", dtype, "baseline diag")


def test_baseline_alg1_large_n_graph_capture():
    """The n > 64 Alg. 1 path is sync-free too: it captures into a CUDA graph."""
    W = (torch.randn(3, 128, 128, device="cuda", dtype=torch.float64) / 12)
    X0 = torch.empty_like(W)
    X.expm_into(W, X0, 1e-12, "baseline")
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        X.expm_into(W, X0, 1e-12, "baseline")
    W.mul_(7.0)
    g.replay()
    torch.cuda.synchronize()
    ref = X.expm_baseline(W.clone(), 1e-12)
    assert torch.equal(X0, ref.value)


def test_baseline_cost_ratio_vs_sastre():
    """The paper's claim on the reference's own bands: Alg. 1 needs
    1.6-2.4x the products of the Sastre route on flow-norm matrices."""
    W = torch.as_tensor(WL.generate("C1", batch=512)).cuda()
    base = X.expm_baseline(W, 1e-8).mults.sum().item()
    sas = X.expm(W, 1e-8).mults.sum().item()
    assert 1.3 <= base / sas <= 3.0, (base, sas)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_large_path_nonfinite(dtype):
    """n > 64 (GEMM pipeline): NaN input and overflowing results raise NonFiniteError,
    the healthy matrices of the same batch are unaffected."""
    rng = np.random.default_rng(5)
    W = rng.uniform(-1, 1, (3, 96, 96))
    W /= np.abs(W).sum(axis=1).max(axis=1)[:, None, None]
    W[1, 3, 4] = np.nan
    W[2] = np.diag(np.full(96, 800.0 if dtype == torch.float64 else 100.0))   # e^W overflows
    Wt = torch.as_tensor(W).to(device="cuda", dtype=dtype)
    with pytest.raises(X.NonFiniteError):
        X.expm(Wt, 1e-6)
    r = X.expm(Wt, 1e-6, check_finite=False)
    assert r.nonfinite.tolist() == [False, True, True]
    good = X.expm(Wt[:1], 1e-6).value
    assert torch.equal(good[0], r.value[0])


# ---------------------------------------------------------------------------
# the reference's acceptance criteria (test_acceptance.py) on the GPU path
# ---------------------------------------------------------------------------

def test_acceptance_04_forward_accuracy_vs_scipy():
    """Criterion 4 (test_acceptance.py:124-139): error <= 1e-7 at eps = 1e-8,
    here against scipy's Pade expm (the reference's own cross-check oracle,
    test_oracle.py:110-122)."""
    sla = pytest.importorskip("scipy.linalg")
    rng = np.random.default_rng(9000)
    norms = np.geomspace(1e-2, 10.0, 60)
    for i, target in enumerate(norms):
        n = (8, 16, 32, 64)[i % 4]
        a = rng.uniform(-1, 1, (n, n))
        W = a * target / np.abs(a).sum(axis=0).max()
        ref = sla.expm(W)
        for scheme in ("sastre", "ps"):
            got = _run(W[None], 1e-8, scheme).value[0].cpu().numpy()
            err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            assert err <= 1e-7, (n, target, scheme, err)


def test_acceptance_07_selector_sanity():
    """Criterion 7 (test_acceptance.py:201-219)."""
    rng = np.random.default_rng(7)
    Ws = []
    for _ in range(40):
        n = int(rng.integers(1, 16))
        a = rng.uniform(-1, 1, (n, n))
        W = np.zeros((16, 16))
        W[:n, :n] = a * (10.0 ** rng.uniform(-6, 2)) / np.abs(a).sum(axis=0).max()
        Ws.append(W)
    Wt = np.stack(Ws)
    for scheme in ("sastre", "ps"):
        r = _run(Wt, 1e-8, scheme, check_finite=False)
        s = r.plan.s.cpu().numpy()
        e = (r.plan.e1 + r.plan.e2).cpu().numpy()
        assert (s >= 0).all() and (s <= 20).all()
        assert (s[e <= 1e-8] == 0).all()
        assert int(_run(np.array([[[1e60]]]), 1e-8, scheme, check_finite=False).plan.s[0]) == 20
        costs = [_run(Wt[:10, :12, :12], eps, scheme).mults.cpu().numpy() for eps in (1e-12, 1e-8, 1e-4)]
        assert (costs[0] >= costs[1]).all() and (costs[1] >= costs[2]).all()


def test_acceptance_08_logdet_equals_trace():
    """Criterion 8 (test_acceptance.py:226-249): log det e^W = tr W."""
    rng = np.random.default_rng(8)
    for n in (4, 16, 40, 96):
        a = rng.uniform(-1, 1, (6, n, n))
        W = a * (rng.uniform(0.5, 2.0, 6) / np.abs(a).sum(axis=1).max(axis=1))[:, None, None]
        X_ = X.expm(torch.as_tensor(W).cuda(), 1e-12).value
        sign, logdet = torch.linalg.slogdet(X_)
        tr = np.trace(W, axis1=1, axis2=2)
        assert (sign.cpu().numpy() == 1.0).all()
        np.testing.assert_allclose(logdet.cpu().numpy(), tr, rtol=0, atol=1e-8 * np.abs(tr).max() + 1e-12)


def test_cuda_graph_capture_and_replay():
    """expm_into / expm_lowrank_into (n <= 64) are capturable: no host sync,
    no allocation.  A captured graph replayed on new inputs gives the same
    results as eager calls (the serving-loop pattern: CUDA graphs instead of a
    tracing compiler)."""
    from paper_2512_20777_b200 import workloads as WL2
    W = torch.as_tensor(WL.generate("C2", indices=np.arange(4096)), device="cuda")
    Xg = torch.empty_like(W)
    plan = {"m": torch.empty(4096, dtype=torch.int8, device="cuda"),
            "s": torch.empty(4096, dtype=torch.int8, device="cuda"),
            "mults": torch.empty(4096, dtype=torch.int32, device="cuda"),
            "nonfinite": torch.empty(4096, dtype=torch.uint8, device="cuda")}
    X.expm_into(W, Xg, 2.0 ** -24, "sastre", plan)  # warm (kernel attributes set outside capture)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        X.expm_into(W, Xg, 2.0 ** -24, "sastre", plan)
    W.copy_(torch.as_tensor(WL.generate("C2", indices=np.arange(4096, 8192)), device="cuda"))
    g.replay()
    torch.cuda.synchronize()
    ref = X.expm(W.clone(), 2.0 ** -24)
    assert torch.equal(Xg, ref.value)
    assert torch.equal(plan["m"], ref.plan.m) and torch.equal(plan["mults"], ref.mults)

    A1, A2 = WL2.generate_lowrank(np.arange(512))
    a1 = torch.as_tensor(A1, device="cuda")
    a2 = torch.as_tensor(A2, device="cuda")
    xo = torch.empty(512, 64, 64, dtype=torch.float64, device="cuda")
    X.expm_lowrank_into(a1, a2, xo, 2.0 ** -53)
    torch.cuda.synchronize()
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        X.expm_lowrank_into(a1, a2, xo, 2.0 ** -53)
    A1b, A2b = WL2.generate_lowrank(np.arange(512, 1024))
    a1.copy_(torch.as_tensor(A1b))
    a2.copy_(torch.as_tensor(A2b))
    g2.replay()
    torch.cuda.synchronize()
    ref2 = X.expm_lowrank(X.LowRankPair(a1.clone(), a2.clone()), 2.0 ** -53)
    assert torch.equal(xo, ref2.value)


@pytest.mark.parametrize("n,B,dtype", [(80, 7, torch.float64), (600, 5, torch.float32), (16, 1001, torch.float32)])
def test_expm_host_pageable_ragged(n, B, dtype):
    """expm_host (the C pipelined entry) with pageable input, batch sizes that
    are not multiples of the chunking (4-matrix alignment), the large-n path
    (and the int8-slice path at n = 600): identical to the device call."""
    rng = np.random.default_rng(n + B)
    W = torch.as_tensor((rng.standard_normal((B, n, n)) * (3.0 / n ** 0.5)).astype(
        np.float32 if dtype == torch.float32 else np.float64))
    host = X.expm_host(W, 2.0 ** -24 if dtype == torch.float32 else 1e-12)
    dev = X.expm(W.cuda(), 2.0 ** -24 if dtype == torch.float32 else 1e-12)
    assert torch.equal(host.value, dev.value.cpu())
    assert torch.equal(host.plan.s, dev.plan.s.cpu()) and torch.equal(host.mults, dev.mults.cpu())


@pytest.mark.parametrize("n,B,dtype", [(256, 24, torch.float32), (200, 9, torch.float64), (2048, 6, torch.float32)])
def test_cuda_graph_capture_large_n(n, B, dtype):
    """The large-n pipeline (n > 64) is sync-free: the device bucket scheduler
    (k_bucket) keeps every stage's slot count on the device, so the whole call
    captures into a CUDA graph (a host synchronisation inside capture fails).
    Replayed on inputs with a different (m, s) mix, the graph gives exactly the
    eager result: n = 256 fp32 (FFMA GEMM), n = 200 fp64 (DMMA GEMM), n = 2048
    fp32 (exact int8-slice tcgen05 GEMM)."""
    eps = 2.0 ** -24 if dtype == torch.float32 else 2.0 ** -53

    def batch(seed, lo, hi):
        g = torch.Generator().manual_seed(seed)
        W = torch.randn(B, n, n, generator=g, dtype=torch.float64)
        tgt = 10.0 ** (torch.rand(B, generator=g, dtype=torch.float64) * (hi - lo) + lo)
        return (W * (tgt / W.abs().sum(dim=-2).amax(dim=-1))[:, None, None]).to(dtype).cuda()

    W = batch(1, -1.0, 0.5)          # mostly s = 0
    Xg = torch.empty_like(W)
    plan = {"m": torch.empty(B, dtype=torch.int8, device="cuda"), "s": torch.empty(B, dtype=torch.int8, device="cuda"),
            "mults": torch.empty(B, dtype=torch.int32, device="cuda"),
            "nonfinite": torch.empty(B, dtype=torch.uint8, device="cuda")}
    X.expm_into(W, Xg, eps, "sastre", plan)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        X.expm_into(W, Xg, eps, "sastre", plan)
    W.copy_(batch(2, 0.0, 2.7))      # s up to ~8: more squaring levels than at capture time
    g.replay()
    torch.cuda.synchronize()
    ref = X.expm(W.clone(), eps)
    assert int(ref.plan.s.max()) >= 3
    assert torch.equal(Xg, ref.value)
    assert torch.equal(plan["s"], ref.plan.s) and torch.equal(plan["mults"], ref.mults)


def test_cuda_graph_capture_timegrid():
    """expm_timegrid for n > 64 is sync-free too (shared powers, device bucketing of the squarings)."""
    A, t = WL.c3_factors()
    Ad = torch.as_tensor(A, device="cuda")
    td = torch.as_tensor(t[:64], device="cuda")
    K, n = 64, 256
    out = torch.empty(K, n, n, device="cuda")
    plan = {k: torch.empty(K, dtype=dt, device="cuda") for k, dt in (("m", torch.int8), ("s", torch.int8),
                                                                     ("mults", torch.int32),
                                                                     ("nonfinite", torch.uint8))}
    wsb = int(X._lib.lib().expmb_timegrid_workspace_bytes(K, n, 0))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    X.expm_timegrid(Ad, td, 2.0 ** -24, check_finite=False, out=out, plan=plan, workspace=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        X.expm_timegrid(Ad, td, 2.0 ** -24, check_finite=False, out=out, plan=plan, workspace=ws)
    td.copy_(torch.as_tensor(t[64:128]))
    g.replay()
    torch.cuda.synchronize()
    ref = X.expm_timegrid(Ad, td.clone(), 2.0 ** -24)
    assert torch.equal(out, ref.value) and torch.equal(plan["s"], ref.plan.s)
