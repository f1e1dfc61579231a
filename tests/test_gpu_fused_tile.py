"""The one-CTA-per-matrix kernel for 64 < n <= 128 (fused_tile.cuh) runs the
same device code as the bucketed GEMM pipeline in the same order, so its
results must be bit-identical to the pipeline's (EXPMB_FUSED_TILE=0, run in a
subprocess because the switch is read once per process) -- and, through the
ragged-order tests, within the bar of the oracle."""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest
import torch

import paper_2512_20777_b200 as X
from oracle import expm_oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2512_20777_b200 as X
d = np.load(sys.argv[2])
W = torch.as_tensor(d["W"]).cuda()
r = X.expm(W, float(d["eps"]), str(d["scheme"]), check_finite=False)
np.savez(sys.argv[3], value=r.value.cpu().numpy(), m=r.plan.m.cpu().numpy(), s=r.plan.s.cpu().numpy(),
         norms=r.plan.norms.cpu().numpy())
"""


@pytest.mark.parametrize("n", [65, 96, 128])
@pytest.mark.parametrize("dtype,scheme", [(torch.float64, "sastre"), (torch.float32, "sastre"),
                                          (torch.float64, "ps")])
def test_fused_tile_bit_identical_to_pipeline(n, dtype, scheme):
    rng = np.random.default_rng(n)
    B = 40
    W = rng.standard_normal((B, n, n))
    W *= (10.0 ** rng.uniform(-4, 2.3, B) / np.abs(W).sum(axis=1).max(axis=1))[:, None, None]
    W = W.astype(np.float32 if dtype == torch.float32 else np.float64)
    eps = 2.0 ** -24 if dtype == torch.float32 else 1e-12
    res = {}
    with tempfile.TemporaryDirectory() as td:
        np.savez(os.path.join(td, "in.npz"), W=W, eps=eps, scheme=scheme)
        for path, flag in (("fused", "1"), ("pipe", "0")):   # 1: the fused kernel for fp32 too
            env = dict(os.environ, EXPMB_FUSED_TILE=flag)
            out = os.path.join(td, f"{path}.npz")
            subprocess.run([sys.executable, "-c", _CHILD, ROOT, os.path.join(td, "in.npz"), out],
                           env=env, check=True, timeout=600)
            res[path] = dict(np.load(out))
    fused, pipe = res["fused"], res["pipe"]
    assert np.array_equal(fused["m"], pipe["m"]) and np.array_equal(fused["s"], pipe["s"])
    assert np.array_equal(fused["value"], pipe["value"])
    assert np.array_equal(np.nan_to_num(fused["norms"], nan=-1.0), np.nan_to_num(pipe["norms"], nan=-1.0))
    # and within the bar of the oracle on a few of them
    for i in range(0, B, 13):
        want = O.expm(np.asarray(W[i], np.float64), eps, scheme,
                      tol_floor=2.0 ** -24 if dtype == torch.float32 else 2.0 ** -53)
        got = np.asarray(fused["value"][i], np.float64)
        err = np.abs(got - want.value).sum(axis=0).max() / np.abs(want.value).sum(axis=0).max()
        assert err <= (1e-5 if dtype == torch.float32 else 1e-12), (i, err)


def test_fused_tile_select_and_graph():
    """Plan-only selection and CUDA-graph capture through the fused tile kernel."""
    W = torch.randn(50, 100, 100, device="cuda", dtype=torch.float64) / 4
    full = X.expm(W, 1e-12)
    sel = X.select_sastre(W, 1e-12)
    assert torch.equal(sel.m, full.plan.m) and torch.equal(sel.s, full.plan.s)
    out = torch.empty_like(W)
    X.expm_into(W, out, 1e-12)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        X.expm_into(W, out, 1e-12)
    W.mul_(3.0)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, X.expm(W.clone(), 1e-12).value)
