"""Low-rank path without a GPU: the C ABI's argument checks and the kernel's
host/device ladder against the oracle (engine.py:224-244), the Python
boundary's shape validation (engine.py:166-181)."""
import math

import numpy as np
import pytest
import torch

from conftest import lowrank_cases
from oracle import expm_oracle as O
from paper_2512_20777_b200 import _lib
import paper_2512_20777_b200 as ex


def test_lowrank_argument_errors_are_synchronous():
    L = _lib.lib()

    def call(b=1, n=8, t=2, dt=1, eps=1e-8):
        return L.expmb_expm_lowrank(None, None, None, b, n, t, dt, eps, *([None] * 6), None, 0, None)
    assert call(eps=2.0 ** -54) == _lib.ERR_TOLERANCE
    assert call(dt=0, eps=2.0 ** -25) == _lib.ERR_TOLERANCE
    assert call(eps=float("nan")) == _lib.ERR_TOLERANCE
    assert call(dt=5) == _lib.ERR_DTYPE
    assert call(t=9) == _lib.ERR_SHAPE          # t > n
    assert call(t=0) == _lib.ERR_SHAPE
    assert call(n=0, t=0) == _lib.ERR_SHAPE
    assert call(n=64, t=33) == _lib.ERR_WORKSPACE   # t > 32 keeps its t x t operands in a workspace
    assert L.expmb_lowrank_workspace_bytes(4, 64, 32, 1) == 0
    assert L.expmb_lowrank_workspace_bytes(4, 64, 33, 1) > 4 * 9 * 33 * 33 * 8
    assert call(b=0) == 0


def _oracle_pick(nv, nv2, eps):
    try:
        m, e1, e2, used = O.select_lowrank_from_norms(nv, nv2, eps)
        return 0, m, e1, e2
    except O.LowRankOrderError:
        return -1, None, None, None


def test_lowrank_selector_matches_oracle():
    rng = np.random.default_rng(11)
    epss = (1e-12, 1e-8, 1e-4, 2.0 ** -24, 2.0 ** -53, 0.3)
    for it in range(20000):
        nv = float(10.0 ** rng.uniform(-9, 2))
        nv2 = nv * nv * float(10.0 ** rng.uniform(-4, 0))
        if it % 101 == 0:
            nv2 = 0.0
        eps = epss[it % len(epss)]
        rc, m, e1, e2 = _lib.select_lowrank_host(nv, None, eps)
        want = _oracle_pick(nv, nv2, eps)
        if rc == 1:
            rc, m, e1, e2 = _lib.select_lowrank_host(nv, nv2, eps)
        else:
            assert want[1] == 1, (nv, eps)   # only rung m=1 decides without V^2
        assert rc == want[0], (nv, nv2, eps)
        if rc == 0:
            assert m == want[1], (nv, nv2, eps)
            for a, b in ((e1, want[2]), (e2, want[3])):
                assert a == b or abs(a - b) <= 1e-12 * abs(b), (a, b)


def test_lowrank_selector_golden(lowrank_golden):
    g = lowrank_golden
    for i, name, A1, A2, X, eps in lowrank_cases(g):
        nv, nv2 = float(g["norm1"][i]), float(g["norm2"][i])
        if g["raised"][i]:
            V = A2 @ A1
            nv, nv2 = O.one_norm(V), O.one_norm(V @ V)
        rc, m, e1, e2 = _lib.select_lowrank_host(nv, None, eps)
        if rc == 1:
            rc, m, e1, e2 = _lib.select_lowrank_host(nv, nv2, eps)
        if g["raised"][i]:
            assert rc == -1, name
        else:
            assert rc == 0 and m == g["m"][i], name
            assert abs(e1 - g["e1"][i]) <= 1e-12 * abs(g["e1"][i]), name


def test_lowrank_mults_ledger():
    # t x t products: V^2 + V^3..V^j + (k-1) Horner stages (poly.py:155)
    for m, want in ((1, 0), (2, 1), (4, 2), (8, 4), (15, 6), (16, 6), (20, 7), (25, 8), (30, 9)):
        V = np.random.default_rng(m).uniform(-1, 1, (3, 3)) * 0.1
        ledger = [0]
        O._mm(V, V, ledger) if m >= 2 else None
        O._ps_eval([O.inv_factorial(i + 1) for i in range(m + 1)], V, ledger, {1: V, 2: V @ V} if m >= 2 else {})
        assert ledger[0] == want, m


def test_lowrank_pair_validation():
    z = torch.zeros
    with pytest.raises(ex.MatrixError):
        ex.LowRankPair(z(4, 2), z(3, 4))
    with pytest.raises(ex.MatrixError):
        ex.LowRankPair(z(2, 4), z(4, 2))            # t > n
    with pytest.raises(ex.MatrixError):
        ex.LowRankPair(z(4, 2), z(2, 4, dtype=torch.float64))
    with pytest.raises(ex.MatrixError):
        ex.LowRankPair(z(3, 4, 2), z(2, 2, 4))      # batch shapes differ
    p = ex.LowRankPair(z(5, 8, 2), z(5, 2, 8))
    assert (p.n, p.t) == (8, 2)
    with pytest.raises(RuntimeError):
        ex.expm_lowrank(p, 1e-8)                    # CPU tensors: no fallback


def test_timegrid_argument_errors_are_synchronous():
    L = _lib.lib()

    def call(K=4, n=128, dt=1, eps=1e-8, scheme=0, ws=None, wsb=0):
        return L.expmb_expm_timegrid(None, None, None, K, n, dt, eps, scheme, *([None] * 7), ws, wsb, None)
    assert call(eps=2.0 ** -54) == _lib.ERR_TOLERANCE
    assert call(dt=0, eps=2.0 ** -25) == _lib.ERR_TOLERANCE
    assert call(dt=4) == _lib.ERR_DTYPE
    assert call(scheme=2) == _lib.ERR_SCHEME      # Alg. 1 has no time-grid form
    assert call(n=0) == _lib.ERR_SHAPE
    assert call(K=0) == 0
    assert call() == _lib.ERR_WORKSPACE
    # workspace: 16 binary64 powers + one scratch matrix per time point (+ plans)
    need = L.expmb_timegrid_workspace_bytes(4, 128, 1)
    assert need >= 16 * 128 * 128 * 8 + 4 * 128 * 128 * 8
    assert L.expmb_timegrid_workspace_bytes(4, 16, 0) >= 4 * 16 * 16 * 4
