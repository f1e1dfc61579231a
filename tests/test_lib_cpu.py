"""CPU-side checks of the C ABI (no GPU needed): load, exports, selector parity."""
import ctypes
import math
import re
import os

import numpy as np
import pytest

from paper_2512_20777_b200 import _lib
from oracle import expm_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    hdr = open(os.path.join(ROOT, "include", "expmb.h")).read()
    declared = set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(expmb_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTS), declared
    for name in declared:
        assert hasattr(L, name), name
    assert L.expmb_version() >= 100


def test_unit_roundoff():
    L = _lib.lib()
    assert L.expmb_unit_roundoff(_lib.EXPMB_F64) == 2.0 ** -53
    assert L.expmb_unit_roundoff(_lib.EXPMB_F32) == 2.0 ** -24


def test_argument_errors_are_synchronous():
    """Validation happens before any device work (select.py:72-79, engine.py:137)."""
    L = _lib.lib()
    args = lambda eps=1e-8, dt=1, sch=0, n=4, b=1: (None, None, b, n, dt, eps, sch, *([None] * 7), None, 0, None)
    assert L.expmb_expm(*args(eps=2.0 ** -54)) == _lib.ERR_TOLERANCE
    assert L.expmb_expm(*args(eps=float("nan"))) == _lib.ERR_TOLERANCE
    assert L.expmb_expm(*args(dt=0, eps=2.0 ** -25)) == _lib.ERR_TOLERANCE
    assert L.expmb_expm(*args(sch=7)) == _lib.ERR_SCHEME
    assert L.expmb_expm(*args(dt=3)) == _lib.ERR_DTYPE
    assert L.expmb_expm(*args(n=0)) == _lib.ERR_SHAPE
    assert L.expmb_expm(*args(b=0)) == 0          # empty batch is a no-op
    assert L.expmb_expm(*args(n=128)) == _lib.ERR_WORKSPACE
    assert L.expmb_workspace_bytes(4, 16, 0, 0) == 256
    assert L.expmb_workspace_bytes(4, 256, 0, 0) > 7 * 4 * 256 * 256 * 4


def _oracle_plan_from_norms(norms, eps, scheme):
    """Run the oracle ladder on synthetic power norms via a diagonal-free trick:
    reuse oracle.select's arithmetic by monkeypatching one_norm on fake powers."""
    tables = O.PS_TABLES if scheme == "ps" else O.SASTRE_TABLES
    norm1 = norms[0]
    if norm1 == 0.0:
        return 0, 0, 0.0, 0.0
    log_eps = math.log2(eps)
    lw = {p + 1: O._log2(v) for p, v in enumerate(norms)}
    l1 = l2 = math.inf
    m = tables.orders[-1]
    finished = False
    for i, mi in enumerate(tables.orders):
        m = mi
        j, k = tables.block_pows[i], tables.block_counts[i]
        lc1, lc2 = tables.log_tails[2 * i], tables.log_tails[2 * i + 1]
        if mi == 1:
            l1 = lc1 + 2 * lw[1]
            l2 = lc2 + 3 * lw[1]
        elif scheme == "ps":
            l1 = lc1 + k * lw[j] + lw[1]
            l2 = lc2 + k * lw[j] + lw[2]
        else:
            l1 = lc1 + k * lw[j]
            l2 = lc2 + k * lw[j]
            if j * k == mi:
                l1 += lw[1]
                l2 += lw[2]
            else:
                l2 += lw[1]
        if float(np.logaddexp2(l1, l2)) <= log_eps:
            finished = True
            break
    s = 0
    if not finished:
        for t, l in ((1, l1), (2, l2)):
            if l == -math.inf:
                continue
            s = max(s, math.ceil((l - log_eps) / (m + t)))
        s = min(s, O.MAX_SCALING)
    with np.errstate(over="ignore"):
        return m, s, float(np.exp2(l1)), float(np.exp2(l2))


@pytest.mark.parametrize("scheme", ["sastre", "ps"])
def test_host_selector_matches_oracle_ladder(scheme):
    """The kernels' __host__ __device__ selector == select.py's ladder on 20k norm sets."""
    rng = np.random.default_rng(5 if scheme == "sastre" else 6)
    code = _lib.EXPMB_SASTRE if scheme == "sastre" else _lib.EXPMB_PS
    mism = 0
    for it in range(20000):
        n1 = float(10.0 ** rng.uniform(-9, 4))
        # submultiplicative power norms with random slack (and exact zeros sometimes)
        ratios = 10.0 ** rng.uniform(-3, 0, 3)
        norms = [n1, n1 * n1 * ratios[0]]
        norms.append(norms[1] * n1 * ratios[1])
        norms.append(norms[2] * n1 * ratios[2])
        if it % 97 == 0:
            norms[1] = 0.0
            norms[2] = norms[3] = 0.0
        eps = (1e-12, 1e-8, 1e-4, 2.0 ** -24, 2.0 ** -53)[it % 5]
        want = _oracle_plan_from_norms(norms, eps, scheme)
        m, s, e1, e2, have = _lib.select_host(norms, eps, code)
        assert (m, s) == want[:2], (norms, eps, want, (m, s))
        for a, b in ((e1, want[2]), (e2, want[3])):
            assert a == b or (math.isinf(a) and math.isinf(b)) or abs(a - b) <= 1e-12 * abs(b)
    assert mism == 0


def test_host_selector_golden(golden):
    """Selector on the reference's own plans (norms recomputed here in binary64)."""
    offs = golden["offsets"]
    for i in range(len(golden["names"])):
        if golden["raised"][i] or str(golden["scheme"][i]) == "baseline":
            continue
        n = int(golden["n"][i])
        W = golden["W"][offs[i]:offs[i + 1]].reshape(n, n)
        scheme = str(golden["scheme"][i])
        norms = [O.one_norm(W)]
        P = W
        for _ in range(3):
            P = P @ W
            norms.append(O.one_norm(P))
        code = _lib.EXPMB_SASTRE if scheme == "sastre" else _lib.EXPMB_PS
        m, s, e1, e2, _ = _lib.select_host(norms, float(golden["eps"][i]), code)
        assert (m, s) == (golden["m"][i], golden["s"][i]), golden["names"][i]


def test_int8_slice_workspace_switch(monkeypatch):
    """The int8-slice path (fp32, n >= 512 by default) adds its slice planes
    and statistics to the large-n workspace; EXPMB_I8=0 removes them."""
    L = _lib.lib()
    monkeypatch.delenv("EXPMB_I8", raising=False)
    on = L.expmb_workspace_bytes(8, 1024, _lib.EXPMB_F32, _lib.EXPMB_SASTRE)
    monkeypatch.setenv("EXPMB_I8", "0")
    off = L.expmb_workspace_bytes(8, 1024, _lib.EXPMB_F32, _lib.EXPMB_SASTRE)
    # 8 slice planes of n x n bytes per matrix at least
    assert on - off >= 8 * 8 * 1024 * 1024
    monkeypatch.delenv("EXPMB_I8", raising=False)
    # fp64 and small orders never use it
    assert L.expmb_workspace_bytes(8, 1024, _lib.EXPMB_F64, 0) == L.expmb_workspace_bytes(8, 1024, _lib.EXPMB_F64, 0)
    monkeypatch.setenv("EXPMB_I8", "0")
    small_off = L.expmb_workspace_bytes(8, 256, _lib.EXPMB_F32, 0)
    monkeypatch.delenv("EXPMB_I8", raising=False)
    assert L.expmb_workspace_bytes(8, 256, _lib.EXPMB_F32, 0) == small_off
