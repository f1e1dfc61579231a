"""Pin the CPU oracle against the reference's own outputs (tests/golden)."""
import math

import numpy as np
import pytest

from oracle import expm_oracle as O


def _cases(g):
    offs = g["offsets"]
    for i in range(len(g["names"])):
        n = int(g["n"][i])
        W = g["W"][offs[i]:offs[i + 1]].reshape(n, n)
        X = g["X"][offs[i]:offs[i + 1]].reshape(n, n)
        yield i, str(g["names"][i]), W, X, float(g["eps"][i]), str(g["scheme"][i])


def test_golden_count(golden):
    assert len(golden["names"]) >= 300


def test_oracle_bit_exact_vs_reference(golden):
    """Same (m, s, e1, e2, mults) and the same binary64 value, bit for bit."""
    for i, name, W, X, eps, scheme in _cases(golden):
        if golden["raised"][i]:
            with pytest.raises(O.NonFiniteError):
                O.expm_baseline(W, eps) if scheme == "baseline" else O.expm(W, eps, scheme)
            continue
        r = O.expm_baseline(W, eps) if scheme == "baseline" else O.expm(W, eps, scheme)
        assert (r.m, r.s, r.mults) == (golden["m"][i], golden["s"][i], golden["mults"][i]), name
        assert r.e1 == golden["e1"][i] or (math.isinf(r.e1) and math.isinf(golden["e1"][i])), name
        assert r.e2 == golden["e2"][i] or (math.isinf(r.e2) and math.isinf(golden["e2"][i])), name
        assert np.array_equal(r.value, X), name


def test_named_plans(golden):
    want = {("zero4", "sastre"): (0, 0, 0), ("diag1e-5", "sastre"): (1, 0, 0),
            ("diag1", "sastre"): (15, 0, 4), ("diag1_n5", "ps"): (12, 0, 5),
            ("diag12.57", "sastre"): (15, 3, 7), ("nilpotent2", "sastre"): (2, 0, 1)}
    got = {}
    for i, name, W, X, eps, scheme in _cases(golden):
        got[(name, scheme)] = (int(golden["m"][i]), int(golden["s"][i]), int(golden["mults"][i]))
    for k, v in want.items():
        assert got[k] == v, k


def test_tolerance_floor():
    with pytest.raises(O.ToleranceError):
        O.expm(np.eye(2), 2.0 ** -54)
    with pytest.raises(O.ToleranceError):
        O.expm(np.eye(2), float("nan"))
    O.expm(np.eye(2), 2.0 ** -53)
    with pytest.raises(O.ToleranceError):
        O.expm(np.eye(2), 2.0 ** -25, tol_floor=2.0 ** -24)


def test_scaling_cap():
    assert O.select(np.diag([1e30] * 4), 1e-8).s == 20
    assert O.select(np.array([[1e60]]), 1e-8, "ps").s == 20


def test_b16_and_tables():
    assert f"{O.B16:.15e}" == "2.608368698098256e-14"
    assert O.SASTRE_TABLES.orders == (1, 2, 4, 8, 15)
    assert [O.budget(m, "sastre") for m in (1, 2, 4, 8, 15)] == [0, 1, 2, 3, 4]
    assert [O.budget(m, "ps") for m in (6, 9, 12, 16)] == [3, 4, 5, 6]
