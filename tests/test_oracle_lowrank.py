"""Pin the oracle's low-rank restatement (engine.py:159-270) against the
reference's own outputs (tests/golden/lowrank_golden.npz)."""
import math

import numpy as np
import pytest

from conftest import lowrank_cases
from oracle import expm_oracle as O


def test_lowrank_golden_count(lowrank_golden):
    assert len(lowrank_golden["names"]) >= 100
    # every order of the ladder and the error path are exercised
    ms = set(int(m) for m in lowrank_golden["m"])
    assert set(O.LOWRANK_ORDERS) | {0, -1} <= ms


def test_lowrank_oracle_bit_exact(lowrank_golden):
    g = lowrank_golden
    for i, name, A1, A2, X, eps in lowrank_cases(g):
        if g["raised"][i]:
            with pytest.raises(O.LowRankOrderError):
                O.expm_lowrank(A1, A2, eps)
            continue
        r = O.expm_lowrank(A1, A2, eps)
        assert (r.m, r.mults, r.rect_mults) == (g["m"][i], g["mults"][i], g["rect_mults"][i]), name
        assert r.e1 == g["e1"][i] and r.e2 == g["e2"][i], name
        assert r.norm1 == g["norm1"][i], name
        assert r.norm2 == g["norm2"][i] or (math.isnan(r.norm2) and math.isnan(g["norm2"][i])), name
        assert np.array_equal(r.value, X), name


def test_lowrank_named(lowrank_golden):
    g = lowrank_golden
    got = {str(g["names"][i]): (int(g["m"][i]), int(g["mults"][i])) for i in range(len(g["names"]))}
    assert got["zero_factor"] == (0, 0)
    assert got["nilpotent_v0"] == (0, 0)
    assert got["psi_1x1"][0] in O.LOWRANK_ORDERS
    assert got["norm_too_large"] == (-1, -1)


def test_lowrank_validation():
    with pytest.raises(O.MatrixError):
        O.expm_lowrank(np.zeros((4, 2)), np.zeros((3, 4)), 1e-8)
    with pytest.raises(O.MatrixError):
        O.expm_lowrank(np.zeros((2, 4)), np.zeros((4, 2)), 1e-8)
    with pytest.raises(O.MatrixError):
        O.expm_lowrank(np.full((4, 2), np.nan), np.zeros((2, 4)), 1e-8)
    with pytest.raises(O.ToleranceError):
        O.expm_lowrank(np.zeros((4, 2)), np.zeros((2, 4)), 2.0 ** -54)


def test_lowrank_value_identity():
    # e^(A1 A2) with V = A2 A1 = 0 is I + A1 A2 exactly
    r = O.expm_lowrank(np.array([[1.0], [0.0]]), np.array([[0.0, 3.0]]), 1e-8)
    assert np.array_equal(r.value, np.array([[1.0, 3.0], [0.0, 1.0]]))
