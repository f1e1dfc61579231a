"""Constants and tables of the reference, restated for the product side.

Same values as expmkit (select.py:55-56, :112-141; poly.py:75-118, :233-241);
the CUDA kernels carry identical literals in csrc/select.cuh and
csrc/fused_small.cuh.  tests/test_tables.py checks all three agree.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

UNIT_ROUNDOFF = 2.0 ** -53          # select.py:55
UNIT_ROUNDOFF_F32 = 2.0 ** -24      # same rule at fp32 working precision
MAX_SCALING = 20                    # select.py:56
SCHEME_PS = "ps"                    # select.py:59
SCHEME_SASTRE = "sastre"            # select.py:60


def inv_factorial(n: int) -> float:
    return float(Fraction(1, math.factorial(n)))


@dataclass(frozen=True)
class CoeffSet:
    """poly.py:104-118."""
    t8: tuple
    t15p: tuple
    b16: float


_T8 = (4.980119205559973e-3, 1.992047682223989e-2, 7.665265321119147e-2,
       8.765009801785554e-1, 1.225521150112075e-1, 2.974307204847627e0)
_T15P = (4.018761610201036e-4, 2.945531440279683e-3, -8.709066576837676e-3,
         4.017568440673568e-1, 3.230762888122312e-2, 5.768988513026145e0,
         2.338576034271299e-2, 2.381070373870987e-1, 2.224209172496374e0,
         -5.792361707073261e0, -4.130276365929783e-2, 1.040801735231354e1,
         -6.331712455883370e1, 3.484665863364574e-1, 1.0, 1.0)
EXP_COEFFS = CoeffSet(t8=_T8, t15p=_T15P, b16=_T15P[0] ** 4)


def _log2(x: float) -> float:
    return math.log2(x) if x > 0.0 else -math.inf


@dataclass(frozen=True)
class SelectionTables:
    """select.py:95-109."""
    orders: tuple
    block_pows: tuple
    block_counts: tuple
    tails: tuple
    log_tails: tuple = field(init=False)

    def __post_init__(self):
        object.__setattr__(self, "log_tails", tuple(_log2(c) for c in self.tails))


PS_TABLES = SelectionTables(
    orders=(1, 2, 4, 6, 9, 12, 16), block_pows=(1, 2, 2, 3, 3, 4, 4),
    block_counts=(1, 1, 2, 2, 3, 3, 4),
    tails=tuple(inv_factorial(i) for i in (2, 3, 3, 4, 5, 6, 7, 8, 10, 11, 13, 14, 17, 18)))
SASTRE_TABLES = SelectionTables(
    orders=(1, 2, 4, 8, 15), block_pows=(1, 2, 2, 2, 2), block_counts=(1, 1, 2, 4, 8),
    tails=tuple(inv_factorial(i) for i in (2, 3, 3, 4, 5, 6, 9, 10))
    + (abs(inv_factorial(16) - EXP_COEFFS.b16), inv_factorial(17)))

_SASTRE_BUDGET = {1: 0, 2: 1, 4: 2, 8: 3, 15: 4}


class MatrixError(ValueError):
    """matrix.py:31."""


class NonFiniteError(MatrixError):
    """matrix.py:35."""


class ToleranceError(ValueError):
    """select.py:64."""


class LowRankOrderError(ArithmeticError):
    """engine.py:60 -- no order on LOWRANK_ORDERS meets the tolerance."""


LOWRANK_ORDERS = (1, 2, 4, 8, 15, 16, 20, 25, 30)   # engine.py:195
SCHEME_LOWRANK = "lowrank"                         # select.py:61


@dataclass(frozen=True)
class PsShape:
    """poly.py:125-134."""
    m: int
    j: int
    k: int

    @property
    def mults(self) -> int:
        return (self.j - 1) + (self.k - 1)


def ps_shape(m: int) -> PsShape:
    """poly.py:136-146."""
    if m < 1:
        raise MatrixError("Paterson-Stockmeyer shape needs degree >= 1")
    j = math.isqrt(m)
    if j * j < m:
        j += 1
    return PsShape(m=m, j=j, k=-(-m // j))


def sastre_budget(m: int) -> int:
    """poly.py:236-241."""
    try:
        return _SASTRE_BUDGET[m]
    except KeyError:
        raise MatrixError(f"no evaluation formula for order {m}") from None
