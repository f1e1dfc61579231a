"""CPU oracle for the batched scaled-Taylor exponential -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2512_20777_b200``) never imports anything under ``oracle/`` and fails
loudly when its CUDA library is missing.

It is a plain NumPy restatement of the reference package ``expmkit``
(``/root/reference/pkg/src/expmkit``), one binary64 matrix at a time, with
the same operation order as the reference so that its outputs agree with the
reference bit for bit on the committed golden vectors
(``tests/golden/make_golden.py`` generated them by importing the reference;
``tests/test_oracle_golden.py`` pins this module against them).

Parity pinned: yes (golden vectors from the reference itself).

Reference map (file:line under /root/reference/pkg/src/expmkit):
  * UNIT_ROUNDOFF / MAX_SCALING ............ select.py:55-56
  * check_tolerance ........................ select.py:72-79
  * tables (SASTRE_TABLES / PS_TABLES) ..... select.py:112-141
  * _select ladder + scaling rule .......... select.py:164-220
  * T8 / T15+ coefficients, b16 ............ poly.py:75-118
  * ps_shape / ps_eval ..................... poly.py:136-182
  * eval_low_order / eval_t8 / eval_t15p ... poly.py:189-230
  * sastre_budget .......................... poly.py:233-241
  * expm driver ............................ engine.py:119-152
  * squaring ............................... engine.py:80-87
  * expm_baseline (Alg. 1) .................. engine.py:90-116
  * finiteness semantics (_wrap) ........... matrix.py:56-57, 95-102
  * expm_lowrank / LowRankPair checks ...... engine.py:159-270
  * phi1 coefficients 1/(i+1)! ............. poly.py:62-66
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

UNIT_ROUNDOFF = 2.0 ** -53          # select.py:55
MAX_SCALING = 20                    # select.py:56
SCHEME_PS = "ps"
SCHEME_SASTRE = "sastre"


class MatrixError(ValueError):
    """matrix.py:31 -- invalid shape/argument."""


class NonFiniteError(MatrixError):
    """matrix.py:35 -- NaN/Inf on entry or produced by an operation."""


class ToleranceError(ValueError):
    """select.py:64 -- tolerance NaN or below the unit roundoff."""


def inv_factorial(n: int) -> float:
    """poly.py:44-46: 1/n! correctly rounded to binary64."""
    return float(Fraction(1, math.factorial(n)))


# poly.py:75-101 -- published binary64 literals of the evaluation formulas.
T8_COEFFS = (
    4.980119205559973e-3, 1.992047682223989e-2, 7.665265321119147e-2,
    8.765009801785554e-1, 1.225521150112075e-1, 2.974307204847627e0,
)
T15P_COEFFS = (
    4.018761610201036e-4, 2.945531440279683e-3, -8.709066576837676e-3,
    4.017568440673568e-1, 3.230762888122312e-2, 5.768988513026145e0,
    2.338576034271299e-2, 2.381070373870987e-1, 2.224209172496374e0,
    -5.792361707073261e0, -4.130276365929783e-2, 1.040801735231354e1,
    -6.331712455883370e1, 3.484665863364574e-1, 1.0, 1.0,
)
B16 = T15P_COEFFS[0] ** 4           # poly.py:118


def _log2(x: float) -> float:
    """select.py:82-83."""
    return math.log2(x) if x > 0.0 else -math.inf


@dataclass(frozen=True)
class Tables:
    """select.py:95-109."""
    orders: tuple
    block_pows: tuple
    block_counts: tuple
    tails: tuple
    log_tails: tuple = field(init=False)

    def __post_init__(self):
        object.__setattr__(self, "log_tails", tuple(_log2(c) for c in self.tails))


PS_TABLES = Tables(                 # select.py:112-125
    orders=(1, 2, 4, 6, 9, 12, 16),
    block_pows=(1, 2, 2, 3, 3, 4, 4),
    block_counts=(1, 1, 2, 2, 3, 3, 4),
    tails=tuple(inv_factorial(i) for i in (2, 3, 3, 4, 5, 6, 7, 8, 10, 11, 13, 14, 17, 18)),
)
SASTRE_TABLES = Tables(             # select.py:130-141
    orders=(1, 2, 4, 8, 15),
    block_pows=(1, 2, 2, 2, 2),
    block_counts=(1, 1, 2, 4, 8),
    tails=tuple(inv_factorial(i) for i in (2, 3, 3, 4, 5, 6, 9, 10))
    + (abs(inv_factorial(16) - B16), inv_factorial(17)),
)
SASTRE_BUDGET = {0: 0, 1: 0, 2: 1, 4: 2, 8: 3, 15: 4}   # poly.py:233-241 (+ m=0)


def ps_shape(m: int):
    """poly.py:136-146: (j, k) with j = ceil(sqrt(m)), k = ceil(m / j)."""
    j = math.isqrt(m)
    if j * j < m:
        j += 1
    return j, -(-m // j)


def budget(m: int, scheme: str) -> int:
    if m == 0:
        return 0
    if scheme == SCHEME_PS:
        j, k = ps_shape(m)
        return (j - 1) + (k - 1)
    return SASTRE_BUDGET[m]


def check_tolerance(eps: float, floor: float = UNIT_ROUNDOFF) -> float:
    """select.py:72-79 (``floor`` = 2^-24 for the fp32 extension)."""
    eps = float(eps)
    if math.isnan(eps) or eps < floor:
        raise ToleranceError(f"tolerance {eps!r} below unit roundoff {floor:.3e}")
    return eps


def _wrap(a: np.ndarray) -> np.ndarray:
    """matrix.py:95-102: every derived matrix is re-validated."""
    if not np.isfinite(a).all():
        raise NonFiniteError("operation produced non-finite entries")
    return a


def one_norm(a: np.ndarray) -> float:
    """matrix.py:149-151."""
    return float(np.abs(a).sum(axis=0).max())


def _mm(a, b, ledger):
    """matrix.py:139-146: one charged product."""
    with np.errstate(over="ignore", invalid="ignore"):
        c = a @ b
    ledger[0] += 1
    return _wrap(c)


def _scale(a, s):
    """matrix.py:159-167: exact ldexp."""
    return a if s == 0 else _wrap(np.ldexp(a, -s))


@dataclass
class Plan:
    """select.py:144-161 (powers kept as arrays)."""
    m: int
    s: int
    e1: float
    e2: float
    powers: dict
    norms: dict


def select(W: np.ndarray, eps: float, scheme: str = SCHEME_SASTRE, ledger=None) -> Plan:
    """select.py:164-220 restated line for line."""
    tables = PS_TABLES if scheme == SCHEME_PS else SASTRE_TABLES
    if ledger is None:
        ledger = [0]
    norm1 = one_norm(W)
    powers = {1: W}
    norms = {1: norm1}
    if norm1 == 0.0:
        return Plan(0, 0, 0.0, 0.0, powers, norms)
    log_eps = math.log2(eps)
    lw = {1: _log2(norm1)}
    l1 = l2 = math.inf
    m = tables.orders[-1]
    finished = False
    for i, m_i in enumerate(tables.orders):
        m = m_i
        j = tables.block_pows[i]
        k = tables.block_counts[i]
        lc1 = tables.log_tails[2 * i]
        lc2 = tables.log_tails[2 * i + 1]
        if m_i == 1:
            l1 = lc1 + 2 * lw[1]
            l2 = lc2 + 3 * lw[1]
        else:
            for p in range(2, j + 1):
                if p not in powers:
                    powers[p] = _mm(powers[p - 1], W, ledger)
                    norms[p] = one_norm(powers[p])
                    lw[p] = _log2(norms[p])
            if scheme == SCHEME_PS:
                l1 = lc1 + k * lw[j] + lw[1]
                l2 = lc2 + k * lw[j] + lw[2]
            else:
                l1 = lc1 + k * lw[j]
                l2 = lc2 + k * lw[j]
                if j * k == m_i:
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
            s1 = math.ceil((l - log_eps) / (m + t))
            if s1 > s:
                s = s1
        if s > MAX_SCALING:
            s = MAX_SCALING
    with np.errstate(over="ignore"):
        e1, e2 = float(np.exp2(l1)), float(np.exp2(l2))
    return Plan(m, s, e1, e2, powers, norms)


def _ps_eval(coeffs, A, ledger, powers):
    """poly.py:149-182."""
    m = len(coeffs) - 1
    eye = np.eye(A.shape[0])
    if m == 0:
        return coeffs[0] * eye
    j, k = ps_shape(m)
    pw = dict(powers)
    pw[1] = A
    for p in range(2, j + 1):
        if p not in pw:
            pw[p] = _mm(pw[p - 1], A, ledger)

    def block(lo, hi):
        acc = _wrap(eye * float(coeffs[lo]))
        for t in range(1, hi - lo + 1):
            acc = _wrap(acc + _wrap(pw[t] * float(coeffs[lo + t])))
        return acc

    q = block((k - 1) * j, m)
    for r in range(k - 2, -1, -1):
        q = _wrap(_mm(q, pw[j], ledger) + block(r * j, r * j + j - 1))
    return q


def _eval_low(A, m, a2, ledger):
    """poly.py:189-201."""
    eye = np.eye(A.shape[0])
    if m == 1:
        return _wrap(A + eye)
    if m == 2:
        return _wrap(_wrap(_wrap(a2 / 2.0) + A) + eye)
    inner = _wrap(_wrap(_wrap(_wrap(a2 / 4.0) + A) / 3.0) + eye)
    return _wrap(_wrap(_wrap(_mm(inner, a2, ledger) / 2.0) + A) + eye)


def _lc(*terms):
    """Left-to-right sum of (coef, matrix) / matrix terms, as numpy does."""
    acc = None
    for t in terms:
        v = t if isinstance(t, np.ndarray) else _wrap(t[1] * float(t[0]))
        acc = v if acc is None else _wrap(acc + v)
    return acc


def _eval_t8(A, a2, ledger):
    """poly.py:204-212."""
    c = T8_COEFFS
    eye = np.eye(A.shape[0])
    y02 = _mm(a2, _lc((c[0], a2), (c[1], A)), ledger)
    prod = _mm(_lc(y02, (c[2], a2), (c[3], A)), _lc(y02, (c[4], a2)), ledger)
    return _lc(prod, (c[5], y02), _wrap(a2 / 2.0), A, eye)


def _eval_t15p(A, a2, ledger):
    """poly.py:215-230."""
    c = T15P_COEFFS
    eye = np.eye(A.shape[0])
    y02 = _mm(a2, _lc((c[0], a2), (c[1], A)), ledger)
    y12 = _lc(_mm(_lc(y02, (c[2], a2), (c[3], A)), _lc(y02, (c[4], a2)), ledger),
              (c[5], y02), (c[6], a2))
    y22 = _lc(_mm(_lc(y12, (c[7], a2), (c[8], A)), _lc(y12, (c[9], y02), (c[10], A)), ledger),
              (c[11], y12), (c[12], y02), (c[13], a2), (c[14], A), (c[15], eye))
    return y22


@dataclass
class Result:
    value: np.ndarray
    m: int
    s: int
    e1: float
    e2: float
    norm1: float
    norm2: float
    mults: int


def expm(W, eps: float, scheme: str = SCHEME_SASTRE, tol_floor: float = UNIT_ROUNDOFF) -> Result:
    """engine.py:119-152 restated.  ``W`` is upcast to binary64 exactly."""
    W = np.array(W, dtype=np.float64)
    if W.ndim != 2 or W.shape[0] != W.shape[1]:
        raise MatrixError(f"expected a square 2-d array, got shape {W.shape}")
    if W.shape[0] < 1:
        raise MatrixError("matrix order must be at least 1")
    if not np.isfinite(W).all():
        raise NonFiniteError("matrix entries must be finite")
    if scheme not in (SCHEME_PS, SCHEME_SASTRE):
        raise MatrixError(f"unknown scheme {scheme!r}; expected 'ps' or 'sastre'")
    eps = check_tolerance(eps, tol_floor)
    ledger = [0]
    plan = select(W, eps, scheme, ledger)
    B = _scale(W, plan.s)
    scaled = {p: _scale(P, plan.s * p) for p, P in plan.powers.items()}
    n = W.shape[0]
    if plan.m == 0:
        X = np.eye(n)
    elif scheme == SCHEME_PS:
        X = _ps_eval([inv_factorial(i) for i in range(plan.m + 1)], B, ledger, scaled)
    elif plan.m in (1, 2, 4):
        X = _eval_low(B, plan.m, scaled.get(2), ledger)
    elif plan.m == 8:
        X = _eval_t8(B, scaled[2], ledger)
    else:
        X = _eval_t15p(B, scaled[2], ledger)
    for _ in range(plan.s):                       # engine.py:80-87
        X = _mm(X, X, ledger)
    return Result(X, plan.m, plan.s, plan.e1, plan.e2, plan.norms[1],
                  plan.norms.get(2, float("nan")), ledger[0])


def expm_batch(Wb, eps: float, scheme: str = SCHEME_SASTRE, tol_floor: float = UNIT_ROUNDOFF):
    """Caller loop over a [B, n, n] stack (the reference's batching, bench.py:272-309).

    Returns (values[B,n,n] f64, m[B], s[B], e1[B], e2[B], mults[B], nonfinite[B]).
    Matrices whose evaluation raises NonFiniteError are flagged, not fatal
    (the reference suite records them as NaN rows, bench.py:280-284).
    """
    Wb = np.asarray(Wb)
    B, n = Wb.shape[0], Wb.shape[-1]
    out = np.full((B, n, n), np.nan)
    m = np.zeros(B, np.int64)
    s = np.zeros(B, np.int64)
    e1 = np.zeros(B)
    e2 = np.zeros(B)
    mults = np.zeros(B, np.int64)
    bad = np.zeros(B, bool)
    for i in range(B):
        try:
            r = expm(Wb[i], eps, scheme, tol_floor)
        except NonFiniteError:
            bad[i] = True
            continue
        out[i], m[i], s[i], e1[i], e2[i], mults[i] = r.value, r.m, r.s, r.e1, r.e2, r.mults
    return out, m, s, e1, e2, mults, bad


def near_threshold(norm1: float, norm2: float, eps: float, scheme: str = SCHEME_SASTRE,
                   margin: float = 1e-4) -> bool:
    """True when the (m, s) decision would flip if log2 ||W||_1 or log2 ||W^2||_1
    moved by ``margin`` (SURVEY.md 8(d) "(m,s) parity exemption").  Sastre only
    needs ||W||_1 and ||W^2||_1 (select.py:228-234)."""
    base = _plan_from_norms(norm1, norm2, eps)
    for d1 in (-margin, 0.0, margin):
        for d2 in (-margin, 0.0, margin):
            n1 = norm1 * 2.0 ** d1
            n2 = norm2 * 2.0 ** d2
            if _plan_from_norms(n1, n2, eps) != base:
                return True
    return False


def plan_from_power_norms(norms: dict, eps: float, scheme: str = SCHEME_SASTRE):
    """The (m, s) that select.py:164-220 picks from given power norms
    ``norms[p] = ||W^p||_1`` (p = 1..4 as the ladder needs them; no products)."""
    tables = PS_TABLES if scheme == SCHEME_PS else SASTRE_TABLES
    if norms[1] == 0.0:
        return (0, 0)
    log_eps = math.log2(eps)
    lw = {p: _log2(v) for p, v in norms.items()}
    l1 = l2 = math.inf
    m = tables.orders[-1]
    for i, m_i in enumerate(tables.orders):
        m = m_i
        j, k = tables.block_pows[i], tables.block_counts[i]
        lc1, lc2 = tables.log_tails[2 * i], tables.log_tails[2 * i + 1]
        if m_i == 1:
            l1, l2 = lc1 + 2 * lw[1], lc2 + 3 * lw[1]
        elif scheme == SCHEME_PS:
            l1, l2 = lc1 + k * lw[j] + lw[1], lc2 + k * lw[j] + lw[2]
        else:
            l1, l2 = lc1 + k * lw[j], lc2 + k * lw[j]
            if j * k == m_i:
                l1 += lw[1]
                l2 += lw[2]
            else:
                l2 += lw[1]
        if float(np.logaddexp2(l1, l2)) <= log_eps:
            return (m, 0)
    s = 0
    for tt, l in ((1, l1), (2, l2)):
        if l == -math.inf:
            continue
        s = max(s, math.ceil((l - log_eps) / (m + tt)))
    return (m, min(s, MAX_SCALING))


def near_threshold_powers(W, eps: float, scheme: str = SCHEME_SASTRE, margin: float = 1e-4) -> bool:
    """``near_threshold`` for either scheme from the matrix itself: the plan
    flips if any power norm ||W^p||_1 (p = 1..4 for PS, 1..2 for Sastre)
    moves by ``margin`` log2 units."""
    W = np.asarray(W, np.float64)
    P, norms = W, {1: one_norm(W)}
    for p in range(2, (4 if scheme == SCHEME_PS else 2) + 1):
        P = P @ W
        norms[p] = one_norm(P)
    base = plan_from_power_norms(norms, eps, scheme)
    for p in norms:
        for d in (-margin, margin):
            nn = dict(norms)
            nn[p] = norms[p] * 2.0 ** d
            if plan_from_power_norms(nn, eps, scheme) != base:
                return True
    return False


def _plan_from_norms(norm1: float, norm2: float, eps: float):
    """Sastre ladder of select.py:180-219 on given norms (no products)."""
    if norm1 == 0.0:
        return (0, 0)
    t = SASTRE_TABLES
    log_eps = math.log2(eps)
    lw1, lw2 = _log2(norm1), _log2(norm2)
    l1 = l2 = math.inf
    m = 15
    for i, m_i in enumerate(t.orders):
        m = m_i
        j, k = t.block_pows[i], t.block_counts[i]
        lc1, lc2 = t.log_tails[2 * i], t.log_tails[2 * i + 1]
        if m_i == 1:
            l1, l2 = lc1 + 2 * lw1, lc2 + 3 * lw1
        else:
            l1, l2 = lc1 + k * lw2, lc2 + k * lw2
            if j * k == m_i:
                l1 += lw1
                l2 += lw2
            else:
                l2 += lw1
        if float(np.logaddexp2(l1, l2)) <= log_eps:
            return (m, 0)
    s = 0
    for tt, l in ((1, l1), (2, l2)):
        if l == -math.inf:
            continue
        s = max(s, math.ceil((l - log_eps) / (m + tt)))
    return (m, min(s, MAX_SCALING))


def expm_baseline(W, eps: float, tol_floor: float = UNIT_ROUNDOFF) -> Result:
    """engine.py:90-116 restated: norm-halving scaling, term accumulation until
    the next term's 1-norm is <= eps, s squarings; mults = m + s."""
    W = np.array(W, dtype=np.float64)
    if not np.isfinite(W).all():
        raise NonFiniteError("matrix entries must be finite")
    eps = check_tolerance(eps, tol_floor)
    ledger = [0]
    s = 0
    norm1 = one_norm(W)
    while math.ldexp(norm1, -s) >= 0.5:
        s += 1
    B = _scale(W, s)
    n = W.shape[0]
    X = np.eye(n)
    Y = B
    k = 2
    while one_norm(Y) > eps:
        X = _wrap(X + Y)
        Y = _wrap(_mm(B, Y, ledger) / k)
        k += 1
    for _ in range(s):
        X = _mm(X, X, ledger)
    return Result(X, k - 2, s, one_norm(Y), 0.0, norm1, float("nan"), ledger[0])


# ---------------------------------------------------------------------------
# Low-rank path (engine.py:159-270): W = A1 A2, e^W = I + A1 psi(V) A2, V = A2 A1
# ---------------------------------------------------------------------------

LOWRANK_ORDERS = (1, 2, 4, 8, 15, 16, 20, 25, 30)                  # engine.py:195
LOG2_FACT = [math.lgamma(i + 1) / math.log(2.0) for i in range(40)]  # engine.py:260


class LowRankOrderError(ArithmeticError):
    """engine.py:60 -- no order on the ladder meets the tolerance (no scaling)."""


def _power_bound_log(q: int, lw1: float, lw2: float) -> float:
    """engine.py:263-265: log2 of ||V^2||^(q//2) ||V||^(q%2)."""
    return (q // 2) * lw2 + (q % 2) * lw1


def select_lowrank_from_norms(nv: float, nv2, eps: float):
    """The order ladder of engine.py:224-244 on given norms.  ``nv2`` may be a
    callable producing ||V^2||_1 lazily (the reference forms V^2 only when
    rung m=1 fails).  Returns (m, e1, e2, used_v2) or raises LowRankOrderError."""
    if nv == 0.0:
        return 0, 0.0, 0.0, False
    log_eps = math.log2(eps)
    lw1 = math.log2(nv) if nv > 0 else -math.inf
    lw2 = None
    used = False
    for m in LOWRANK_ORDERS:
        if m >= 2 and lw2 is None:
            n2 = nv2() if callable(nv2) else nv2
            used = True
            lw2 = math.log2(n2) if n2 > 0 else -math.inf
        if m == 1:
            l1 = 2 * lw1 - LOG2_FACT[3]
            l2 = 3 * lw1 - LOG2_FACT[4]
        else:
            l1 = _power_bound_log(m + 1, lw1, lw2) - LOG2_FACT[m + 2]
            l2 = _power_bound_log(m + 2, lw1, lw2) - LOG2_FACT[m + 3]
        if float(np.logaddexp2(l1, l2)) <= log_eps:
            with np.errstate(over="ignore"):
                return m, float(np.exp2(l1)), float(np.exp2(l2)), used
    raise LowRankOrderError(f"||V||_1 = {nv:.6g} admits no order <= {LOWRANK_ORDERS[-1]} at tolerance {eps:.3g}")


@dataclass
class LowRankResult:
    value: np.ndarray
    m: int
    e1: float
    e2: float
    norm1: float
    norm2: float
    mults: int
    rect_mults: int


def expm_lowrank(a1, a2, eps: float, tol_floor: float = UNIT_ROUNDOFF) -> LowRankResult:
    """engine.py:198-257 restated (LowRankPair validation engine.py:166-181)."""
    a1 = np.array(a1, dtype=np.float64)
    a2 = np.array(a2, dtype=np.float64)
    if a1.ndim != 2 or a2.ndim != 2:
        raise MatrixError("low-rank factors must be 2-d arrays")
    n, t = a1.shape
    if a2.shape != (t, n):
        raise MatrixError(f"factor shapes incompatible: {a1.shape} and {a2.shape}")
    if t > n:
        raise MatrixError(f"inner rank {t} exceeds order {n}")
    if not (np.isfinite(a1).all() and np.isfinite(a2).all()):
        raise MatrixError("low-rank factors must be finite")
    eps = check_tolerance(eps, tol_floor)
    ledger = [0]
    V = _wrap(a2 @ a1)
    nv = one_norm(V)
    powers = {1: V}
    norms = {}

    def v2():
        powers[2] = _mm(V, V, ledger)
        norms[2] = one_norm(powers[2])
        return norms[2]

    m, e1, e2, _ = select_lowrank_from_norms(nv, v2, eps)
    if m == 0:
        psi = np.eye(t)
    else:
        psi = _ps_eval([inv_factorial(i + 1) for i in range(m + 1)], V, ledger, powers)
    out = _wrap(np.eye(n) + a1 @ (psi @ a2))
    return LowRankResult(out, m, e1, e2, nv, norms.get(2, float("nan")), ledger[0], 3)


def lowrank_near_threshold(nv: float, nv2: float, eps: float, margin: float = 1e-4) -> bool:
    """True when the low-rank order would change if log2 ||V||_1 or log2 ||V^2||_1
    moved by ``margin`` (the same exemption as ``near_threshold``)."""
    def pick(a, b):
        try:
            return select_lowrank_from_norms(a, b, eps)[0]
        except LowRankOrderError:
            return -1
    base = pick(nv, nv2)
    for d1 in (-margin, 0.0, margin):
        for d2 in (-margin, 0.0, margin):
            if pick(nv * 2.0 ** d1, nv2 * 2.0 ** d2) != base:
                return True
    return False
