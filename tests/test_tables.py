"""Constants: product tables == oracle == the literals compiled into the kernels."""
import os
import re

from oracle import expm_oracle as O
import paper_2512_20777_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_product_tables_match_oracle():
    assert P.SASTRE_TABLES.log_tails == O.SASTRE_TABLES.log_tails
    assert P.PS_TABLES.log_tails == O.PS_TABLES.log_tails
    assert P.EXP_COEFFS.t8 == O.T8_COEFFS and P.EXP_COEFFS.t15p == O.T15P_COEFFS
    assert P.EXP_COEFFS.b16 == O.B16
    assert P.UNIT_ROUNDOFF == O.UNIT_ROUNDOFF and P.MAX_SCALING == O.MAX_SCALING
    assert [P.ps_shape(m).mults for m in (1, 2, 4, 6, 9, 12, 16)] == [0, 1, 2, 3, 4, 5, 6]
    assert [P.sastre_budget(m) for m in (1, 2, 4, 8, 15)] == [0, 1, 2, 3, 4]


def _hex_cases(src, fn):
    body = src[src.index(fn):]
    body = body[:body.index("}\n}")]
    return [float.fromhex(h) for h in re.findall(r"(-?0x1\.[0-9a-f]+p[+-]\d+)", body)]


def test_kernel_literals_match_python():
    src = open(os.path.join(ROOT, "paper_2512_20777_b200", "csrc", "select.cuh")).read()
    assert tuple(_hex_cases(src, "double sastre_log_tail")) == O.SASTRE_TABLES.log_tails
    assert tuple(_hex_cases(src, "double ps_log_tail")) == O.PS_TABLES.log_tails
    fs = open(os.path.join(ROOT, "paper_2512_20777_b200", "csrc", "fused_small.cuh")).read()
    t8 = re.search(r"kT8\[6\] = \{([^}]*)\}", fs).group(1)
    t15 = re.search(r"kT15\[16\] = \{([^}]*)\}", fs).group(1)
    assert tuple(float(x) for x in t8.replace("\n", " ").split(",")) == O.T8_COEFFS
    assert tuple(float(x) for x in t15.replace("\n", " ").split(",")) == O.T15P_COEFFS
    inv = re.search(r"kInvFact\[17\] = \{([^}]*)\}", fs).group(1)
    assert [float.fromhex(x.strip()) for x in inv.split(",")] == [O.inv_factorial(i) for i in range(17)]
