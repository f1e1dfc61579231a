"""expmkit_b200 -- B200-native batched matrix exponential (arXiv 2512.20777).

Drop-in for the reference hot path ``expmkit.expm`` (engine.py:119-152),
batched over a leading tensor dimension, computed by hand-written sm_100a
CUDA kernels in libexpmb.so (C ABI: include/expmb.h).
"""

from .tables import (  # noqa: F401
    EXP_COEFFS, MAX_SCALING, PS_TABLES, SASTRE_TABLES, SCHEME_PS, SCHEME_SASTRE, UNIT_ROUNDOFF,
    UNIT_ROUNDOFF_F32, CoeffSet, MatrixError, NonFiniteError, PsShape, SelectionTables,
    ToleranceError, ps_shape, sastre_budget, LOWRANK_ORDERS, LowRankOrderError, SCHEME_LOWRANK,
)
from .api import (  # noqa: F401
    EvalPlan, ExpmResult, HostPipeline, SCHEME_BASELINE, check_tolerance, expm, expm_baseline, expm_host, expm_into, select_ps, select_sastre,
    LowRankPair, expm_lowrank, expm_lowrank_into, expm_timegrid,
)

__version__ = "0.1.0"
