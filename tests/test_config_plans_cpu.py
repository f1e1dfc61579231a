"""CPU check of the committed per-matrix config plans (tests/golden/config_plans.npz,
made by the unmodified reference's select_sastre): the oracle's ladder over
the reference's own norms reproduces every (m, s), and the fixture covers
every matrix of every config."""
import os

import numpy as np

from oracle import expm_oracle as O
from paper_2512_20777_b200 import workloads as WL

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fixture_complete_and_oracle_ladder_agrees():
    g = np.load(os.path.join(ROOT, "tests", "golden", "config_plans.npz"))
    for key, cfg in WL.CONFIGS.items():
        m, s, n1, n2 = g[f"{key}_m"], g[f"{key}_s"], g[f"{key}_n1"], g[f"{key}_n2"]
        assert m.shape == (cfg.batch,) and s.shape == (cfg.batch,)
        for i in range(cfg.batch):
            norms = {1: float(n1[i])}
            if np.isfinite(n2[i]):
                norms[2] = float(n2[i])
            elif m[i] > 1:
                raise AssertionError((key, i, "W^2 missing"))
            if m[i] <= 1 and 2 not in norms:
                norms[2] = 0.0  # the m = 1 rung never reads ||W^2||_1
            assert O.plan_from_power_norms(norms, cfg.eps) == (int(m[i]), int(s[i])), (key, i)
        assert g[f"{key}_near"].sum() <= max(8, cfg.batch // 4096)
