"""The reference's accuracy suite on the GPU: plans and
ledgers equal the oracle's, errors at the suite tolerance, reports in the
reference's formats."""
import math

import numpy as np
import pytest

from oracle import expm_oracle as O
from paper_2512_20777_b200 import suite as S

pytestmark = pytest.mark.gpu


def test_suite_subset_on_gpu(tmp_path):
    cfg = S.SuiteConfig(eps=1e-8, sizes=(8, 16, 64), kinds=(S.KIND_DIAG, S.KIND_DENSE, S.KIND_ROTATION,
                                                             S.KIND_TRIANGULAR),
                        schemes=S.SCHEMES, norm_min=2.84e-4, norm_max=12.8, norm_count=6, base_seed=2024)
    recs = S.run_suite_gpu(cfg)
    assert len(recs) == len(cfg.specs()) * 3
    for r in recs:
        W = S.gen_matrix(r.generator)
        want = O.expm_baseline(W, cfg.eps) if r.scheme == "baseline" else O.expm(W, cfg.eps, r.scheme)
        assert (r.m, r.s, r.square_mults) == (want.m, want.s, want.mults), (r.generator, r.scheme)
        assert math.isfinite(r.rel_err) and r.rel_err <= 1e-6, (r.generator, r.scheme, r.rel_err)
    S.emit_reports(recs, tmp_path / "gpu.csv", tmp_path / "gpu.json")
    back = S.read_records_csv(tmp_path / "gpu.csv")
    assert [(b.m, b.s, b.square_mults) for b in back] == [(r.m, r.s, r.square_mults) for r in recs]
