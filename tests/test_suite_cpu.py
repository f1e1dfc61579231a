"""The reference-format suite runner without a GPU: its
restated generator and spec list against the reference's own (golden
fixture from tests/golden/make_golden.py), and the CSV / summary formats."""
import json
import math
import os

import numpy as np
import pytest

from paper_2512_20777_b200 import suite as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sg():
    return np.load(os.path.join(ROOT, "tests", "golden", "suite_golden.npz"))


def test_default_suite_specs_match_reference(sg):
    specs = S.default_suite_config().specs()
    assert len(specs) == len(sg["spec_kind"]) == 300
    for i, sp in enumerate(specs):
        assert sp.kind == str(sg["spec_kind"][i]) and sp.n == int(sg["spec_n"][i])
        assert sp.target_norm == float(sg["spec_norm"][i]) and sp.seed == int(sg["spec_seed"][i])


def test_generator_bit_identical(sg):
    offs = sg["offsets"]
    for i in range(len(sg["sample_kind"])):
        sp = S.GeneratorSpec(str(sg["sample_kind"][i]), int(sg["sample_n"][i]), float(sg["sample_norm"][i]),
                             int(sg["sample_seed"][i]))
        W = S.gen_matrix(sp)
        want = sg["W"][offs[i]:offs[i + 1]].reshape(sp.n, sp.n)
        assert np.array_equal(W, want), sp.kind


def test_csv_and_summary_formats(tmp_path):
    sp = S.GeneratorSpec("random_dense", 8, 0.5, 123)
    recs = [S.BenchRecord(sp, "sastre", 8, 0, 3, 1.25e-12, 1e-4), S.BenchRecord(sp, "ps", 9, 0, 4, 2e-12, 2e-4),
            S.BenchRecord(sp, "baseline", 12, 1, 13, math.nan, 0.0)]
    c, j = tmp_path / "r.csv", tmp_path / "s.json"
    S.emit_reports(recs, c, j)
    lines = open(c).read().splitlines()
    assert lines[0] == ",".join(S.CSV_COLUMNS)
    assert lines[1] == "random_dense,8,0.5,123,sastre,8,0,3,1.25e-12,0.0001"
    back = S.read_records_csv(c)
    assert [(r.scheme, r.m, r.s, r.square_mults) for r in back] == [("sastre", 8, 0, 3), ("ps", 9, 0, 4),
                                                                      ("baseline", 12, 1, 13)]
    summ = json.load(open(j))
    assert summ["records"] == 3 and summ["matrices"] == 1
    assert summ["schemes"]["baseline"]["failures"] == 1 and summ["schemes"]["sastre"]["total_mults"] == 3
    assert set(summ["schemes"]["ps"]) == {"records", "failures", "total_mults", "mean_rel_err", "max_rel_err",
                                          "mean_m", "mean_s", "m_quantiles", "s_quantiles", "total_wall_time_s"}
