"""Reference (m, s) plans for EVERY matrix of the five BASELINE.json configs.

Run in the build container, where the reference package is importable:

    python tests/golden/make_config_plans.py [--jobs 8]

It regenerates each config's seeded inputs (paper_2512_20777_b200/workloads.py,
the same bytes the GPU tests and bench.py feed the CUDA path), upcasts them to
binary64 exactly as the reference would (matrix.py:51), and runs the
UNMODIFIED reference selector ``expmkit.select_sastre`` (select.py:228-234)
on each matrix.  Only W^2 is formed per matrix, so the whole corpus
(1024 + 65536 + 4096 + 64 + 256 matrices) takes about a minute.

Output: tests/golden/config_plans.npz with, per config Ck:
    Ck_m, Ck_s          int8   the reference's selected order / scaling
    Ck_e1, Ck_e2        fp64   EvalPlan.e1 / e2
    Ck_n1, Ck_n2        fp64   ||W||_1, ||W^2||_1 (NaN when W^2 was not formed)
    Ck_near             bool   the plan flips if log2 ||W||_1 or log2 ||W^2||_1
                               moves by 1e-4 (SURVEY.md 8(d) exemption), computed
                               from the reference's own norms
Nothing on the GPU box reads /root/reference; only this script does.
"""

from __future__ import annotations

import argparse
import math
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

OUT = os.path.join(ROOT, "tests", "golden", "config_plans.npz")


def _plans(args):
    key, lo, hi = args
    import expmkit  # noqa: E402
    from expmkit import Matrix  # noqa: E402

    from oracle import expm_oracle as O
    from paper_2512_20777_b200 import workloads as WL

    cfg = WL.CONFIGS[key]
    W = WL.generate(key, indices=np.arange(lo, hi))
    out = []
    for i in range(W.shape[0]):
        p = expmkit.select_sastre(Matrix(np.asarray(W[i], np.float64)), cfg.eps)
        n1 = float(p.cached_norms[1])
        n2 = float(p.cached_norms.get(2, math.nan))
        near = False
        if n1 != 0.0 and math.isfinite(n1):
            nn2 = n2 if math.isfinite(n2) else O.one_norm(np.asarray(W[i], np.float64) @ np.asarray(W[i], np.float64))
            near = O.near_threshold(n1, nn2, cfg.eps)
        out.append((p.m, p.s, p.e1, p.e2, n1, n2, near))
    return key, lo, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    args = ap.parse_args()
    from paper_2512_20777_b200 import workloads as WL

    tasks = []
    for key in args.configs.split(","):
        cfg = WL.CONFIGS[key]
        step = {"C1": 256, "C2": 4096, "C3": 512, "C4": 8, "C5": 8}[key]
        tasks += [(key, lo, min(cfg.batch, lo + step)) for lo in range(0, cfg.batch, step)]
    res = {}
    with ProcessPoolExecutor(args.jobs) as pool:
        for key, lo, out in pool.map(_plans, tasks):
            res.setdefault(key, {})[lo] = out
    arrays = {}
    for key, parts in res.items():
        rows = [r for lo in sorted(parts) for r in parts[lo]]
        m, s, e1, e2, n1, n2, near = zip(*rows)
        arrays[f"{key}_m"] = np.array(m, np.int8)
        arrays[f"{key}_s"] = np.array(s, np.int8)
        arrays[f"{key}_e1"] = np.array(e1, np.float64)
        arrays[f"{key}_e2"] = np.array(e2, np.float64)
        arrays[f"{key}_n1"] = np.array(n1, np.float64)
        arrays[f"{key}_n2"] = np.array(n2, np.float64)
        arrays[f"{key}_near"] = np.array(near, bool)
        hist = {}
        for a, b in zip(m, s):
            hist[(a, b)] = hist.get((a, b), 0) + 1
        print(key, len(rows), "near", int(np.sum(near)), dict(sorted(hist.items())))
    if os.path.exists(OUT):  # keep configs not regenerated this run
        old = np.load(OUT)
        for k in old.files:
            arrays.setdefault(k, old[k])
    np.savez_compressed(OUT, **arrays)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
