"""Generate the golden vectors that pin the oracle (and, through it, the CUDA path).

Run in the build container, where the reference package is importable:

    python tests/golden/make_golden.py

It imports the UNMODIFIED reference ``expmkit`` from /root/reference/pkg/src
and records, for every case, what the reference's own ``expm`` returns
(engine.py:119-152): the value, (m, s), e1/e2, ``mults`` -- or that it raised
NonFiniteError.  The cases restate the reference tests' golden inputs
(test_select.py:61-139, test_engine.py:109-130, test_acceptance.py:211-212)
plus seeded random / structured matrices from the reference's own generator
kinds (bench.py:100-143) over the orders, tolerances and norms the tests use.

Output: tests/golden/expm_golden.npz (ragged cases concatenated with offsets).
Nothing on the GPU box reads /root/reference; only this script does.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import expmkit  # noqa: E402
from expmkit import GeneratorSpec, Matrix, NonFiniteError, gen_matrix  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "expm_golden.npz")


def cases():
    # named golden inputs from the reference tests
    named = [
        ("zero4", np.zeros((4, 4)), 1e-8),
        ("diag1e-5", np.diag([1e-5] * 4), 1e-8),
        ("diag1", np.diag([1.0] * 4), 1e-8),
        ("diag1_n5", np.diag([1.0] * 5), 1e-8),
        ("diag12.57", np.diag([12.57] * 4), 1e-8),
        ("diag1e30", np.diag([1e30] * 4), 1e-8),
        ("scalar1e60", np.array([[1e60]]), 1e-8),
        ("nilpotent2", np.array([[0.0, 1.0], [0.0, 0.0]]), 1e-8),
        ("diag1_floor", np.diag([1.0] * 4), 2.0 ** -53),
        ("overflow", np.diag([1e300, 1.0]), 1e-8),
        ("scalar_neg", np.array([[-3.5]]), 1e-12),
    ]
    for name, W, eps in named:
        yield name, W, eps
    rng = np.random.default_rng(20251220)
    sizes = (1, 2, 3, 5, 8, 13, 16, 17, 24, 31, 32, 33, 48, 64)
    epss = (1e-12, 1e-8, 1e-4, 2.0 ** -24, 2.0 ** -53)
    for i in range(120):
        n = sizes[i % len(sizes)]
        if n >= 48 and i % 3:
            n = sizes[i % 8]
        target = float(10.0 ** rng.uniform(-7, 2.6))
        arr = rng.uniform(-1, 1, (n, n))
        W = arr * (target / np.abs(arr).sum(axis=0).max())
        yield f"rand{i}", W, epss[i % len(epss)]
    kinds = ("diag", "random_dense", "nonnormal_triangular", "nilpotent_perturbed", "rotation_block")
    for i in range(60):
        kind = kinds[i % len(kinds)]
        n = (2, 4, 7, 16, 20, 32)[i % 6]
        target = float(10.0 ** rng.uniform(-4, 2.2))
        spec = GeneratorSpec(kind=kind, n=n, target_norm=target, seed=777 + i)
        W = gen_matrix(spec).a.copy()
        yield f"{kind}{i}", W, epss[(i // 5) % len(epss)]


def main():
    names, ns, epss, schemes = [], [], [], []
    ms, ss, e1s, e2s, mults, raised = [], [], [], [], [], []
    ins, outs = [], []
    for name, W, eps in cases():
        for scheme in ("sastre", "ps", "baseline"):
            if scheme == "baseline" and (W.shape[0] > 64 or not np.isfinite(W).all() or np.abs(W).max() > 1e12):
                continue
            names.append(name)
            ns.append(W.shape[0])
            epss.append(eps)
            schemes.append(scheme)
            ins.append(np.asarray(W, np.float64).ravel())
            try:
                r = (expmkit.expm_baseline(Matrix(W), eps) if scheme == "baseline"
                     else expmkit.expm(Matrix(W), eps, scheme))
            except NonFiniteError:
                raised.append(True)
                ms.append(-1); ss.append(-1); e1s.append(math.nan); e2s.append(math.nan)
                mults.append(-1)
                outs.append(np.full(W.size, np.nan))
                continue
            raised.append(False)
            ms.append(r.plan.m); ss.append(r.plan.s)
            e1s.append(r.plan.e1); e2s.append(r.plan.e2)
            mults.append(r.mults)
            outs.append(r.value.a.ravel().copy())
    offs = np.concatenate([[0], np.cumsum([a.size for a in ins])])
    np.savez_compressed(
        OUT,
        names=np.array(names), n=np.array(ns), eps=np.array(epss),
        scheme=np.array(schemes), m=np.array(ms), s=np.array(ss),
        e1=np.array(e1s), e2=np.array(e2s), mults=np.array(mults),
        raised=np.array(raised), offsets=offs,
        W=np.concatenate(ins), X=np.concatenate(outs),
    )
    print(f"wrote {len(names)} cases, {offs[-1]} entries -> {OUT}")


if __name__ == "__main__":
    main()
