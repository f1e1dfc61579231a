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
OUT_LR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lowrank_golden.npz")
OUT_SUITE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "suite_golden.npz")


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


def lowrank_cases():
    """expm_lowrank (engine.py:198-257) inputs: the reference tests' factors
    (test_engine.py:241-318, test_acceptance.py:257-270), a nilpotent pair
    with V = 0, and seeded random factors over orders, ranks and norms."""
    from expmkit import LowRankPair  # noqa: F401
    n = 6
    a1 = np.zeros((n, 1)); a1[0, 0] = 1.0
    a2 = np.zeros((1, n)); a2[0, 0] = 1.0
    yield "projector", a1, a2, 1e-8
    yield "zero_factor", np.zeros((5, 2)), np.ones((2, 5)), 1e-8
    rng = np.random.default_rng(53)
    a1 = rng.uniform(-1, 1, (64, 8)); a2 = rng.uniform(-1, 1, (8, 64))
    a2 *= 2.0 / np.abs(a2 @ a1).sum(axis=0).max()
    yield "matches_reference", a1, a2, 1e-8
    rng = np.random.default_rng(59)
    a1 = rng.uniform(-1, 1, (16, 2)); a2 = rng.uniform(-1, 1, (2, 16))
    a2 *= 1.0 / np.abs(a2 @ a1).sum(axis=0).max()
    yield "order_minimal", a1, a2, 1e-8
    yield "norm_too_large", np.eye(4, 2) * 10.0, np.eye(2, 4) * 10.0, 1e-8
    yield "psi_1x1", np.array([[1.5]]), np.array([[1.0]]), 1e-8
    yield "nilpotent_v0", np.array([[1.0], [0.0]]), np.array([[0.0, 1.0]]), 1e-8
    for i, target in enumerate((0.5, 1.0, 2.0, 3.5, 5.0)):
        pair = gen_matrix(GeneratorSpec(kind="lowrank_pair", n=64, target_norm=target, seed=500 + i))
        yield f"criterion9_{i}", pair.a1.copy(), pair.a2.copy(), 1e-8
    rng = np.random.default_rng(20251221)
    sizes = (1, 2, 3, 5, 8, 13, 16, 17, 31, 33, 64, 65, 100, 128)
    epss = (1e-12, 1e-8, 1e-4, 2.0 ** -24, 2.0 ** -53)
    for i in range(90):
        n = sizes[i % len(sizes)]
        t = int(rng.integers(1, min(n, 32) + 1))
        target = float(10.0 ** rng.uniform(-4, 1.5))
        a1 = rng.uniform(-1, 1, (n, t)); a2 = rng.uniform(-1, 1, (t, n))
        vn = np.abs(a2 @ a1).sum(axis=0).max()
        if vn > 0:
            a2 *= target / vn
        yield f"lr_rand{i}", a1, a2, epss[i % len(epss)]


def main_lowrank():
    names, ns, ts, epss, ms, e1s, e2s, mults, rects, raised = [], [], [], [], [], [], [], [], [], []
    a1s, a2s, outs, nv1, nv2 = [], [], [], [], []
    for name, a1, a2, eps in lowrank_cases():
        names.append(name); ns.append(a1.shape[0]); ts.append(a1.shape[1]); epss.append(eps)
        a1s.append(np.asarray(a1, np.float64).ravel()); a2s.append(np.asarray(a2, np.float64).ravel())
        try:
            r = expmkit.expm_lowrank(expmkit.LowRankPair(a1, a2), eps)
        except expmkit.LowRankOrderError:
            raised.append(True)
            ms.append(-1); e1s.append(math.nan); e2s.append(math.nan); mults.append(-1); rects.append(-1)
            nv1.append(math.nan); nv2.append(math.nan)
            outs.append(np.full(a1.shape[0] ** 2, np.nan))
            continue
        raised.append(False)
        ms.append(r.plan.m); e1s.append(r.plan.e1); e2s.append(r.plan.e2)
        mults.append(r.mults); rects.append(r.rect_mults)
        nv1.append(r.plan.cached_norms.get(1, math.nan)); nv2.append(r.plan.cached_norms.get(2, math.nan))
        outs.append(r.value.a.ravel().copy())
    offs = np.concatenate([[0], np.cumsum([a.size for a in a1s])])
    oo = np.concatenate([[0], np.cumsum([a.size for a in outs])])
    np.savez_compressed(
        OUT_LR, names=np.array(names), n=np.array(ns), t=np.array(ts), eps=np.array(epss),
        m=np.array(ms), e1=np.array(e1s), e2=np.array(e2s), mults=np.array(mults),
        rect_mults=np.array(rects), raised=np.array(raised), norm1=np.array(nv1), norm2=np.array(nv2),
        offsets=offs, out_offsets=oo, A1=np.concatenate(a1s), A2=np.concatenate(a2s),
        X=np.concatenate(outs),
    )
    print(f"wrote {len(names)} low-rank cases -> {OUT_LR}")


def main_suite():
    """The reference's suite plumbing (bench.py:60-251): the default config's
    spec list (kinds, orders, norms, derived seeds) and the generated matrices
    of a sample of specs covering every generator kind."""
    from expmkit.bench import GeneratorSpec as GS, default_suite_config, gen_matrix as gm
    cfg = default_suite_config()
    specs = cfg.specs()
    sample = [GS(kind=k, n=n, target_norm=t, seed=1000 + i)
              for i, (k, n, t) in enumerate([("diag", 8, 0.3), ("random_dense", 16, 2.5),
                                             ("nonnormal_triangular", 12, 7.0), ("nilpotent_perturbed", 9, 1.1),
                                             ("rotation_block", 10, 4.0), ("random_dense", 33, 1e-3)])]
    mats = [gm(sp).a.ravel() for sp in sample]
    offs = np.concatenate([[0], np.cumsum([m.size for m in mats])])
    np.savez_compressed(
        OUT_SUITE,
        spec_kind=np.array([sp.kind for sp in specs]), spec_n=np.array([sp.n for sp in specs]),
        spec_norm=np.array([sp.target_norm for sp in specs]),
        spec_seed=np.array([sp.seed for sp in specs], dtype=np.uint64),
        sample_kind=np.array([sp.kind for sp in sample]), sample_n=np.array([sp.n for sp in sample]),
        sample_norm=np.array([sp.target_norm for sp in sample]),
        sample_seed=np.array([sp.seed for sp in sample], dtype=np.uint64),
        offsets=offs, W=np.concatenate(mats))
    print(f"wrote {len(specs)} suite specs + {len(sample)} generated matrices -> {OUT_SUITE}")


if __name__ == "__main__":
    main()
    main_lowrank()
    main_suite()
