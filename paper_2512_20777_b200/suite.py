"""GPU runs of the reference's accuracy suite, emitted in the reference's own
report formats.

The reference's harness (``expmkit.bench``: ``gen_matrix`` bench.py:100-143,
``SuiteConfig.specs`` bench.py:218-230, ``run_suite`` bench.py:272-309,
``write_records_csv`` / ``summarize`` bench.py:363-451) runs every (matrix,
scheme) cell on the CPU, one matrix at a time.  Here the same suite -- the
same matrices, bit for bit, from a restatement of its generator -- runs
batched on the GPU (one ``expm`` / ``expm_baseline`` call per (order,
scheme)), and the records are written with the reference's CSV columns and
JSON summary keys, so the reference's ``expm profile --csv`` and summary
tooling consume GPU results unchanged.

Truth for ``rel_err`` (relative Frobenius error, oracle.py:149-156): the
reference uses its double-double Taylor oracle (out of scope here, SURVEY
§2); this module uses ``scipy.linalg.expm`` in binary64, whose own error
(~1e-15 relative) is far below the suite's errors at its tolerances
(default 1e-8).  Records of matrices whose truth is not finite carry NaN,
as the reference's do.
"""

from __future__ import annotations

import csv
import json
import math
import time
from dataclasses import dataclass

import numpy as np

KIND_DIAG = "diag"
KIND_DENSE = "random_dense"
KIND_TRIANGULAR = "nonnormal_triangular"
KIND_NILPOTENT = "nilpotent_perturbed"
KIND_ROTATION = "rotation_block"
KINDS = (KIND_DIAG, KIND_DENSE, KIND_TRIANGULAR, KIND_NILPOTENT, KIND_ROTATION)
SCHEMES = ("baseline", "ps", "sastre")

# bench.py:363-364
CSV_COLUMNS = ("generator_kind", "n", "target_norm", "seed", "scheme",
               "m", "s", "square_mults", "rel_err", "wall_time_s")


@dataclass(frozen=True)
class GeneratorSpec:
    """bench.py:60-86 (the low-rank kind is exercised through expm_lowrank)."""
    kind: str
    n: int
    target_norm: float
    seed: int
    noise: float = 1e-8


def _scaled(arr: np.ndarray, target: float) -> np.ndarray:
    norm = float(np.abs(arr).sum(axis=0).max())
    if norm == 0.0:
        raise ValueError("generated matrix is zero; cannot hit a positive norm")
    return arr * (target / norm)


def gen_matrix(spec: GeneratorSpec) -> np.ndarray:
    """The reference generator (bench.py:100-143) restated: Philox(seed) draws
    in the same order, so the matrices are bit-identical."""
    rng = np.random.Generator(np.random.Philox(spec.seed))
    n = spec.n
    if spec.kind == KIND_DIAG:
        d = rng.uniform(-1.0, 1.0, n)
        if not np.abs(d).max() > 0:
            d[0] = 1.0
        return np.diag(d * (spec.target_norm / np.abs(d).max()))
    if spec.kind == KIND_DENSE:
        return _scaled(rng.uniform(-1.0, 1.0, (n, n)), spec.target_norm)
    if spec.kind == KIND_TRIANGULAR:
        a = np.triu(rng.uniform(-1.0, 1.0, (n, n)))
        a[np.diag_indices(n)] *= 0.25
        i = np.arange(n)
        return _scaled(a * 0.5 ** np.maximum(i[None, :] - i[:, None], 0), spec.target_norm)
    if spec.kind == KIND_NILPOTENT:
        a = np.triu(rng.uniform(-1.0, 1.0, (n, n)), 1)
        if spec.noise > 0:
            a = a + spec.noise * rng.uniform(-1.0, 1.0, (n, n))
        return _scaled(a, spec.target_norm)
    if spec.kind == KIND_ROTATION:
        a = np.zeros((n, n))
        for i, theta in enumerate(rng.uniform(0.25, 1.0, n // 2)):
            a[2 * i, 2 * i + 1] = theta
            a[2 * i + 1, 2 * i] = -theta
        return _scaled(a, spec.target_norm)
    raise ValueError(f"unknown generator kind {spec.kind!r}")


def _derive_seed(base: int, index: int) -> int:
    """bench.py:233-234."""
    return int(np.random.SeedSequence([base, index]).generate_state(1, np.uint64)[0])


@dataclass(frozen=True)
class SuiteConfig:
    """bench.py:150-230 (the fields the runner uses)."""
    eps: float
    sizes: tuple
    kinds: tuple
    schemes: tuple
    norm_min: float
    norm_max: float
    norm_count: int
    norm_scale: str = "log"
    base_seed: int = 0
    noise: float = 1e-8

    def norm_grid(self) -> np.ndarray:
        if self.norm_count == 1:
            return np.array([self.norm_min])
        if self.norm_scale == "log":
            return np.geomspace(self.norm_min, self.norm_max, self.norm_count)
        return np.linspace(self.norm_min, self.norm_max, self.norm_count)

    def specs(self) -> list:
        out, index = [], 0
        for kind in self.kinds:
            for n in self.sizes:
                for target in self.norm_grid():
                    out.append(GeneratorSpec(kind, int(n), float(target), _derive_seed(self.base_seed, index),
                                             self.noise))
                    index += 1
        return out


def default_suite_config(eps: float = 1e-8, base_seed: int = 2024) -> SuiteConfig:
    """bench.py:237-251: 300 matrices, 1-norms log-spaced over [2.84e-4, 12.8], orders 8..64."""
    return SuiteConfig(eps=eps, sizes=(8, 16, 32, 64), kinds=(KIND_DIAG, KIND_DENSE, KIND_ROTATION),
                       schemes=SCHEMES, norm_min=2.84e-4, norm_max=12.8, norm_count=25, norm_scale="log",
                       base_seed=base_seed)


@dataclass(frozen=True)
class BenchRecord:
    """bench.py:254-265."""
    generator: GeneratorSpec
    scheme: str
    m: int
    s: int
    square_mults: int
    rel_err: float
    wall_time: float


def _truth(W: np.ndarray):
    import scipy.linalg
    with np.errstate(all="ignore"):
        try:
            X = scipy.linalg.expm(W)
        except (ValueError, OverflowError, np.linalg.LinAlgError):
            return None
    return X if np.isfinite(X).all() else None


def run_suite_gpu(config: SuiteConfig, device: str = "cuda") -> list:
    """Every (matrix, scheme) cell of the suite on the GPU, batched per
    (order, scheme); records in the reference's order (spec, then scheme).
    ``wall_time`` is the batch's wall time divided by its size."""
    import torch

    from . import api
    specs = config.specs()
    mats = [gen_matrix(sp) for sp in specs]
    truth = [_truth(W) for W in mats]
    cell = {}
    for n in sorted({sp.n for sp in specs}):
        idx = [i for i, sp in enumerate(specs) if sp.n == n]
        Wb = torch.as_tensor(np.stack([mats[i] for i in idx]), device=device)
        for scheme in config.schemes:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if scheme == "baseline":
                res = api.expm_baseline(Wb, config.eps, check_finite=False)
            else:
                res = api.expm(Wb, config.eps, scheme, check_finite=False)
            torch.cuda.synchronize()
            per = (time.perf_counter() - t0) / len(idx)
            X = res.value.cpu().numpy()
            m = res.plan.m.cpu().numpy()
            s = res.plan.s.cpu().numpy()
            mults = res.mults.cpu().numpy()
            bad = res.nonfinite.cpu().numpy()
            for k, i in enumerate(idx):
                cell[(i, scheme)] = (X[k], int(m[k]), int(s[k]), int(mults[k]), bool(bad[k]), per)
    records = []
    for i, sp in enumerate(specs):
        for scheme in config.schemes:
            X, m, s, mults, bad, per = cell[(i, scheme)]
            if bad:  # the reference records a driver failure as a NaN row (bench.py:281-283)
                records.append(BenchRecord(sp, scheme, 0, 0, 0, math.nan, 0.0))
                continue
            if scheme == "baseline":
                m = mults - s  # the int8 plan outputs saturate; mults = m + s does not
            T = truth[i]
            err = math.nan if T is None else float(np.linalg.norm(X - T) / np.linalg.norm(T))
            records.append(BenchRecord(sp, scheme, m, s, mults, err, per))
    return records


def write_records_csv(records, path) -> None:
    """bench.py:367-376: the reference's columns and number formatting."""
    with open(path, "w", newline="", encoding="ascii") as f:
        w = csv.writer(f)
        w.writerow(CSV_COLUMNS)
        for r in records:
            w.writerow([r.generator.kind, r.generator.n, repr(r.generator.target_norm), r.generator.seed,
                        r.scheme, r.m, r.s, r.square_mults, repr(r.rel_err), repr(r.wall_time)])


def read_records_csv(path) -> list:
    """bench.py:379-397."""
    out = []
    with open(path, newline="", encoding="ascii") as f:
        rd = csv.reader(f)
        if tuple(next(rd, ())) != CSV_COLUMNS:
            raise ValueError("unexpected CSV header")
        for row in rd:
            sp = GeneratorSpec(row[0], int(row[1]), float(row[2]), int(row[3]))
            out.append(BenchRecord(sp, row[4], int(row[5]), int(row[6]), int(row[7]), float(row[8]),
                                   float(row[9])))
    return out


def _quantiles(values) -> dict:
    if not values:
        return {"p25": 0.0, "p50": 0.0, "p75": 0.0, "max": 0.0}
    q25, q50, q75 = np.percentile(values, [25, 50, 75])
    return {"p25": float(q25), "p50": float(q50), "p75": float(q75), "max": float(max(values))}


def summarize(records) -> dict:
    """bench.py:408-437 (without the optional profile block)."""
    per = {}
    for sch in sorted({r.scheme for r in records}):
        rows = [r for r in records if r.scheme == sch]
        errs = [r.rel_err for r in rows if math.isfinite(r.rel_err)]
        per[sch] = {
            "records": len(rows),
            "failures": sum(1 for r in rows if not math.isfinite(r.rel_err)),
            "total_mults": sum(r.square_mults for r in rows),
            "mean_rel_err": float(np.mean(errs)) if errs else 0.0,
            "max_rel_err": float(max(errs)) if errs else 0.0,
            "mean_m": float(np.mean([r.m for r in rows])) if rows else 0.0,
            "mean_s": float(np.mean([r.s for r in rows])) if rows else 0.0,
            "m_quantiles": _quantiles([r.m for r in rows]),
            "s_quantiles": _quantiles([r.s for r in rows]),
            "total_wall_time_s": float(sum(r.wall_time for r in rows)),
        }
    return {"records": len(records),
            "matrices": len({(r.generator.kind, r.generator.n, r.generator.target_norm, r.generator.seed)
                             for r in records}),
            "schemes": per}


def emit_reports(records, csv_path, summary_path) -> None:
    """bench.py:446-451."""
    write_records_csv(records, csv_path)
    with open(summary_path, "w", encoding="ascii") as f:
        json.dump(summarize(records), f, indent=2)
        f.write("\n")


def main(argv=None) -> int:
    """python -m paper_2512_20777_b200.suite --csv out.csv --summary out.json
    (the reference CLI's ``expm bench`` with the default suite, on the GPU)."""
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--csv", required=True)
    ap.add_argument("--summary", required=True)
    ap.add_argument("--eps", type=float, default=1e-8)
    ap.add_argument("--seed", type=int, default=2024)
    a = ap.parse_args(argv)
    t0 = time.perf_counter()
    recs = run_suite_gpu(default_suite_config(a.eps, a.seed))
    emit_reports(recs, a.csv, a.summary)
    print(f"{len(recs)} records in {time.perf_counter() - t0:.1f} s -> {a.csv}, {a.summary}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
