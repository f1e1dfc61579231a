"""Seeded synthetic inputs for the five BASELINE.json configurations.

SURVEY.md 8(d) fixes the recipe; every draw comes from
``np.random.default_rng([config, chunk])`` so any subset of a batch can be
regenerated independently (the parity tests regenerate the matrices they
check on the CPU; bench.py regenerates whole batches).  N(0, v) means
variance v.  "1-norm log-uniform in [a, b]" means
target = 10**U(log10 a, log10 b) and A <- A * target / ||A||_1.

No public dataset is involved (BASELINE.json configs are synthetic).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    key: str
    batch: int
    n: int
    dtype: str        # "f32" | "f64"
    eps: float
    chunk: int        # matrices per seeded chunk
    desc: str


CONFIGS = {
    "C1": Config("C1", 1024, 64, "f64", 2.0 ** -53, 64,
                 "batch 1024 of 64x64 fp64 dense N(0,1), 1-norm log-U[1e-3,1e2], tol 2^-53"),
    "C2": Config("C2", 65536, 16, "f32", 2.0 ** -24, 1024,
                 "batch 65536 of 16x16 fp32 skew-symmetric (B-B^T)/2, 1-norm log-U[1e-2,10], tol 2^-24"),
    "C3": Config("C3", 4096, 256, "f32", 2.0 ** -24, 4096,
                 "exp(t_k A), A 256x256 fp32 N(0,1/n)-0.5I, t_k~U[0,4], 4096 times, tol 2^-24"),
    "C4": Config("C4", 64, 1024, "f64", 2.0 ** -53, 1,
                 "batch 64 of 1024x1024 fp64 non-normal (upper N(0,n^-1/2), diag U[-5,5], "
                 "lower N(0,0.01 n^-1/2)), 1-norm log-U[1,500], tol 2^-53"),
    "C5": Config("C5", 256, 2048, "f32", 2.0 ** -24, 1,
                 "batch 256 of 2048x2048 fp32 N(0,1/n) scaled by log-U[0.1,50], tol 2^-24"),
}


def _colnorm(a: np.ndarray) -> np.ndarray:
    return np.abs(a).sum(axis=-2).max(axis=-1)


def _logu(rng, lo, hi, size):
    return 10.0 ** rng.uniform(math.log10(lo), math.log10(hi), size)


def _chunk(cfg: Config, c: int) -> np.ndarray:
    """Matrices [c*chunk, (c+1)*chunk) of a config, in its dtype."""
    n = cfg.n
    if cfg.key == "C1":
        rng = np.random.default_rng([1, c])
        a = rng.standard_normal((cfg.chunk, n, n))
        t = _logu(rng, 1e-3, 1e2, cfg.chunk)
        return a * (t / _colnorm(a))[:, None, None]
    if cfg.key == "C2":
        rng = np.random.default_rng([2, c])
        b = rng.standard_normal((cfg.chunk, n, n))
        a = (b - np.swapaxes(b, -1, -2)) / 2.0
        t = _logu(rng, 1e-2, 10.0, cfg.chunk)
        return (a * (t / _colnorm(a))[:, None, None]).astype(np.float32)
    if cfg.key == "C3":
        A, t = c3_factors()
        return (t[:, None, None] * A[None, :, :]).astype(np.float32)
    if cfg.key == "C4":
        rng = np.random.default_rng([4, c])
        up = np.triu(rng.standard_normal((n, n)) * n ** -0.25, 1)
        dg = np.diag(rng.uniform(-5.0, 5.0, n))
        lo = np.tril(rng.standard_normal((n, n)) * (0.1 * n ** -0.25), -1)
        a = up + dg + lo
        t = _logu(rng, 1.0, 500.0, 1)[0]
        return (a * (t / _colnorm(a)))[None]
    if cfg.key == "C5":
        rng = np.random.default_rng([5, c])
        a = rng.standard_normal((n, n)) * n ** -0.5
        f = _logu(rng, 0.1, 50.0, 1)[0]
        return (a * f).astype(np.float32)[None]
    raise KeyError(cfg.key)


def c3_factors():
    """C3's shared matrix A (fp32) and times t_k (fp32)."""
    n = 256
    rng = np.random.default_rng([3, 0])
    A = (rng.standard_normal((n, n)) * n ** -0.5 - 0.5 * np.eye(n)).astype(np.float32)
    t = np.random.default_rng([3, 1]).uniform(0.0, 4.0, 4096).astype(np.float32)
    return A, t


def generate(key: str, indices=None, batch: int | None = None) -> np.ndarray:
    """Inputs of config ``key`` (all of them, the first ``batch``, or ``indices``)."""
    cfg = CONFIGS[key]
    if indices is None:
        indices = np.arange(cfg.batch if batch is None else batch)
    indices = np.asarray(indices)
    out = np.empty((len(indices), cfg.n, cfg.n), np.float32 if cfg.dtype == "f32" else np.float64)
    if cfg.key == "C3":
        A, t = c3_factors()
        out[:] = (t[indices][:, None, None] * A[None]).astype(np.float32)
        return out
    cache = {}
    for k, i in enumerate(indices):
        c, r = divmod(int(i), cfg.chunk)
        if c not in cache:
            cache.clear()
            cache[c] = _chunk(cfg, c)
        out[k] = cache[c][r]
    return out


def useful_flops(m, s, n: int, scheme: str = "sastre") -> float:
    """sum over matrices of (budget(m) + s) * 2 n^3."""
    from .tables import ps_shape
    m = np.asarray(m).astype(np.int64).ravel()
    s = np.asarray(s).astype(np.int64).ravel()
    if scheme == "ps":
        b = np.array([0 if mm <= 1 else ps_shape(int(mm)).mults for mm in m])
    else:
        lut = {0: 0, 1: 0, 2: 1, 4: 2, 8: 3, 15: 4}
        b = np.array([lut[int(mm)] for mm in m])
    return float(((b + s) * 2.0 * n ** 3).sum())


# ---------------------------------------------------------------------------
# Low-rank flow-layer workload (not a BASELINE.json config)
# ---------------------------------------------------------------------------

LOWRANK = Config("LR", 16384, 64, "f64", 2.0 ** -53, 1024,
                 "batch 16384 low-rank flow weights W = A1 A2, n 64, t 8 (the reference generator's n/8, "
                 "bench.py:134-142), factors U[-1,1], ||A2 A1||_1 log-U[1e-2,3], fp64, tol 2^-53")
LOWRANK_T = 8


def _lowrank_chunk(c: int):
    cfg, n, t = LOWRANK, LOWRANK.n, LOWRANK_T
    rng = np.random.default_rng([9, c])
    a1 = rng.uniform(-1.0, 1.0, (cfg.chunk, n, t))
    a2 = rng.uniform(-1.0, 1.0, (cfg.chunk, t, n))
    target = _logu(rng, 1e-2, 3.0, cfg.chunk)
    a2 *= (target / _colnorm(a2 @ a1))[:, None, None]
    return a1, a2


def generate_lowrank(indices) -> tuple[np.ndarray, np.ndarray]:
    """(A1 [B,n,t], A2 [B,t,n]) fp64 for the given global indices of LR."""
    indices = np.asarray(indices)
    n, t = LOWRANK.n, LOWRANK_T
    A1 = np.empty((len(indices), n, t))
    A2 = np.empty((len(indices), t, n))
    cache = {}
    for k, i in enumerate(indices):
        c, r = divmod(int(i), LOWRANK.chunk)
        if c not in cache:
            cache.clear()
            cache[c] = _lowrank_chunk(c)
        A1[k], A2[k] = cache[c][0][r], cache[c][1][r]
    return A1, A2
