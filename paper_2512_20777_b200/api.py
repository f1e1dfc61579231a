"""Batched drop-in for ``expmkit.expm`` (engine.py:119-152) on B200.

    res = expm(W, eps, scheme="sastre")      # W: cuda tensor [..., n, n] fp32/fp64
    res.value   -> tensor [..., n, n]        (ExpmResult.value)
    res.plan.m / .s / .e1 / .e2              (EvalPlan, select.py:144-161)
    res.mults   -> int32 tensor [...]        (ExpmResult.mults = budget(m) + s)
    res.wall_time                            (seconds, host clock around the call)

Error behaviour follows the reference: ToleranceError for eps NaN or below
the dtype's unit roundoff (select.py:72-79), MatrixError for non-square /
empty input and unknown schemes (matrix.py:52-55, engine.py:137),
NonFiniteError when an input or any produced matrix is not finite
(matrix.py:56-57, 95-102) -- raised after the batch completes, listing the
offending batch indices.  CPU tensors raise: there is no CPU fallback.

The compute is the registered custom op ``expmkit_b200::expm`` over the C ABI
of libexpmb.so (include/expmb.h).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import torch

from . import _lib
from .tables import (LowRankOrderError, MatrixError, NonFiniteError, SCHEME_LOWRANK, SCHEME_PS, SCHEME_SASTRE,
                     ToleranceError, UNIT_ROUNDOFF, UNIT_ROUNDOFF_F32)

_SCHEMES = {SCHEME_SASTRE: _lib.EXPMB_SASTRE, SCHEME_PS: _lib.EXPMB_PS}
SCHEME_BASELINE = "baseline"  # select.py:58


@dataclass
class EvalPlan:
    """Batched select.py:144-161 (tensors instead of scalars)."""
    m: torch.Tensor       # int8 [...]
    s: torch.Tensor       # int8 [...]
    scheme: str
    e1: torch.Tensor      # float64 [...]
    e2: torch.Tensor      # float64 [...]
    norms: torch.Tensor   # float64 [..., 2]: ||W||_1, ||W^2||_1 (NaN if W^2 never formed)


@dataclass
class ExpmResult:
    """Batched engine.py:64-77."""
    value: torch.Tensor
    plan: EvalPlan
    mults: torch.Tensor   # int32 [...]
    wall_time: float
    nonfinite: torch.Tensor  # bool [...]
    rect_mults: int = 0      # engine.py:77 (3 on the low-rank path)


def unit_roundoff(dtype: torch.dtype) -> float:
    return UNIT_ROUNDOFF_F32 if dtype == torch.float32 else UNIT_ROUNDOFF


def check_tolerance(eps: float, dtype: torch.dtype = torch.float64) -> float:
    """select.py:72-79, with the fp32 floor for fp32 inputs."""
    eps = float(eps)
    floor = unit_roundoff(dtype)
    if math.isnan(eps) or eps < floor:
        raise ToleranceError(
            f"tolerance {eps!r} below unit roundoff {floor:.3e}; "
            f"sub-roundoff accuracy cannot be guaranteed in {str(dtype).replace('torch.', '')}")
    return eps


def _raise_rc(rc: int):
    if rc == _lib.ERR_TOLERANCE:
        raise ToleranceError(_lib.strerror(rc))
    if rc in (_lib.ERR_SHAPE, _lib.ERR_SCHEME, _lib.ERR_DTYPE, _lib.ERR_UNSUPPORTED):
        raise MatrixError(_lib.strerror(rc))
    raise RuntimeError(f"libexpmb: {_lib.strerror(rc)} (code {rc})")


def _launch(W: torch.Tensor, X: torch.Tensor, eps: float, scheme_code: int,
            m, s, e1, e2, norms, mults, nonfinite) -> None:
    """One C-ABI call on the current stream (all pointers device memory)."""
    L = _lib.lib()
    B = W.shape[0]
    n = W.shape[-1]
    dt = _lib.EXPMB_F32 if W.dtype == torch.float32 else _lib.EXPMB_F64
    wsb = L.expmb_workspace_bytes(B, n, dt, scheme_code)
    ws = torch.empty(max(int(wsb), 1), dtype=torch.uint8, device=W.device) if wsb else None
    stream = torch.cuda.current_stream(W.device).cuda_stream

    def p(t):
        return None if t is None else t.data_ptr()

    with torch.cuda.device(W.device):  # the library launches on the current device
        rc = L.expmb_expm(W.data_ptr(), X.data_ptr(), B, n, dt, float(eps), scheme_code,
                          p(m), p(s), p(e1), p(e2), p(norms), p(mults), p(nonfinite),
                          p(ws), int(wsb), stream)
    if rc != 0:
        _raise_rc(rc)


@torch.library.custom_op("expmkit_b200::expm", mutates_args=())
def _expm_op(W: torch.Tensor, eps: float, scheme: int) -> tuple[
        torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor,
        torch.Tensor, torch.Tensor]:
    B = W.shape[0]
    dev = W.device
    X = torch.empty_like(W)
    m = torch.empty(B, dtype=torch.int8, device=dev)
    s = torch.empty(B, dtype=torch.int8, device=dev)
    e1 = torch.empty(B, dtype=torch.float64, device=dev)
    e2 = torch.empty(B, dtype=torch.float64, device=dev)
    norms = torch.empty(B, 2, dtype=torch.float64, device=dev)
    mults = torch.empty(B, dtype=torch.int32, device=dev)
    nonfinite = torch.empty(B, dtype=torch.uint8, device=dev)
    _launch(W, X, eps, scheme, m, s, e1, e2, norms, mults, nonfinite)
    return X, m, s, e1, e2, norms, mults, nonfinite


@_expm_op.register_fake
def _(W, eps, scheme):
    B = W.shape[0]
    return (torch.empty_like(W), W.new_empty(B, dtype=torch.int8), W.new_empty(B, dtype=torch.int8),
            W.new_empty(B, dtype=torch.float64), W.new_empty(B, dtype=torch.float64),
            W.new_empty(B, 2, dtype=torch.float64), W.new_empty(B, dtype=torch.int32),
            W.new_empty(B, dtype=torch.uint8))


_PLAN_SPEC = {"m": (torch.int8, 1), "s": (torch.int8, 1), "e1": (torch.float64, 1), "e2": (torch.float64, 1),
              "norms": (torch.float64, 2), "mults": (torch.int32, 1), "nonfinite": (torch.uint8, 1),
              "flags": (torch.uint8, 1)}


def _check_plan(plan: dict | None, B: int, device: torch.device, keys) -> dict:
    """Caller-provided plan tensors are written through raw pointers: check
    dtype, size, device and contiguity before any launch."""
    plan = plan or {}
    for k, v in plan.items():
        if k not in keys:
            raise MatrixError(f"unknown plan key {k!r}; expected {sorted(keys)}")
        if v is None:
            continue
        dt, per = _PLAN_SPEC[k]
        if (not isinstance(v, torch.Tensor) or v.dtype != dt or v.numel() != B * per or v.device != device
                or not v.is_contiguous()):
            raise MatrixError(f"plan[{k!r}] must be a contiguous {dt} tensor of {B * per} elements on {device}")
    return plan


def _validate(W: torch.Tensor, eps: float, scheme: str, allow_baseline: bool = False) -> tuple[torch.Tensor, int]:
    if not isinstance(W, torch.Tensor):
        raise MatrixError(f"expected a torch.Tensor, got {type(W).__name__}")
    if W.dim() < 2 or W.shape[-1] != W.shape[-2]:
        raise MatrixError(f"expected [..., n, n] square matrices, got shape {tuple(W.shape)}")
    if W.shape[-1] < 1:
        raise MatrixError("matrix order must be at least 1")
    if scheme not in _SCHEMES and not (allow_baseline and scheme == SCHEME_BASELINE):
        raise MatrixError(f"unknown scheme {scheme!r}; expected 'ps' or 'sastre'")
    if W.dtype not in (torch.float32, torch.float64):
        raise MatrixError(f"dtype must be float32 or float64, got {W.dtype}")
    if W.device.type != "cuda":
        raise RuntimeError("expmkit_b200.expm runs on CUDA tensors only (no CPU fallback)")
    check_tolerance(eps, W.dtype)
    Wc = W.reshape(-1, W.shape[-1], W.shape[-1])
    if not Wc.is_contiguous() or Wc.data_ptr() % 16:
        Wc = Wc.contiguous().clone()
    return Wc, _SCHEMES.get(scheme, _lib.EXPMB_BASELINE)


def expm(W: torch.Tensor, eps: float, scheme: str = SCHEME_SASTRE, check_finite: bool = True) -> ExpmResult:
    """Selected-order scaled-Taylor exponential of every matrix in ``W``.

    Mirrors engine.py:119-152 per matrix; ``scheme`` selects the Sastre
    evaluation formulas (orders 1,2,4,8,15+) or Paterson-Stockmeyer (1..16).
    """
    t0 = time.perf_counter()
    Wc, code = _validate(W, eps, scheme)
    lead = W.shape[:-2]
    n = W.shape[-1]
    X, m, s, e1, e2, norms, mults, nonfinite = torch.ops.expmkit_b200.expm(Wc, float(eps), code)
    bad = nonfinite.bool()
    if check_finite and Wc.shape[0] > 0 and bool(bad.any()):
        idx = torch.nonzero(bad).flatten()[:8].tolist()
        raise NonFiniteError(f"operation produced non-finite entries (batch indices {idx}...)")
    plan = EvalPlan(m.reshape(lead), s.reshape(lead), scheme, e1.reshape(lead), e2.reshape(lead),
                    norms.reshape(*lead, 2))
    return ExpmResult(X.reshape(*lead, n, n), plan, mults.reshape(lead), time.perf_counter() - t0,
                      bad.reshape(lead))


def expm_baseline(W: torch.Tensor, eps: float, check_finite: bool = True) -> ExpmResult:
    """Alg. 1, the paper's comparator (engine.py:90-116): scale until the
    1-norm is below 1/2, add Taylor terms B^k/k! until the next term's 1-norm
    is at most eps, square back.  plan.m = terms added, plan.e1 = the norm of
    the first term not added, mults = m + s (test_engine.py:83-97).  Any n:
    fused per-matrix kernels for n <= 64, the GEMM pipeline above (term stages
    over device-resident active lists, every squaring level in one
    cooperative launch; no host synchronisation)."""
    t0 = time.perf_counter()
    Wc, code = _validate(W, eps, SCHEME_BASELINE, allow_baseline=True)
    lead, n = W.shape[:-2], W.shape[-1]
    X, m, s, e1, e2, norms, mults, nonfinite = torch.ops.expmkit_b200.expm(Wc, float(eps), code)
    bad = nonfinite.bool()
    if check_finite and Wc.shape[0] > 0 and bool(bad.any()):
        idx = torch.nonzero(bad).flatten()[:8].tolist()
        raise NonFiniteError(f"operation produced non-finite entries (batch indices {idx}...)")
    plan = EvalPlan(m.reshape(lead), s.reshape(lead), SCHEME_BASELINE, e1.reshape(lead), e2.reshape(lead),
                    norms.reshape(*lead, 2))
    return ExpmResult(X.reshape(*lead, n, n), plan, mults.reshape(lead), time.perf_counter() - t0,
                      bad.reshape(lead))


def expm_into(W: torch.Tensor, X: torch.Tensor, eps: float, scheme: str = SCHEME_SASTRE,
              plan: dict | None = None) -> None:
    """Allocation-free variant for steady-state loops and CUDA graphs:
    writes e^W into the preallocated ``X`` (same shape/dtype) and, if given,
    into the plan tensors of ``plan`` (keys m, s, e1, e2, norms, mults, nonfinite).
    No host synchronisation for any n (capturable in a CUDA graph)."""
    Wc, code = _validate(W, eps, scheme, allow_baseline=True)
    if X.shape != W.shape or X.dtype != W.dtype or not X.is_contiguous() or X.device != W.device:
        raise MatrixError("X must be a contiguous tensor shaped and typed like W, on W's device")
    plan = _check_plan(plan, Wc.shape[0], W.device, ("m", "s", "e1", "e2", "norms", "mults", "nonfinite"))
    _launch(Wc, X.view(Wc.shape), eps, code, plan.get("m"), plan.get("s"), plan.get("e1"),
            plan.get("e2"), plan.get("norms"), plan.get("mults"), plan.get("nonfinite"))


class HostPipeline:
    """Reusable host-buffer pipeline (pinned output + device staging buffers
    allocated once), for serving loops that call the reference's calling
    convention -- host memory in, host memory out (engine.py:119-152) -- over
    and over.  ``run`` splits the batch into ``chunks`` pieces pipelined over
    three CUDA streams, so the host->device copy of chunk c+1, the
    exponentials of chunk c and the device->host copy of chunk c-1 overlap
    (PCIe is full duplex)."""

    def __init__(self, batch: int, n: int, dtype: torch.dtype = torch.float32, chunks: int = 8,
                 device: int | torch.device | None = None):
        self.dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.B, self.n, self.dtype = int(batch), int(n), dtype
        B = self.B
        self.out = torch.empty((B, n, n), dtype=dtype, pin_memory=True)
        self.host = {k: torch.empty(shape, dtype=dt, pin_memory=True) for k, shape, dt in (
            ("m", (B,), torch.int8), ("s", (B,), torch.int8), ("e1", (B,), torch.float64),
            ("e2", (B,), torch.float64), ("norms", (B, 2), torch.float64), ("mults", (B,), torch.int32),
            ("nonfinite", (B,), torch.uint8))}
        self.Wd = torch.empty((B, n, n), dtype=dtype, device=self.dev)
        self.Xd = torch.empty_like(self.Wd)
        self.pd = {k: torch.empty(v.shape, dtype=v.dtype, device=self.dev) for k, v in self.host.items()}
        self.streams = [torch.cuda.Stream(self.dev) for _ in range(3)]
        c = max(1, min(int(chunks), B, 256)) if B else 1  # expmb_expm_pipelined caps chunks at 256
        self._nchunks = c
        # chunk bounds on multiples of 4 matrices keep every slice 16-byte aligned
        self.bounds = sorted({min(B, ((B * k) // c) // 4 * 4) for k in range(c)} | {B})
        if self.bounds[0] != 0:
            self.bounds = [0] + self.bounds
        # per-chunk C-ABI argument tuples and events, built once (the Python
        # per-chunk overhead otherwise dominated beyond ~8 chunks)
        L = _lib.lib()
        self._dt = _lib.EXPMB_F32 if dtype == torch.float32 else _lib.EXPMB_F64
        cmax = max((b - a for a, b in zip(self.bounds[:-1], self.bounds[1:])), default=0)
        self._wsb = {code: int(L.expmb_workspace_bytes(cmax, n, self._dt, code)) for code in (0, 1, 2)}
        self._ws = torch.empty(max(max(self._wsb.values()), 1), dtype=torch.uint8, device=self.dev)
        esz = self.Wd.element_size()
        self._chunks = []
        for a, b in zip(self.bounds[:-1], self.bounds[1:]):
            if a == b:
                continue
            ptrs = [self.pd[k].data_ptr() + a * self.pd[k][0:1].numel() * self.pd[k].element_size()
                    for k in ("m", "s", "e1", "e2", "norms", "mults", "nonfinite")]
            self._chunks.append((a, b, self.Wd.data_ptr() + a * n * n * esz, self.Xd.data_ptr() + a * n * n * esz,
                                 ptrs, torch.cuda.Event(), torch.cuda.Event()))
        self.h2d_bytes = B * n * n * self.Wd.element_size()
        self.d2h_bytes = self.h2d_bytes + sum(v.numel() * v.element_size() for v in self.host.values())

    def run(self, W: torch.Tensor, eps: float, scheme: str = SCHEME_SASTRE, check_finite: bool = True) -> ExpmResult:
        t0 = time.perf_counter()
        if not isinstance(W, torch.Tensor) or W.device.type != "cpu":
            raise MatrixError("HostPipeline.run takes a CPU tensor; use expm() for device tensors")
        n = self.n
        lead = W.shape[:-2]
        Wf = W.reshape(-1, n, n)
        if Wf.shape[0] != self.B or W.dtype != self.dtype:
            raise MatrixError(f"pipeline built for {self.B} x {n}x{n} {self.dtype}, got {tuple(W.shape)} {W.dtype}")
        if not Wf.is_contiguous():
            Wf = Wf.contiguous()
        check_tolerance(eps, W.dtype)
        code = _SCHEMES.get(scheme, _lib.EXPMB_BASELINE if scheme == SCHEME_BASELINE else None)
        if code is None:
            raise MatrixError(f"unknown scheme {scheme!r}; expected 'ps' or 'sastre'")
        L = _lib.lib()
        wsp, wsb = self._ws.data_ptr(), self._wsb[code]
        s_in, s_comp, s_out = self.streams
        s_in.wait_stream(torch.cuda.current_stream(self.dev))
        # the chunk loop runs in C (expmb_expm_pipelined): every host->device
        # copy queued first, each chunk's expm on s_comp after its copy, its
        # result copied back on s_out while later chunks compute
        p = [self.pd[k].data_ptr() for k in ("m", "s", "e1", "e2", "norms", "mults", "nonfinite")]
        with torch.cuda.device(self.dev):
            rc = L.expmb_expm_pipelined(Wf.data_ptr(), self.out.data_ptr(), self.Wd.data_ptr(), self.Xd.data_ptr(),
                                        self.B, n, self._dt, float(eps), code, *p, self._nchunks, wsp, wsb,
                                        s_in.cuda_stream, s_comp.cuda_stream, s_out.cuda_stream)
        if rc != 0:
            _raise_rc(rc)
        with torch.cuda.stream(s_out):  # the small plan arrays: one copy each, after the last chunk
            s_out.wait_stream(s_comp)
            for k, v in self.host.items():
                v.copy_(self.pd[k], non_blocking=True)
        s_out.synchronize()
        h = self.host
        bad = h["nonfinite"].bool()
        if check_finite and self.B > 0 and bool(bad.any()):
            idx = torch.nonzero(bad).flatten()[:8].tolist()
            raise NonFiniteError(f"operation produced non-finite entries (batch indices {idx}...)")
        plan = EvalPlan(h["m"].reshape(lead), h["s"].reshape(lead), scheme, h["e1"].reshape(lead),
                        h["e2"].reshape(lead), h["norms"].reshape(*lead, 2))
        return ExpmResult(self.out.reshape(*lead, n, n), plan, h["mults"].reshape(lead), time.perf_counter() - t0,
                          bad.reshape(lead))


def expm_host(W: torch.Tensor, eps: float, scheme: str = SCHEME_SASTRE, chunks: int = 8,
              device: int | torch.device | None = None, check_finite: bool = True) -> ExpmResult:
    """One-off host-buffer call: CPU tensor ``[..., n, n]`` in, pinned CPU
    tensor out (see HostPipeline; results alias that pipeline's buffers)."""
    if not isinstance(W, torch.Tensor) or W.device.type != "cpu":
        raise MatrixError("expm_host takes a CPU tensor; use expm() for device tensors")
    if W.dim() < 2 or W.shape[-1] != W.shape[-2] or W.shape[-1] < 1:
        raise MatrixError(f"expected [..., n, n] square matrices, got shape {tuple(W.shape)}")
    n = W.shape[-1]
    pipe = HostPipeline(W.numel() // (n * n), n, W.dtype, chunks, device)
    return pipe.run(W, eps, scheme, check_finite)


@torch.library.custom_op("expmkit_b200::select", mutates_args=())
def _select_op(W: torch.Tensor, eps: float, scheme: int) -> tuple[
        torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
    B, n = W.shape[0], W.shape[-1]
    dev = W.device
    m = torch.empty(B, dtype=torch.int8, device=dev)
    s = torch.empty(B, dtype=torch.int8, device=dev)
    e1 = torch.empty(B, dtype=torch.float64, device=dev)
    e2 = torch.empty(B, dtype=torch.float64, device=dev)
    norms = torch.empty(B, 2, dtype=torch.float64, device=dev)
    mults = torch.empty(B, dtype=torch.int32, device=dev)
    nonfinite = torch.empty(B, dtype=torch.uint8, device=dev)
    L = _lib.lib()
    dt = _lib.EXPMB_F32 if W.dtype == torch.float32 else _lib.EXPMB_F64
    wsb = int(L.expmb_workspace_bytes(B, n, dt, scheme))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        rc = L.expmb_select(W.data_ptr(), B, n, dt, float(eps), scheme, m.data_ptr(), s.data_ptr(), e1.data_ptr(),
                            e2.data_ptr(), norms.data_ptr(), mults.data_ptr(), nonfinite.data_ptr(), ws.data_ptr(),
                            wsb, torch.cuda.current_stream(dev).cuda_stream)
    if rc != 0:
        _raise_rc(rc)
    return m, s, e1, e2, norms, mults, nonfinite


@_select_op.register_fake
def _(W, eps, scheme):
    B = W.shape[0]
    return (W.new_empty(B, dtype=torch.int8), W.new_empty(B, dtype=torch.int8), W.new_empty(B, dtype=torch.float64),
            W.new_empty(B, dtype=torch.float64), W.new_empty(B, 2, dtype=torch.float64),
            W.new_empty(B, dtype=torch.int32), W.new_empty(B, dtype=torch.uint8))


def _select(W: torch.Tensor, eps: float, scheme: str, check_finite: bool) -> EvalPlan:
    Wc, code = _validate(W, eps, scheme)
    lead = W.shape[:-2]
    m, s, e1, e2, norms, _, nonfinite = torch.ops.expmkit_b200.select(Wc, float(eps), code)
    if check_finite and Wc.shape[0] > 0 and bool(nonfinite.any()):
        idx = torch.nonzero(nonfinite).flatten()[:8].tolist()
        raise NonFiniteError(f"operation produced non-finite entries (batch indices {idx}...)")
    return EvalPlan(m.reshape(lead), s.reshape(lead), scheme, e1.reshape(lead), e2.reshape(lead),
                    norms.reshape(*lead, 2))


def select_sastre(W: torch.Tensor, eps: float, check_finite: bool = True) -> EvalPlan:
    """select.py:228-234, batched: ||W||_1, W^2 and ||W^2||_1 only where the
    ladder needs them, then the (m, s) choice -- no exponential is formed
    (expmb_select).  Raises NonFiniteError like the reference when the input
    or W^2 is not finite (matrix.py:56-57, 95-102)."""
    return _select(W, eps, SCHEME_SASTRE, check_finite)


def select_ps(W: torch.Tensor, eps: float, check_finite: bool = True) -> EvalPlan:
    """select.py:223-225, batched: the Paterson-Stockmeyer ladder (W^2, W^3,
    W^4 as needed), plan only."""
    return _select(W, eps, SCHEME_PS, check_finite)


# ---------------------------------------------------------------------------
# Low-rank path: engine.py:159-257
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class LowRankPair:
    """Batched engine.py:159-191: W = A1 A2 with a1 [..., n, t], a2 [..., t, n],
    1 <= t <= n, on the same CUDA device and dtype (fp32/fp64).  Shapes are
    checked here (MatrixError, engine.py:168-178); the finiteness check of
    engine.py:179-180 runs on the device inside ``expm_lowrank`` so building a
    pair never synchronises the host."""
    a1: torch.Tensor
    a2: torch.Tensor

    def __post_init__(self):
        a1, a2 = self.a1, self.a2
        if not isinstance(a1, torch.Tensor) or not isinstance(a2, torch.Tensor):
            raise MatrixError("low-rank factors must be torch tensors")
        if a1.dim() < 2 or a2.dim() < 2:
            raise MatrixError("low-rank factors must be (batched) 2-d arrays")
        n, t = a1.shape[-2], a1.shape[-1]
        if tuple(a2.shape[-2:]) != (t, n) or a1.shape[:-2] != a2.shape[:-2]:
            raise MatrixError(f"factor shapes incompatible: {tuple(a1.shape)} and {tuple(a2.shape)}")
        if t > n:
            raise MatrixError(f"inner rank {t} exceeds order {n}")
        if t < 1:
            raise MatrixError("inner rank must be at least 1")
        if a1.dtype != a2.dtype or a1.dtype not in (torch.float32, torch.float64):
            raise MatrixError("factors must share dtype float32 or float64")

    @property
    def n(self) -> int:
        return self.a1.shape[-2]

    @property
    def t(self) -> int:
        return self.a1.shape[-1]


@torch.library.custom_op("expmkit_b200::expm_lowrank", mutates_args=())
def _expm_lowrank_op(A1: torch.Tensor, A2: torch.Tensor, eps: float) -> tuple[
        torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
    B, n, t = A1.shape
    dev = A1.device
    X = torch.empty(B, n, n, dtype=A1.dtype, device=dev)
    m = torch.empty(B, dtype=torch.int8, device=dev)
    e1 = torch.empty(B, dtype=torch.float64, device=dev)
    e2 = torch.empty(B, dtype=torch.float64, device=dev)
    norms = torch.empty(B, 2, dtype=torch.float64, device=dev)
    mults = torch.empty(B, dtype=torch.int32, device=dev)
    flags = torch.empty(B, dtype=torch.uint8, device=dev)
    L = _lib.lib()
    dt = _lib.EXPMB_F32 if A1.dtype == torch.float32 else _lib.EXPMB_F64
    wsb = int(L.expmb_lowrank_workspace_bytes(B, n, t, dt))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev) if wsb else None
    with torch.cuda.device(dev):
        rc = L.expmb_expm_lowrank(A1.data_ptr(), A2.data_ptr(), X.data_ptr(), B, n, t, dt, float(eps),
                                  m.data_ptr(), e1.data_ptr(), e2.data_ptr(), norms.data_ptr(), mults.data_ptr(),
                                  flags.data_ptr(), None if ws is None else ws.data_ptr(), wsb,
                                  torch.cuda.current_stream(dev).cuda_stream)
    if rc != 0:
        _raise_rc(rc)
    return X, m, e1, e2, norms, mults, flags


@_expm_lowrank_op.register_fake
def _(A1, A2, eps):
    B, n, t = A1.shape
    return (A1.new_empty(B, n, n), A1.new_empty(B, dtype=torch.int8), A1.new_empty(B, dtype=torch.float64),
            A1.new_empty(B, dtype=torch.float64), A1.new_empty(B, 2, dtype=torch.float64),
            A1.new_empty(B, dtype=torch.int32), A1.new_empty(B, dtype=torch.uint8))


def expm_lowrank(pair: LowRankPair, eps: float) -> ExpmResult:
    """Batched engine.py:198-257: e^(A1 A2) = I + A1 psi(V) A2, V = A2 A1, at
    the smallest order on LOWRANK_ORDERS whose two-term bound meets eps (no
    scaling; plan.s = 0, plan.scheme = "lowrank").  ``mults`` counts the t x t
    products, ``rect_mults`` = 3 (A2 A1 and the two assembly products).

    Raises, after the batch completes: MatrixError when a factor holds
    NaN/Inf (engine.py:179-180), LowRankOrderError when no order qualifies
    (engine.py:236-240), NonFiniteError when V, psi or the result is not
    finite (matrix.py:95-102).  Any 1 <= t <= n: t <= 32 runs one CTA per
    matrix with every t x t operand in shared memory; larger inner ranks keep
    the t x t operands in a device workspace (lowrank_large.cuh)."""
    t0 = time.perf_counter()
    if not isinstance(pair, LowRankPair):
        pair = LowRankPair(*pair)
    a1, a2 = pair.a1, pair.a2
    if a1.device.type != "cuda" or a2.device != a1.device:
        raise RuntimeError("expmkit_b200.expm_lowrank runs on CUDA tensors only (no CPU fallback)")
    check_tolerance(eps, a1.dtype)
    lead, n, t = a1.shape[:-2], pair.n, pair.t
    A1 = a1.reshape(-1, n, t).contiguous()
    A2 = a2.reshape(-1, t, n).contiguous()
    X, m, e1, e2, norms, mults, flags = torch.ops.expmkit_b200.expm_lowrank(A1, A2, float(eps))
    if A1.shape[0] > 0 and bool(flags.any()):
        f = flags.cpu()
        if bool((f & _lib.LR_BAD_INPUT).any()):
            raise MatrixError("low-rank factors must be finite")
        i = int(torch.nonzero(f).flatten()[0])
        if int(f[i]) & _lib.LR_NO_ORDER:
            nv = float(norms[i, 0])
            raise LowRankOrderError(
                f"||V||_1 = {nv:.6g} admits no order <= 30 at tolerance {float(eps):.3g}; "
                f"the factored path runs unscaled (batch index {i})")
        raise NonFiniteError(f"operation produced non-finite entries (batch index {i})")
    plan = EvalPlan(m.reshape(lead), torch.zeros_like(m).reshape(lead), SCHEME_LOWRANK, e1.reshape(lead),
                    e2.reshape(lead), norms.reshape(*lead, 2))
    return ExpmResult(X.reshape(*lead, n, n), plan, mults.reshape(lead), time.perf_counter() - t0,
                      flags.bool().reshape(lead), rect_mults=3)


def expm_lowrank_into(A1: torch.Tensor, A2: torch.Tensor, X: torch.Tensor, eps: float,
                      plan: dict | None = None, workspace: torch.Tensor | None = None) -> None:
    """Allocation-free, synchronisation-free ``expm_lowrank`` for steady-state
    loops and CUDA graphs: A1 [B,n,t], A2 [B,t,n], X [B,n,n] contiguous CUDA
    tensors; plan tensors (keys m, e1, e2, norms, mults, flags) are optional.
    Errors are left in plan["flags"] (EXPMB_LR_* bits) instead of raised.  For
    t > 32 a preallocated ``workspace`` (expmb_lowrank_workspace_bytes) keeps the
    call allocation-free."""
    LowRankPair(A1, A2)
    B, n, t = A1.shape
    if X.shape != (B, n, n) or X.dtype != A1.dtype or not (A1.is_contiguous() and A2.is_contiguous()
                                                             and X.is_contiguous()):
        raise MatrixError("X must be contiguous [B, n, n] of the factors' dtype; factors contiguous")
    if A1.device.type != "cuda" or A2.device != A1.device or X.device != A1.device:
        raise MatrixError("A1, A2 and X must be on the same CUDA device")
    check_tolerance(eps, A1.dtype)
    plan = _check_plan(plan, B, A1.device, ("m", "e1", "e2", "norms", "mults", "flags"))

    def p(k):
        v = plan.get(k)
        return None if v is None else v.data_ptr()
    L = _lib.lib()
    dt = _lib.EXPMB_F32 if A1.dtype == torch.float32 else _lib.EXPMB_F64
    wsb = int(L.expmb_lowrank_workspace_bytes(B, n, t, dt))
    if wsb and (workspace is None or not isinstance(workspace, torch.Tensor) or workspace.dtype != torch.uint8
                or workspace.device != A1.device or workspace.numel() < wsb or not workspace.is_contiguous()):
        if workspace is not None:
            raise MatrixError(f"workspace must be a contiguous uint8 tensor of >= {wsb} bytes on {A1.device}")
        workspace = torch.empty(wsb, dtype=torch.uint8, device=A1.device)
    with torch.cuda.device(A1.device):
        rc = L.expmb_expm_lowrank(
            A1.data_ptr(), A2.data_ptr(), X.data_ptr(), B, n, t, dt, float(eps),
            p("m"), p("e1"), p("e2"), p("norms"), p("mults"), p("flags"),
            workspace.data_ptr() if wsb else None, wsb, torch.cuda.current_stream(A1.device).cuda_stream)
    if rc != 0:
        _raise_rc(rc)


# ---------------------------------------------------------------------------
# Time grid: e^(t_k A) for one A and many t_k
# ---------------------------------------------------------------------------

def expm_timegrid(A: torch.Tensor, times: torch.Tensor, eps: float, scheme: str = SCHEME_SASTRE,
                  check_finite: bool = True, out: torch.Tensor | None = None, plan: dict | None = None,
                  workspace: torch.Tensor | None = None) -> ExpmResult:
    """value[k] = e^(times[k] * A), each what ``expm`` returns for the
    materialised matrix times[k] * A (engine.py:119-152 per time point).

    For n > 64 the powers A^1..A^16 are formed once (binary64) and a time point
    costs its s_k squarings plus one fused linear combination, instead of
    budget(m_k) + s_k products.  ``out`` / ``plan`` / ``workspace`` may be
    preallocated for steady-state loops (``expmb_timegrid_workspace_bytes``)."""
    t0 = time.perf_counter()
    if not isinstance(A, torch.Tensor) or A.dim() != 2 or A.shape[0] != A.shape[1] or A.shape[0] < 1:
        raise MatrixError("A must be a square [n, n] tensor")
    if scheme not in _SCHEMES:
        raise MatrixError(f"unknown scheme {scheme!r}; expected 'ps' or 'sastre'")
    if A.dtype not in (torch.float32, torch.float64):
        raise MatrixError(f"dtype must be float32 or float64, got {A.dtype}")
    if A.device.type != "cuda":
        raise RuntimeError("expmkit_b200.expm_timegrid runs on CUDA tensors only (no CPU fallback)")
    check_tolerance(eps, A.dtype)
    n = A.shape[0]
    A = A.contiguous()
    t = torch.as_tensor(times).to(device=A.device, dtype=A.dtype).reshape(-1).contiguous()
    K = t.shape[0]
    dev = A.device
    if out is not None and (not isinstance(out, torch.Tensor) or tuple(out.shape) != (K, n, n)
                            or out.dtype != A.dtype or out.device != dev or not out.is_contiguous()
                            or out.data_ptr() % 16):
        raise MatrixError(f"out must be a contiguous, 16-byte aligned ({K}, {n}, {n}) {A.dtype} tensor on {dev}")
    X = out if out is not None else torch.empty(K, n, n, dtype=A.dtype, device=dev)
    if plan is not None:
        _check_plan(plan, K, dev, ("m", "s", "e1", "e2", "norms", "mults", "nonfinite"))
    if plan is None:
        plan = {"m": torch.empty(K, dtype=torch.int8, device=dev), "s": torch.empty(K, dtype=torch.int8, device=dev),
                "e1": torch.empty(K, dtype=torch.float64, device=dev),
                "e2": torch.empty(K, dtype=torch.float64, device=dev),
                "norms": torch.empty(K, 2, dtype=torch.float64, device=dev),
                "mults": torch.empty(K, dtype=torch.int32, device=dev),
                "nonfinite": torch.empty(K, dtype=torch.uint8, device=dev)}
    L = _lib.lib()
    dt = _lib.EXPMB_F32 if A.dtype == torch.float32 else _lib.EXPMB_F64
    wsb = int(L.expmb_timegrid_workspace_bytes(K, n, dt))
    if workspace is not None and (not isinstance(workspace, torch.Tensor) or workspace.dtype != torch.uint8
                                  or workspace.device != dev or not workspace.is_contiguous()):
        raise MatrixError(f"workspace must be a contiguous uint8 tensor on {dev}")
    if workspace is None or workspace.numel() < wsb:
        workspace = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)

    def p(k):
        v = plan.get(k)
        return None if v is None else v.data_ptr()
    with torch.cuda.device(dev):
        rc = L.expmb_expm_timegrid(A.data_ptr(), t.data_ptr(), X.data_ptr(), K, n, dt, float(eps), _SCHEMES[scheme],
                                   p("m"), p("s"), p("e1"), p("e2"), p("norms"), p("mults"), p("nonfinite"),
                                   workspace.data_ptr(), wsb, torch.cuda.current_stream(dev).cuda_stream)
    if rc != 0:
        _raise_rc(rc)
    bad = plan["nonfinite"].bool() if plan.get("nonfinite") is not None else torch.zeros(K, dtype=torch.bool,
                                                                                          device=dev)
    if check_finite and K > 0 and bool(bad.any()):
        idx = torch.nonzero(bad).flatten()[:8].tolist()
        raise NonFiniteError(f"operation produced non-finite entries (time indices {idx}...)")
    ep = EvalPlan(plan.get("m"), plan.get("s"), scheme, plan.get("e1"), plan.get("e2"), plan.get("norms"))
    return ExpmResult(X, ep, plan.get("mults"), time.perf_counter() - t0, bad)
