#!/usr/bin/env python
"""Benchmark: batched matrix exponentials/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One "step" = one call of the hot path (expm over the whole batch of the
config).  Default workload: BASELINE.json configs[1] = C2 (65536 x 16x16 fp32
skew-symmetric, tol 2^-24); the same line carries ``per_config`` with C1, C3,
C4 and C5 measured the same way (fewer steps).  Under torchrun (N > 1) the
config's fixed global batch is split into rank-ordered shards
(shard.shard_range; strong scaling, ``--scaling weak`` gives every rank a full
batch), with no collective on the data path; the step time is the max over
ranks of device time, and ``e2e_gather`` repeats the step with the final NCCL
gather of every result into rank 0.

Printed JSON line (rank 0):
  value        whole-job exps/s with inputs resident in HBM (device-timed)
  e2e          exps/s through the public API from pinned host memory, H2D of W
               and D2H of e^W + plan inside the timed region
  roofline     dominant kernel vs its bound (HBM bytes or useful FLOPs)
  cpu_baseline the reference's CPU path on this host (the unmodified expmkit
               from baseline/_ref, else the oracle port)
`--impl reference` times that CPU path alone, on the same config.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2512_20777_b200 import workloads as WL  # noqa: E402

L2_BYTES = 126 * 1024 * 1024


def _make_l2_flush(flush):
    """Write a buffer 2x the L2 (evicting everything); BENCH_FLUSH=writeread
    adds a read pass so the L2 is left holding clean lines."""
    import torch
    sink = torch.empty(1, dtype=flush.dtype, device=flush.device)

    # measured on B200: the read pass changes nothing (C2 90.0 vs 89.9 us, C1
    # 153.4 vs 153.3 us), so the default is the contract's plain write
    read_back = os.environ.get("BENCH_FLUSH", "write") == "writeread"

    def l2_flush():
        flush.zero_()
        if read_back:
            torch.sum(flush, dim=0, keepdim=True, out=sink)
    return l2_flush
# matrices per CPU-baseline sample (our line) and per reference-arm step:
# the whole batch where it finishes in about a second, bounded samples above
CPU_SAMPLE = {"C1": 1024, "C2": 65536, "C3": 512, "C4": 6, "C5": 3}
REF_STEP = {"C1": 1024, "C2": 65536, "C3": 256, "C4": 2, "C5": 1}


def _peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver) + our pipe microbenchmarks."""
    out = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        out["hbm_gbs"] = float(d["hbm_gbs"])
        out["hbm_src"] = "MEASURED_PEAKS.json"
    pp = os.path.join(ROOT, "profiles", "peaks.json")
    if os.path.exists(pp):
        for line in open(pp):
            line = line.strip()
            if line.startswith("{") and "pipe" in line:
                d = json.loads(line)
                out[d["pipe"]] = float(d["tflops"])
    out.setdefault("ffma_fp32", 74.4)
    out.setdefault("dfma_fp64", 37.2)
    # fp64: the faster of the two fp64 pipes (DFMA, DMMA tensor core) -- the
    # products run on DMMA
    fp32 = {k: v for k, v in out.items() if k.startswith(("ffma_fp32", "ffma2_fp32")) and isinstance(v, float)}
    out["fp32_src"] = max(fp32, key=fp32.get)
    out["fp32"] = fp32[out["fp32_src"]]
    fp64 = {k: v for k, v in out.items() if k.startswith(("dfma_fp64", "dmma_")) and isinstance(v, float)}
    out["fp64_src"] = max(fp64, key=fp64.get)
    out["fp64"] = fp64[out["fp64_src"]]
    if "tcgen05_i8_m128n256" in out:
        out["i8_tops"], out["i8_src"] = out["tcgen05_i8_m128n256"], "profiles/peaks.json tcgen05_i8_m128n256 (tools/peaks.cu, measured on B200)"
    else:
        out["i8_tops"], out["i8_src"] = 4500.0, "nominal dense int8 (tcgen05 i8 probe not yet run)"
    return out


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def mark(self, which):
        (self.__dict__.setdefault("marks", {}))[which] = time.perf_counter()

    def _run_nvml(self):
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        bits = {"hw_slowdown": getattr(N, "nvmlClocksEventReasonHwSlowdown", 0x8),
                "hw_thermal_slowdown": getattr(N, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(N, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": getattr(N, "nvmlClocksEventReasonSwPowerCap", 0x4)}
        while not self._stop.is_set():
            sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
            try:
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            act = [k for k, b in bits.items() if r & b]
            self.rows.append([str(sm), str(mx), "", *["Active" if k in act else "Not Active" for k in bits],
                              time.perf_counter()])
            self._stop.wait(0.001)

    def _run(self):
        try:
            import pynvml  # noqa: F401
            return self._run_nvml()
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                r = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                    "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if r.returncode == 0 and r.stdout.strip():
                    self.rows.append([x.strip() for x in r.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        marks = getattr(self, "marks", {})
        if "start" in marks and "end" in marks:
            inwin = [r for r in self.rows if len(r) > 7 and marks["start"] <= r[7] <= marks["end"]]
            if inwin:
                self.rows = inwin
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU side (the reference's own CPU path) -- rank 0 only
# ---------------------------------------------------------------------------

_CPU = {}  # the sample a forked worker pool reads (copy-on-write, no pickling)


def reference_impl():
    """The CPU implementation the baselines time: the UNMODIFIED reference
    package ``expmkit`` installed under baseline/_ref (pip --target, see
    DESIGN.md) when present -- kind "reference" -- else the oracle's
    restatement of it (oracle/expm_oracle.py, pinned bit-exactly to the
    reference's outputs) -- kind "port"."""
    p = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(p, "expmkit")):
        if p not in sys.path:
            sys.path.insert(0, p)
        try:
            import expmkit
            return "reference", expmkit
        except Exception:
            pass
    from oracle import expm_oracle
    return "port", expm_oracle


def _cpu_worker_init():
    # one BLAS thread per worker process (the pool supplies the parallelism;
    # forked workers inherit the parent's already-initialised BLAS pool)
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _cpu_range(args):
    """expm (engine.py:119-152) on matrices [lo, hi) of the forked sample."""
    lo, hi = args
    kind, mod = reference_impl()
    W, eps = _CPU["W"], _CPU["eps"]
    if kind == "reference":
        for i in range(lo, hi):
            mod.expm(mod.Matrix(W[i]), eps, "sastre")
    else:
        for i in range(lo, hi):
            mod.expm(W[i], eps)
    return hi - lo


def cpu_reference_rate(key: str, count: int | None = None, cores: int | None = None, repeats: int = 1):
    """exps/s of the reference's CPU path (binary64, as the reference computes
    every dtype) on the first ``count`` matrices of config ``key``.  Orders
    <= 256: a forked process pool with one BLAS thread per worker, the
    reference harness's own sharding (bench.py:303-306); larger orders: one
    process, BLAS threads on every core.  Returns (rates per repeat, cores,
    kind, sample description)."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    cfg = WL.CONFIGS[key]
    count = min(cfg.batch, count or CPU_SAMPLE[key])
    cores = cores or os.cpu_count() or 1
    kind, _ = reference_impl()
    _CPU["W"] = WL.generate(key, indices=np.arange(count)).astype(np.float64)
    _CPU["eps"] = cfg.eps
    rates = []
    if cfg.n > 256:
        for _ in range(repeats):
            t0 = time.perf_counter()
            done = _cpu_range((0, count))
            rates.append(done / (time.perf_counter() - t0))
        mode = "one process, multithreaded BLAS"
        used = cores
    else:
        step = max(1, min(256, -(-count // (cores * 4))))
        ranges = [(a, min(count, a + step)) for a in range(0, count, step)]
        with ProcessPoolExecutor(max_workers=cores, mp_context=mp.get_context("fork"),
                                 initializer=_cpu_worker_init) as pool:
            list(pool.map(_cpu_range, [(0, 1)] * cores))  # warm every worker (imports)
            for _ in range(repeats):
                t0 = time.perf_counter()
                done = sum(pool.map(_cpu_range, ranges))
                rates.append(done / (time.perf_counter() - t0))
        mode = f"fork pool x{cores}, 1 BLAS thread each (reference bench.py:303-306)"
        used = cores
    what = "unmodified expmkit from baseline/_ref" if kind == "reference" else "oracle port of expmkit"
    sample = (f"{count} of {cfg.batch} matrices of {key} ({cfg.n}x{cfg.n}, binary64 as the reference computes; "
              f"{what}; {mode})")
    return rates, used, kind, sample


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------

def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path
    (the unmodified expmkit from baseline/_ref, else the oracle port) on this
    host's cores, on the same config / metric as our arm.  Each step
    exponentiates REF_STEP[config] matrices of the config (C1, C2: the whole
    batch, so the config is the same; larger orders: a bounded sample)."""
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    cfg = WL.CONFIGS[args.config]
    count = REF_STEP[args.config]
    t0 = time.perf_counter()
    rates, cores, kind, sample = cpu_reference_rate(args.config, count, repeats=args.warmup + args.steps)
    wall = time.perf_counter() - t0
    rates = rates[args.warmup:]
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": "matrix exponentials/s", "value": value, "unit": "exps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * count / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md 8(d) recipe)",
        "config": {"workload": f"{cfg.key}: {cfg.desc}", "batch": cfg.batch, "n": cfg.n, "eps": cfg.eps,
                   "matrices_per_step": count, "same_config": count == cfg.batch,
                   "parallelism": "cpu process pool (reference bench.py:303-306)" if cfg.n <= 256
                   else "one process, multithreaded BLAS"},
        "cpu_baseline": {"value": value, "unit": "exps/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "exps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Low-rank path: --config LR
# ---------------------------------------------------------------------------

def _cpu_lr_chunk(args):
    A1, A2, eps = args
    kind, mod = reference_impl()
    for i in range(A1.shape[0]):
        if kind == "reference":
            mod.expm_lowrank(mod.LowRankPair(A1[i], A2[i]), eps)
        else:
            mod.expm_lowrank(A1[i], A2[i], eps)
    return A1.shape[0]


def cpu_lowrank_rate(count: int = 4096, cores: int | None = None):
    """pairs/s of the reference's expm_lowrank (oracle port) over a process pool."""
    from concurrent.futures import ProcessPoolExecutor
    cores = cores or os.cpu_count() or 1
    A1, A2 = WL.generate_lowrank(np.arange(count))
    eps = WL.LOWRANK.eps
    parts = np.array_split(np.arange(count), max(1, min(count, cores * 4)))
    with ProcessPoolExecutor(max_workers=cores, initializer=_cpu_worker_init) as pool:
        list(pool.map(_cpu_lr_chunk, [(A1[:1], A2[:1], eps)] * min(cores, 2)))
        t0 = time.perf_counter()
        done = sum(pool.map(_cpu_lr_chunk, [(A1[p], A2[p], eps) for p in parts]))
        dt = time.perf_counter() - t0
    kind, _ = reference_impl()
    return done / dt, cores, (f"{done} pairs of LR (n 64, t 8, fp64; "
                              f"{'unmodified expmkit' if kind == 'reference' else 'oracle port'}; "
                              f"process pool x{cores}, 1 BLAS thread each)")


def run_lowrank(args):
    cfg = WL.LOWRANK
    n, t = cfg.n, WL.LOWRANK_T
    ws, rank, local = _dist_env()
    base = {"metric": "low-rank matrix exponentials/s", "unit": "exps/s", "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "steps": args.steps, "warmup": max(3, args.warmup)}
    if args.impl == "reference":
        if rank != 0:
            return
        for _ in range(args.warmup):
            cpu_lowrank_rate(512)
        rates = []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            r, cores, sample = cpu_lowrank_rate()
            rates.append(r)
        value = statistics.median(rates)
        line = dict(base, impl="reference", value=value, n_gpus=args.gpus,
                    ms_per_step=1e3 * (time.perf_counter() - t0) / max(1, args.steps),
                    config={"workload": f"LR: {cfg.desc}", "batch": cfg.batch, "n": n, "t": t, "eps": cfg.eps},
                    cpu_baseline={"value": value, "unit": "exps/s", "cores": cores, "kind": reference_impl()[0],
                                  "sample": sample},
                    e2e={"value": value, "unit": "exps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        print(json.dumps(line), flush=True)
        return
    import torch
    import torch.distributed as dist
    import paper_2512_20777_b200 as XP
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    B = args.batch or cfg.batch
    A1h, A2h = WL.generate_lowrank(np.arange(rank * B, (rank + 1) * B))
    A1h, A2h = torch.from_numpy(A1h), torch.from_numpy(A2h)
    A1, A2 = A1h.to(dev), A2h.to(dev)
    Xd = torch.empty(B, n, n, dtype=torch.float64, device=dev)
    plan = {"m": torch.empty(B, dtype=torch.int8, device=dev), "e1": torch.empty(B, dtype=torch.float64, device=dev),
            "e2": torch.empty(B, dtype=torch.float64, device=dev),
            "norms": torch.empty(B, 2, dtype=torch.float64, device=dev),
            "mults": torch.empty(B, dtype=torch.int32, device=dev),
            "flags": torch.empty(B, dtype=torch.uint8, device=dev)}
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    l2_flush = _make_l2_flush(flush)
    stream = torch.cuda.current_stream(dev)

    def step():
        XP.expm_lowrank_into(A1, A2, Xd, cfg.eps, plan)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    assert not plan["flags"].any(), "flagged matrices in the LR bench batch"
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        time.sleep(0.05)
        clk.mark("start")
        # (busy-wait: the SM clock stays up; ~0.5 ms per step covers the host's
        # per-call overhead)
        torch.cuda._sleep(int(2_000_000 + min(args.steps, 200) * 1_000_000))
        # one untimed step right after the hold: the first kernel after a
        # memory-idle spin runs ~2x slow (measured: C2 204 vs 80 us, C1 333 vs
        # 145 us), an artifact of the hold, not of the step
        l2_flush()
        step()
        for i in range(args.steps):
            l2_flush()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        clk.mark("end")
    tot = torch.tensor([sum(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = float(tot.item()) / args.steps
    value = ws * B / (ms_per_step * 1e-3)

    # e2e: pinned host factors in, pinned e^W + plan out, 8 chunks over 3 streams
    A1p, A2p = A1h.pin_memory(), A2h.pin_memory()
    Xp = torch.empty(B, n, n, dtype=torch.float64, pin_memory=True)
    ph = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in plan.items()}
    streams = [torch.cuda.Stream(dev) for _ in range(3)]
    bounds = [B * c // 8 for c in range(9)]

    def e2e_step():
        for c in range(8):
            a, b = bounds[c], bounds[c + 1]
            st = streams[c % 3]
            with torch.cuda.stream(st):
                A1[a:b].copy_(A1p[a:b], non_blocking=True)
                A2[a:b].copy_(A2p[a:b], non_blocking=True)
                XP.expm_lowrank_into(A1[a:b], A2[a:b], Xd[a:b], cfg.eps, {k: v[a:b] for k, v in plan.items()})
                Xp[a:b].copy_(Xd[a:b], non_blocking=True)
                for k, v in plan.items():
                    ph[k][a:b].copy_(v[a:b], non_blocking=True)
        torch.cuda.synchronize()

    for _ in range(2):
        e2e_step()
    if ws > 1:
        dist.barrier()
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    et = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_value = ws * B / (float(et.item()) / args.steps * 1e-3)
    h2d = (A1h.numel() + A2h.numel()) * 8
    d2h = Xp.numel() * 8 + sum(v.numel() * v.element_size() for v in ph.values())
    if rank == 0:
        pk = _peaks()
        hbm_bytes = B * (2 * n * t + n * n) * 8
        gbs = hbm_bytes / (ms_per_step * 1e-3) / 1e9
        ms_ = plan["m"].cpu().numpy()
        mults = plan["mults"].long().cpu().numpy()
        flops = float(B * (2 * t * t * n * 2 + 2 * n * n * t) + (mults * 2 * t ** 3).sum())
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic_LR.json")
        traffic = json.load(open(tpath)).get("dram_bytes_per_launch") if os.path.exists(tpath) else None
        roof = {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": gbs / pk["hbm_gbs"], "traffic": traffic, "peak_source": pk["hbm_src"],
                "algorithmic_bytes_per_launch": hbm_bytes, "kernel": "expm_lowrank_dmma_kernel (DMMA)",
                "other": {"bound": "fp64", "achieved": flops / (ms_per_step * 1e-3) / 1e12,
                          "peak": pk["fp64"], "peak_source": pk["fp64_src"], "unit": "TFLOP/s",
                          "useful_flops_per_launch": flops}}
        cpu = None
        if not args.no_cpu_baseline and ws == 1:  # the CPU baseline is an N=1 measurement
            r, cores, sample = cpu_lowrank_rate()
            cpu = {"value": r, "unit": "exps/s", "cores": cores, "kind": reference_impl()[0], "sample": sample}
        hist = {}
        for mm in ms_.tolist():
            hist[str(mm)] = hist.get(str(mm), 0) + 1
        line = dict(base, value=value, n_gpus=ws, ms_per_step=ms_per_step,
                    config={"workload": f"LR: {cfg.desc}", "batch_per_gpu": B, "global_batch": ws * B, "n": n,
                            "t": t, "eps": cfg.eps, "l2": "flushed between steps (252 MB write)",
                            "timing": "per-step CUDA events, host queue primed",
                            "parallelism": f"batch-sharded x{ws}, no collective on the hot path"},
                    hbm_gbs=gbs, roofline=roof, cpu_baseline=cpu,
                    e2e={"value": e2e_value, "unit": "exps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                         "ms_per_step": float(et.item()) / args.steps},
                    gpu_launches=args.steps, clocks=clk.summary(), order_histogram=hist,
                    mults_total=int(mults.sum()), rect_mults_total=3 * B)
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def _launch_count(key, m, s, n, dtype="f64"):
    """Kernels of ours launched by one expm call (host orchestration is deterministic
    and sync-free): n <= 64 one fused kernel.  n > 64 (one chunk): colsum, two
    k_select, k_bucket, elem, nonfinite, finish + one launch per product stage:
    W^2, E1..E3 and every squaring level up to the cap of 20 (levels beyond the
    batch's largest s find an empty device-side bucket and exit at once).  On
    the int8-slice path (fp32, n >= 320, n % 16 == 0) a product stage is four
    kernels (prep, route, int8 stage, FFMA GEMM for routed-away products)."""
    if n <= 64:
        return 1
    stages = 4 + 20
    per = 4 if (dtype == "f32" and n >= 320 and n % 16 == 0 and os.environ.get("EXPMB_I8", "") != "0") else 1
    return int(7 + stages * per)


def _shard_indices(cfg, rank: int, ws: int, scaling: str, batch: int = 0) -> np.ndarray:
    """Global indices of this rank's matrices.  Strong (the
    default): the config's fixed global batch split into contiguous rank-ordered
    shards (shard.shard_range; C3: disjoint time points).  Weak: every rank
    exponentiates a full batch of its own (indices rank*B ..)."""
    from paper_2512_20777_b200.shard import shard_range
    if scaling == "strong":
        lo, hi = shard_range(rank, ws, batch or cfg.batch)
        return np.arange(lo, hi)
    B = batch or cfg.batch
    idx = np.arange(rank * B, (rank + 1) * B)
    return idx % cfg.batch if cfg.key == "C3" else idx


def measure(key: str, args, steps: int, warmup: int, cpu: bool, timegrid: bool = False):
    """Device-timed and end-to-end throughput of one config on this rank's shard;
    the JSON dict on rank 0 (None elsewhere)."""
    import torch
    import torch.distributed as dist
    import paper_2512_20777_b200 as XP
    from paper_2512_20777_b200.shard import gather_to_rank0, max_over_ranks

    ws, rank, local = _dist_env()
    dev = torch.device("cuda", local)
    cfg = WL.CONFIGS[key]
    dtype = torch.float32 if cfg.dtype == "f32" else torch.float64
    esz = 4 if cfg.dtype == "f32" else 8
    idx = _shard_indices(cfg, rank, ws, args.scaling, args.batch)
    B = len(idx)
    G = B * ws if args.scaling == "weak" else (args.batch or cfg.batch)
    tg = timegrid and cfg.key == "C3"
    if tg:
        # time-grid path: inputs are A and this rank's times only
        A_h, t_all = WL.c3_factors()
        A_h, t_h = torch.from_numpy(A_h), torch.from_numpy(t_all[idx % cfg.batch])
        A_d, t_d = A_h.to(dev), t_h.to(dev)
        tg_ws = torch.empty(max(1, int(XP._lib.lib().expmb_timegrid_workspace_bytes(B, cfg.n, 0))),
                            dtype=torch.uint8, device=dev)
        Wh = None
        Xd = torch.empty(B, cfg.n, cfg.n, dtype=dtype, device=dev)
    else:
        Wh = torch.from_numpy(WL.generate(cfg.key, indices=idx))
        W = Wh.to(dev)
        Xd = torch.empty_like(W)
    plan = {"m": torch.empty(B, dtype=torch.int8, device=dev), "s": torch.empty(B, dtype=torch.int8, device=dev),
            "e1": torch.empty(B, dtype=torch.float64, device=dev), "e2": torch.empty(B, dtype=torch.float64, device=dev),
            "norms": torch.empty(B, 2, dtype=torch.float64, device=dev),
            "mults": torch.empty(B, dtype=torch.int32, device=dev),
            "nonfinite": torch.empty(B, dtype=torch.uint8, device=dev)}
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    l2_flush = _make_l2_flush(flush)
    stream = torch.cuda.current_stream(dev)

    def step():
        if tg:
            XP.expm_timegrid(A_d, t_d, cfg.eps, args.scheme, check_finite=False, out=Xd, plan=plan,
                             workspace=tg_ws)
        else:
            XP.expm_into(W, Xd, cfg.eps, args.scheme, plan)

    for _ in range(max(3, warmup)):
        step()
    torch.cuda.synchronize()
    m = plan["m"].cpu().numpy(); s = plan["s"].cpu().numpy()
    assert not plan["nonfinite"].any(), "non-finite results in the bench batch"
    if args.scheme == "baseline":  # mults = m + s (the int8 m/s outputs saturate; mults does not)
        flops = float(plan["mults"].double().sum().item()) * 2.0 * cfg.n ** 3
    else:
        flops = WL.useful_flops(m, s, cfg.n, args.scheme)

    # ---- device-timed steps, L2 flushed between steps ----------------------
    def timed(fn, k):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            time.sleep(0.05)  # let the sampler start
            clk.mark("start")
            # hold the device briefly so the host queues all K steps ahead of it:
            # the per-step events then bracket device work only (host launch cost
            # is what the e2e number below measures); busy-wait keeps the SM clock up
            torch.cuda._sleep(int(2_000_000 + min(k, 200) * 1_000_000))
            # one untimed step right after the hold: the first kernel after a
            # memory-idle spin runs ~2x slow (measured: C2 204 vs 80 us), an
            # artifact of the hold, not of the step
            l2_flush()
            fn()
            for i in range(k):
                l2_flush()
                evs[i][0].record(stream)
                fn()
                evs[i][1].record(stream)
            torch.cuda.synchronize()
            clk.mark("end")
        ms = [a.elapsed_time(b) for a, b in evs]
        tot = max_over_ranks(sum(ms), dev) if ws > 1 else sum(ms)
        return tot / k, ms, clk.summary()

    ms_per_step, step_ms, clocks = timed(step, steps)
    if os.environ.get("BENCH_STEP_TIMES"):
        print(f"{key} step ms:", " ".join(f"{x:.4f}" for x in step_ms), file=sys.stderr)
    value = G / (ms_per_step * 1e-3)

    # ---- with the final NCCL gather of e^W to rank 0 (N > 1) ---------------
    gather = None
    if ws > 1:
        def step_gather():
            step()
            gather_to_rank0(Xd, G)
        g_ms, _, _ = timed(step_gather, max(2, steps // 2))
        gather = {"value": G / (g_ms * 1e-3), "unit": "exps/s", "ms_per_step": g_ms,
                  "gather_bytes": G * cfg.n * cfg.n * esz,
                  "what": "each step + dist.gather of every rank's e^W into rank 0 (NCCL, rank order)"}

    # ---- end-to-end through the public API from pinned host memory --------
    if tg:
        Ap, tp_ = A_h.pin_memory(), t_h.pin_memory()
        Xp = torch.empty(B, cfg.n, cfg.n, dtype=dtype, pin_memory=True)
        php = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in plan.items()}

        class _TgPipe:
            h2d_bytes = Ap.numel() * Ap.element_size() + tp_.numel() * tp_.element_size()
            d2h_bytes = Xp.numel() * Xp.element_size() + sum(v.numel() * v.element_size() for v in php.values())

            def run(self, *_a, **_k):
                A_d.copy_(Ap, non_blocking=True)
                t_d.copy_(tp_, non_blocking=True)
                XP.expm_timegrid(A_d, t_d, cfg.eps, args.scheme, check_finite=False, out=Xd, plan=plan,
                                 workspace=tg_ws)
                Xp.copy_(Xd, non_blocking=True)
                for k, v in plan.items():
                    php[k].copy_(v, non_blocking=True)
        pipe = _TgPipe()
        Wp = None
    else:
        Wp = Wh.pin_memory()
        # chunked so copies overlap compute (tools/e2e_large_probe.py: C4 1056 ->
        # 1231 exps/s at 4 chunks, C3 61.6k -> 85.1k and C5 305 -> 358 at 8)
        pipe = XP.HostPipeline(B, cfg.n, dtype, chunks=8 if (cfg.n <= 64 or B >= 128) else 4, device=dev)

    def e2e_step():
        pipe.run(Wp, cfg.eps, args.scheme, check_finite=False)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e2e_ms = []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        torch.cuda.synchronize()
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_t = max_over_ranks(sum(e2e_ms), dev) / steps if ws > 1 else sum(e2e_ms) / steps
    e2e = {"value": G / (e2e_t * 1e-3), "unit": "exps/s", "h2d_bytes_per_step": pipe.h2d_bytes,
           "d2h_bytes_per_step": pipe.d2h_bytes, "ms_per_step": e2e_t}
    mults_total = int(plan["mults"].long().sum().item())
    del pipe, Wp, Xd, plan, flush
    if not tg:
        del W, Wh
    torch.cuda.empty_cache()
    if rank != 0:
        return None

    pk = _peaks()
    hbm_bytes = 2 * B * cfg.n * cfg.n * esz
    tflops = flops / (ms_per_step * 1e-3) / 1e12
    gbs = hbm_bytes / (ms_per_step * 1e-3) / 1e9
    cpeak, cpeak_name = (pk["fp32"], pk["fp32_src"]) if cfg.dtype == "f32" else (pk["fp64"], pk["fp64_src"])
    t_hbm = hbm_bytes / (pk["hbm_gbs"] * 1e9)
    t_cmp = flops / (cpeak * 1e12)
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg.key}.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("dram_bytes_per_launch")
    hbm_roof = {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": gbs / pk["hbm_gbs"], "traffic": traffic, "peak_source": pk["hbm_src"],
                "algorithmic_bytes_per_launch": hbm_bytes}
    cmp_roof = {"bound": "fp32_ffma" if cfg.dtype == "f32" else "fp64", "achieved": tflops,
                "peak": cpeak, "unit": "TFLOP/s", "frac": tflops / cpeak,
                "peak_source": f"profiles/peaks.json {cpeak_name} (tools/peaks.cu, measured on B200)",
                "useful_flops_per_launch": flops}
    # fp32 n <= 16 runs its products as 3xTF32 mma.sync (3 x 1.648e9 TC flops
    # at 266.6 TF/s = 18.5 us < the 20.5 us HBM floor): the binding roofline is
    # HBM.  Elsewhere: the larger of the two lower bounds.
    tc_products = cfg.dtype == "f32" and cfg.n <= 16 and args.scheme == "sastre"
    hbm_binds = t_hbm >= t_cmp or tc_products
    roof = dict(hbm_roof if hbm_binds else cmp_roof)
    if cfg.n <= 16:
        roof["kernel"] = ("w16::expm_w16_kernel (warp-batched, 3xTF32 mma.sync)" if tc_products and cfg.n == 16
                          else "expm_fused_kernel<float,16,...> (3xTF32 mma.sync)" if tc_products else "expm_fused_kernel")
    elif cfg.n <= 64:
        roof["kernel"] = "expm_dmma_kernel (DMMA)" if cfg.dtype == "f64" else "expm_fused_kernel"
    else:
        roof["kernel"] = "gemm_stage_kernel" + (" (DMMA)" if cfg.dtype == "f64" else " (FFMA2)")
    roof["other"] = cmp_roof if hbm_binds else hbm_roof
    if (cfg.dtype == "f32" and cfg.n >= 320 and cfg.n % 16 == 0 and os.environ.get("EXPMB_I8", "") != "0"
            and not tg):
        # products run as exact int8-slice GEMMs on tcgen05 (gemm_i8.cuh): ten
        # int8 slice-pair products per fp32 product; the FFMA peak stays the
        # useful-flop yardstick, the int8 view is reported beside it
        i8_ops = 10.0 * flops
        ffma_view = dict(roof)
        ffma_view.pop("other", None)
        ipk, isrc = pk["i8_tops"], pk["i8_src"]
        roof = {"bound": "tensor", "achieved": i8_ops / (ms_per_step * 1e-3) / 1e12, "peak": ipk,
                "unit": "TOPS", "frac": i8_ops / (ms_per_step * 1e-3) / 1e12 / ipk, "traffic": traffic,
                "traffic_note": "DRAM bytes of ONE stage launch (profiles/ncu_traffic_C5.json); a step is 24 stage "
                                "launches, per-stage bytes in profiles/stage_metrics_C5_r02.txt",
                "peak_source": isrc, "executed_int8_ops_per_launch": i8_ops,
                "kernel": "i8::k_i8_stage (persistent int8-slice tcgen05 stage, split epilogue) after i8::k_i8_prep; "
                          "gemm_stage_kernel for routed-away products",
                "other": ffma_view}
    if tg:
        # the time-grid path skips the evaluation products: its roofline is over
        # the flops it executes (squarings, shared powers in fp64, the fused
        # combination); useful_flops stays the reference's ledger
        n3 = 2.0 * cfg.n ** 3
        ex_flops = float(np.asarray(s, np.int64).sum()) * n3 + 15 * n3 + B * 16 * 2.0 * cfg.n ** 2
        ex_tf = ex_flops / (ms_per_step * 1e-3) / 1e12
        roof = {"bound": "fp32_ffma", "achieved": ex_tf, "peak": cpeak, "unit": "TFLOP/s", "frac": ex_tf / cpeak,
                "peak_source": "profiles/peaks.json (tools/peaks.cu, measured on B200)",
                "executed_flops_per_launch": ex_flops, "traffic": None,
                "kernel": "gemm_stage_kernel (FFMA2) squarings + k_tg_combine",
                "other": {"reference_ledger_flops_per_launch": flops, "ledger_tflops": tflops}}
    cpu_line = None
    if cpu and ws == 1:  # the CPU baseline is an N=1 measurement
        rates, cores, kind, sample = cpu_reference_rate(cfg.key)
        cpu_line = {"value": rates[0], "unit": "exps/s", "cores": cores, "kind": kind, "sample": sample}
    hist = {}
    for mm, ss in zip(m.tolist(), s.tolist()):
        hist[f"{mm},{ss}"] = hist.get(f"{mm},{ss}", 0) + 1
    launches = (10 + int(np.asarray(s).max())) if tg else _launch_count(cfg.key, m, s, cfg.n, cfg.dtype)
    return {
        "metric": "matrix exponentials/s", "value": value, "unit": "exps/s", "n_gpus": ws,
        "steps": steps, "warmup": max(3, warmup), "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": cfg.dtype, "data": "synthetic (seeded, SURVEY.md 8(d) recipe)",
        "config": {"workload": f"{cfg.key}: {cfg.desc}", "batch_per_gpu": B, "global_batch": G,
                   "n": cfg.n, "eps": cfg.eps, "scheme": args.scheme, "l2": "flushed between steps (252 MB write)",
                   "path": "time grid: shared powers + per-time squarings (expm_timegrid)" if tg else "batched expm",
                   "timing": "per-step CUDA events around each call, host queue primed (device held by a sleep "
                             "before the first step), max over ranks",
                   "parallelism": (f"{args.scaling} scaling: " + ("fixed global batch split into rank-ordered "
                                   "shards" if args.scaling == "strong" else "a full batch per rank")
                                   + f" x{ws}, no collective on the hot path")},
        "useful_tflops": tflops, "hbm_gbs": gbs,
        "roofline": roof,
        "cpu_baseline": cpu_line,
        "e2e": e2e,
        "e2e_gather": gather,
        "gpu_launches": launches * steps,
        "clocks": clocks,
        "plan_histogram": hist,
        "mults_total": mults_total,
    }


PER_CONFIG = {"C1": (10, 3), "C3": (5, 3), "C4": (4, 3), "C5": (3, 3)}  # (steps, warmup) of the side lines


def run_ours(args):
    import torch
    import torch.distributed as dist
    ws, rank, local = _dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    line = measure(args.config, args, args.steps, args.warmup, cpu=not args.no_cpu_baseline,
                   timegrid=bool(args.timegrid))
    if args.per_config and args.config == "C2" and not args.timegrid:
        # the other BASELINE.json configs, each measured the same way (fewer steps)
        per = {}
        for key, (k, w) in PER_CONFIG.items():
            r = measure(key, args, k, w, cpu=not args.no_cpu_baseline)
            if rank == 0:
                per[key] = {f: r[f] for f in ("value", "ms_per_step", "steps", "useful_tflops", "hbm_gbs",
                                              "roofline", "e2e", "e2e_gather", "cpu_baseline", "clocks",
                                              "gpu_launches", "plan_histogram")}
                per[key]["config"] = r["config"]["workload"]
                per[key]["global_batch"] = r["config"]["global_batch"]
        if rank == 0:
            line["per_config"] = per
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(WL.CONFIGS) + ["LR"],
                    help="C1..C5 = BASELINE.json configs; LR = the low-rank path (SURVEY 8(f) rank 2)")
    ap.add_argument("--batch", type=int, default=0, help="override batch per GPU")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--timegrid", action="store_true",
                    help="C3 through expm_timegrid (one A, many t_k: shared powers, SURVEY 8(f) rank 3)")
    ap.add_argument("--scheme", default="sastre", choices=["sastre", "ps", "baseline"],
                    help="evaluation route (baseline = Alg. 1, the paper's comparator)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's global batch split over the ranks (default); weak: a batch per rank")
    ap.add_argument("--per-config", dest="per_config", action="store_true", default=True,
                    help="with the default C2 line, also measure C1, C3, C4, C5 into 'per_config' (default)")
    ap.add_argument("--no-per-config", dest="per_config", action="store_false")
    args = ap.parse_args()
    if args.config == "LR":
        run_lowrank(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
