#!/usr/bin/env python
"""Benchmark: batched matrix exponentials/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One "step" = one call of the hot path (expm over the whole batch of the
config).  Default workload: BASELINE.json configs[1] = C2 (65536 x 16x16 fp32
skew-symmetric, tol 2^-24).  Under torchrun (N > 1) every rank exponentiates
its own batch (global indices rank*B .. rank*B+B-1; weak scaling, no
collective on the data path); the step time is the max over ranks.

Printed JSON line (rank 0):
  value       whole-job exps/s with inputs resident in HBM (device-timed)
  e2e         exps/s through the public API from pinned host memory, H2D of W
              and D2H of e^W + plan inside the timed region
  roofline    dominant kernel vs its bound (HBM bytes and useful FLOPs)
  cpu_baseline the CPU oracle port timed on this host (bounded sample)
`--impl reference` times the reference algorithm's CPU port (oracle/) instead.
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
CPU_SAMPLE = {"C1": 1024, "C2": 16384, "C3": 48, "C4": 6, "C5": 3}


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
# CPU side (the oracle port of the reference algorithm) -- rank 0 only
# ---------------------------------------------------------------------------

def _cpu_worker_init():
    # one BLAS thread per worker process (the pool supplies the parallelism;
    # forked workers inherit the parent's already-initialised BLAS pool)
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _cpu_chunk(args):
    W, eps = args
    from oracle import expm_oracle as O
    for i in range(W.shape[0]):
        O.expm(W[i], eps)
    return W.shape[0]


def cpu_reference_rate(key: str, count: int | None = None, cores: int | None = None):
    """exps/s of the reference algorithm (oracle port, binary64 as the reference)
    on `count` matrices of config `key`, sharded over a process pool the way
    the reference's own harness shards (bench.py:303-306)."""
    from concurrent.futures import ProcessPoolExecutor
    cfg = WL.CONFIGS[key]
    count = count or CPU_SAMPLE[key]
    cores = cores or os.cpu_count() or 1
    W = WL.generate(key, indices=np.arange(count)).astype(np.float64)
    if cfg.n >= 256:
        # large orders: one process, BLAS threads on every core (BASELINE.md mode 1)
        t0 = time.perf_counter()
        done = _cpu_chunk((W, cfg.eps))
        dt = time.perf_counter() - t0
        mode = "serial expm loop, multithreaded BLAS"
    else:
        # small orders: process pool, one BLAS thread each (reference bench.py:303-306; mode 2)
        pieces = np.array_split(W, max(1, min(count, cores * 4)))
        with ProcessPoolExecutor(max_workers=cores, initializer=_cpu_worker_init) as pool:
            list(pool.map(_cpu_chunk, [(pieces[0][:1], cfg.eps)] * min(cores, 2)))  # warm workers
            t0 = time.perf_counter()
            done = sum(pool.map(_cpu_chunk, [(p, cfg.eps) for p in pieces]))
            dt = time.perf_counter() - t0
        mode = f"process pool x{cores}, 1 BLAS thread each"
    return done / dt, cores, f"{done} matrices of {key} ({cfg.n}x{cfg.n}, fp64 as the reference computes; {mode})"


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------

def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    cfg = WL.CONFIGS[args.config]
    count = CPU_SAMPLE[args.config]
    for _ in range(args.warmup):
        cpu_reference_rate(args.config, max(1, count // 8))
    rates = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r, cores, sample = cpu_reference_rate(args.config, count)
        rates.append(r)
    wall = time.perf_counter() - t0
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": "matrix exponentials/s", "value": value, "unit": "exps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.key}: {cfg.desc}", "batch": cfg.batch, "n": cfg.n, "eps": cfg.eps,
                   "parallelism": "cpu process pool (reference bench.py:303-306)"},
        "cpu_baseline": {"value": value, "unit": "exps/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "exps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Low-rank path: --config LR
# ---------------------------------------------------------------------------

def _cpu_lr_chunk(args):
    A1, A2, eps = args
    from oracle import expm_oracle as O
    for i in range(A1.shape[0]):
        O.expm_lowrank(A1[i], A2[i], eps)
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
    return done / dt, cores, f"{done} pairs of LR (n 64, t 8, fp64; process pool x{cores}, 1 BLAS thread each)"


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
                    cpu_baseline={"value": value, "unit": "exps/s", "cores": cores, "kind": "port", "sample": sample},
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
                "algorithmic_bytes_per_launch": hbm_bytes, "kernel": "expm_lowrank_kernel<double,8>",
                "other": {"bound": "fp64_dfma", "achieved": flops / (ms_per_step * 1e-3) / 1e12,
                          "peak": pk["dfma_fp64"], "unit": "TFLOP/s", "useful_flops_per_launch": flops}}
        cpu = None
        if not args.no_cpu_baseline and ws == 1:  # the CPU baseline is an N=1 measurement
            r, cores, sample = cpu_lowrank_rate()
            cpu = {"value": r, "unit": "exps/s", "cores": cores, "kind": "port", "sample": sample}
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
    """Kernels of ours launched by one expm call (host orchestration is deterministic):
    n > 64: colsum, two k_select, elem, nonfinite, finish + one launch per product
    stage (W^2, E1..E3 as present, one per squaring level); on the int8-slice path
    (fp32, n >= 512) a product stage is five kernels (stats, route, slice,
    int8 GEMM, FFMA GEMM for routed-away products)."""
    if n <= 64:
        return 1
    m = np.asarray(m); s = np.asarray(s)
    stages = 1 + int((m >= 4).any()) + int((m >= 8).any()) + int((m >= 15).any()) + int(s.max())
    per = 5 if (dtype == "f32" and n >= 512 and n % 16 == 0 and os.environ.get("EXPMB_I8", "") != "0") else 1
    return int(6 + stages * per)


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2512_20777_b200 as XP

    ws, rank, local = _dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = WL.CONFIGS[args.config]
    B = args.batch or cfg.batch
    dtype = torch.float32 if cfg.dtype == "f32" else torch.float64
    esz = 4 if cfg.dtype == "f32" else 8
    # this rank's shard of the global batch (seeded chunks -> independent of N)
    if cfg.key == "C3":
        idx = np.arange(B) % cfg.batch
    else:
        idx = np.arange(rank * B, (rank + 1) * B)
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

    tg = bool(getattr(args, "timegrid", False)) and cfg.key == "C3"
    if tg:
        # time-grid path: inputs are A and the times only
        A_h, t_all = WL.c3_factors()
        A_h, t_h = torch.from_numpy(A_h), torch.from_numpy(t_all[idx])
        A_d, t_d = A_h.to(dev), t_h.to(dev)
        tg_ws = torch.empty(max(1, int(XP._lib.lib().expmb_timegrid_workspace_bytes(B, cfg.n, 0))),
                            dtype=torch.uint8, device=dev)
        del W

    def step():
        if tg:
            XP.expm_timegrid(A_d, t_d, cfg.eps, args.scheme, check_finite=False, out=Xd, plan=plan,
                             workspace=tg_ws)
        else:
            XP.expm_into(W, Xd, cfg.eps, args.scheme, plan)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    m = plan["m"].cpu().numpy(); s = plan["s"].cpu().numpy()
    assert not plan["nonfinite"].any(), "non-finite results in the bench batch"
    if args.scheme == "baseline":  # mults = m + s (the int8 m/s outputs saturate; mults does not)
        flops = float(plan["mults"].double().sum().item()) * 2.0 * cfg.n ** 3
    else:
        flops = WL.useful_flops(m, s, cfg.n, args.scheme)

    # ---- device-timed steps, L2 flushed between steps ----------------------
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        time.sleep(0.05)  # let the sampler start
        clk.mark("start")
        # hold the device briefly so the host queues all K steps ahead of it:
        # the per-step events then bracket device work only (host launch cost
        # is what the e2e number below measures)
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
    step_ms = [a.elapsed_time(b) for a, b in evs]
    if os.environ.get("BENCH_STEP_TIMES"):
        print("step ms:", " ".join(f"{x:.4f}" for x in step_ms), file=sys.stderr)
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot.item())
    ms_per_step = total_ms / args.steps
    value = ws * B / (ms_per_step * 1e-3)

    # ---- end-to-end through the public API from pinned host memory --------
    # HostPipeline: H2D of W, expm, D2H of e^W + plan, chunked over 3 streams
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
        # chunked so copies overlap compute (measured on B200, tools/e2e_large_probe.py:
        # C4 1056 -> 1231 exps/s at 4 chunks, C3 61.6k -> 85.1k and C5 305 -> 358 at 8)
        pipe = XP.HostPipeline(B, cfg.n, dtype, chunks=8 if (cfg.n <= 64 or B >= 128) else 4, device=dev)

    def e2e_step():
        pipe.run(Wp, cfg.eps, args.scheme, check_finite=False)

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
        torch.cuda.synchronize()
        e2e_ms.append(1e3 * (time.perf_counter() - t0))
    et = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_value = ws * B / (float(et.item()) / args.steps * 1e-3)
    h2d = pipe.h2d_bytes
    d2h = pipe.d2h_bytes

    gather_ms = None
    if ws > 1:
        # the final rank-ordered gather of results to rank 0 (reported, not in the step)
        from paper_2512_20777_b200.shard import gather_to_rank0
        dist.barrier()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        full = gather_to_rank0(Xd, ws * B)
        g1.record(stream)
        torch.cuda.synchronize()
        from paper_2512_20777_b200.shard import max_over_ranks
        gather_ms = max_over_ranks(g0.elapsed_time(g1), dev)
        del full

    if rank == 0:
        pk = _peaks()
        hbm_bytes = 2 * B * cfg.n * cfg.n * esz
        tflops = flops / (ms_per_step * 1e-3) / 1e12
        gbs = hbm_bytes / (ms_per_step * 1e-3) / 1e9
        cpeak = pk["ffma_fp32"] if cfg.dtype == "f32" else pk["dfma_fp64"]
        t_hbm = hbm_bytes / (pk["hbm_gbs"] * 1e9)
        t_cmp = flops / (cpeak * 1e12)
        traffic = None
        tp = os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg.key}.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        hbm_roof = {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": gbs / pk["hbm_gbs"], "traffic": traffic, "peak_source": pk["hbm_src"],
                    "algorithmic_bytes_per_launch": hbm_bytes}
        cmp_roof = {"bound": "fp32_ffma" if cfg.dtype == "f32" else "fp64_dfma", "achieved": tflops,
                    "peak": cpeak, "unit": "TFLOP/s", "frac": tflops / cpeak,
                    "peak_source": "profiles/peaks.json (tools/peaks.cu, measured on B200)",
                    "useful_flops_per_launch": flops}
        # fp32 n <= 16 runs its products as 3xTF32 mma.sync (3 x 1.648e9 TC flops
        # at 266.6 TF/s = 18.5 us < the 20.5 us HBM floor): the binding
        # roofline is HBM.  Elsewhere: the larger of the two lower bounds.
        tc_products = cfg.dtype == "f32" and cfg.n <= 16 and args.scheme == "sastre"
        hbm_binds = t_hbm >= t_cmp or tc_products
        roof = dict(hbm_roof if hbm_binds else cmp_roof)
        if cfg.n <= 16:
            roof["kernel"] = "expm_fused_kernel<float,16,2,8,0,2,2> (3xTF32 mma.sync)" if tc_products else "expm_fused_kernel"
        elif cfg.n <= 64:
            roof["kernel"] = "expm_dmma_kernel (DMMA)" if cfg.dtype == "f64" else "expm_fused_kernel"
        else:
            roof["kernel"] = "gemm_stage_kernel" + (" (DMMA)" if cfg.dtype == "f64" else " (FFMA2)")
        roof["other"] = cmp_roof if hbm_binds else hbm_roof
        if cfg.dtype == "f32" and cfg.n >= 512 and cfg.n % 16 == 0 and os.environ.get("EXPMB_I8", "") != "0":
            # products run as exact int8-slice GEMMs on tcgen05 (gemm_i8.cuh): ten
            # int8 slice-pair products per fp32 product; the FFMA peak stays the
            # useful-flop yardstick, the int8 view is reported beside it
            i8_ops = 10.0 * flops
            ffma_view = dict(roof)
            ffma_view.pop("other", None)
            roof = {"bound": "tensor", "achieved": i8_ops / (ms_per_step * 1e-3) / 1e12, "peak": 4500.0,
                    "unit": "TOPS", "frac": i8_ops / (ms_per_step * 1e-3) / 1e12 / 4500.0, "traffic": None,
                    "peak_source": "nominal dense int8 (no measured int8 peak on this pool)",
                    "executed_int8_ops_per_launch": i8_ops,
                    "kernel": "i8::k_i8_stage (int8-slice tcgen05) + gemm_stage_kernel for routed-away products",
                    "other": ffma_view}
        if tg:
            # the time-grid path skips the evaluation products: its roofline is
            # over the flops it executes (squarings, shared powers in fp64, the
            # fused combination); useful_flops stays the reference's ledger
            n3 = 2.0 * cfg.n ** 3
            ex_flops = float(np.asarray(s, np.int64).sum()) * n3 + 15 * n3 + B * 16 * 2.0 * cfg.n ** 2
            ex_tf = ex_flops / (ms_per_step * 1e-3) / 1e12
            roof = {"bound": "fp32_ffma", "achieved": ex_tf, "peak": cpeak, "unit": "TFLOP/s", "frac": ex_tf / cpeak,
                    "peak_source": "profiles/peaks.json (tools/peaks.cu, measured on B200)",
                    "executed_flops_per_launch": ex_flops, "traffic": None,
                    "kernel": "gemm_stage_kernel (FFMA2) squarings + k_tg_combine",
                    "other": {"reference_ledger_flops_per_launch": flops, "ledger_tflops": tflops}}
        cpu = None
        if not args.no_cpu_baseline and ws == 1:  # the CPU baseline is an N=1 measurement
            r, cores, sample = cpu_reference_rate(cfg.key)
            cpu = {"value": r, "unit": "exps/s", "cores": cores, "kind": "port", "sample": sample}
        hist = {}
        for mm, ss in zip(m.tolist(), s.tolist()):
            hist[f"{mm},{ss}"] = hist.get(f"{mm},{ss}", 0) + 1
        line = {
            "metric": "matrix exponentials/s", "value": value, "unit": "exps/s", "n_gpus": ws,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": cfg.dtype, "data": "synthetic (seeded, SURVEY.md 8(d) recipe)",
            "config": {"workload": f"{cfg.key}: {cfg.desc}", "batch_per_gpu": B, "global_batch": ws * B,
                       "n": cfg.n, "eps": cfg.eps, "scheme": args.scheme, "l2": "flushed between steps (252 MB write)",
                       "path": "time grid: shared powers + per-time squarings (expm_timegrid)" if tg else "batched expm",
                       "timing": "per-step CUDA events around each call, host queue primed (device held by a sleep before the first step)",
                       "parallelism": f"batch-sharded x{ws}, no collective on the hot path"},
            "useful_tflops": tflops, "hbm_gbs": gbs,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "exps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": float(et.item()) / args.steps},
            "gpu_launches": (10 + int(np.asarray(s).max()) if tg else _launch_count(cfg.key, m, s, cfg.n, cfg.dtype)) * args.steps,
            "clocks": clk.summary(),
            "plan_histogram": hist,
            "mults_total": int(plan["mults"].long().sum().item()),
            "gather_ms": gather_ms,
        }
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
                    help="evaluation route (baseline = Alg. 1, the paper's comparator; n <= 64)")
    args = ap.parse_args()
    if args.config == "LR":
        run_lowrank(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
