#!/usr/bin/env python
"""Summarise an ncu --set full report into the text committed under profiles/.

usage: python tools/ncu_summary.py report.ncu-rep kernel_substring out.txt [note] [units_per_launch]

units_per_launch (e.g. matrices per launch) adds warp instructions per unit.
"""
import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    vals = rows[2]
    return hdr, units, vals


def main():
    rep, ksub, outp = sys.argv[1:4]
    note = sys.argv[4] if len(sys.argv) > 4 else ""
    n_units = float(sys.argv[5]) if len(sys.argv) > 5 else 0.0
    hdr, units, vals = raw(rep)
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    lines = [f"# ncu --set full summary: {os.path.basename(rep)}", f"kernel: {d.get('Kernel Name', '?')}", note, ""]
    for k in KEYS:
        if k in d:
            lines.append(f"{k:70s} {d[k]:>16s} {u.get(k, '')}")
    if n_units > 0 and "smsp__inst_executed.sum" in d:
        lines.append(f"{'warp instructions per unit':70s} {float(d['smsp__inst_executed.sum'].replace(',', '')) / n_units:16.1f}")
    stalls = [(k, d[k]) for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    stalls = sorted(stalls, key=lambda kv: -float(kv[1].replace(",", "") or 0))
    tot = sum(float(v.replace(",", "") or 0) for _, v in stalls) or 1
    lines.append("")
    lines.append("warp stall samples (share):")
    for k, v in stalls[:10]:
        lines.append(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * float(v) / tot:5.1f}%")
    try:
        import ncu_lines as NL
        import contextlib
        buf = io.StringIO()
        sys.argv = ["ncu_lines", rep, ksub, "15"]
        with contextlib.redirect_stdout(buf):
            NL.main()
        lines.append("")
        lines.append("instructions / stall samples by source line:")
        lines.extend("  " + x for x in buf.getvalue().splitlines())
    except Exception as ex:  # pragma: no cover
        lines.append(f"(line attribution unavailable: {ex})")
    open(outp, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
