#!/usr/bin/env python
"""Summarise an ncu --set full report (raw page) into the handful of numbers
the roofline needs.  Usage: ncu_summary.py report.ncu-rep [more.ncu-rep ...]"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__grid_size",
    "launch__block_size",
    "lts__t_bytes.sum",
    "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[rows[0].index("Kernel Name")][:80] if "Kernel Name" in rows[0] else "?"}
        for k in KEYS:
            if k in rows[0]:
                i = rows[0].index(k)
                rec[k] = f"{r[i]} {rows[1][i]}".strip()
        # any tensor-pipe metric, whatever its exact name on this ncu
        for i, name in enumerate(rows[0]):
            if "pipe_tensor" in name and "pct" in name and name not in rec:
                rec[name] = f"{r[i]} {rows[1][i]}".strip()
        out.append(rec)
    return out


if __name__ == "__main__":
    res = {p: summarize(p) for p in sys.argv[1:]}
    print(json.dumps(res, indent=1))
