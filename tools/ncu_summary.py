"""Summarise an `ncu --set full` report: per launch, the time, SM clock, tensor-pipe activity,
DRAM and L2 traffic, and the pipe/memory throughputs (JSON on stdout).

    python tools/ncu_summary.py gpurun_out/gemm_final.ncu-rep > profiles/r01_gemm_ncu_summary.json
"""
from __future__ import annotations

import csv
import json
import subprocess
import sys

METRICS = {
    "dur_us": ("gpu__time_duration.sum", {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", {"Ghz": 1, "GHz": 1, "Mhz": 1e-3, "MHz": 1e-3}),
    # the tensor-pipe utilisation (B200_PROFILING.md): cycles the tcgen05 pipe is busy over elapsed cycles
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", {}),
    # kept for reference only: the TPC triage section's realtime counter (reads ~half of the
    # above on the 2-CTA MMAs — it is not the utilisation figure)
    "tpc_triage_tensor_realtime_pct": ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", {}),
    "mem_tensor_active_pct": ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", {}),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", {}),
    "dram_throughput_pct": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", {}),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", {}),
    "dram_read_bytes": ("dram__bytes_read.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
    "dram_write_bytes": ("dram__bytes_write.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
    "l2_sectors": ("lts__t_sectors.sum", {}),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", {}),
    "registers": ("launch__registers_per_thread", {}),
    "grid": ("launch__grid_size", {}),
}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in rows[2:]:
        d = {"kernel": r[idx["Kernel Name"]].split("(")[0].replace("void ", "")}
        for key, (metric, scale) in METRICS.items():
            if metric not in idx:
                continue
            raw = r[idx[metric]].replace(",", "")
            try:
                v = float(raw)
            except ValueError:
                continue
            d[key] = v * scale.get(units[idx[metric]], 1.0) if scale else v
        res.append(d)
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
