"""Modeled vs measured DRAM traffic per fused kernel.

For each LLaMa-3.1-8B projection shape (m = 8192, r = 16, p = 0.1) every launcher runs
under ncu (one warm launch, --clock-control none) and its dram__bytes_read/write are set
next to the reference's analytic model (lorasched costmodel ``fused_lora``, mirrored
byte-for-byte by paper_2510_00206_b200.costmodel) and this design's ``b200_built``.

    python tools/traffic_report.py [--out profiles/r01_traffic_report]    # on the GPU box
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [("q/o", 4096, 4096), ("k/v", 4096, 1024), ("gate/up", 4096, 14336), ("down", 14336, 4096)]
# launcher -> (kbench name, ncu kernel regex, model kernel name, pass)
LAUNCHERS = [
    ("①", "dropout_down_fwd", "lf_down_kernel", "dropout_down_proj_fused", "forward"),
    ("②", "base_fwd", "lf_gemm", "base_gemm_epilogue_fused", "forward"),
    ("③", "grad_up", "lf_gradup_kernel|lf_finalize_kernel", "grad_up_fused", "backward"),
    ("④", "grad_down", "lf_dgrad_a_kernel", "grad_down_fused", "backward"),
    ("⑤", "grad_input", "lf_gemm", "grad_base_accum_fused", "backward"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
         "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def measure(m, k, n, only, regex):
    """(read B, written B, µs) of the last launch group of `only` (ncu, serialized)."""
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "--csv", "-k", f"regex:{regex}",
           sys.executable, os.path.join(ROOT, "tools", "kbench.py"), "--m", str(m), "--k", str(k), "--n", str(n),
           "--p", "0.1", "--bits", "--iters", "1", "--only", only]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600).stdout
    rows = [r for r in csv.reader(out.splitlines()) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    launches: dict = {}
    for r in rows[1:]:
        d = launches.setdefault(int(r[ii]), {"kernel": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    seq = [launches[i] for i in sorted(launches)]
    # ③ is two kernels (main + split-K finalize): the last launch of each name
    last = {}
    for d in seq:
        last[d["kernel"].split("(")[0]] = d
    rd = sum(d["dram__bytes_read.sum"] for d in last.values())
    wr = sum(d["dram__bytes_write.sum"] for d in last.values())
    us = sum(d["gpu__time_duration.sum"] for d in last.values())
    return rd, wr, us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "traffic_report"))
    args = ap.parse_args()
    from paper_2510_00206_b200 import costmodel as cm

    m, r = 8192, 16
    rows = []
    for label, k, n in SHAPES:
        shape = cm.GemmShape(m, k, n, r, 2)
        for sym, only, regex, model_name, ps in LAUNCHERS:
            ref = {x.kernel: x for x in cm.traffic(shape, ps, "fused_lora").kernels}[model_name]
            built = {x.kernel: x for x in cm.traffic(shape, ps, "b200_built").kernels}[model_name]
            rd, wr, us = measure(m, k, n, only, regex)
            rows.append({"shape": label, "k": k, "n": n, "kernel": f"{sym} {model_name}", "dram_read": rd,
                         "dram_write": wr, "us": us, "model_b200_built": built.total_bytes,
                         "model_ref_fused_lora": ref.total_bytes})
            print(json.dumps(rows[-1]), flush=True)
    with open(args.out + ".json", "w") as f:
        json.dump(rows, f, indent=1)
    lines = ["# DRAM traffic per fused kernel: ncu measured vs modeled (m = 8192, r = 16, p = 0.1)", "",
             "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, one warm launch per",
             "launcher through the C ABI (tools/kbench.py); `ref fused_lora` = the reference's analytic model",
             "(lorasched costmodel, ls/costmodel.py:250-277, mirrored byte-exactly), `b200_built` = this design.", "",
             "| shape | kernel | measured MB | model b200_built MB | measured / built | ref fused_lora MB | µs |",
             "|---|---|---|---|---|---|---|"]
    for r_ in rows:
        meas = r_["dram_read"] + r_["dram_write"]
        lines.append(f"| {r_['shape']} | {r_['kernel']} | {meas / 1e6:.1f} | {r_['model_b200_built'] / 1e6:.1f} | "
                     f"{meas / r_['model_b200_built']:.2f} | {r_['model_ref_fused_lora'] / 1e6:.1f} | {r_['us']:.1f} |")
    tot_m = sum(r_["dram_read"] + r_["dram_write"] for r_ in rows)
    tot_b = sum(r_["model_b200_built"] for r_ in rows)
    tot_r = sum(r_["model_ref_fused_lora"] for r_ in rows)
    lines += ["", f"All shapes: measured {tot_m / 1e9:.2f} GB, b200_built model {tot_b / 1e9:.2f} GB "
                  f"({tot_m / tot_b:.2f}x), reference fused_lora model {tot_r / 1e9:.2f} GB "
                  f"(measured / ref model = {tot_m / tot_r:.2f})."]
    with open(args.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
