"""DRAM traffic of the lf_gemm_kernel launches of one bench step, from an ncu capture.

    ncu --set full --clock-control none -k regex:lf_gemm -c 14 -o gpurun_out/gemm_step \\
        python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline
    python tools/ncu_traffic.py gpurun_out/gemm_step.ncu-rep [c2|c4] > profiles/gemm_traffic[_c4].json

The first 14 GEMM launches are one step of the config in bench.py's order (a shared-input
group's ② launches, then its ⑤ launches; single projections ② then ⑤), default c2; for c4
capture `bench.py --config c4` (the --metrics of METRICS suffice).
Algorithmic bytes per launch follow SURVEY.md §8(d): ② 2(mk+kn+mr+rn)+2mn, ⑤ 2(mn+kn+mr+kr)+2mk.
"""
from __future__ import annotations

import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]


def main():
    rep = sys.argv[1]
    config = sys.argv[2] if len(sys.argv) > 2 else "c2"
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if "lf_gemm" not in d.get("Kernel Name", ""):
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        u = dict(zip(hdr, units))
        rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale.get(u["dram__bytes_read.sum"], 1)
        wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale.get(u["dram__bytes_write.sum"], 1)
        t = float(d["gpu__time_duration.sum"].replace(",", ""))
        tu = u["gpu__time_duration.sum"]
        t_us = {"nsecond": t / 1e3, "ns": t / 1e3, "usecond": t, "us": t, "msecond": t * 1e3, "ms": t * 1e3}[tu]
        launches.append({"kernel": d["Kernel Name"][:60], "dram_read": rd, "dram_write": wr, "dur_us": t_us})
    import bench  # noqa: E402  (bench order)

    m, r = bench.tokens_per_gpu(config), 16
    shapes = {name: (k, n) for name, k, n, _ in bench.projections(config)}
    grouped = os.environ.get("LF_BENCH_GROUP", "1") != "0"
    order = []  # bench.fused_step: a shared-input group runs all forwards, then all backwards
    by_grp: dict = {}
    for name, k, n, grp in bench.projections(config):
        by_grp.setdefault(grp, []).append(name)
    # a group's ② is one launch over the concatenated outputs (lf_base_fwd_group) when every
    # width tiles; its ⑤ one launch over the concatenated reduction dims while that stays
    # <= 12288 (lf_gemm.cu gemm_launch_group), else one launch per projection
    for grp, names in by_grp.items():
        if grouped and grp in bench.SHARED_INPUT_GROUPS and len(names) > 1:
            ns = [shapes[nm][1] for nm in names]
            fwd_one = all(n_ % 256 == 0 for n_ in ns)
            bwd_one = sum(ns) <= 12288 and all(n_ % 64 == 0 for n_ in ns)
            order += [(tuple(names), "base_fwd")] if fwd_one else [((nm,), "base_fwd") for nm in names]
            order += [(tuple(names), "grad_input")] if bwd_one else [((nm,), "grad_input") for nm in names]
        else:
            for nm in names:
                order += [((nm,), "base_fwd"), ((nm,), "grad_input")]
    alg = []
    for names, kind in order:
        k = shapes[names[0]][0]
        ns = [shapes[nm][1] for nm in names]
        if kind == "base_fwd":  # X once, every W_j / Ŝ_j / B_j once, every Y_j written once
            b = 2 * m * k + sum(2 * (k * n_ + m * r + r * n_) + 2 * m * n_ for n_ in ns)
        else:  # every dY_j / W_j / dŜ_j / A_j once, dX written once
            b = sum(2 * (m * n_ + k * n_ + m * r + k * r) for n_ in ns) + 2 * m * k
        alg.append(("/".join(names) + f" {kind}", b))
    n = min(len(launches), len(alg))
    dram = sum(l["dram_read"] + l["dram_write"] for l in launches[:n])
    algb = sum(a for _, a in alg[:n])
    print(json.dumps({
        "source": os.path.basename(rep) + f" (ncu --clock-control none, one {config.upper()} bench step)",
        "launches": n,
        "dram_bytes_per_launch": dram / n if n else None,
        "algorithmic_bytes_per_launch": algb / n if n else None,
        "dram_over_algorithmic": dram / algb if algb else None,
        "per_launch": [dict(l, algorithmic=a[1], launcher=a[0]) for l, a in zip(launches[:n], alg[:n])],
    }, indent=1))


if __name__ == "__main__":
    main()
