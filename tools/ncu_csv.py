"""Summarise an `ncu --csv --metrics ...` launch list (stdin): one line per launch with
duration (µs) and DRAM bytes (GB), units normalised from ncu's 'Metric Unit' column."""
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "second": 1e6,
         "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}

rows = [r for r in csv.reader(sys.stdin) if len(r) > 10]
if not rows:
    sys.exit(0)
hdr = rows[0]
ki, mi, vi, ui, ii = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
launches: dict = {}
for r in rows[1:]:
    d = launches.setdefault(r[ii], {"kernel": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for d in launches.values():
    name = d["kernel"].split("(")[0].replace("void ", "")[-24:]
    us = d.get("gpu__time_duration.sum")
    gb = d.get("dram__bytes_read.sum")
    print(f"{tag} {name} {us:.1f}us" + (f" read {gb:.2f}GB" if gb is not None else ""))
