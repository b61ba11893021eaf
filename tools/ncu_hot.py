"""Top stall-sampled SASS instructions of one kernel in an ncu report (read here, no GPU)."""
import csv, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = None, []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
f = lambda x: float(x) if x not in ("", None) else 0.0
tot = sum(f(r[i_s]) for r in data)
print("total samples", tot, "instructions", len(data))
for i in sorted(range(len(data)), key=lambda i: -f(data[i][i_s]))[:n]:
    print(f"{f(data[i][i_s]):6.0f}  {data[i][0][-5:]}  {data[i][1][:70]:70s} <- {data[i-1][1][:50]}")
