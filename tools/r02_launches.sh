# ncu launch list (gpu__time_duration per kernel) of one graphed bench step, summarised per launch
# usage: r02_launches.sh CONFIG [TAG] (environment variables pass through)
CFG=${1:-c2}; TAG=${2:-}
OUT=gpurun_out/launch_$CFG$TAG; mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-multi > /dev/null 2>&1
python - $OUT/launches.csv $CFG <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]; idx = {h: i for i, h in enumerate(hdr)}
out = [(r[idx["Kernel Name"]][:60], float(r[idx["Metric Value"]].replace(",", ""))) for r in rows[hi + 1:] if len(r) >= len(hdr)]
# one step = from the last lf_routes_kernel on (each step starts with the routing table)
starts = [i for i, (n, _) in enumerate(out) if "lf_routes_kernel" in n]
step = out[starts[-2]:starts[-1]] if len(starts) >= 2 else out[-60:]
tot = {}
for n, v in step:
    key = n.split("(")[0].replace("void ", "")
    tot[key] = tot.get(key, 0) + v
    if "gemm" in n:
        print(f"{v/1000:9.1f} us  {n}")
print("step total (serialised) %.3f ms" % (sum(v for _, v in step) / 1e6))
for k_, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {v/1e6:8.4f} ms  {k_}")
PY
