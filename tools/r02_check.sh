# GPU parity suite, then one C2 bench line with its step breakdown
timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-multi > gpurun_out/r02_bd_c2.json 2>gpurun_out/r02_bd_c2.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r02_bd_c2.json"))
b = d["step_breakdown"]
print("ms_per_step", round(d["ms_per_step"], 4), "span", round(b["span_ms_per_step"], 4), "clk", d["clocks"]["sm_mhz"],
      "unfused x", round(d["unfused_torch"]["speedup"], 3), "e2e ms", round(d["e2e"]["ms_per_step"], 2))
for k, v in b["parts"].items():
    print(f'{v["ms_per_step"]:8.4f} {v.get("kernels_per_step", "")!s:5} {k}')
PY
