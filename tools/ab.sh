# Interleaved whole-step A/B on one box: ab.sh "<args A>" "<args B>" [rounds] [extra bench args]
# prints each run and the median ms/step per variant (box-to-box spread is +-5%; in-box ~1%)
A="$1"; B="$2"; N=${3:-3}; EXTRA="$4"
for i in $(seq $N); do
  for v in A B; do
    args=$([ $v = A ] && echo "$A" || echo "$B")
    env $args python bench.py $EXTRA --no-cpu-baseline --no-e2e --no-multi > gpurun_out/ab_$v$i.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_$v$i.json'));print('$v', '$args', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], {n:round(x['ms_per_step'],3) for n,x in d['per_kernel'].items()})"
  done
done
python - <<PY
import json, statistics
for v, a in (("A", "$A"), ("B", "$B")):
    ms = [json.load(open(f"gpurun_out/ab_{v}{i}.json"))["ms_per_step"] for i in range(1, $N + 1)]
    print("median", v, a, round(statistics.median(ms), 4), [round(x, 3) for x in ms])
PY
