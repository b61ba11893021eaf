# FusedMultiLoRAGroup in C3 (bench grouping) and C5 (decoder): interleaved --no-group vs group
for i in 1 2; do
  for g in --no-group ""; do
    python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-multi $g > gpurun_out/c3$g$i.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/c3$g$i.json'));print('c3 $g', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['unfused_torch']['speedup'],3), {n:round(x['ms_per_step'],3) for n,x in d['per_kernel'].items()})"
  done
done
for i in 1 2; do
  for g in 0 1; do
    LF_DECODER_GROUPS=$g python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/c5_$g$i.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/c5_$g$i.json'));print('c5 groups=$g', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], round(d['unfused_torch']['speedup'],3))"
  done
done
