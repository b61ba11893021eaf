# shared-input groups: API/parity tests, then bench A/B (--group vs --no-group) on C2 and C4
timeout 900 python -m pytest tests/test_api_gpu.py tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -4
for cfg in c2 c4; do
  st=10; [ $cfg = c4 ] && st=5
  for grp in --no-group --group; do
    python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-multi $grp > gpurun_out/r02_grp_${cfg}${grp}.json 2>gpurun_out/r02_grp_${cfg}${grp}.err
    python -c "import json;d=json.load(open('gpurun_out/r02_grp_${cfg}${grp}.json'));k=d['per_kernel'];print('$cfg $grp', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], 'unf', round(d['unfused_torch']['speedup'],3), round(d['unfused_torch']['speedup_vs_graph'] or 0,3), 'e2e', round(d['e2e']['ms_per_step'],2), {n:round(v['ms_per_step'],3) for n,v in k.items()})" || tail -5 gpurun_out/r02_grp_${cfg}${grp}.err
  done
done
