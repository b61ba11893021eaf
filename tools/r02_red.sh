# accumulate via L2 red.add (v4.bf16x2) instead of a register read-modify-write: parity + kbench + benches
set -x
OUT=gpurun_out/red; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "accum or full_size or kernels_match" > $OUT/pytest.txt 2>&1; echo "pytest rc=$?"
tail -5 $OUT/pytest.txt
timeout 900 python -m pytest tests/test_api_gpu.py -q -x -m gpu > $OUT/pytest_api.txt 2>&1; echo "pytest api rc=$?"
tail -5 $OUT/pytest_api.txt
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-multi > $OUT/bench_c2.json 2> $OUT/bench_c2.err
python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-multi > $OUT/bench_c4.json 2> $OUT/bench_c4.err
for c in c2 c4; do python -c "import json;d=json.load(open('$OUT/bench_$c.json'));k=d['per_kernel'];b=d['step_breakdown']['parts'];print('$c', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], 'unf', round(d['unfused_torch']['speedup'],3), 'roof', round(d['roofline']['frac'],3), {n:round(v['ms_per_step'],4) for n,v in k.items()}); [print('   %8.4f %s' % (v['ms_per_step'], n)) for n,v in b.items()]"; done
