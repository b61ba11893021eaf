# GPU parity suite + a short default bench (round 2 iteration loop)
set -x
python -m pytest tests -q -m gpu -x --timeout 1500 "$@" > gpurun_out/r02_pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r02_pytest_gpu.txt
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r02_bench_c2.json
