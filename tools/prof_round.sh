set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:lf_gemm -c 14 -o gpurun_out/gemm_step python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/gemm_step.log 2>&1
ncu --set full --import-source on --clock-control none -k 'regex:lf_down|lf_gradup|lf_dgrad_a' -c 3 -o gpurun_out/lowrank_step python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/lowrank_step.log 2>&1
ls -la gpurun_out/
