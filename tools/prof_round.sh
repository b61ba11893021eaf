# round profile: headline bench line, ncu launch list of the same command, ncu --set full of the
# top kernel (one ② launch) and of the streaming kernels (①③④ of the q projection)
set -x
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-multi --no-graph > gpurun_out/launches_final.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lf_gemm -s 14 -c 2 -o gpurun_out/gemm_final python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-multi --no-graph > gpurun_out/gemm_final.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:lf_down|lf_gradup|lf_dgrad_a' -s 21 -c 3 -o gpurun_out/lowrank_final python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-multi --no-graph > gpurun_out/lowrank_final.log 2>&1
ls -la gpurun_out/ | tail -5
