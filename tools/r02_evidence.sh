# Round-2 evidence on one box: GPU suite, bench lines for every config + the reference arm,
# the ncu launch list of the headline command, GEMM / streaming-kernel ncu captures.
set -x
OUT=gpurun_out/ev; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4 > $OUT/pytest_gpu.txt
python bench.py --steps 20 --warmup 5 > $OUT/bench_c2.json 2> $OUT/bench_c2.err
python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c1.json 2> $OUT/bench_c1.err
python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
python bench.py --config c4 --steps 6 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
python bench.py --config c5 --steps 4 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err
python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-multi > /dev/null 2>&1
ncu --set full --clock-control none -k regex:lf_gemm -c 9 -o $OUT/gemm_step \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-multi --no-graph > /dev/null 2>&1
ncu --set full --clock-control none -k "regex:lf_(down|gradup|finalize|dgrad_a)" -c 24 -o $OUT/lowrank_step \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-multi --no-graph > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:lf_gemm -c 9 -o $OUT/gemm_step_c4 \
  python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:lf_gemm -c 2 -o $OUT/gemm_step_c1 \
  python bench.py --config c1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
# summarise on the box (the .ncu-rep files exceed gpurun's 64 MiB copy-back)
python tools/ncu_summary.py $OUT/gemm_step.ncu-rep > $OUT/gemm_ncu_summary.json
python tools/ncu_summary.py $OUT/lowrank_step.ncu-rep > $OUT/lowrank_ncu_summary.json
python tools/ncu_traffic.py $OUT/gemm_step.ncu-rep c2 > $OUT/gemm_traffic.json
python tools/ncu_traffic.py $OUT/gemm_step_c4.ncu-rep c4 > $OUT/gemm_traffic_c4.json
python tools/ncu_traffic.py $OUT/gemm_step_c1.ncu-rep c1 > $OUT/gemm_traffic_c1.json
rm -f $OUT/*.ncu-rep
ls -la $OUT
