#!/bin/bash
# end-of-round measurement set: bench lines for C1/C2(+C3)/C4/C5 and the reference arm, the ncu
# launch list of the headline command, full-set captures of one C2 step's GEMMs and streaming kernels
set -x
timeout 900 python bench.py > gpurun_out/final_c2.log 2>&1
timeout 600 python bench.py --config c1 > gpurun_out/final_c1.log 2>&1
timeout 900 python bench.py --config c4 > gpurun_out/final_c4.log 2>&1
timeout 1200 python bench.py --config c5 > gpurun_out/final_c5.log 2>&1
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-multi --no-graph > gpurun_out/launches_final.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lf_gemm -c 14 -o gpurun_out/gemm_step python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-multi --no-graph > gpurun_out/gemm_step.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:lf_down|lf_gradup|lf_dgrad_a|lf_finalize' -c 4 -o gpurun_out/lowrank_final python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-multi --no-graph > gpurun_out/lowrank_final.log 2>&1
ls -la gpurun_out/
