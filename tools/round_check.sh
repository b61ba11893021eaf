timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 500 python bench.py > gpurun_out/bench_c2.log 2>&1; echo c2=$?
timeout 500 python bench.py --config c4 --steps 20 --no-multi > gpurun_out/bench_c4.log 2>&1; echo c4=$?
timeout 900 python bench.py --config c5 --steps 4 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
