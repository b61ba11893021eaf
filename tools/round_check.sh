export LF_BENCH_SHARE_GPU=1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_n2.log 2>&1; echo n2=$?
tail -c 600 gpurun_out/bench_n2.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 3 --warmup 3 --impl reference > gpurun_out/bench_n2_ref.log 2>&1; echo n2ref=$?
tail -c 300 gpurun_out/bench_n2_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --config c5 --layers 2 --mb-per-rank 1 --steps 2 --warmup 3 > gpurun_out/bench_n2_c5.log 2>&1; echo n2c5=$?
tail -c 400 gpurun_out/bench_n2_c5.log
