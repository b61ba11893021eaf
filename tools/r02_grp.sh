# group GEMMs (N-concat ②, K-concat ⑤): parity, then whole-step A/B vs the per-projection path
set -x
OUT=gpurun_out/grp; mkdir -p $OUT
timeout 900 python -m pytest tests/test_api_gpu.py tests/test_gpu_parity.py -q -x -m gpu > $OUT/pytest.txt 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest.txt
bash tools/ab.sh "LF_GROUP_GEMM=0" "LF_GROUP_GEMM=1" 3
bash tools/ab.sh "LF_GROUP_GEMM=0" "LF_GROUP_GEMM=1" 2 "--config c4 --steps 5 --warmup 3"
