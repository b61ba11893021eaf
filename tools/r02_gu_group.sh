# ③ group launch: parity (group tests), then interleaved A/B (LF_GROUP_UP=0|1) on C2 and C3, per-launch ncu
timeout 900 python -m pytest tests/test_api_gpu.py tests/test_gpu_parity.py tests/test_decoder.py -q -x -m gpu 2>&1 | tail -3
bash tools/ab.sh "LF_GROUP_UP=0" "LF_GROUP_UP=1" 3 2>&1 | tail -2
bash tools/ab.sh "LF_GROUP_UP=0" "LF_GROUP_UP=1" 2 "--config c3 --steps 10 --warmup 3" 2>&1 | tail -2
LF_GROUP_UP=1 bash tools/r02_launches.sh c2 _gu1 | grep -v gemm | head -16
