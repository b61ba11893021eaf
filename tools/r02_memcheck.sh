# compute-sanitizer memcheck (and racecheck on ①'s shared-memory keep-bit ring) over the group
# tests, the parity matrix, the multi-adapter dB block copies and the capturable graphs
OUT=gpurun_out/memcheck; mkdir -p $OUT
{
echo "# compute-sanitizer --tool memcheck / racecheck (round 2 HEAD)"
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_api_gpu.py -q -x -m gpu -k "group or copy_column or capturable" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|out of bounds" | head
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "kernels_match and (c1 or multi4 or single)" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|out of bounds" | head
compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "kernels_match and c1 and packed" 2>&1 | grep -E "passed|failed|RACECHECK SUMMARY|ERROR SUMMARY|hazard" | head
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_graphs.py -q -x -m gpu 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|out of bounds" | head
} > $OUT/memcheck.txt 2>&1
cat $OUT/memcheck.txt
