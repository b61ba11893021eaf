# CTA-pair clusters (LF_CL=2) vs two pairs sharing B by TMA multicast (LF_CL=4):
# parity under each forced schedule, then per-GEMM time A/B and ncu L2/DRAM traffic.
set -x
for sched in 1 2; do
  LF_CL=4 LF_SCHED=$sched timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k \
    "test_kernels_match_oracle or test_module_api or test_shared_adapter or test_max_segments or test_microbatch_beyond or test_frozen" 2>&1 | tail -3
  LF_CL=4 LF_SCHED=$sched LF_WIDE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k \
    "test_kernels_match_oracle or test_module_api or test_max_segments" 2>&1 | tail -3
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "full_size" 2>&1 | tail -3
for shape in ${SHAPES:-"16384 8192 28672" "16384 28672 8192" "16384 8192 8192" "8192 4096 14336" "8192 14336 4096" "8192 4096 4096"}; do
  set -- $shape
  for cl in 2 4; do
    LF_CL=$cl timeout 300 python tools/kbench.py --m $1 --k $2 --n $3 --p 0.1 --bits --iters 20 --rounds 2 --graph --only base_fwd,grad_input 2>&1 | tail -2 | sed "s/^/cl=$cl /"
  done
done
for shape in "16384 8192 28672" "8192 14336 4096"; do
  set -- $shape
  for cl in 2 4; do
    LF_CL=$cl timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sectors.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:lf_gemm -s 2 -c 2 --csv python tools/kbench.py --m $1 --k $2 --n $3 --p 0.1 --bits --iters 1 --only base_fwd,grad_input 2>/dev/null | python -c "
import sys,csv
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; mi=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit'); ki=h.index('Kernel Name')
for r in rows[1:]: print('cl=$cl m=$1 k=$2 n=$3', r[ki][:40], r[mi], r[vi], r[ui])"
  done
done
