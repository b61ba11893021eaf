# 256x512 (LF_WIDE=1) vs 256x256 (LF_WIDE=0) GEMM tiles: ncu serialized time, clock, DRAM, L2 sectors
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "every_case and wide" 2>&1 | tail -2
ONLY=${ONLY:-grad_input}
for shape in ${SHAPES:-"8192 4096 4096" "8192 14336 4096" "8192 4096 14336" "16384 8192 8192" "16384 8192 28672" "16384 28672 8192"}; do
  set -- $shape
  for w in 0 1; do
    LF_WIDE=$w timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sectors.sum --clock-control none -k regex:lf_gemm -s 3 -c 1 --csv python tools/kbench.py --m $1 --k $2 --n $3 --p 0.1 --bits --iters 1 --only $ONLY 2>/dev/null | python -c "
import sys,csv
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; mi=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
print('$ONLY m=$1 k=$2 n=$3 wide=$w', '  '.join(f'{r[mi].split(\".\")[0]}={r[vi]}{r[ui]}' for r in rows[1:]))"
  done
done
