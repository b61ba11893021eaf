# ① variants: parity of the last build listed, then kbench (graphed) per shape interleaved
# across builds.   usage: r02_down_ab.sh a.so b.so ...
LIBS="$@"; LAST=${@: -1}
OUT=gpurun_out/dab; mkdir -p $OUT
LF_LIB=$LAST timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "kernels_match or explicit or bit_exact or packed or keep_bits or golden or module_api" > $OUT/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.txt
for r in 1 2; do
for shp in "8192 4096" "8192 14336" "16384 8192" "16384 28672"; do
  set -- $shp
  for L in $LIBS; do
    LF_LIB=$L python tools/kbench.py --m $1 --k $2 --n 4096 --bits --graph --iters 20 --only dropout_down_fwd 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$L'.split('/')[-1], d['kernel'], d['m'], d['k'], d['us'])"
  done
done
done | tee $OUT/kbench.txt
