#!/bin/bash
# A/B of library variants built into _variants/*.so (same sources, different -D flags)
LIB=paper_2510_00206_b200/liblorafusion_b200.so
cp $LIB /tmp/lib_orig.so
for v in _variants/*.so; do
  cp $v $LIB
  for shp in "1024 4096 1024" "8192 4096 1024" "8192 4096 4096" "8192 4096 14336"; do set -- $shp
    timeout 120 python tools/kbench.py --m $1 --k $2 --n $3 --p 0.1 --bits --iters 50 --only ${ONLY:-dropout_down_fwd,grad_up,grad_down,grad_input,base_fwd} \
      | python -c "import sys,json; print('$v m=$1 k=$2 n=$3', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
  done
done
cp /tmp/lib_orig.so $LIB
