#!/bin/bash
# GEMM raster group sweep (LF_GROUP) at the C2 shapes
for shape in "4096 4096" "4096 14336" "14336 4096"; do
  set -- $shape
  for g in ${GS:-4 8 16 32}; do
    LF_GROUP=$g python tools/kbench.py --m 8192 --k $1 --n $2 --p 0.1 --bits --only base_fwd,grad_input --iters 20 \
      | python -c "import sys,json; print('G=$g k=$1 n=$2', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
  done
done
