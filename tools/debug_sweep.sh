#!/bin/bash
# LF_DEBUG bit sweep over the memory-bound kernels (timings only; results are invalid with flags set)
FLAGS=${FLAGS:-"0 1 2 4 8 12 16 33 35 51"}
ONLY=${ONLY:-dropout_down_fwd,grad_up,grad_down}
K=${K:-4096}; N=${N:-4096}
for f in $FLAGS; do
  LF_DEBUG=$f python tools/kbench.py --m 8192 --k $K --n $N --p 0.1 --bits --only $ONLY --iters 40 \
    | python -c "import sys,json; print('LF_DEBUG=$f', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
done
