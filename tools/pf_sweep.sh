#!/bin/bash
# L2-prefetch distance sweep for the streaming kernels (LF_PF_UNITS)
ONLY=${ONLY:-grad_down}; K=${K:-4096}; N=${N:-4096}
for pf in ${PFS:-0 2 4 8 16}; do
  LF_PF_UNITS=$pf python tools/kbench.py --m 8192 --k $K --n $N --p 0.1 --bits --only $ONLY --iters 40 \
    | python -c "import sys,json; print('PF=$pf k=$K n=$N', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
done
