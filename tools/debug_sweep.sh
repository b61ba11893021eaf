#!/bin/bash
# LF_DEBUG bit sweep over the memory-bound kernels (timings only; results are invalid with flags set)
for f in 0 1 2 4 8 12 16 33 35 51; do
  for a in "--p 0.1 --bits"; do
    LF_DEBUG=$f python tools/kbench.py --m 8192 --k 4096 --n 4096 $a --only dropout_down_fwd,grad_up,grad_down \
      | python -c "import sys,json; print('LF_DEBUG=$f', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
  done
done
