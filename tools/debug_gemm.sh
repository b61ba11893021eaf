#!/bin/bash
# LF_DEBUG sweep of the masked dX GEMM (timings only)
for f in 0 192 2048; do
  LF_DEBUG=$f python tools/kbench.py --m 8192 --k 4096 --n 4096 --p 0.1 --bits --only grad_input \
    | python -c "import sys,json; print('masked LF_DEBUG=$f', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
  LF_DEBUG=$f python tools/kbench.py --m 8192 --k 4096 --n 4096 --p 0 --only grad_input \
    | python -c "import sys,json; print('plain  LF_DEBUG=$f', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
done
