#!/bin/bash
# LF_DEBUG sweep of the masked dX GEMM (timings only); args: k n
K=${1:-4096}; N=${2:-4096}
for f in 0 2048 192; do
  LF_DEBUG=$f python tools/kbench.py --m 8192 --k $K --n $N --p 0.1 --bits --only grad_input,cublas_dgrad --iters 30 \
    | python -c "import sys,json; print('masked LF_DEBUG=$f', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
done
for f in 0 2048; do
  LF_DEBUG=$f python tools/kbench.py --m 8192 --k $K --n $N --p 0 --only grad_input --iters 30 \
    | python -c "import sys,json; print('plain  LF_DEBUG=$f', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
done
