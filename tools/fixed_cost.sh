#!/bin/bash
# GPU-side fixed vs marginal cost of the streaming kernels (timed loop captured as one CUDA
# graph: no per-call host cost): m sweep at the k/v and q shapes
for n in 1024 4096; do
for m in 128 1024 4096 8192 16384 32768; do
  timeout 120 python tools/kbench.py --graph --m $m --k 4096 --n $n --p 0.1 --bits --iters 50 --only ${ONLY:-dropout_down_fwd,keep_bits,grad_up,grad_down,torch_copy_x} \
    | python -c "import sys,json; print('n=$n m=$m', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
done; done
