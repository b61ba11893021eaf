#!/bin/bash
# LF_DEBUG ablations of ③/④ (GPU time via graph capture; results invalid with flags set)
for shp in "8192 4096" "32768 1024" "16384 4096"; do set -- $shp
for f in 0 2 16 18 1 32 33 51; do
  LF_DEBUG=$f timeout 120 python tools/kbench.py --graph --m $1 --k 4096 --n $2 --p 0.1 --bits --iters 50 --only grad_up,grad_down \
    | python -c "import sys,json; print('m=$1 n=$2 LF_DEBUG=$f', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
done; done
