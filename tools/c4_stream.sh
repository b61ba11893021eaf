#!/bin/bash
# ①③④ (and the Philox floor) at the C4 shapes, GPU time via graph capture
for shp in "16384 8192 8192" "16384 8192 1024" "16384 8192 28672" "16384 28672 8192" "2048 8192 28672" "2048 28672 8192"; do set -- $shp
  timeout 200 python tools/kbench.py --graph --m $1 --k $2 --n $3 --p 0.1 --bits --iters 20 --only dropout_down_fwd,keep_bits,grad_up,grad_down,torch_copy_x \
    | python -c "import sys,json; print('m=$1 k=$2 n=$3', ' '.join(f\"{d['kernel']}={d['us']}/{d['gbs']}\" for d in map(json.loads, sys.stdin)))"
done
