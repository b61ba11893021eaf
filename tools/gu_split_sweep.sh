#!/bin/bash
# ③ n-split sweep (LF_GU_NSPLIT forces it; 0 = launcher heuristic), GPU time via graph capture
# SHAPES: ';'-separated "m k n r"
IFS=';' read -ra SH <<< "${SHAPES:-16384 8192 28672 16;8192 4096 14336 16;8192 4096 4096 16;16384 8192 8192 16;16384 28672 8192 16}"
for shp in "${SH[@]}"; do read -r m k n r <<< "$shp"
for ns in ${NS:-0 4 8 9 14 16 28 32 56 112 224}; do
  LF_GU_NSPLIT=$ns timeout 120 python tools/kbench.py --graph --m $m --k $k --n $n --r ${r:-16} --p 0.1 --bits --iters 20 --only grad_up \
    | python -c "import sys,json; print('m=$m k=$k n=$n r=${r:-16} ns=$ns', ' '.join(f\"{d['kernel']}={d['us']} {d['gbs']}GB/s\" for d in map(json.loads, sys.stdin)))"
done; done
