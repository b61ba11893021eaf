#!/bin/bash
# per-kernel timings at the C2 projection shapes (q, gate/up, down)
./tools/tma_stream 2>&1 | tail -2
for shape in "4096 4096" "4096 14336" "14336 4096" "4096 1024"; do
  set -- $shape
  python tools/kbench.py --m 8192 --k $1 --n $2 --p 0.1 --bits --iters 40 | python -c "import sys,json; print('k=$1 n=$2', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
done
