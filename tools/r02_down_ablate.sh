# ① ablations (LF_DEBUG): 4096 = fixed keep pattern instead of Philox, 8192 = no shared-memory
# mask pass, 1 = no MMA, 2 = no partial-sum flush; p = 0 = no mask warps at all
for r in 1 2; do
for shp in "8192 4096" "8192 14336"; do
  set -- $shp
  for d in ${DBGS:-0 4096 8192 12288 1 2}; do
    LF_DEBUG=$d python tools/kbench.py --m $1 --k $2 --n 4096 --bits --graph --iters 20 --only dropout_down_fwd | python -c "
import sys,json
d=json.loads(sys.stdin.readline()); print('dbg=$d', d['m'], d['k'], d['us'])"
  done
  python tools/kbench.py --m $1 --k $2 --n 4096 --p 0.0 --graph --iters 20 --only dropout_down_fwd | python -c "
import sys,json
d=json.loads(sys.stdin.readline()); print('p=0', d['m'], d['k'], d['us'])"
done
done
