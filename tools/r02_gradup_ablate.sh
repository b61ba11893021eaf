# ③ ablations (LF_DEBUG): 1 = no dŜ MMA, 32 = no dB MMA, 2 = no partial-sum / dB flush;
# beside torch's read-only reduction of a same-size tensor (the streaming floor)
for r in 1 2; do
for shp in "8192 4096 4096" "8192 14336 4096" "8192 4096 14336"; do
  set -- $shp
  for d in 0 1 32 33 2 35; do
    LF_DEBUG=$d python tools/kbench.py --m $1 --n $2 --k $3 --bits --graph --iters 20 --only grad_up | python -c "
import sys,json
d=json.loads(sys.stdin.readline()); print('dbg=$d', d['m'], d['n'], d['us'], d.get('gbs'))"
  done
done
python tools/kbench.py --m 8192 --k 4096 --n 4096 --graph --iters 20 --only torch_sum_x,torch_copy_x | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print(d['kernel'], d['m'], d['k'], d['us'], d.get('gbs'))"
python tools/kbench.py --m 8192 --k 14336 --n 4096 --graph --iters 20 --only torch_sum_x | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print(d['kernel'], d['m'], d['k'], d['us'], d.get('gbs'))"
done
