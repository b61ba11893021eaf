# fixed cost vs bandwidth of the streaming kernels: time at m = 4k..32k (k = n = 4096)
for m in 4096 8192 16384 32768; do
  timeout 200 python tools/kbench.py --m $m --k 4096 --n 4096 --p 0.1 --bits --iters 30 --only dropout_down_fwd,grad_up,grad_down,torch_sum_x,torch_copy_x | python -c "
import sys,json
print('m=$m', ' '.join('%s=%.1fus(%.0fGB/s)'%(d['kernel'],d['us'],d['gbs']) for d in map(json.loads,sys.stdin)))"
done
for m in 4096 8192 16384 32768; do
  timeout 200 python tools/kbench.py --m $m --k 4096 --n 4096 --p 0.0 --iters 30 --only dropout_down_fwd,grad_down | python -c "
import sys,json
print('p0 m=$m', ' '.join('%s=%.1fus(%.0fGB/s)'%(d['kernel'],d['us'],d['gbs']) for d in map(json.loads,sys.stdin)))"
done
