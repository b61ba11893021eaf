# ④ with packed keep bits: which part of the mask path costs (LF_DEBUG knobs, results invalid)
#   4 = skip fence.proxy.async, 8 = skip the smem apply, 64 = stages bypass the mask warps
for dbg in 0 4 8 12 64; do
  LF_DEBUG=$dbg timeout 120 python tools/kbench.py --m 16384 --k 4096 --n 4096 --p 0.1 --bits --iters 30 --only grad_down,dropout_down_fwd | python -c "
import sys,json
print('debug=$dbg', ' '.join('%s=%.1fus'%(d['kernel'],d['us']) for d in map(json.loads,sys.stdin)))"
done
