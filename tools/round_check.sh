timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -3
for c in c1 c2; do for g in --graph --no-graph; do timeout 300 python bench.py --config $c $g --steps 20 --no-multi --no-e2e --no-cpu-baseline 2>&1 | python -c "
import sys,json
ls=[l for l in sys.stdin if l.startswith('{')]
if not ls: print('$c $g FAILED'); sys.exit()
d=json.loads(ls[-1]); r=d['roofline']
print('$c $g ms %.3f'%d['ms_per_step'], 'unf x%.3f'%d['unfused_torch']['speedup'], 'launches', d['gpu_launches'], d['clocks']['sm_mhz'], {k:round(v['ms_per_step'],3) for k,v in r['per_kernel'].items()})"; done; done
