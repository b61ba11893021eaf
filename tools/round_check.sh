timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 120 python tools/host_overhead.py
timeout 300 python bench.py --config c1 --steps 30 --no-multi --no-e2e --no-cpu-baseline 2>&1 | python -c "
import sys,json
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']
print('c1 ms %.3f'%d['ms_per_step'], 'unf x%.3f'%d['unfused_torch']['speedup'], {k:round(v['ms_per_step'],3) for k,v in r['per_kernel'].items()})"
