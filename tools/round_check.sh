sed -i 's/--p 0.1 --bits --iters 1/--p 0 --iters 1/' tools/wide_ab.sh
SHAPES="8192 14336 4096:16384 8192 8192:16384 28672 8192" 
for shape in "8192 14336 4096" "16384 8192 8192" "16384 28672 8192"; do
  set -- $shape
  for w in 0 1; do
    LF_WIDE=$w timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:lf_gemm -s 3 -c 1 --csv python tools/kbench.py --m $1 --k $2 --n $3 --p 0 --iters 1 --only grad_input 2>/dev/null | python tools/ncu_csv.py "p0 grad_input m=$1 k=$2 n=$3 wide=$w"
  done
done
timeout 800 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 400 python bench.py --no-e2e --no-cpu-baseline --steps 20 | python -c "
import sys,json
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']
print('c2 ms %.3f unf %.3f'%(d['ms_per_step'], d['unfused_torch']['speedup']), {k:round(v['ms_per_step'],3) for k,v in r['per_kernel'].items()}, d['clocks']['sm_mhz'], 'c3', round(d['multi_lora']['ms_per_step'],3), round(d['multi_lora']['unfused_torch']['speedup'],3))"
timeout 400 python bench.py --config c4 --no-multi --no-e2e --no-cpu-baseline --steps 10 | python -c "
import sys,json
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']
print('c4 ms %.3f unf %.3f'%(d['ms_per_step'], d['unfused_torch']['speedup']), {k:round(v['ms_per_step'],3) for k,v in r['per_kernel'].items()}, d['clocks']['sm_mhz'])"
