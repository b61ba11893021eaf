# C3 step's raw kernel list (LF_BREAKDOWN_NAMES) and an ncu capture of the split ① at the q shape
OUT=gpurun_out/c3list; mkdir -p $OUT
LF_BREAKDOWN_NAMES=1 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c3.json 2> $OUT/c3.err
grep "\[breakdown\]" $OUT/c3.err > $OUT/c3_kernels.txt
ncu --set full --clock-control none -k regex:lf_down -s 3 -c 1 -o $OUT/down \
  python tools/kbench.py --m 8192 --k 4096 --n 4096 --bits --iters 1 --only dropout_down_fwd > /dev/null 2>&1
python tools/ncu_summary.py $OUT/down.ncu-rep > $OUT/down_split_ncu.json
ncu -i $OUT/down.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h,u,r=rows[0],rows[1],rows[2]
keep=('sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
      'smsp__issue_active.avg.pct_of_peak_sustained_active','sm__issue_active.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.pct_of_peak_sustained_active')
for i,x in enumerate(h):
    if x in keep or x.startswith('smsp__average_warps_issue_stalled') and 'per_issue_active' in x:
        try:
            if float(r[i].replace(',',''))>0.3: print(x, r[i])
        except ValueError: pass
" > $OUT/down_split_pipes.txt
rm -f $OUT/*.ncu-rep
cat $OUT/c3_kernels.txt | head -30; cat $OUT/down_split_ncu.json; cat $OUT/down_split_pipes.txt
