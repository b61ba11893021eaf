# DRAM traffic / L2 hit rate of the q/k/v group dgrad: masked (p = 0.1) vs unmasked (p = 0), both schedules
M=dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.sum
for cfg in "LF_SCHED=0" "LF_SCHED=1"; do
for p in 0.1 0.0; do
  env $cfg ncu --metrics $M --clock-control none -k regex:lf_gemm -s 1 -c 1 --csv \
    python tools/grp_bench.py --m 8192 --k 4096 --ns 4096,1024,1024 --p $p --only dgrad_group --iters 1 --rounds 1 2>/dev/null \
    | python -c "
import sys,csv
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; iv=h.index('Metric Name'); iu=h.index('Metric Value'); ik=h.index('Kernel Name')
print('$cfg p=$p', rows[1][ik][:40], {r[iv]: r[iu] for r in rows[1:]})"
done
done
