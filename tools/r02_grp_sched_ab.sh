# masked / unmasked q/k/v group dgrad (C2 shapes) under tile-schedule and raster overrides
OUT=gpurun_out/gsched; mkdir -p $OUT
for rnd in 1 2; do
for cfg in "LF_SCHED=0" "LF_SCHED=1" "LF_SCHED=2" "LF_GROUP=4" "LF_GROUP=16" "LF_SCHED=1 LF_GROUP=16"; do
  for p in 0.1 0.0; do
    echo "== $cfg p=$p" >> $OUT/ab.txt
    env $cfg python tools/grp_bench.py --m 8192 --k 4096 --ns 4096,1024,1024 --p $p --only dgrad_group,dgrad_separate --rounds 1 >> $OUT/ab.txt 2>&1
  done
done
done
cat $OUT/ab.txt
