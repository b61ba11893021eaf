# raster group G x schedule for the long-K GEMMs (ncu serialized launch time + DRAM reads)
for shape in "16384 28672 8192" "16384 8192 28672" "8192 14336 4096"; do
  set -- $shape
  for cfg in "LF_SCHED=2 LF_GROUP=2" "LF_SCHED=2 LF_GROUP=4" "LF_SCHED=2 LF_GROUP=8" "LF_SCHED=2 LF_GROUP=16" "LF_SCHED=2 LF_GROUP=32"; do
    env $cfg timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:"lf_gemm" -s 2 -c 2 --csv python tools/kbench.py --m $1 --k $2 --n $3 --p 0.1 --bits --iters 1 --only base_fwd 2>/dev/null | python tools/ncu_csv.py "m=$1 k=$2 n=$3 $cfg"
  done
done
