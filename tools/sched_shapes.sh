# static vs CLC-dynamic GEMM schedule per shape (ncu serialized launch times + DRAM reads)
for shape in "8192 4096 4096" "8192 4096 1024" "8192 4096 14336" "8192 14336 4096" "16384 8192 8192" "16384 8192 1024" "16384 8192 28672" "16384 28672 8192" "2048 4096 4096"; do
  set -- $shape
  for s in 0 1; do
    LF_SCHED=$((s+1)) timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:"lf_gemm" -c 4 --csv python tools/kbench.py --m $1 --k $2 --n $3 --p 0.1 --bits --iters 1 --only base_fwd,grad_input 2>/dev/null | python tools/ncu_csv.py "m=$1 k=$2 n=$3 sched=$((s+1))"
  done
done
