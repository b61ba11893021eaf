# ncu full set with source of the masked q/k/v group dgrad (C2) and the q-alone masked dgrad, summarised on the box
OUT=gpurun_out/gncu; mkdir -p $OUT
ncu --set full --import-source on --clock-control none -k regex:lf_gemm -s 2 -c 1 -o $OUT/grp \
  python tools/grp_bench.py --m 8192 --k 4096 --ns 4096,1024,1024 --p 0.1 --only dgrad_group --iters 1 --rounds 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:lf_gemm -s 3 -c 1 -o $OUT/q \
  python tools/kbench.py --m 8192 --k 4096 --n 4096 --bits --iters 1 --only grad_input > /dev/null 2>&1
for K in grp q; do
  python tools/ncu_summary.py $OUT/$K.ncu-rep > $OUT/${K}_summary.json
  ncu -i $OUT/$K.ncu-rep --page source --csv --print-source sass > $OUT/${K}_sass.csv 2>&1
done
rm -f $OUT/*.ncu-rep
cat $OUT/grp_summary.json $OUT/q_summary.json
