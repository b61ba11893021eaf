# ① (lf_down_kernel) beside the bare keep-bit generator: full ncu set with source, summarised on the box
OUT=gpurun_out/dncu; mkdir -p $OUT
ncu --set full --import-source on --clock-control none -k regex:"lf_down" -s 3 -c 1 -o $OUT/d \
  python tools/kbench.py --m 8192 --k 4096 --n 4096 --bits --iters 1 --only dropout_down_fwd,keep_bits > /dev/null 2>&1
python tools/ncu_summary.py $OUT/d.ncu-rep > $OUT/summary.json
ncu -i $OUT/d.ncu-rep --page raw --csv > $OUT/raw.csv 2>&1
ncu -i $OUT/d.ncu-rep --page source --csv --print-source sass -k regex:lf_down > $OUT/down_sass.csv 2>&1
ncu -i $OUT/d.ncu-rep --page source --csv --print-source sass -k regex:lf_keep > $OUT/keep_sass.csv 2>&1
rm -f $OUT/*.ncu-rep
cat $OUT/summary.json
