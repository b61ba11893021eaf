# ncu --set full (with source) of ① lf_down_kernel and the bare keep-bit generator at the C2 q shape;
# exported on the box (raw metrics, SASS source page with per-instruction stall samples)
OUT=gpurun_out/down; mkdir -p $OUT
ncu --set full --import-source on --clock-control none -k regex:lf_down_kernel -s 2 -c 1 -o $OUT/down \
  python tools/kbench.py --m 8192 --k 4096 --n 4096 --p 0.1 --bits --iters 1 --only dropout_down_fwd > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:lf_keep_bits -s 2 -c 1 -o $OUT/keepbits \
  python tools/kbench.py --m 8192 --k 4096 --n 4096 --p 0.1 --bits --iters 1 --only keep_bits > /dev/null 2>&1
for K in down keepbits; do
  ncu -i $OUT/$K.ncu-rep --page raw --csv > $OUT/${K}_raw.csv
  ncu -i $OUT/$K.ncu-rep --page source --csv --print-source sass > $OUT/${K}_sass.csv 2>&1
  ncu -i $OUT/$K.ncu-rep --page details --csv > $OUT/${K}_details.csv 2>&1
done
ls -la $OUT
