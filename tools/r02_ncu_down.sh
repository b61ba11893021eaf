# ncu --set full (with source) of ① lf_down_kernel and the bare keep-bit generator at the C2 q shape
ncu --set full --import-source on --clock-control none -k regex:lf_down_kernel -s 2 -c 1 -o gpurun_out/r02_down \
  python tools/kbench.py --m 8192 --k 4096 --n 4096 --p 0.1 --bits --iters 1 --only dropout_down_fwd > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:lf_keep_bits -s 1 -c 1 -o gpurun_out/r02_keepbits \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-multi > /dev/null 2>&1
ls -la gpurun_out/r02_down.ncu-rep gpurun_out/r02_keepbits.ncu-rep
