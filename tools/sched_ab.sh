# dynamic (CLC) vs static persistent tile schedule: parity suite, then DRAM traffic + time
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
K=${1:-8192}; N=${2:-28672}; M=${3:-16384}
for cfg in "LF_SCHED=2" "LF_SCHED=1"; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/kbench.py --m $M --k $K --n $N --p 0.1 --bits --iters 10 --rounds 2 --power --only base_fwd,cublas_fwd,grad_input,cublas_dgrad | cut -c1-200
  env $cfg timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:"lf_gemm|nvjet" -c 3 python tools/kbench.py --m $M --k $K --n $N --p 0.1 --bits --iters 1 --only base_fwd,grad_input,cublas_fwd 2>&1 | grep -E "^  [a-z]|dram__|gpu__time" | cut -c1-90
done
