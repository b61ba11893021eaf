# C4 gate-shape GEMM: DRAM traffic and time vs raster group / persistence (ncu + CUDA events)
K=${1:-8192}; N=${2:-28672}; M=${3:-16384}
for cfg in "LF_GROUP=8" "LF_GROUP=4" "LF_GROUP=16" "LF_NONPERSIST=1" "LF_NONPERSIST=1 LF_GROUP=4"; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/kbench.py --m $M --k $K --n $N --p 0.1 --bits --iters 10 --rounds 2 --power --only base_fwd,cublas_fwd,grad_input,cublas_dgrad | cut -c1-200
  env $cfg timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:"lf_gemm|nvjet" -c 4 python tools/kbench.py --m $M --k $K --n $N --p 0.1 --bits --iters 1 --only base_fwd,grad_input,cublas_fwd 2>&1 | grep -E "^  [a-z]|dram__|gpu__time" | cut -c1-90
done
