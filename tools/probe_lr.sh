set -x
for shp in "4096 4096" "4096 1024" "4096 14336" "14336 4096"; do set -- $shp
  timeout 120 python tools/kbench.py --m 8192 --k $1 --n $2 --p 0.1 --bits --iters 50 --only dropout_down_fwd,keep_bits,grad_up,grad_down,torch_copy_x >> gpurun_out/lr_probe.txt 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/kbench.py --m 8192 --k $1 --n $2 --p 0.1 --bits --iters 3 --only dropout_down_fwd,grad_up,grad_down > gpurun_out/lr_ncu_$1_$2.csv 2>&1
done
