#!/bin/bash
# A/B of library variants built into _variants/*.so (same sources, different -D flags):
#   LF_EXTRA_NVCC="-D..." python -m paper_2510_00206_b200.build --force; cp the .so to _variants/<name>.so
# SHAPES: ';'-separated "m k n r" tuples
LIB=paper_2510_00206_b200/liblorafusion_b200.so
cp $LIB /tmp/lib_orig.so
IFS=';' read -ra SH <<< "${SHAPES:-1024 4096 1024 16;8192 4096 1024 16;8192 4096 4096 16;8192 4096 14336 16}"
for v in _variants/*.so; do
  cp $v $LIB
  for shp in "${SH[@]}"; do
    read -r m k n r <<< "$shp"
    timeout 120 python tools/kbench.py ${KB_ARGS} --m $m --k $k --n $n --r ${r:-16} --p 0.1 --bits --iters 50 --only ${ONLY:-dropout_down_fwd,grad_up,grad_down,grad_input,base_fwd} \
      | python -c "import sys,json; print('$v m=$m k=$k n=$n r=${r:-16}', ' '.join(f\"{d['kernel']}={d['us']}\" for d in map(json.loads, sys.stdin)))"
  done
done
cp /tmp/lib_orig.so $LIB
