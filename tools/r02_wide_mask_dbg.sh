# where the wide masked dgrad's time goes (C4 q and down shapes): full / no TMEM mask pass (64) /
# no LoRA at all (2048) / unmasked p = 0 — kbench graphed, two rounds
for shp in "16384 8192 8192" "16384 28672 8192"; do
  set -- $shp
  for r in 1 2; do
    for dbg in 0 64 2048; do
      LF_DEBUG=$dbg python tools/kbench.py --m $1 --k $2 --n $3 --bits --graph --iters 5 --only grad_input 2>&1 | tail -1 | sed "s/^/dbg=$dbg /"
    done
    python tools/kbench.py --m $1 --k $2 --n $3 --p 0 --graph --iters 5 --only grad_input 2>&1 | tail -1 | sed "s/^/p=0 /"
    python tools/kbench.py --m $1 --k $2 --n $3 --graph --iters 5 --only base_fwd 2>&1 | tail -1 | sed "s/^/fwd /"
  done
done
