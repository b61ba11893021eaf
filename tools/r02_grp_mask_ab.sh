# masked q/k/v group dgrad (C2): where partial j of the next tile goes in (LF_DEBUG 256 / 512 /
# 1024 = after / a quarter / three quarters into the main loop; default half-way), x schedule
for rnd in 1 2; do
for cfg in "LF_DEBUG=0" "LF_DEBUG=512" "LF_DEBUG=1024" "LF_DEBUG=256" "LF_SCHED=1" "LF_SCHED=1 LF_DEBUG=512"; do
  env $cfg python tools/grp_bench.py --m 8192 --k 4096 --ns 4096,1024,1024 --p 0.1 --only dgrad_group --rounds 1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$cfg', d['variant'], d['us'])"
done
done
