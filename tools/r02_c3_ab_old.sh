# C3 whole step, interleaved on one box: the tree before the round-2 C3 work (_old = commit 682ed7e,
# a git worktree built in place) vs HEAD
for i in 1 2 3; do
  (cd _old && python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-multi 2>/dev/null) | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('old', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['unfused_torch']['speedup'])"
  python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-multi 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('head', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['unfused_torch']['speedup'])"
done
