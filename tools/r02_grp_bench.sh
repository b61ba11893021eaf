# group GEMM variants vs per-projection launches (graphed, interleaved); schedule A/B
for s in 0 1 2; do echo "LF_SCHED=$s"; LF_SCHED=$s python tools/grp_bench.py --m 8192 --k 4096 --ns 4096,1024,1024 --p 0.1 --rounds 3; done
for s in 0 1; do echo "LF_SCHED=$s"; LF_SCHED=$s python tools/grp_bench.py --m 8192 --k 4096 --ns 4096,1024,1024 --p 0.0 --rounds 2; done
