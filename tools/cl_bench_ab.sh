# cluster occupancy by cluster size, then whole-step A/B of the multicast GEMM (LF_CL) on one box
./tools/cluster_occupancy
for i in 1 2; do
for cl in 2 4; do
  LF_CL=$cl python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-multi > gpurun_out/r02_clab_c2_cl$cl.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r02_clab_c2_cl$cl.json'));k=d['per_kernel'];print('c2 cl=$cl', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {n:round(v['ms_per_step'],3) for n,v in k.items()})"
done
done
for cl in 2 4; do
  LF_CL=$cl python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_clab_c4_cl$cl.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r02_clab_c4_cl$cl.json'));k=d['per_kernel'];print('c4 cl=$cl', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['unfused_torch']['speedup'],3), {n:round(v['ms_per_step'],3) for n,v in k.items()})"
done
