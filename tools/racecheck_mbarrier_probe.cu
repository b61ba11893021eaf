// Control for profiles/r02_memcheck.txt:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_00206_b200/csrc -I include \
//        tools/racecheck_mbarrier_probe.cu -o /tmp/rc && compute-sanitizer --tool racecheck /tmp/rc
// Does compute-sanitizer racecheck model mbarrier arrive/wait? warp 0 writes smem, arrives;
// warp 1 waits on the barrier phase, then reads. A correct producer/consumer hand-off.
#include <cstdint>
#include <cstdio>
#include "lf_device.cuh"
using namespace lf;
__global__ void k(uint64_t* out) {
  __shared__ uint64_t data[32 * 8];
  __shared__ uint64_t bar_full, bar_empty;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(&bar_full, 1); mbar_init(&bar_empty, 1); fence_barrier_init(); }
  __syncthreads();
  uint32_t ph = 0;
  for (int it = 0; it < 8; ++it) {
    if (warp == 0) {
      mbar_wait(&bar_empty, ph ^ 1);
      sts64(smem_u32(&data[lane]), (uint64_t)it * 100 + lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_full);
    } else {
      mbar_wait(&bar_full, ph);
      const uint64_t v = lds64(smem_u32(&data[lane]));
      out[it * 32 + lane] = v;
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_empty);
    }
    ph ^= 1;
  }
}
int main() {
  uint64_t* out;
  cudaMalloc(&out, 8 * 32 * 8);
  k<<<1, 64>>>(out);
  uint64_t h[256];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int it = 0; it < 8; ++it) for (int l = 0; l < 32; ++l) bad += h[it * 32 + l] != (uint64_t)it * 100 + l;
  printf("bad %d err %s\n", bad, cudaGetErrorString(cudaGetLastError()));
}
