// Standalone throughput of Philox4x32-10 on sm_100a, with no TMA / MMA pipeline around it:
//   pure      — the bare 10-round generator (4 words per call)
//   masks     — ①'s philox_masks<CH> (Philox -> SWAR keep test -> bf16 lane masks + packed
//               bits), the per-row state (philox_row) hoisted out of the loop as in ①
//   masks_row — the same with philox_row recomputed per call group (the generator kernel's shape)
// at 2 / 4 / 8 / 16 warps per SMSP. Prints µs per 8192 x 4096 mask (the C2 q projection).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2510_00206_b200/csrc \
//        tools/philox_bench.cu -o /tmp/philox_bench && /tmp/philox_bench
#include <cstdio>

#include "lf_device.cuh"

using namespace lf;

template <int MODE, int CH>
__global__ void __launch_bounds__(256) bench(LfSegDev seg, int rows, int cols, uint32_t* sink) {
  uint32_t acc = 0;
  const int groups_per_row = cols / (8 * CH);  // a power of two: row / group by shift and mask
  const int lg = __ffs(groups_per_row) - 1;
  const int total = rows * groups_per_row;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  PhiloxRow pr = philox_row(seg, (uint32_t)t);
  for (int i = t; i < total; i += gridDim.x * blockDim.x) {
    const int row = i >> lg, cg = i & (groups_per_row - 1);
    if constexpr (MODE == 0) {
      uint32_t c0[CH], c1[CH], c2[CH], c3[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) { c0[j] = cg * CH + j; c1[j] = row; c2[j] = pr.c2; c3[j] = pr.c3; }
#pragma unroll
      for (int r = 0; r < 10; ++r)
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const uint64_t p0 = (uint64_t)0xD2511F53u * c0[j];
          const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2[j];
          const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1[j] ^ pr.k0[r];
          const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3[j] ^ pr.k1[r];
          c1[j] = (uint32_t)p1; c3[j] = (uint32_t)p0; c0[j] = n0; c2[j] = n2;
        }
#pragma unroll
      for (int j = 0; j < CH; ++j) acc ^= c0[j] ^ c1[j] ^ c2[j] ^ c3[j];
    } else {
      if constexpr (MODE == 2) pr = philox_row(seg, (uint32_t)row);
      else pr.c1 = (uint32_t)row;
      uint32_t msk[CH][4];
      const uint64_t bits = philox_masks<CH>(pr, cg * 8 * CH, msk);
#pragma unroll
      for (int j = 0; j < CH; ++j) acc ^= msk[j][0] ^ msk[j][1] ^ msk[j][2] ^ msk[j][3];
      acc += (uint32_t)bits ^ (uint32_t)(bits >> 32);
    }
  }
  sink[t] = acc;  // observable: no dead-code elimination
}

template <int MODE, int CH>
float run(int rows, int cols, int blocks) {
  LfSegDev s{};
  s.thr = 2 * 3276;
  s.key0 = 1234;
  uint32_t* sink;
  cudaMalloc(&sink, (size_t)blocks * 256 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 20; ++w) bench<MODE, CH><<<blocks, 256>>>(s, rows, cols, sink);  // clocks up
  cudaEventRecord(a);
  const int it = 20;
  for (int w = 0; w < it; ++w) bench<MODE, CH><<<blocks, 256>>>(s, rows, cols, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(sink);
  return ms * 1000.f / it / (rows / 8192.f);  // per 8192 x 4096 mask
}

int main() {
  const int rows = 8 * 8192, cols = 4096;  // 8 C2 q-projection masks per launch (33.5 M elements each)
  for (int wps : {2, 4, 8, 16}) {  // warps per SMSP (256-thread blocks = 8 warps = 2 per SMSP)
    const int blocks = 148 * wps / 2;
    printf("{\"warps_per_smsp\": %d, \"pure_ch4_us\": %.2f, \"masks_ch4_us\": %.2f, \"masks_row_ch4_us\": %.2f, "
           "\"pure_ch8_us\": %.2f, \"masks_ch8_us\": %.2f, \"masks_row_ch8_us\": %.2f}\n",
           wps, run<0, 4>(rows, cols, blocks), run<1, 4>(rows, cols, blocks), run<2, 4>(rows, cols, blocks),
           run<0, 8>(rows, cols, blocks), run<1, 8>(rows, cols, blocks), run<2, 8>(rows, cols, blocks));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
