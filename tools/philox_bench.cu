// Standalone throughput of the ① mask generator (philox_masks<CH>: Philox4x32-10 ->
// SWAR keep test -> lane masks + packed bits) with no TMA / MMA pipeline around it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2510_00206_b200/csrc \
//        tools/philox_bench.cu -o tools/philox_bench && tools/philox_bench
#include <cstdio>

#include "lf_device.cuh"

using namespace lf;

template <int CH>
__global__ void __launch_bounds__(256) bench(LfSegDev seg, int rows, int cols, uint32_t* sink) {
  uint32_t acc = 0;
  const int chunks_per_row = cols / (8 * CH);
  const int total = rows * chunks_per_row;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int row = i / chunks_per_row, cg = i - row * chunks_per_row;
    const PhiloxRow pr = philox_row(seg, (uint32_t)row);
    uint32_t msk[CH][4];
    const uint64_t bits = philox_masks<CH>(pr, cg * 8 * CH, msk);
#pragma unroll
    for (int j = 0; j < CH; ++j) acc ^= msk[j][0] ^ msk[j][1] ^ msk[j][2] ^ msk[j][3];
    acc += (uint32_t)bits ^ (uint32_t)(bits >> 32);
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;  // observable: no dead-code elimination
}

template <int CH>
float run(int rows, int cols, int blocks) {
  LfSegDev s{};
  s.thr = 2 * 3276;
  s.key0 = 1234;
  uint32_t* sink;
  cudaMalloc(&sink, (size_t)blocks * 256 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) bench<CH><<<blocks, 256>>>(s, rows, cols, sink);
  cudaEventRecord(a);
  const int it = 20;
  for (int w = 0; w < it; ++w) bench<CH><<<blocks, 256>>>(s, rows, cols, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(sink);
  return ms * 1000.f / it;
}

int main() {
  const int rows = 8192, cols = 4096;  // the C2 q-projection mask: 33.5 M elements
  for (int bps : {2, 4, 8}) {
    const int blocks = 148 * bps;
    printf("{\"blocks\": %d, \"ch4_us\": %.2f, \"ch8_us\": %.2f, \"elements\": %d}\n", blocks,
           run<4>(rows, cols, blocks), run<8>(rows, cols, blocks), rows * cols);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
