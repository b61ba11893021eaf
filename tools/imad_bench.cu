// Throughput of the 32x32->64 multiply forms a Philox round can use on sm_100a:
// IMAD.WIDE.U32 (one instruction, hi+lo) vs IMAD.HI.U32 + IMAD (two instructions).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/imad_bench.cu -o tools/imad_bench
#include <cstdio>
#include <cstdint>

template <int MODE>
__global__ void __launch_bounds__(256) k(uint32_t seed, uint32_t* out, int iters) {
  uint32_t a[8], h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = seed + threadIdx.x * 8 + i; h[i] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        const uint64_t p = (uint64_t)a[i] * 0xD2511F53u;  // IMAD.WIDE.U32
        h[i] ^= (uint32_t)(p >> 32);
        a[i] = (uint32_t)p ^ h[i];
      } else if (MODE == 1) {
        uint32_t hi, lo;
        asm volatile("mul.hi.u32 %0, %1, 0xD2511F53;" : "=r"(hi) : "r"(a[i]));
        asm volatile("mul.lo.u32 %0, %1, 0xD2511F53;" : "=r"(lo) : "r"(a[i]));
        h[i] ^= hi;
        a[i] = lo ^ h[i];
      } else {
        a[i] = a[i] * 0xD2511F53u ^ h[i];  // IMAD only (lower bound)
        h[i] += a[i];
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= a[i] ^ h[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
float run(int blocks, int iters) {
  uint32_t* out;
  cudaMalloc(&out, blocks * 256 * 4);
  k<MODE><<<blocks, 256>>>(1, out, iters);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<blocks, 256>>>(1, out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double mults = (double)blocks * 256 * iters * 8;
  const double per_clk_sm = mults / (ms * 1e-3) / (clk * 1e3) / 148;  // at the nominal max clock
  printf("mode %d: %.3f ms, %.1f multiplies/clk/SM (at %d MHz nominal)\n", MODE, ms, per_clk_sm, clk / 1000);
  return ms;
}

int main() {
  const int blocks = 148 * 8, iters = 4096;
  run<0>(blocks, iters);
  run<1>(blocks, iters);
  run<2>(blocks, iters);
  return 0;
}
