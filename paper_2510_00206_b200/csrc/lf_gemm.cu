// lf_gemm.cu — ② base_gemm_epilogue_fused and ⑤ grad_base_accum_fused on sm_100a.
//
// Reference contract: ls/costmodel.py:262-264 (Y = X·W + α·S·B written once) and
// ls/costmodel.py:273-277 (dX = dY·Wᵀ + mask ⊙ LoRA term, one dX write);
// paper design PAPER.md:457-463.
//
// B200 design: persistent, warp-specialised tcgen05 GEMM, one CTA per SM.
//   warp 0      TMA producer (one lane): A/B tiles into a STAGES-deep smem ring
//   warp 1      MMA issuer (one lane): tcgen05.mma 128xBNx16, fp32 accumulators in TMEM,
//               double-buffered so the epilogue of tile i overlaps the main loop of tile i+1
//   warps 2..5  epilogue: tcgen05.ld -> (mask ⊙ LoRA accumulator) -> bf16 -> global
// The low-rank up-projection is NOT an epilogue GEMM: [X | Ŝ]·[W | B_cat]ᵀ — the
// rank-R LoRA operands are streamed as extra K-blocks into the same accumulator, so
// the output tile is written exactly once and the epilogue stays a pure convert.
// With dropout in the backward (⑤, p > 0) the mask multiplies the LoRA term only,
// so that term goes to a second TMEM accumulator and is folded in by the epilogue.
#include "lf_device.cuh"
#include "lf_kernels.h"

namespace lf {

template <int BN, bool B_MN, bool MASKED, int STAGES>
struct GemmCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;  // 16 KB, K-major SW128
  static constexpr int B_BYTES = BN * BK * 2;  // BN x 128 B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int ACC_COLS = MASKED ? 2 * BN : BN;
  static constexpr int TMEM_COLS = 2 * ACC_COLS;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
  static_assert(TMEM_COLS <= 512 && (TMEM_COLS & (TMEM_COLS - 1)) == 0, "TMEM budget");
  static_assert(BN % 64 == 0 && BN <= 256, "BN");
};

// grouped raster: GROUP m-tiles share each n-column sweep so W tiles stay L2-hot
__device__ __forceinline__ void gemm_tile_coords(int t, int tiles_m, int tiles_n, int& mb, int& nb) {
  constexpr int G = 8;
  const int per_group = G * tiles_n;
  const int g = t / per_group;
  const int first_m = g * G;
  const int gm = min(G, tiles_m - first_m);
  const int r = t - g * per_group;
  mb = first_m + r % gm;
  nb = r / gm;
}

template <int BN, bool B_MN, bool MASKED, int STAGES>
__global__ void __launch_bounds__(192, 1)
    lf_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
                   const __grid_constant__ GemmArgs args) {
  using Cfg = GemmCfg<BN, B_MN, MASKED, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (args.routes) {
      tma_prefetch_desc(&tmA2);
      tma_prefetch_desc(&tmB2);
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int tiles = args.tiles_m * args.tiles_n;
  const int nkb = (args.K + Cfg::BK - 1) / Cfg::BK;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int mb, nb;
        gemm_tile_coords(t, args.tiles_m, args.tiles_n, mb, nb);
        const int m0 = mb * Cfg::BM, n0 = nb * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sA = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sB = sA + Cfg::A_BYTES;
          mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          tma_load_2d(sA, &tmA, &full[stage], kb * Cfg::BK, m0);
          if constexpr (!B_MN) {
            tma_load_2d(sB, &tmB, &full[stage], kb * Cfg::BK, n0);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i) tma_load_2d(sB + i * 8192, &tmB, &full[stage], n0 + 64 * i, kb * Cfg::BK);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (args.routes) {
          const LfRoute rt = args.routes[mb];
          for (int c = rt.col_lo; c < rt.col_hi; c += 64) {
            const int nsub = min(4, (rt.col_hi - c) >> 4);
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sA = smem + stage * Cfg::STAGE_BYTES;
            uint8_t* sB = sA + Cfg::A_BYTES;
            mbar_arrive_expect_tx(&full[stage], nsub * (Cfg::BM * 32 + BN * 32));
            for (int j = 0; j < nsub; ++j) {
              tma_load_2d(sA + j * (Cfg::BM * 32), &tmA2, &full[stage], c + 16 * j, m0);
              if constexpr (!B_MN) {
                tma_load_2d(sB + j * (BN * 32), &tmB2, &full[stage], c + 16 * j, n0);
              } else {
#pragma unroll
                for (int i = 0; i < BN / 64; ++i)
                  tma_load_2d(sB + j * (BN / 64) * 2048 + i * 2048, &tmB2, &full[stage], n0 + 64 * i, c + 16 * j);
              }
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = make_idesc_bf16(Cfg::BM, BN, false, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        int mb, nb;
        gemm_tile_coords(t, args.tiles_m, args.tiles_n, mb, nb);
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * Cfg::ACC_COLS;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sA = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sB = sA + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = make_sdesc(sA + kk * 32, 16, 1024, kLayoutSW128);
            const uint64_t bd = B_MN ? make_sdesc(sB + kk * 2048, 8192, 1024, kLayoutSW128)
                                     : make_sdesc(sB + kk * 32, 16, 1024, kLayoutSW128);
            umma_bf16(d, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (args.routes) {
          const LfRoute rt = args.routes[mb];
          const uint32_t dl = MASKED ? d + BN : d;
          uint32_t accum = MASKED ? 0u : 1u;
          for (int c = rt.col_lo; c < rt.col_hi; c += 64) {
            const int nsub = min(4, (rt.col_hi - c) >> 4);
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t sA = smem_u32(smem + stage * Cfg::STAGE_BYTES);
            const uint32_t sB = sA + Cfg::A_BYTES;
            for (int j = 0; j < nsub; ++j) {
              const uint64_t ad = make_sdesc(sA + j * (Cfg::BM * 32), 16, 256, kLayoutSW32);
              const uint64_t bd = B_MN ? make_sdesc(sB + j * (BN / 64) * 2048, 2048, 1024, kLayoutSW128)
                                       : make_sdesc(sB + j * (BN * 32), 16, 256, kLayoutSW32);
              umma_bf16(dl, ad, bd, idesc, accum);
              accum = 1u;
            }
            umma_commit(&empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const uint32_t q = warp & 3u;  // TMEM lane quadrant this warp may access
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      int mb, nb;
      gemm_tile_coords(t, args.tiles_m, args.tiles_n, mb, nb);
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const int row = mb * Cfg::BM + (int)(q * 32 + lane);
      const int n0 = nb * BN;
      bool lora_on = false;
      int seg = -1;
      if constexpr (MASKED) {
        if (args.routes) {
          const LfRoute rt = args.routes[mb];
          lora_on = rt.col_lo < rt.col_hi;
          seg = find_segment(args.segs, rt.seg_lo, rt.seg_hi, row);
        }
      }
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * Cfg::ACC_COLS;
      __nv_bfloat16* crow = reinterpret_cast<__nv_bfloat16*>(args.C) + (int64_t)row * args.ldc;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        tmem_ld32(taddr + c, v);
        float f[32];
        if constexpr (MASKED) {
          uint32_t u[32];
          if (lora_on) tmem_ld32(taddr + BN + c, u);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
          if (lora_on && seg >= 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int col = n0 + c + 8 * j;
              uint32_t bits;
              if (args.segs.mask_mode == 2) {
                bits = (row < args.M) ? explicit_keep8(args.segs.mask + (int64_t)row * args.segs.ld_mask, col, args.N)
                                      : 0u;
              } else {
                const LfSegDev& s = args.segs.seg[seg];
                bits = s.thr ? philox_keep8((uint32_t)col >> 3, (uint32_t)row, s) : 0xFFu;
              }
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if ((bits >> e) & 1u) f[8 * j + e] += __uint_as_float(u[8 * j + e]);
            }
          }
        } else {
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
        }
        if (row < args.M) {
          const int col0 = n0 + c;
          uint4 pk[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            pk[j] = make_uint4(pack_bf16x2(f[8 * j + 0], f[8 * j + 1]), pack_bf16x2(f[8 * j + 2], f[8 * j + 3]),
                               pack_bf16x2(f[8 * j + 4], f[8 * j + 5]), pack_bf16x2(f[8 * j + 6], f[8 * j + 7]));
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (col0 + 8 * j < args.N) *reinterpret_cast<uint4*>(crow + col0 + 8 * j) = pk[j];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

template <int BN, bool B_MN, bool MASKED, int STAGES>
static int launch_one(const GemmMaps& maps, const GemmArgs& args, int num_sms, cudaStream_t stream) {
  using Cfg = GemmCfg<BN, B_MN, MASKED, STAGES>;
  auto kern = lf_gemm_kernel<BN, B_MN, MASKED, STAGES>;
  static bool configured = false;  // per instantiation; attribute set is idempotent
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES) != cudaSuccess)
      return -1;
    configured = true;
  }
  const int tiles = args.tiles_m * args.tiles_n;
  const int grid = tiles < num_sms ? tiles : num_sms;
  kern<<<grid, 192, Cfg::SMEM_BYTES, stream>>>(maps.a, maps.b, maps.a2, maps.b2, args);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int gemm_launch(GemmKind kind, const GemmMaps& maps, const GemmArgs& a, int num_sms, cudaStream_t stream) {
  GemmArgs args = a;
  switch (kind) {
    case kGemmFwd:
      args.tiles_m = (args.M + 127) / 128;
      args.tiles_n = (args.N + 255) / 256;
      return launch_one<256, false, false, 4>(maps, args, num_sms, stream);
    case kGemmDgrad:
      args.tiles_m = (args.M + 127) / 128;
      args.tiles_n = (args.N + 255) / 256;
      return launch_one<256, true, false, 4>(maps, args, num_sms, stream);
    case kGemmDgradMasked:
      args.tiles_m = (args.M + 127) / 128;
      args.tiles_n = (args.N + 127) / 128;
      return launch_one<128, true, true, 6>(maps, args, num_sms, stream);
  }
  return -1;
}

}  // namespace lf
