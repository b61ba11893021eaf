// lf_lowrank.cu — the X-streaming low-rank kernels and the routing/mask utilities.
//
//   ① lf_down_kernel  — dropout_down_proj_fused (ls/costmodel.py:258-261)
//       Ŝ = bf16( s_seg · (M⊙X)·A_catᵀ ) : X is read once, the mask is regenerated in
//       registers (never stored), only the m x R result is written.
//   ④ lf_dgrad_a_kernel — grad_down_fused (ls/costmodel.py:270-272)
//       dA_cat += dŜᵀ·(M⊙X)  — X re-read once, mask regenerated, no mk-sized output.
//   lf_routes_kernel  — adapter_routing_table (ls/costmodel.py:279-281): 16 B per 128-row tile.
//   lf_mask_kernel    — materialises SPEC.md §3's keep mask (parity tests / explicit-mask callers).
//
// Both streaming kernels are HBM-bound (≈ r FLOP/B). They still run the inner products
// on the tensor cores (tcgen05, fp32 accumulators in TMEM): at r = 16 keeping pace with
// 6.5 TB/s needs ~105 TFLOP/s, beyond the FP32 pipes. X tiles arrive by TMA; when
// dropout is active four "mask" warps zero the dropped bf16 lanes of each tile in shared
// memory (Philox4x32-10, 8 keep bits per call = one 16-byte chunk) before the single
// MMA-issuing thread consumes it.
#include "lf_device.cuh"
#include "lf_kernels.h"

namespace lf {

// ------------------------------------------------------------------------------------
// shared helpers
// ------------------------------------------------------------------------------------
__device__ __forceinline__ bool tile_needs_mask(const LfSegTable& t, const LfRoute& rt) {
  if (t.mask_mode == 2) return rt.col_lo < rt.col_hi;
  if (t.mask_mode == 0) return false;
  for (int i = rt.seg_lo; i <= rt.seg_hi; ++i)
    if (t.seg[i].thr) return true;
  return false;
}

// finalize one row of a split-K reduced m x R result: scale own-segment columns, zero the
// rest, write bf16, and return the partial-sum workspace to zero.
__device__ __forceinline__ void finalize_row(const LfSegTable& t, const LfRoute& rt, int row, float* ws,
                                             __nv_bfloat16* out) {
  const int rtot = t.rtot;
  const int seg = find_segment(t, rt.seg_lo, rt.seg_hi, row);
  const int own0 = seg >= 0 ? t.seg[seg].col0 : 0;
  const int own1 = seg >= 0 ? t.seg[seg].col0 + t.seg[seg].ncol : 0;
  const float scale = seg >= 0 ? t.seg[seg].scale : 0.f;
  float* wrow = ws + (int64_t)row * rtot;
  __nv_bfloat16* orow = out + (int64_t)row * rtot;
  for (int c = 0; c < rtot; c += 8) {
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const bool in_range = c >= rt.col_lo && c < rt.col_hi;
    if (in_range) {
      const float4 a = ld_cg_f4(wrow + c), b = ld_cg_f4(wrow + c + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
      *reinterpret_cast<float4*>(wrow + c) = make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(wrow + c + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const bool own = c >= own0 && c < own1;
    const float s = own ? scale : 0.f;
    *reinterpret_cast<uint4*>(orow + c) = make_uint4(pack_bf16x2(v[0] * s, v[1] * s), pack_bf16x2(v[2] * s, v[3] * s),
                                                     pack_bf16x2(v[4] * s, v[5] * s), pack_bf16x2(v[6] * s, v[7] * s));
  }
}

// ------------------------------------------------------------------------------------
// ① dropout + down projection
// ------------------------------------------------------------------------------------
namespace down {
constexpr int X_BYTES = 128 * 64 * 2;  // 16 KB
// 2 CTAs / SM (register bound): ~2 x 100 KB of X tiles in flight per SM
constexpr int SMEM_BUDGET = 100 * 1024;
}  // namespace down

void down_config(int rtot, int* stages, int* stage_bytes) {
  *stage_bytes = down::X_BYTES + rtot * 128;
  int s = down::SMEM_BUDGET / *stage_bytes;
  *stages = s < 2 ? 2 : (s > 8 ? 8 : s);
}

constexpr int kDownThreads = 320;  // producer, MMA, 8 mask warps (2 per row quadrant; 4 also do the epilogue)

__global__ void __launch_bounds__(kDownThreads, 2)
    lf_down_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ DownArgs args, int STAGES, int STAGE_BYTES) {
  using namespace down;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* masked = empty + STAGES;
  uint64_t* tfull = masked + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int mt = blockIdx.x;
  const int m0 = mt * 128;
  const int nkb = (args.k + 63) / 64;
  const int kb0 = (int)((int64_t)blockIdx.y * nkb / args.ksplit);
  const int kb1 = (int)((int64_t)(blockIdx.y + 1) * nkb / args.ksplit);
  const LfRoute rt = args.routes[mt];
  const int N = rt.col_hi - rt.col_lo;
  const bool has_work = N > 0 && kb1 > kb0;
  const bool need_mask = has_work && tile_needs_mask(args.segs, rt);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&masked[s], 8);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
    if (has_work) {
      tma_prefetch_desc(&tmX);
      tma_prefetch_desc(&tmA);
    }
  }
  // one accumulator: spreading the K-steps over several (summed in the epilogue) was
  // measured to make no difference on B200 — these pipelines are TMA/mask bound
  constexpr int NACC = 1;
  uint32_t tmem_cols = 32;
  while ((int)tmem_cols < NACC * args.rtot) tmem_cols <<= 1;
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && has_work) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sX = smem + stage * STAGE_BYTES;
        uint8_t* sA = sX + X_BYTES;
        mbar_arrive_expect_tx(&full[stage], X_BYTES + N * 128);
        tma_load_2d(sX, &tmX, &full[stage], kb * 64, m0);
        for (int j = 0; j < N / 16; ++j) tma_load_2d(sA + j * 2048, &tmA, &full[stage], kb * 64, rt.col_lo + 16 * j);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && has_work) {
      const uint32_t idesc = make_idesc_bf16(128, (uint32_t)N, false, false);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(need_mask ? &masked[stage] : &full[stage], phase);
        tc_fence_after();
        const uint32_t sX = smem_u32(smem + stage * STAGE_BYTES);
        const uint32_t sA = sX + X_BYTES;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (!(args.segs.debug & 1))
          umma_bf16(tmem + (kk % NACC) * args.rtot, make_sdesc(sX + kk * 32, 16, 1024, kLayoutSW128),
                    make_sdesc(sA + kk * 32, 16, 1024, kLayoutSW128), idesc, (kb > kb0 || kk >= NACC) ? 1u : 0u);
        }
        umma_commit(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      umma_commit(tfull);
    }
    __syncwarp();
  } else {
    // mask warps 2..9: thread <-> tile row 32*(warp&3) + lane, half = which 4 of the row's 8
    // 16-byte chunks it masks; warps 2..5 (half 0) also run the epilogue
    const uint32_t q = warp & 3u;
    const int half = warp >= 6 ? 1 : 0;
    const int rit = (int)(q * 32 + lane);
    const int row = m0 + rit;
    const int seg = row < args.m ? find_segment(args.segs, rt.seg_lo, rt.seg_hi, row) : -1;
    if (need_mask) {
      const bool my_mask = seg >= 0 && (args.segs.mask_mode == 2 || args.segs.seg[seg].thr != 0);
      const bool explicit_mask = args.segs.mask_mode == 2;
      const PhiloxRow pr = philox_row(args.segs.seg[seg >= 0 ? seg : 0], (uint32_t)row);
      uint8_t* bits_row = args.segs.bits ? args.segs.bits + (int64_t)row * args.segs.ld_bits : nullptr;
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        // the keep bits depend only on (row, column, seed, offset): generate them while the
        // tile is still in flight, so Philox latency overlaps the TMA instead of adding to it
        const int col = kb * 64 + 32 * half;
        uint32_t bits = ~0u;
        if (my_mask) {
          if (explicit_mask) {
            const uint8_t* mrow = args.segs.mask + (int64_t)row * args.segs.ld_mask;
            bits = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c) bits |= explicit_keep8(mrow, col + 8 * c, args.k) << (8 * c);
          } else {
            bits = (uint32_t)keep_bits_philox<4>(pr, col);
          }
        }
        mbar_wait(&full[stage], phase);
        if (my_mask) {
          if (!(args.segs.debug & 8) && bits != ~0u)
            apply_chunks_sw128<4>(smem + stage * STAGE_BYTES, rit, 4 * half, bits);
          // Philox runs once per step: ④ and ⑤ read these bits instead
          if (!explicit_mask && bits_row) {
            const int b0 = kb * 8 + 4 * half;
            if (b0 + 4 <= (int)args.segs.ld_bits && ((reinterpret_cast<uintptr_t>(bits_row + b0) & 3u) == 0)) {
              *reinterpret_cast<uint32_t*>(bits_row + b0) = bits;
            } else {
              for (int i = 0; i < 4; ++i)
                if (b0 + i < (int)args.segs.ld_bits) bits_row[b0 + i] = (uint8_t)(bits >> (8 * i));
            }
          }
        }
        if (!(args.segs.debug & 4)) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&masked[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
    if (has_work && half == 0) {
      mbar_wait(tfull, 0);
      tc_fence_after();
      const uint32_t taddr = tmem + ((q * 32u) << 16);
      float* wrow = args.ws + (int64_t)row * args.rtot + rt.col_lo;
      for (int c = 0; c < N; c += 16) {
        float s[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) s[j] = 0.f;
        for (int a = 0; a < NACC; ++a) {
          uint32_t v[16];
          tmem_ld16(taddr + a * args.rtot + c, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) s[j] += __uint_as_float(v[j]);
        }
        if (row < args.m && !(args.segs.debug & 2)) {
#pragma unroll
          for (int j = 0; j < 16; j += 4) red_add_v4(wrow + c + j, s[j], s[j + 1], s[j + 2], s[j + 3]);
        }
      }
    }
    // split-K partials are complete in the workspace once this grid retires; the
    // lf_finalize_kernel launched behind it scales, masks and converts them
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
}

// Split-K epilogue shared by ① and ③: per row, scale the own-segment columns of the fp32
// partial sums by s = scaling / (1 - p), zero every other column, write bf16, and return
// the workspace to zero. One thread per row.
__global__ void __launch_bounds__(128) lf_finalize_kernel(const __grid_constant__ LfSegTable segs,
                                                          const LfRoute* __restrict__ routes, float* ws,
                                                          __nv_bfloat16* out) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= segs.m || (segs.debug & 16)) return;
  finalize_row(segs, routes[row / LF_TILE_M], row, ws, out);
}

int finalize_launch(const LfSegTable& segs, const LfRoute* routes, float* ws, void* out, cudaStream_t stream) {
  lf_finalize_kernel<<<(segs.m + 127) / 128, 128, 0, stream>>>(segs, routes, ws,
                                                                 reinterpret_cast<__nv_bfloat16*>(out));
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int down_launch(const CUtensorMap& tm_x, const CUtensorMap& tm_a, const DownArgs& args, int num_sms,
                cudaStream_t stream) {
  int stages = 0, stage_bytes = 0;
  down_config(args.rtot, &stages, &stage_bytes);
  const int smem = stages * stage_bytes + 1024 + 256;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(lf_down_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess)
      return -1;
    configured = true;
  }
  dim3 grid((args.m + 127) / 128, args.ksplit);
  lf_down_kernel<<<grid, kDownThreads, smem, stream>>>(tm_x, tm_a, args, stages, stage_bytes);
  if (cudaGetLastError() != cudaSuccess) return -1;
  return finalize_launch(args.segs, args.routes, args.ws, args.s_hat, stream);
}

// ------------------------------------------------------------------------------------
// ④ dA_cat += dŜᵀ · (M⊙X)
// ------------------------------------------------------------------------------------
// ④ keep bits without ①'s packed mask (explicit uint8 mask or Philox regenerated): out of
// line so the rarely used path does not bloat the kernel's hot loops
__device__ __noinline__ void dgrad_a_keep_slow(const LfSegTable& t, int seg, int row, int col, int ncols,
                                               uint64_t& b0, uint64_t& b1) {
  if (t.mask_mode == 2) {
    b0 = keep_bits64_explicit(t, row, col, ncols);
    b1 = keep_bits64_explicit(t, row, col + 64, ncols);
  } else {
    const PhiloxRow pr = philox_row(t.seg[seg], (uint32_t)row);
    b0 = keep_bits64_philox(pr, col);
    b1 = keep_bits64_philox(pr, col + 64);
  }
}

namespace dga {
constexpr int X_BYTES = 2 * 128 * 64 * 2;  // two 64-column SW128 boxes of 128 rows = 32 KB
constexpr int MAX_SMEM = 200 * 1024;
}  // namespace dga

__global__ void __launch_bounds__(192, 2)
    lf_dgrad_a_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmD,
                      const __grid_constant__ GradDownArgs args, int stages, int stage_bytes) {
  using namespace dga;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* masked = empty + stages;
  uint64_t* tfull = masked + stages;
  uint64_t* tzero = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tzero + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int kt = blockIdx.x;
  const int tiles_m = (args.m + 127) / 128;
  const int mt0 = (int)((int64_t)blockIdx.y * tiles_m / args.m_split);
  const int mt1 = (int)((int64_t)(blockIdx.y + 1) * tiles_m / args.m_split);
  const int rtot = args.rtot;
  // independent accumulators for consecutive K-steps (see ①); 2 CTAs / SM share 512 columns
  const int NACC = 4 * rtot <= 256 ? 4 : 2;
  uint32_t tmem_cols = 32;
  while ((int)tmem_cols < NACC * rtot) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&masked[s], 4);
    }
    mbar_init(tfull, 1);
    mbar_init(tzero, 4);
    fence_barrier_init();
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmD);
  }
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int mt = mt0; mt < mt1; ++mt) {
        const LfRoute rt = args.routes[mt];
        const int N = rt.col_hi - rt.col_lo;
        if (N <= 0) continue;
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sX = smem + stage * stage_bytes;
        uint8_t* sD = sX + X_BYTES;
        mbar_arrive_expect_tx(&full[stage], X_BYTES + (N / 16) * 4096);
        tma_load_2d(sX, &tmX, &full[stage], kt * 128, mt * 128);
        tma_load_2d(sX + 16384, &tmX, &full[stage], kt * 128 + 64, mt * 128);
        for (int j = 0; j < N / 16; ++j) tma_load_2d(sD + j * 4096, &tmD, &full[stage], rt.col_lo + 16 * j, mt * 128);
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(tzero, 0);
      tc_fence_after();
      int stage = 0;
      uint32_t phase = 0;
      for (int mt = mt0; mt < mt1; ++mt) {
        const LfRoute rt = args.routes[mt];
        const int N = rt.col_hi - rt.col_lo;
        if (N <= 0) continue;
        const bool need_mask = tile_needs_mask(args.segs, rt);
        mbar_wait(need_mask ? &masked[stage] : &full[stage], phase);
        tc_fence_after();
        const uint32_t sX = smem_u32(smem + stage * stage_bytes);
        const uint32_t sD = sX + X_BYTES;
        const uint32_t idesc = make_idesc_bf16(128, (uint32_t)N, true, true);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (!(args.segs.debug & 1))
          umma_bf16(tmem + (kk % NACC) * rtot + rt.col_lo, make_sdesc(sX + kk * 2048, 16384, 1024, kLayoutSW128),
                    make_sdesc(sD + kk * 512, 4096, 256, kLayoutSW32), idesc, 1u);
        }
        umma_commit(&empty[stage]);
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
      umma_commit(tfull);
    }
    __syncwarp();
  } else {
    const uint32_t q = warp & 3u;
    const uint32_t taddr = tmem + ((q * 32u) << 16);
    // zero the accumulator so every MMA may accumulate
    {
      uint32_t z[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) z[i] = 0u;
      for (int c = 0; c < NACC * rtot; c += 16) tmem_st16(taddr + c, z);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tzero);
    }
    const int rit = (int)(q * 32 + lane);
    // keep bits of this thread's row in m-tile `mt` (128 columns of k-tile kt); false = keep all
    auto fetch_bits = [&](int mt, uint64_t& b0, uint64_t& b1) -> bool {
      b0 = b1 = ~0ull;
      const LfRoute rt = args.routes[mt];
      if (!tile_needs_mask(args.segs, rt)) return false;
      const int row = mt * 128 + rit;
      const int seg = row < args.m ? find_segment(args.segs, rt.seg_lo, rt.seg_hi, row) : -1;
      if (!(seg >= 0 && (args.segs.mask_mode == 2 || args.segs.seg[seg].thr != 0))) return false;
      if (args.segs.mask_mode == 1 && args.segs.bits) {
        const uint8_t* rb = args.segs.bits + (int64_t)row * args.segs.ld_bits;
        b0 = load_bits64(rb, kt * 16, (int)args.segs.ld_bits);
        b1 = load_bits64(rb, kt * 16 + 8, (int)args.segs.ld_bits);
      } else {
        dgrad_a_keep_slow(args.segs, seg, row, kt * 128, args.k, b0, b1);
      }
      return true;
    };
    auto next_tile = [&](int mt) {
      while (mt < mt1 && args.routes[mt].col_hi <= args.routes[mt].col_lo) ++mt;
      return mt;
    };
    int stage = 0;
    uint32_t phase = 0;
    uint32_t touched = 0;  // 16-column groups that received contributions
    // software pipeline: the keep bits of the next m-tile are fetched while this one is masked
    int cur = next_tile(mt0);
    uint64_t cb0 = ~0ull, cb1 = ~0ull;
    bool cmask = cur < mt1 ? fetch_bits(cur, cb0, cb1) : false;
    while (cur < mt1) {
      const int nxt = next_tile(cur + 1);
      uint64_t nb0 = ~0ull, nb1 = ~0ull;
      const bool nmask = nxt < mt1 ? fetch_bits(nxt, nb0, nb1) : false;
      const LfRoute rt = args.routes[cur];
      for (int c = rt.col_lo; c < rt.col_hi; c += 16) touched |= 1u << (c >> 4);
      if (tile_needs_mask(args.segs, rt)) {
        mbar_wait(&full[stage], phase);
        if (cmask) {
          uint8_t* sX = smem + stage * stage_bytes;
          if (!(args.segs.debug & 8)) {
            apply_row_sw128(sX, rit, cb0);
            apply_row_sw128(sX + 16384, rit, cb1);
          }
        }
        if (!(args.segs.debug & 4)) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&masked[stage]);
      }
      if (++stage == stages) { stage = 0; phase ^= 1; }
      cur = nxt;
      cb0 = nb0;
      cb1 = nb1;
      cmask = nmask;
    }
    if (touched) {
      mbar_wait(tfull, 0);
      tc_fence_after();
      const int kcol = kt * 128 + rit;
      for (int g = 0; g < rtot / 16; ++g) {
        if (!((touched >> g) & 1u)) continue;
        float s[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) s[j] = 0.f;
        for (int a = 0; a < NACC; ++a) {
          uint32_t v[16];
          tmem_ld16(taddr + a * rtot + g * 16, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) s[j] += __uint_as_float(v[j]);
        }
        if (kcol < args.k) {
#pragma unroll
          for (int j = 0; j < 16; ++j) red_add_f32(args.da + (int64_t)(g * 16 + j) * args.k + kcol, s[j]);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
}

void grad_down_config(int rtot, int* stages, int* stage_bytes) {
  *stage_bytes = dga::X_BYTES + (rtot / 16) * 4096;
  int s = (110 * 1024) / *stage_bytes;
  *stages = s < 2 ? 2 : (s > 4 ? 4 : s);
}

int grad_down_launch(const CUtensorMap& tm_x, const CUtensorMap& tm_ds, const GradDownArgs& args, int num_sms,
                     cudaStream_t stream) {
  (void)num_sms;
  int stages = 0, stage_bytes = 0;
  grad_down_config(args.rtot, &stages, &stage_bytes);
  const int smem = stages * stage_bytes + 1024 + 256;
  static int configured = 0;
  if (configured < smem) {
    if (cudaFuncSetAttribute(lf_dgrad_a_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dga::MAX_SMEM + 2048) !=
        cudaSuccess)
      return -1;
    configured = dga::MAX_SMEM + 2048;
  }
  dim3 grid((args.k + 127) / 128, args.m_split);
  lf_dgrad_a_kernel<<<grid, 192, smem, stream>>>(tm_x, tm_ds, args, stages, stage_bytes);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ------------------------------------------------------------------------------------
// routing table and explicit keep mask
// ------------------------------------------------------------------------------------
__global__ void lf_routes_kernel(const __grid_constant__ LfSegTable segs, LfRoute* routes, int ntiles) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int r0 = t * LF_TILE_M;
  const int r1 = min(segs.m, r0 + LF_TILE_M);
  int lo = -1, hi = -2;
  for (int i = 0; i < segs.nseg; ++i) {
    const LfSegDev& s = segs.seg[i];
    if (s.row0 < s.row1 && s.row0 < r1 && s.row1 > r0) {
      if (lo < 0) lo = i;
      hi = i;
    }
  }
  LfRoute r;
  if (lo < 0) {
    r.seg_lo = 0; r.seg_hi = -1; r.col_lo = 0; r.col_hi = 0;
  } else {
    r.seg_lo = lo; r.seg_hi = hi;
    r.col_lo = segs.seg[lo].col0;
    r.col_hi = segs.seg[hi].col0 + segs.seg[hi].ncol;
  }
  routes[t] = r;
}

__global__ void lf_mask_kernel(const __grid_constant__ LfSegTable segs, int32_t k, uint8_t* keep) {
  const int groups = (k + 7) / 8;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)segs.m * groups) return;
  const int row = (int)(idx / groups);
  const int g = (int)(idx - (int64_t)row * groups);
  uint32_t bits = 0xFFu;
  const int seg = find_segment(segs, 0, segs.nseg - 1, row);
  if (seg >= 0 && segs.mask_mode == 1 && segs.seg[seg].thr)
    bits = philox_keep8((uint32_t)g, (uint32_t)row, segs.seg[seg]);
  uint8_t* out = keep + (int64_t)row * k + g * 8;
  for (int e = 0; e < 8; ++e)
    if (g * 8 + e < k) out[e] = (uint8_t)((bits >> e) & 1u);
}

int routes_launch(const LfSegTable& segs, int32_t* routes, int ntiles, cudaStream_t stream) {
  if (ntiles <= 0) return 0;
  lf_routes_kernel<<<(ntiles + 127) / 128, 128, 0, stream>>>(segs, reinterpret_cast<LfRoute*>(routes), ntiles);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int mask_launch(const LfSegTable& segs, int32_t k, uint8_t* keep, cudaStream_t stream) {
  const int64_t total = (int64_t)segs.m * ((k + 7) / 8);
  if (total <= 0) return 0;
  lf_mask_kernel<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(segs, k, keep);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace lf
