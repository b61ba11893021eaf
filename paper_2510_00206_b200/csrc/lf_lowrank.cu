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
#include <cstdlib>

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

// ------------------------------------------------------------------------------------
// ① dropout + down projection
// ------------------------------------------------------------------------------------
#ifndef LF_DOWN_MINB
#define LF_DOWN_MINB 2  // resident CTAs per SM (register bound)
#endif
#ifndef LF_DOWN_SMEM_KB
#define LF_DOWN_SMEM_KB 100
#endif
#ifndef LF_DOWN_SPLIT
#define LF_DOWN_SPLIT 1  // Philox keep bits by 4 generator warps running ahead, masks applied by 4 others
#endif
namespace down {
constexpr int X_BYTES = 128 * 64 * 2;  // 16 KB
constexpr int BITS_SLOTS = 8;          // LF_DOWN_SPLIT: keep-bit ring depth (k-blocks the generators run ahead)
constexpr int BITS_SLOT_BYTES = 128 * 8;  // one k-block's 64 keep bits per tile row
// 2 CTAs / SM (register bound): ~2 x 100 KB of X tiles in flight per SM
constexpr int SMEM_BUDGET = LF_DOWN_SMEM_KB * 1024;
}  // namespace down

// wmax: the widest routing hull (LfSegTable::wmax), the most A_cat columns a stage holds
void down_config(int wmax, int* stages, int* stage_bytes) {
  *stage_bytes = down::X_BYTES + wmax * 128;
  int s = down::SMEM_BUDGET / *stage_bytes;
  *stages = s < 2 ? 2 : (s > 8 ? 8 : s);
}

int down_extra_smem(int mask_mode) {
  return (LF_DOWN_SPLIT && mask_mode != 2) ? down::BITS_SLOTS * (down::BITS_SLOT_BYTES + 16) : 0;
}

constexpr int kDownThreads = 320;  // producer, MMA, 8 mask warps (2 per row quadrant; 4 also do the epilogue)

// Stream-K work split shared by ① and ④: the (tile, k-block) units are laid out tile-major
// and every CTA takes one contiguous, equal share, so a single resident wave of CTAs moves
// the same number of bytes each (a per-tile split leaves SMs with 2 CTAs next to SMs with 1).
// A share crossing a tile boundary is walked as per-tile spans, each flushed on its own.
struct UnitSpan {
  int tile, k0, k1;
};
struct UnitWalker {
  int u, u1, per_tile;
  __device__ UnitWalker(int units, int ctas, int cta, int per_tile_) : per_tile(per_tile_) {
    u = (int)((int64_t)cta * units / ctas);
    u1 = (int)((int64_t)(cta + 1) * units / ctas);
  }
  __device__ bool next(UnitSpan& sp) {
    if (u >= u1) return false;
    sp.tile = u / per_tile;
    sp.k0 = u - sp.tile * per_tile;
    sp.k1 = min(per_tile, sp.k0 + (u1 - u));
    u += sp.k1 - sp.k0;
    return true;
  }
};

// EXPLICIT: the keep mask comes from a caller's uint8 mask (mask_mode 2) instead of Philox —
// a separate instantiation, so the Philox hot loop carries no per-k-block mode test
template <bool EXPLICIT>
__global__ void __launch_bounds__(kDownThreads, LF_DOWN_MINB)
    lf_down_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ DownArgs args, int STAGES, int STAGE_BYTES) {
  using namespace down;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  // SPLIT (Philox path): warps 6..9 generate each k-block's keep bits into a ring of
  // BITS_SLOTS slots (bits_full / bits_empty), up to BITS_SLOTS k-blocks ahead of the data;
  // warps 2..5 apply them to the X tiles and flush. Otherwise all 8 mask warps do both.
  constexpr bool SPLIT = LF_DOWN_SPLIT && !EXPLICIT;
  uint8_t* sbits = smem + STAGES * STAGE_BYTES;  // SPLIT: [BITS_SLOTS][128 rows] x 8 bytes
  uint64_t* full = reinterpret_cast<uint64_t*>(sbits + (SPLIT ? BITS_SLOTS * BITS_SLOT_BYTES : 0));
  uint64_t* empty = full + STAGES;
  uint64_t* masked = empty + STAGES;
  uint64_t* tfull = masked + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint64_t* bits_full = tempty + 2;   // [BITS_SLOTS] SPLIT
  uint64_t* bits_empty = bits_full + BITS_SLOTS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bits_empty + BITS_SLOTS);
  __shared__ int s_last;

  const uint32_t warp = warp_id(), lane = lane_id();
  const int nkb = (args.k + 63) / 64;
  const int tiles_m = (args.m + 127) / 128;
  const int units = tiles_m * nkb;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&masked[s], SPLIT ? 4 : 8);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    if constexpr (SPLIT) {
      for (int i = 0; i < BITS_SLOTS; ++i) {
        mbar_init(&bits_full[i], 4);
        mbar_init(&bits_empty[i], 4);
      }
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmA);
  }
  // two accumulators (R columns each): a span's flush overlaps the next span's MMAs
  uint32_t tmem_cols = 32;
  while ((int)tmem_cols < 2 * args.rtot) tmem_cols <<= 1;
  pdl_launch_dependents();
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // the prologue above overlaps the predecessor's tail; global memory only from here
  const uint32_t tmem = *tmem_slot;

  UnitWalker walk(units, (int)gridDim.x, (int)blockIdx.x, nkb);
  UnitSpan sp;
  // With any dropout in the problem EVERY stage passes through the mask warps (full ->
  // masked), whatever its tile needs: a CTA's span may mix p = 0 and p > 0 tiles, and a
  // per-stage choice of barrier would desynchronise `masked`'s phase from the ring's.
  const bool gated = args.segs.mask_mode != 0;
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      while (walk.next(sp)) {
        const LfRoute rt = args.routes[sp.tile];
        const int N = rt.col_hi - rt.col_lo;
        if (N <= 0) continue;
        for (int kb = sp.k0; kb < sp.k1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sX = smem + stage * STAGE_BYTES;
          uint8_t* sA = sX + X_BYTES;
          mbar_arrive_expect_tx(&full[stage], X_BYTES + N * 128);
          tma_load_2d(sX, &tmX, &full[stage], kb * 64, sp.tile * 128);
          for (int j = 0; j < N / 16; ++j) tma_load_2d(sA + j * 2048, &tmA, &full[stage], kb * 64, rt.col_lo + 16 * j);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // whole warp, one elected lane issues (uniform-datapath descriptors)
    int stage = 0, it = 0;
    uint32_t phase = 0;
    while (walk.next(sp)) {
      const LfRoute rt = args.routes[sp.tile];
      const int N = rt.col_hi - rt.col_lo;
      if (N <= 0) continue;
      const int b = it & 1;
      mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + b * args.rtot;
      const uint32_t idesc = make_idesc_bf16(128, (uint32_t)N, false, false);
      for (int kb = sp.k0; kb < sp.k1; ++kb) {
        mbar_wait(gated ? &masked[stage] : &full[stage], phase);
        tc_fence_after();
        const uint32_t sX = smem_u32(smem + stage * STAGE_BYTES);
        const uint64_t ax = make_sdesc(sX, 16, 1024, kLayoutSW128);
        const uint64_t ba = make_sdesc(sX + X_BYTES, 16, 1024, kLayoutSW128);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (!(args.segs.debug & 1))
            umma_bf16_warp(d, sdesc_add(ax, kk * 32), sdesc_add(ba, kk * 32), idesc,
                           (kb > sp.k0 || kk > 0) ? 1u : 0u);
        }
        umma_commit_warp(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      umma_commit_warp(&tfull[b]);
      ++it;
    }
    __syncwarp();
  } else if (SPLIT && warp >= 6) {
    // keep-bit generators (warps 6..9): thread <-> tile row 32*(warp&3) + lane; per k-block
    // the row's 64 keep bits (8 Philox4x32-10 calls) into the ring and to the packed global
    // mask ④ / ⑤ read. They never wait for X, only for a free slot.
    const uint32_t q = warp & 3u;
    const int rit = (int)(q * 32 + lane);
    const uint64_t step_offset = table_offset(args.segs);
    const int nbytes = (int)args.segs.ld_bits;
    int slot = 0;
    uint32_t bphase = 0;
    if (gated) {
      while (walk.next(sp)) {
        const LfRoute rt = args.routes[sp.tile];
        if (rt.col_hi - rt.col_lo <= 0) continue;
        const int row = sp.tile * 128 + rit;
        const int seg = row < args.m ? find_segment(args.segs, rt.seg_lo, rt.seg_hi, row) : -1;
        const bool my_mask = seg >= 0 && args.segs.seg[seg].thr != 0;
        const PhiloxRow pr = philox_row(args.segs.seg[seg >= 0 ? seg : 0], (uint32_t)(row + args.segs.row_base), step_offset);
        // rows of p = 0 segments get all-ones bits (see the unsplit path below)
        uint8_t* bits_row = (seg >= 0 && args.segs.bits) ? args.segs.bits + (int64_t)row * nbytes : nullptr;
        for (int kb = sp.k0; kb < sp.k1; ++kb) {
          uint64_t bits = ~0ull;
          if (my_mask) {
            if (args.segs.debug & 4096) {  // profiling: a fixed pattern instead of Philox
              bits = 0xFBFFFFFEFBFFFFFEull ^ (uint64_t)kb;
            } else {
              uint32_t msk[8][4];  // unused here: the appliers expand the bits themselves
              bits = philox_masks<8>(pr, kb * 64, msk);
            }
          }
          mbar_wait(&bits_empty[slot], bphase ^ 1);
          sts64(smem_u32(sbits + slot * BITS_SLOT_BYTES + rit * 8), bits);
          if (bits_row && !(args.segs.debug & 16384)) store_bits64(bits_row, kb * 8, nbytes, bits);
          __syncwarp();
          if (lane == 0) mbar_arrive(&bits_full[slot]);
          if (++slot == BITS_SLOTS) { slot = 0; bphase ^= 1; }
        }
      }
    }
  } else if (SPLIT) {
    // appliers (warps 2..5): thread <-> tile row; per k-block zero the dropped elements of
    // the whole 128-byte row from the ring's bits, then release stage and slot; each span's
    // partial sums are flushed here too
    const uint32_t q = warp & 3u;
    const int rit = (int)(q * 32 + lane);
    int stage = 0, it = 0, slot = 0;
    uint32_t phase = 0, bphase = 0;
    while (walk.next(sp)) {
      const LfRoute rt = args.routes[sp.tile];
      const int N = rt.col_hi - rt.col_lo;
      const int row = sp.tile * 128 + rit;
      if (N <= 0) {  // no adapter in this row tile: its Ŝ rows are zero (written once, by the span at k = 0)
        if (sp.k0 == 0 && row < args.m) zero_row(args.rtot, row, reinterpret_cast<__nv_bfloat16*>(args.s_hat));
        continue;
      }
      for (int kb = sp.k0; kb < sp.k1; ++kb) {
        if (gated) {
          mbar_wait(&bits_full[slot], bphase);
          const uint64_t bits = lds64(smem_u32(sbits + slot * BITS_SLOT_BYTES + rit * 8));
          mbar_wait(&full[stage], phase);
          if (!(args.segs.debug & 8192)) apply_row_sw128(smem + stage * STAGE_BYTES, rit, bits);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&masked[stage]);
            mbar_arrive(&bits_empty[slot]);
          }
          if (++slot == BITS_SLOTS) { slot = 0; bphase ^= 1; }
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      const int b = it & 1;
      mbar_wait(&tfull[b], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + ((q * 32u) << 16) + b * args.rtot;
      float* wrow = args.ws + (int64_t)row * args.rtot + rt.col_lo;
      for (int c = 0; c < N; c += 16) {
        uint32_t v[16];
        tmem_ld16(taddr + c, v);
        tmem_ld_wait();
        if (row < args.m && !(args.segs.debug & 2)) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            red_add_v4(wrow + c + j, __uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                       __uint_as_float(v[j + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
      tile_contribute(args.segs, rt, sp.tile, rit, sp.k1 - sp.k0, nkb, args.counters, args.ws,
                      reinterpret_cast<__nv_bfloat16*>(args.s_hat), 1, &s_last);
      ++it;
    }
  } else {
    // mask warps 2..9: thread <-> tile row 32*(warp&3) + lane, half = which 4 of the row's 8
    // 16-byte chunks it masks; warps 2..5 (half 0) also flush each span's partial sums
    // (measured: whole rows of alternate stages per thread — 8 Philox streams, half the
    // barrier round trips — ran 1-2% slower than this split)
    const uint32_t q = warp & 3u;
    const int half = warp >= 6 ? 1 : 0;
    const int rit = (int)(q * 32 + lane);
    const uint64_t step_offset = table_offset(args.segs);
    // shared addresses of this thread's four chunks in stage 0 (SW128: chunk c of row r at
    // ((c ^ (r & 7)) * 16); the stage offset is added per k-block
    const uint32_t row0 = smem_u32(smem) + (uint32_t)rit * 128u;
    uint32_t coff[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) coff[c] = row0 + (uint32_t)(((4 * half + c) ^ (rit & 7)) << 4);
    const int nbytes = (int)args.segs.ld_bits;
    int stage = 0, it = 0;
    uint32_t phase = 0;
    while (walk.next(sp)) {
      const LfRoute rt = args.routes[sp.tile];
      const int N = rt.col_hi - rt.col_lo;
      const int row = sp.tile * 128 + rit;
      if (N <= 0) {  // no adapter in this row tile: its Ŝ rows are zero (written once, by the span at k = 0)
        if (half == 0 && sp.k0 == 0 && row < args.m) zero_row(args.rtot, row, reinterpret_cast<__nv_bfloat16*>(args.s_hat));
        continue;
      }
      if (gated) {
        const int seg = row < args.m ? find_segment(args.segs, rt.seg_lo, rt.seg_hi, row) : -1;
        const bool my_mask = seg >= 0 && (EXPLICIT || args.segs.seg[seg].thr != 0);
        const PhiloxRow pr = philox_row(args.segs.seg[seg >= 0 ? seg : 0], (uint32_t)(row + args.segs.row_base), step_offset);
        // Philox runs once per step: ④ and ⑤ read the packed bits written here (4 bytes per
        // k-block and thread; word stores when the row pitch keeps them aligned). Rows of
        // p = 0 segments get all-ones bits, so the group launchers (one mask per projection,
        // no segment table) can apply the bits of every row that carries a LoRA term.
        uint8_t* bits_row = (!EXPLICIT && seg >= 0 && args.segs.bits) ? args.segs.bits + (int64_t)row * nbytes : nullptr;
        const bool bits_words = (nbytes & 3) == 0 && ((reinterpret_cast<uintptr_t>(args.segs.bits) & 3u) == 0);
        for (int kb = sp.k0; kb < sp.k1; ++kb) {
          // the keep bits depend only on (row, column, seed, offset): generate them while the
          // tile is still in flight, so Philox latency overlaps the TMA instead of adding to it
          const int col = kb * 64 + 32 * half;
          uint32_t bits = ~0u;
          uint32_t msk[4][4];
          if (my_mask) {
            if constexpr (EXPLICIT) {
              const uint8_t* mrow = args.segs.mask + (int64_t)row * args.segs.ld_mask;
              bits = 0;
#pragma unroll
              for (int c = 0; c < 4; ++c) bits |= explicit_keep8(mrow, col + 8 * c, args.k) << (8 * c);
            } else if (args.segs.debug & 4096) {  // profiling: a fixed pattern instead of Philox
              bits = 0xFBFFFFFEu ^ (uint32_t)kb;
#pragma unroll
              for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int i = 0; i < 4; ++i) msk[c][i] = (c | i) ? 0xFFFFFFFFu : 0xFFFF0000u;
            } else {
              bits = (uint32_t)philox_masks<4>(pr, col, msk);
            }
          }
          mbar_wait(&full[stage], phase);
          if (my_mask && bits != ~0u && !(args.segs.debug & 8192)) {  // 8192, profiling: no smem pass
            const uint32_t so = (uint32_t)(stage * STAGE_BYTES);
            uint4 v[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) v[c] = lds128(coff[c] + so);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              if constexpr (EXPLICIT)
                sts128(coff[c] + so, apply_keep8(v[c], (bits >> (8 * c)) & 0xFFu));
              else
                sts128(coff[c] + so, make_uint4(v[c].x & msk[c][0], v[c].y & msk[c][1], v[c].z & msk[c][2],
                                                v[c].w & msk[c][3]));
            }
          }
          if (bits_row && !(args.segs.debug & 16384)) {  // 16384, profiling: no keep-bit stores
            const int b0 = kb * 8 + 4 * half;
            if (bits_words && b0 + 4 <= nbytes) {
              *reinterpret_cast<uint32_t*>(bits_row + b0) = bits;
            } else {
              for (int i = 0; i < 4; ++i)
                if (b0 + i < nbytes) bits_row[b0 + i] = (uint8_t)(bits >> (8 * i));
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&masked[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      } else {
        // no dropout anywhere: the MMA consumes the stages straight from `full`; keep the
        // ring position in step with it
        for (int kb = sp.k0; kb < sp.k1; ++kb)
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (half == 0) {
        const int b = it & 1;
        mbar_wait(&tfull[b], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem + ((q * 32u) << 16) + b * args.rtot;
        float* wrow = args.ws + (int64_t)row * args.rtot + rt.col_lo;
        for (int c = 0; c < N; c += 16) {
          uint32_t v[16];
          tmem_ld16(taddr + c, v);
          tmem_ld_wait();
          if (row < args.m && !(args.segs.debug & 2)) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              red_add_v4(wrow + c + j, __uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                         __uint_as_float(v[j + 3]));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
        // the span's partial is in; the CTA that completes the tile finalizes it
        tile_contribute(args.segs, rt, sp.tile, rit, sp.k1 - sp.k0, nkb, args.counters, args.ws,
                        reinterpret_cast<__nv_bfloat16*>(args.s_hat), 1, &s_last);
      }
      ++it;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
}

// Split-K epilogue of ③ (① finalizes in-kernel, see tile_contribute): per row, scale the own-segment columns of the fp32
// partial sums by s = scaling / (1 - p), zero every other column, write bf16, and return
// the workspace to zero. One thread per row.
__global__ void __launch_bounds__(128) lf_finalize_kernel(const __grid_constant__ LfSegTable segs,
                                                          const LfRoute* __restrict__ routes, float* ws,
                                                          __nv_bfloat16* out) {
  pdl_wait();
  pdl_launch_dependents();
  // one thread per 8-column chunk: a single L2 round trip each (one thread per row walked
  // its chunks serially: 60 µs per launch at R = 128, C3)
  const int chunks = segs.rtot / 8;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)segs.m * chunks || (segs.debug & 16)) return;
  const int row = (int)(idx / chunks);
  const int c = (int)(idx - (int64_t)row * chunks) * 8;
  finalize_chunk(segs, routes[row / LF_TILE_M], row, c, ws, out);
}

// the dŜ finalize of several ③ problems (a shared-input group) in one launch
__global__ void __launch_bounds__(128) lf_finalize_group_kernel(const __grid_constant__ GroupFinArgs f) {
  pdl_wait();
  pdl_launch_dependents();
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int j = 0;
  while (j + 1 < f.J && idx >= f.chunk_end[j]) ++j;
  if (idx >= f.chunk_end[j]) return;
  idx -= j ? f.chunk_end[j - 1] : 0;
  const LfSegTable& segs = f.segs[j];
  if (segs.debug & 16) return;
  const int chunks = segs.rtot / 8;
  const int row = (int)(idx / chunks);
  const int c = (int)(idx - (int64_t)row * chunks) * 8;
  finalize_chunk(segs, f.routes[j][row / LF_TILE_M], row, c, f.ws[j], f.out[j]);
}

int finalize_launch(const LfSegTable& segs, const LfRoute* routes, float* ws, void* out, cudaStream_t stream) {
  const int64_t threads = (int64_t)segs.m * (segs.rtot / 8);
  return launch_k(lf_finalize_kernel, dim3((unsigned)((threads + 127) / 128)), dim3(128), 0, stream, segs, routes, ws,
                  reinterpret_cast<__nv_bfloat16*>(out));
}

int down_launch(const CUtensorMap& tm_x, const CUtensorMap& tm_a, const DownArgs& args, int num_sms,
                cudaStream_t stream) {
  int stages = 0, stage_bytes = 0;
  down_config(args.segs.wmax, &stages, &stage_bytes);
  const bool expl = args.segs.mask_mode == 2;
  const int smem = stages * stage_bytes + 1024 + 256 + down_extra_smem(args.segs.mask_mode);
  auto kern = expl ? lf_down_kernel<true> : lf_down_kernel<false>;
  static std::atomic<uint64_t> attr_done[2] = {0, 0};
  if (ensure_smem_attr(kern, 200 * 1024, attr_done[expl ? 1 : 0])) return -1;
  return launch_k(kern, dim3(args.ctas), dim3(kDownThreads), smem, stream, tm_x, tm_a, args, stages, stage_bytes);
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
    const PhiloxRow pr = philox_row(t.seg[seg], (uint32_t)(row + t.row_base), table_offset(t));
    b0 = keep_bits64_philox(pr, col);
    b1 = keep_bits64_philox(pr, col + 64);
  }
}

constexpr int kDgaThreads = 320;  // producer, MMA, 8 mask warps (2 per row quadrant; 4 also flush)

namespace dga {
constexpr int X_BYTES = 2 * 128 * 64 * 2;  // two 64-column SW128 boxes of 128 rows = 32 KB
constexpr int MAX_SMEM = 200 * 1024;
}  // namespace dga

__global__ void __launch_bounds__(kDgaThreads, 2)
    lf_dgrad_a_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmD,
                      const __grid_constant__ CUtensorMap tmK, const __grid_constant__ GradDownArgs args, int stages,
                      int stage_bytes) {
  using namespace dga;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* masked = empty + stages;
  uint64_t* tfull = masked + stages;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint64_t* tzero = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tzero + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int tiles_m = (args.m + 127) / 128;
  const int tiles_k = (args.k + 127) / 128;
  const int rtot = args.rtot;
  // stage: X | dŜ columns (up to the widest routing hull) | keep bits (16 B x 128 rows)
  const int KBITS_OFF = X_BYTES + (args.segs.wmax / 16) * 4096;
  // stream-K over (k-tile, m-tile) units, k-tile major: a span = one k-tile's dAᵀ columns
  // summed over a run of m-tiles. Two zero-initialised accumulators (R columns each).
  const int u0 = (int)((int64_t)blockIdx.x * tiles_m * tiles_k / gridDim.x);
  const int u1 = (int)((int64_t)(blockIdx.x + 1) * tiles_m * tiles_k / gridDim.x);
  uint32_t tmem_cols = 32;
  while ((int)tmem_cols < 2 * rtot) tmem_cols <<= 1;
  // profiling bit 64: stages bypass the mask warps (results invalid)
  auto needs_mask = [&](const LfRoute& rt) { return !(args.segs.debug & 64) && tile_needs_mask(args.segs, rt); };
  // every stage passes through the mask warps when the problem has any dropout (see ①)
  const bool gated = args.segs.mask_mode != 0 && !(args.segs.debug & 64);
  auto live = [&](int u) {  // next unit at or after u whose row tile carries adapters
    while (u < u1 && args.routes[u % tiles_m].col_hi <= args.routes[u % tiles_m].col_lo) ++u;
    return u;
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&masked[s], 8);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    mbar_init(tzero, 4);
    fence_barrier_init();
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmD);
    if (args.bits_tma) tma_prefetch_desc(&tmK);
  }
  pdl_launch_dependents();
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // the prologue above overlaps the predecessor's tail; global memory only from here
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = live(u0); u < u1; u = live(u + 1)) {
        const int mt = u % tiles_m, kt = u / tiles_m;
        const LfRoute rt = args.routes[mt];
        const int N = rt.col_hi - rt.col_lo;
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sX = smem + stage * stage_bytes;
        uint8_t* sD = sX + X_BYTES;
        const bool kbits = args.bits_tma && needs_mask(rt);
        mbar_arrive_expect_tx(&full[stage], X_BYTES + (N / 16) * 4096 + (kbits ? 2048 : 0));
        tma_load_2d(sX, &tmX, &full[stage], kt * 128, mt * 128);
        tma_load_2d(sX + 16384, &tmX, &full[stage], kt * 128 + 64, mt * 128);
        for (int j = 0; j < N / 16; ++j) tma_load_2d(sD + j * 4096, &tmD, &full[stage], rt.col_lo + 16 * j, mt * 128);
        if (kbits) tma_load_2d(sX + KBITS_OFF, &tmK, &full[stage], kt * 16, mt * 128);
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // whole warp, one elected lane issues (uniform-datapath descriptors)
    mbar_wait(tzero, 0);
    tc_fence_after();
    int stage = 0, it = 0;
    uint32_t phase = 0;
    bool open = false;
    for (int u = live(u0); u < u1;) {
      const int mt = u % tiles_m, kt = u / tiles_m;
      const int nxt = live(u + 1);
      const int b = it & 1;
      if (!open) {
        mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        open = true;
      }
      const LfRoute rt = args.routes[mt];
      const int N = rt.col_hi - rt.col_lo;
      mbar_wait(gated ? &masked[stage] : &full[stage], phase);
      tc_fence_after();
      const uint32_t sX = smem_u32(smem + stage * stage_bytes);
      const uint64_t ax = make_sdesc(sX, 16384, 1024, kLayoutSW128);
      const uint64_t bd = make_sdesc(sX + X_BYTES, 4096, 256, kLayoutSW32);
      const uint32_t idesc = make_idesc_bf16(128, (uint32_t)N, true, true);
      const uint32_t d = tmem + b * rtot + rt.col_lo;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (!(args.segs.debug & 1))
          umma_bf16_warp(d, sdesc_add(ax, kk * 2048), sdesc_add(bd, kk * 512), idesc, 1u);
      }
      umma_commit_warp(&empty[stage]);
      if (++stage == stages) { stage = 0; phase ^= 1; }
      if (nxt >= u1 || nxt / tiles_m != kt) {  // span ends: hand the accumulator to the flush
        umma_commit_warp(&tfull[b]);
        ++it;
        open = false;
      }
      u = nxt;
    }
    __syncwarp();
  } else {
    const uint32_t q = warp & 3u;
    const uint32_t taddr = tmem + ((q * 32u) << 16);
    uint32_t z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = 0u;
    // zero both accumulators so every MMA may accumulate (warps 2..5: one per lane quadrant)
    if (warp < 6) {
      for (int c = 0; c < 2 * rtot; c += 16) tmem_st16(taddr + c, z);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tzero);
    }
    const int rit = (int)(q * 32 + lane);
    const int half = warp >= 6 ? 1 : 0;  // which 64-column box of the unit this warp masks
    int stage = 0, it = 0;
    uint32_t phase = 0;
    uint32_t touched = 0;  // 16-column groups of the open span that received contributions
    for (int cur = live(u0); cur < u1;) {
      const int nxt = live(cur + 1);
      const int mt = cur % tiles_m, kt = cur / tiles_m;
      const LfRoute rt = args.routes[mt];
      for (int c = rt.col_lo; c < rt.col_hi; c += 16) touched |= 1u << (c >> 4);
      if (gated) {
        const int row = mt * 128 + rit;
        const int seg = row < args.m ? find_segment(args.segs, rt.seg_lo, rt.seg_hi, row) : -1;
        const bool mine = seg >= 0 && (args.segs.mask_mode == 2 || args.segs.seg[seg].thr != 0);
        uint64_t bits = ~0ull;
        if (mine && !args.bits_tma) {  // fallback: fetched before the wait so it overlaps the TMA
          if (args.segs.mask_mode == 1 && args.segs.bits) {
            bits = load_bits64(args.segs.bits + (int64_t)row * args.segs.ld_bits, kt * 16 + 8 * half,
                               (int)args.segs.ld_bits);
          } else {
            uint64_t b0, b1;
            dgrad_a_keep_slow(args.segs, seg, row, kt * 128, args.k, b0, b1);
            bits = half ? b1 : b0;
          }
        }
        mbar_wait(&full[stage], phase);
        if (mine) {
          uint8_t* sX = smem + stage * stage_bytes;
          if (args.bits_tma) bits = lds64(smem_u32(sX + KBITS_OFF) + (uint32_t)(rit * 16 + half * 8));
          if (!(args.segs.debug & 8)) apply_row_sw128(sX + half * 16384, rit, bits);
        }
        if (!(args.segs.debug & 4)) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&masked[stage]);
      }
      if (++stage == stages) { stage = 0; phase ^= 1; }
      if (half == 0 && (nxt >= u1 || nxt / tiles_m != kt)) {
        // flush the span: dA_catᵀ rows of this k-tile += accumulator, then re-zero it
        const int b = it & 1;
        mbar_wait(&tfull[b], (it >> 1) & 1);
        tc_fence_after();
        const int kcol = kt * 128 + rit;
        for (int g = 0; g < rtot / 16; ++g) {
          if (!((touched >> g) & 1u)) continue;
          uint32_t v[16];
          tmem_ld16(taddr + b * rtot + g * 16, v);
          tmem_ld_wait();
          if (kcol < args.k && !(args.segs.debug & 2)) {
#pragma unroll
            for (int j = 0; j < 16; ++j) red_add_f32(args.da + (int64_t)(g * 16 + j) * args.k + kcol, __uint_as_float(v[j]));
          }
          tmem_st16(taddr + b * rtot + g * 16, z);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
        ++it;
        touched = 0;
      }
      cur = nxt;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
}

// 2 CTAs / SM x ~110 KB rings (with TMA'd keep bits, 2 KB more per stage: 2 stages each).
void grad_down_config(int wmax, bool bits_tma, int* stages, int* stage_bytes) {
  *stage_bytes = dga::X_BYTES + (wmax / 16) * 4096 + (bits_tma ? 2048 : 0);
  static const int budget_kb = [] { const char* e = getenv("LF_DGA_SMEM_KB"); return e ? atoi(e) : 0; }();
  // ~110 KB rings so two CTAs share each SM (with keep bits too: 2 x 2 stages beat one CTA
  // with a 5-stage ring by 18-20%, kbench m = 8192/16384) unless R makes a stage too big
  (void)bits_tma;
  int s = (budget_kb > 0 ? budget_kb * 1024 : 112 * 1024) / *stage_bytes;
  *stages = s < 2 ? 2 : (s > 6 ? 6 : s);
}

int grad_down_launch(const CUtensorMap& tm_x, const CUtensorMap& tm_ds, const CUtensorMap& tm_bits,
                     const GradDownArgs& args, int num_sms, cudaStream_t stream) {
  (void)num_sms;
  int stages = 0, stage_bytes = 0;
  grad_down_config(args.segs.wmax, args.bits_tma != 0, &stages, &stage_bytes);
  const int smem = stages * stage_bytes + 1024 + 256;
  static std::atomic<uint64_t> attr_done{0};
  if (ensure_smem_attr(lf_dgrad_a_kernel, dga::MAX_SMEM + 2048, attr_done)) return -1;
  return launch_k(lf_dgrad_a_kernel, dim3(args.ctas), dim3(kDgaThreads), smem, stream, tm_x, tm_ds, tm_bits, args,
                  stages, stage_bytes);
}

// ------------------------------------------------------------------------------------
// ④ for a shared-input group: dA_j += dŜ_jᵀ·(M_j⊙X), j = 0..J-1, one launch
// ------------------------------------------------------------------------------------
// Units (k-tile, m-tile, projection), projection fastest: the X tile of (k-tile, m-tile) is
// TMA-loaded J times in a row — the first load streams it from DRAM, the others hit L2 —
// and each copy is masked in place with its own projection's keep bits (mask warps), so the
// MMA of projection j reads M_j⊙X. Stream-K as ④: every CTA takes an equal contiguous share
// of the units; a span is one k-tile's run, flushed per projection with red.global.add.
__global__ void __launch_bounds__(kDgaThreads, 2)
    lf_dgrad_a_group_kernel(const __grid_constant__ GroupDownMaps maps, const __grid_constant__ GroupDownArgs args,
                            int stages, int stage_bytes) {
  using namespace dga;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* masked = empty + stages;
  uint64_t* tfull = masked + stages;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint64_t* tzero = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tzero + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int J = args.J;
  const int tiles_m = (args.m + 127) / 128;
  const int tiles_k = (args.k + 127) / 128;
  const int per_k = tiles_m * J;  // units per k-tile
  const int units = tiles_k * per_k;
  const int KBITS_OFF = X_BYTES + (args.rmax / 16) * 4096;
  const int u0 = (int)((int64_t)blockIdx.x * units / gridDim.x);
  const int u1 = (int)((int64_t)(blockIdx.x + 1) * units / gridDim.x);
  uint32_t tmem_cols = 32;
  while ((int)tmem_cols < 2 * args.rsum) tmem_cols <<= 1;
  bool gated = false;
  for (int j = 0; j < J; ++j) gated |= args.masked[j] != 0;
  if (args.debug & 64) gated = false;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&masked[s], 8);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    mbar_init(tzero, 4);
    fence_barrier_init();
    tma_prefetch_desc(&maps.x);
    for (int j = 0; j < J; ++j) {
      tma_prefetch_desc(&maps.d[j]);
      if (args.masked[j]) tma_prefetch_desc(&maps.bits[j]);
    }
  }
  pdl_launch_dependents();
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = u0; u < u1; ++u) {
        const int kt = u / per_k, r = u - kt * per_k, mt = r / J, j = r - mt * J;
        const int R = args.R[j];
        const bool kb = args.masked[j] && gated;
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sX = smem + stage * stage_bytes;
        mbar_arrive_expect_tx(&full[stage], X_BYTES + (R / 16) * 4096 + (kb ? 2048 : 0));
        tma_load_2d(sX, &maps.x, &full[stage], kt * 128, mt * 128);
        tma_load_2d(sX + 16384, &maps.x, &full[stage], kt * 128 + 64, mt * 128);
        for (int g = 0; g < R / 16; ++g) tma_load_2d(sX + X_BYTES + g * 4096, &maps.d[j], &full[stage], 16 * g, mt * 128);
        if (kb) tma_load_2d(sX + KBITS_OFF, &maps.bits[j], &full[stage], kt * 16, mt * 128);
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    mbar_wait(tzero, 0);
    tc_fence_after();
    int stage = 0, it = 0;
    uint32_t phase = 0;
    bool open = false;
    for (int u = u0; u < u1; ++u) {
      const int kt = u / per_k, r = u - kt * per_k, mt = r / J, j = r - mt * J;
      (void)mt;
      const int b = it & 1;
      if (!open) {
        mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        open = true;
      }
      const int R = args.R[j];
      mbar_wait(gated ? &masked[stage] : &full[stage], phase);
      tc_fence_after();
      const uint32_t sX = smem_u32(smem + stage * stage_bytes);
      const uint64_t ax = make_sdesc(sX, 16384, 1024, kLayoutSW128);
      const uint64_t bd = make_sdesc(sX + X_BYTES, 4096, 256, kLayoutSW32);
      const uint32_t idesc = make_idesc_bf16(128, (uint32_t)R, true, true);
      const uint32_t d = tmem + b * args.rsum + args.off[j];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (!(args.debug & 1)) umma_bf16_warp(d, sdesc_add(ax, kk * 2048), sdesc_add(bd, kk * 512), idesc, 1u);
      }
      umma_commit_warp(&empty[stage]);
      if (++stage == stages) { stage = 0; phase ^= 1; }
      if (u + 1 >= u1 || (u + 1) / per_k != kt) {  // span ends: hand the accumulators to the flush
        umma_commit_warp(&tfull[b]);
        ++it;
        open = false;
      }
    }
    __syncwarp();
  } else {
    const uint32_t q = warp & 3u;
    const uint32_t taddr = tmem + ((q * 32u) << 16);
    uint32_t z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = 0u;
    if (warp < 6) {
      for (int c = 0; c < 2 * args.rsum; c += 16) tmem_st16(taddr + c, z);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tzero);
    }
    const int rit = (int)(q * 32 + lane);
    const int half = warp >= 6 ? 1 : 0;
    int stage = 0, it = 0;
    uint32_t phase = 0;
    uint32_t touched = 0;  // projections with contributions in the open span
    for (int u = u0; u < u1; ++u) {
      const int kt = u / per_k, r = u - kt * per_k, mt = r / J, j = r - mt * J;
      touched |= 1u << j;
      if (gated) {
        const int row = mt * 128 + rit;
        mbar_wait(&full[stage], phase);
        if (args.masked[j] && row < args.m) {
          uint8_t* sX = smem + stage * stage_bytes;
          const uint64_t bits = lds64(smem_u32(sX + KBITS_OFF) + (uint32_t)(rit * 16 + half * 8));
          if (!(args.debug & 8)) apply_row_sw128(sX + half * 16384, rit, bits);
        }
        if (!(args.debug & 4)) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&masked[stage]);
      }
      if (++stage == stages) { stage = 0; phase ^= 1; }
      if (half == 0 && (u + 1 >= u1 || (u + 1) / per_k != kt)) {
        const int b = it & 1;
        mbar_wait(&tfull[b], (it >> 1) & 1);
        tc_fence_after();
        const int kcol = kt * 128 + rit;
        for (int jj = 0; jj < J; ++jj) {
          if (!((touched >> jj) & 1u)) continue;
          for (int g = 0; g < args.R[jj] / 16; ++g) {
            uint32_t v[16];
            const uint32_t a = taddr + b * args.rsum + args.off[jj] + g * 16;
            tmem_ld16(a, v);
            tmem_ld_wait();
            if (kcol < args.k && !(args.debug & 2)) {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                red_add_f32(args.da[jj] + (int64_t)(g * 16 + i) * args.k + kcol, __uint_as_float(v[i]));
            }
            tmem_st16(a, z);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
        ++it;
        touched = 0;
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

void grad_down_group_config(int rmax, int* stages, int* stage_bytes) {
  *stage_bytes = dga::X_BYTES + (rmax / 16) * 4096 + 2048;
  const int s = (112 * 1024) / *stage_bytes;
  *stages = s < 2 ? 2 : (s > 6 ? 6 : s);
}

int grad_down_group_launch(const GroupDownMaps& maps, const GroupDownArgs& args, cudaStream_t stream) {
  int stages = 0, stage_bytes = 0;
  grad_down_group_config(args.rmax, &stages, &stage_bytes);
  const int smem = stages * stage_bytes + 1024 + 256;
  static std::atomic<uint64_t> attr_done{0};
  if (ensure_smem_attr(lf_dgrad_a_group_kernel, dga::MAX_SMEM + 2048, attr_done)) return -1;
  return launch_k(lf_dgrad_a_group_kernel, dim3(args.ctas), dim3(kDgaThreads), smem, stream, maps, args, stages,
                  stage_bytes);
}

// ------------------------------------------------------------------------------------
// routing table and explicit keep mask
// ------------------------------------------------------------------------------------
__global__ void lf_routes_kernel(const __grid_constant__ LfSegTable segs, LfRoute* routes, int ntiles) {
  pdl_wait();
  pdl_launch_dependents();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int r0 = t * LF_TILE_M;
  const int r1 = min(segs.m, r0 + LF_TILE_M);
  int lo = -1, hi = -2, c0 = 0, c1 = 0;
  for (int i = 0; i < segs.nseg; ++i) {
    const LfSegDev& s = segs.seg[i];
    if (s.row0 < s.row1 && s.row0 < r1 && s.row1 > r0) {
      // column blocks may be shared by segments of one adapter: take the union's hull
      if (lo < 0) {
        lo = i;
        c0 = s.col0;
        c1 = s.col0 + s.ncol;
      } else {
        c0 = min(c0, s.col0);
        c1 = max(c1, s.col0 + s.ncol);
      }
      hi = i;
    }
  }
  LfRoute r;
  if (lo < 0) {
    r.seg_lo = 0; r.seg_hi = -1; r.col_lo = 0; r.col_hi = 0;
  } else {
    r.seg_lo = lo; r.seg_hi = hi;
    r.col_lo = c0;
    r.col_hi = c1;
  }
  routes[t] = r;
}

__global__ void lf_mask_kernel(const __grid_constant__ LfSegTable segs, int32_t k, uint8_t* keep) {
  pdl_wait();
  pdl_launch_dependents();
  const int groups = (k + 7) / 8;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)segs.m * groups) return;
  const int row = (int)(idx / groups);
  const int g = (int)(idx - (int64_t)row * groups);
  uint32_t bits = 0xFFu;
  const int seg = find_segment(segs, 0, segs.nseg - 1, row);
  if (seg >= 0 && segs.mask_mode == 1 && segs.seg[seg].thr)
    bits = philox_keep8((uint32_t)g, (uint32_t)(row + segs.row_base), segs.seg[seg], table_offset(segs));
  uint8_t* out = keep + (int64_t)row * k + g * 8;
  for (int e = 0; e < 8; ++e)
    if (g * 8 + e < k) out[e] = (uint8_t)((bits >> e) & 1u);
}

// Packed keep bits (SPEC.md §3; bit c of byte j = column 8j + c) of the whole m x k mask,
// one thread per (row, 64-column group). Input-free: it depends only on (seed, offset, row,
// column). Rows outside every dropout segment keep everything.
__global__ void __launch_bounds__(256) lf_keep_bits_kernel(const __grid_constant__ LfSegTable segs, int32_t k,
                                                           uint8_t* bits, int64_t ld) {
  pdl_wait();
  pdl_launch_dependents();
  const int groups = (k + 63) / 64;
  const int64_t total = (int64_t)segs.m * groups;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(idx / groups);
    const int g = (int)(idx - (int64_t)row * groups);
    const int seg = find_segment(segs, 0, segs.nseg - 1, row);
    uint64_t b = ~0ull;
    if (seg >= 0 && segs.seg[seg].thr) {
      uint32_t msk[8][4];
      b = philox_masks<8>(philox_row(segs.seg[seg], (uint32_t)(row + segs.row_base), table_offset(segs)), g * 64, msk);
    }
    uint8_t* out = bits + (int64_t)row * ld + g * 8;
    const int nbytes = min(8, (k - g * 64 + 7) / 8);
    if (nbytes == 8 && ((reinterpret_cast<uintptr_t>(out) & 7u) == 0)) {
      *reinterpret_cast<uint64_t*>(out) = b;
    } else {
      for (int i = 0; i < nbytes; ++i) out[i] = (uint8_t)(b >> (8 * i));
    }
  }
}

int keep_bits_launch(const LfSegTable& segs, int32_t k, uint8_t* bits, int64_t ld, int num_sms, cudaStream_t stream) {
  const int64_t total = (int64_t)segs.m * ((k + 63) / 64);
  if (total <= 0) return 0;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 4LL * num_sms) blocks = 4LL * num_sms;
  return launch_k(lf_keep_bits_kernel, dim3((unsigned)blocks), dim3(256), 0, stream, segs, k, bits, ld);
}

int routes_launch(const LfSegTable& segs, int32_t* routes, int ntiles, cudaStream_t stream) {
  if (ntiles <= 0) return 0;
  return launch_k(lf_routes_kernel, dim3((ntiles + 127) / 128), dim3(128), 0, stream, segs,
                  reinterpret_cast<LfRoute*>(routes), ntiles);
}

int mask_launch(const LfSegTable& segs, int32_t k, uint8_t* keep, cudaStream_t stream) {
  const int64_t total = (int64_t)segs.m * ((k + 7) / 8);
  if (total <= 0) return 0;
  return launch_k(lf_mask_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, stream, segs, k, keep);
}

// Column blocks out of fp32 row-major matrices into contiguous buffers (dB_cat n x R ->
// each adapter's n x r gradient): one launch for every block of a call; blockIdx.y picks the
// block, the x grid strides over its elements (4 floats per thread where alignment allows).
__global__ void __launch_bounds__(256) lf_copy_blocks_kernel(const __grid_constant__ CopyBlocksArgs a) {
  pdl_wait();
  pdl_launch_dependents();
  const CopyBlock& b = a.blk[blockIdx.y];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool vec = ((b.width | b.ld | b.col) & 3) == 0 && ((reinterpret_cast<uintptr_t>(b.src) | reinterpret_cast<uintptr_t>(b.dst)) & 15u) == 0;
  if (vec) {
    const int w4 = b.width >> 2;
    const int64_t total = (int64_t)b.rows * w4;
    for (int64_t i = t0; i < total; i += stride) {
      const int64_t r = i / w4;
      const int c = (int)(i - r * w4) * 4;
      const float4 v = *reinterpret_cast<const float4*>(b.src + r * b.ld + b.col + c);
      *reinterpret_cast<float4*>(b.dst + r * b.width + c) = v;
    }
  } else {
    const int64_t total = (int64_t)b.rows * b.width;
    for (int64_t i = t0; i < total; i += stride) {
      const int64_t r = i / b.width;
      const int c = (int)(i - r * b.width);
      b.dst[r * b.width + c] = b.src[r * b.ld + b.col + c];
    }
  }
}

int copy_blocks_launch(const CopyBlocksArgs& a, int num_sms, cudaStream_t stream) {
  if (a.n <= 0) return 0;
  int64_t most = 0;
  for (int i = 0; i < a.n; ++i) most = max(most, (int64_t)a.blk[i].rows * a.blk[i].width);
  int64_t gx = (most / 4 + 255) / 256;
  const int64_t cap = (4LL * num_sms + a.n - 1) / a.n;  // ~4 CTAs per SM over all blocks
  if (gx > cap) gx = cap;
  if (gx < 1) gx = 1;
  return launch_k(lf_copy_blocks_kernel, dim3((unsigned)gx, (unsigned)a.n), dim3(256), 0, stream, a);
}

}  // namespace lf
