// lf_gemm.cu — ② base_gemm_epilogue_fused and ⑤ grad_base_accum_fused on sm_100a.
//
// Reference contract: ls/costmodel.py:262-264 (Y = X·W + α·S·B written once) and
// ls/costmodel.py:273-277 (dX = dY·Wᵀ + mask ⊙ LoRA term, one dX write);
// paper design PAPER.md:457-463.
//
// B200 design: persistent, warp-specialised tcgen05 GEMM on CTA pairs (cluster 2x1x1,
// cta_group::2). A pair owns a 256x256 output tile: each CTA TMA-loads its 128-row half of
// A and its 128-column half of B into its own shared memory (completion counted on the
// leader's mbarrier), the leader issues tcgen05.mma M=256 N=256 K=16 over both halves, and
// each CTA's TMEM holds the fp32 accumulator of its 128 rows (double-buffered, 2 x 256
// columns) — half the shared-memory operand traffic per FLOP of a single-CTA 128x256 tile.
//   warp 0      TMA producer (one lane per CTA)
//   warp 1      MMA issuer (one lane, leader CTA only) + TMEM allocation (both CTAs)
//   warps 2..9  epilogue, two per TMEM lane quadrant (half the columns each): tcgen05.ld -> bf16
//               -> global (and, for ⑤ with dropout, the mask pass)
// The low-rank up-projection is NOT an epilogue GEMM: [X | Ŝ]·[W | B_cat]ᵀ — the rank-R
// LoRA operands are streamed as extra K-blocks into the same accumulator, so the output
// tile is written exactly once and the epilogue stays a pure convert.
//
// ⑤ with dropout: the mask multiplies only the LoRA term (dX = dY·W + M ⊙ (dŜ·A_cat)),
// so the LoRA K-block of a tile is issued FIRST into its (empty) accumulator, the
// epilogue warps zero the dropped elements of that partial in TMEM (tcgen05.ld → keep
// bits → tcgen05.st), and only then is the main dY·W loop accumulated on top. The LoRA
// block of tile i+1 is issued half-way through tile i's main loop, so its mask pass
// runs while the tensor pipe is busy with tile i.
#include <cstdlib>

#include "lf_device.cuh"
#include "lf_kernels.h"

namespace lf {

constexpr int kEpiWarps = 8;                         // warps 2..9
constexpr int kGemmThreads = 32 * (2 + kEpiWarps);   // producer, MMA, epilogue

// control block after the operand ring: mbarriers, TMEM slot, tile-sequence ring
constexpr int kGemmCtlBytes = 512;
constexpr int kSeqDepth = 6;  // CLC responses in flight / not yet released

// WIDE: 256 x 512 pair tiles — two N = 256 MMAs per K-step share each A slice, one
// 512-column accumulator (no double buffer): 25% less operand traffic from L2 and smem per
// FLOP than 256 x 256, which is what the power-capped long GEMMs (C4) are bound by.
template <bool B_MN, int STAGES, bool WIDE = false>
struct GemmCfg {
  static constexpr int BM = 128;                  // rows per CTA (pair tile: 256)
  static constexpr int BN = WIDE ? 512 : 256;     // pair tile columns; each CTA loads BN/2 of B
  static constexpr int NH = BN / 256;             // N = 256 MMAs per K-step
  static constexpr int NACC = WIDE ? 1 : 2;       // TMEM accumulator buffers
  static constexpr int HBN = BN / 2;
  static constexpr int BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;     // 16 KB, K-major SW128
  static constexpr int B_BYTES = HBN * BK * 2;    // 16 KB (WIDE: 32 KB, two 128-row pieces)
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int ACC_COLS = BN;
  static constexpr int TMEM_COLS = NACC * ACC_COLS;  // 512
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + kGemmCtlBytes + 512 * 16;  // + routing cache
};

// grouped raster: G m-tiles share each n-column sweep so W tiles stay L2-hot
__device__ __forceinline__ void gemm_tile_coords(int t, int tiles_m, int tiles_n, int G, int& mb, int& nb) {
  const int per_group = G * tiles_n;
  const int g = t / per_group;
  const int first_m = g * G;
  const int gm = min(G, tiles_m - first_m);
  const int r = t - g * per_group;
  mb = first_m + r % gm;
  nb = r / gm;
}

struct TileInfo {
  int mb, nb;          // cluster-tile coordinates: rows [mb * NP * 256, +NP * 256), columns [nb * BN, +BN)
  int col_lo, col_hi;  // LoRA K-range: union over the cluster tile's 128-row routes (every pair of
                       // the cluster streams the same stages: the multicast operand is shared)
  int proj, noff;      // GRP forward: projection owning the tile's columns, its first column
  __device__ bool lora() const { return col_hi > col_lo; }
};

constexpr int kSmemRoutes = 512;  // routing entries staged in smem (m <= 65536); beyond: global

// the single-thread producer / MMA roles must not stall on a dependent global load per
// tile: the routing table is staged in shared memory once per CTA
__device__ __forceinline__ LfRoute route_at(const GemmArgs& a, const LfRoute* s_routes, int r) {
  return r < kSmemRoutes ? s_routes[r] : a.routes[r];
}

template <int NP>
__device__ __forceinline__ TileInfo tile_info(const GemmArgs& a, const LfRoute* s_routes, int t) {
  TileInfo ti;
  gemm_tile_coords(t, a.tiles_m, a.tiles_n, a.group, ti.mb, ti.nb);
  ti.col_lo = ti.col_hi = 0;
  if (a.routes && !(a.segs.debug & 2048)) {
    const int tiles128 = (a.M + 127) / 128;
    for (int h = 0; h < 2 * NP; ++h) {
      const int r = 2 * NP * ti.mb + h;
      if (r >= tiles128) break;
      const LfRoute rt = route_at(a, s_routes, r);
      if (rt.col_hi <= rt.col_lo) continue;
      if (ti.col_hi <= ti.col_lo) {
        ti.col_lo = rt.col_lo;
        ti.col_hi = rt.col_hi;
      } else {
        ti.col_lo = min(ti.col_lo, rt.col_lo);
        ti.col_hi = max(ti.col_hi, rt.col_hi);
      }
    }
  }
  return ti;
}

// Fallback keep bits when ① did not leave a packed mask (explicit uint8 mask, or Philox
// regenerated here). Kept out of line: inlined into the unrolled mask pass it multiplies the
// kernel's code size ~15x and the epilogue warps' instruction fetch starts evicting the
// single-thread producer / MMA loops from the instruction cache.
__device__ __noinline__ uint32_t dgrad_keep32_slow(const LfSegTable& t, int seg, int row, int col, int ncols) {
  uint32_t v = 0;
  for (int j = 0; j < 4; ++j) {
    const int cc = col + 8 * j;
    const uint32_t b = (t.mask_mode == 2) ? explicit_keep8(t.mask + (int64_t)row * t.ld_mask, cc, ncols)
                                           : philox_keep8((uint32_t)cc >> 3, (uint32_t)(row + t.row_base), t.seg[seg], table_offset(t));
    v |= b << (8 * j);
  }
  return v;
}

// keep bits (4 bytes = 32 columns, byte j = columns col+8j..col+8j+7) of one row for the
// ⑤ mask pass: the bit-packed mask written by ① when present
__device__ __forceinline__ uint32_t dgrad_keep32(const LfSegTable& t, int seg, int row, int col, int ncols) {
  if (t.mask_mode == 1 && t.bits) {
    const uint8_t* rb = t.bits + (int64_t)row * t.ld_bits;
    const int b0 = col >> 3;
    const int nb = (int)t.ld_bits;
    if (b0 + 4 <= nb && ((reinterpret_cast<uintptr_t>(rb + b0) & 3u) == 0))
      return *reinterpret_cast<const uint32_t*>(rb + b0);
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i)
      if (b0 + i < nb) v |= (uint32_t)rb[b0 + i] << (8 * i);
    return v;
  }
  return dgrad_keep32_slow(t, seg, row, col, ncols);
}

// `accumulate` (lf_grad_input_accum): C += result, the input gradient of projections that
// share X summed by the GEMMs instead of separate elementwise adds. The epilogue hands the
// addition to L2 (red.global.add.noftz.v4.bf16x2: 8 bf16 per lane, each element added once
// per launch, so the sum is deterministic): no load of the old C, no round trip in the
// epilogue — a register read-modify-write cost short-K tiles 30% (k/v dgrad) and did not fit
// the 256 x 512 tiles' registers at all.
__device__ __forceinline__ void red_add_bf16x8(__nv_bfloat16* dst, uint4 v) {
  asm volatile("red.global.add.noftz.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void store_c8(__nv_bfloat16* dst, uint4 v, int accumulate) {
  if (accumulate)
    red_add_bf16x8(dst, v);
  else
    *reinterpret_cast<uint4*>(dst) = v;
}

// Tile sequence of one CTA pair. Dynamic (default): the grid has one cluster per tile; a
// pair starts on its own tile (blockIdx.x / 2) and then takes over not-yet-launched
// clusters' tiles through cluster launch control, in launch order — the tiles in flight
// always form one contiguous window of the raster, so pairs that run slower never drift
// onto data no other pair is reading (a static round-robin persistent schedule let them
// drift and re-read W from DRAM: 15 GB vs 4.8 GB per C4 gate launch, ncu).
// Response i (i >= 1) sits in slot (i-1) % kSeqDepth; every role of both CTAs reads each
// response once, in order, and releases it on the leader's `empty` barrier (19 readers:
// 2 producers, the MMA warp, 16 epilogue warps). Only the leader's producer requests, and
// only after the previous response named a tile, so no request is left unread at exit.
// Static (operands that fit in L2 together, or LF_SCHED=1): tile i = pair + i * npairs.
template <int CL>
struct TileSeq {
  uint64_t* full;   // [kSeqDepth] per CTA: response landed
  uint64_t* empty;  // [kSeqDepth] cluster rank 0: all readers done
  uint8_t* resp;    // [kSeqDepth][16]
  int cluster, nclusters, tiles;
  bool dynamic;

  // every CTA's producer, each pair leader's MMA warp, every CTA's 8 epilogue warps
  static constexpr uint32_t kReaders = CL * (1 + kEpiWarps) + CL / 2;

  __device__ int first() const { return cluster < tiles ? cluster : -1; }
  // cluster rank 0's producer only: ask for response i
  __device__ void request(int i) const {
    if (!dynamic) return;
    const int slot = (i - 1) % kSeqDepth;
    const uint32_t ph = (uint32_t)((i - 1) / kSeqDepth) & 1u;
    mbar_wait(&empty[slot], ph ^ 1u);
    const uint32_t fb = smem_u32(&full[slot]);
#pragma unroll
    for (int c = 0; c < CL; ++c) mbar_arrive_expect_tx_cluster(mapa_shared(fb, c), 16);
    clc_try_cancel_multicast(smem_u32(resp + 16 * slot), fb);
  }
  // every reader: tile of response i (waits for it), or -1 when the grid is exhausted.
  // Warp-wide readers call it with the whole warp; `arrive` = the one lane that releases.
  __device__ int read(int i, bool arrive) const {
    if (!dynamic) {
      const int t = cluster + i * nclusters;
      return t < tiles ? t : -1;
    }
    const int slot = (i - 1) % kSeqDepth;
    const uint32_t ph = (uint32_t)((i - 1) / kSeqDepth) & 1u;
    mbar_wait(&full[slot], ph);
    const int x = clc_first_ctaid_x(smem_u32(resp + 16 * slot));
    fence_proxy_async_smem();  // the next response into this slot is an async-proxy write
    if (arrive) mbar_arrive_cluster(mapa_shared(smem_u32(&empty[slot]), 0));
    return x < 0 ? -1 : (x / CL);
  }
};

// CL = CTAs per cluster: 2 = one CTA pair; 4 = two pairs stacked along M (cluster tile
// 512 x BN) that share the B operand — the pair-0 CTAs TMA-load each B tile once and
// multicast it into both pairs' shared memory (half the B reads from L2 per FLOP), and every
// pair leader's MMA commit releases the stage in all four CTAs.
// GRP (shared-input groups, lf_base_fwd_group / lf_grad_input_group): J = args.nseg
// projections that read the same input in ONE launch. Forward: the projections' output
// columns are concatenated (N segments) — a tile belongs to one projection, takes W_j's rows,
// the LoRA K-block of Ŝ_j / B_j and writes Y_j. Input gradient: their reduction dims are
// concatenated (K segments: dY_j·W_j summed in the accumulator, dX written once) and each
// projection's masked LoRA term M_j ⊙ (dŜ_j·A_j) enters the drained accumulator first: the
// J partials take turns in it (MMA → epilogue masks into registers → next partial), the
// masked sum goes back to TMEM, and the main loop accumulates on top.
template <bool B_MN, bool MASKED, int STAGES, bool WIDE, int CL, bool ACC, bool GRP>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(kGemmThreads, 1)
    lf_gemm_kernel(const __grid_constant__ GemmMaps maps, const __grid_constant__ GemmArgs args) {
  using Cfg = GemmCfg<B_MN, STAGES, WIDE>;
  constexpr int BN = Cfg::BN, HBN = Cfg::HBN, NH = Cfg::NH, NACC = Cfg::NACC;
  constexpr int NP = CL / 2;                                    // CTA pairs per cluster
  constexpr uint16_t kAllCtas = (uint16_t)((1u << CL) - 1u);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);  // pair leader: both halves landed
  uint64_t* empty = full + STAGES;   // every CTA: stage consumed by every pair (multicast commits)
  uint64_t* tfull = empty + STAGES;  // [2] both CTAs: main loop done
  uint64_t* tempty = tfull + 2;      // [2] leader: both CTAs drained the accumulator (16 warps)
  uint64_t* lfull = tempty + 2;      // [2] both CTAs: LoRA partial ready                 MASKED
  uint64_t* lmasked = lfull + 2;     // [2] leader: both CTAs masked their partial (16)  MASKED
  uint64_t* lnext = lmasked + 2;     // [2] leader: both CTAs read partial j < J-1 (16)  MASKED GRP
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lnext + 2);
  uint8_t* ctl = smem + STAGES * Cfg::STAGE_BYTES;
  TileSeq<CL> seq;
  seq.full = reinterpret_cast<uint64_t*>(ctl + 192);
  seq.empty = seq.full + kSeqDepth;
  seq.resp = ctl + 320;
  LfRoute* s_routes = reinterpret_cast<LfRoute*>(ctl + kGemmCtlBytes);  // [kSmemRoutes]
  pdl_launch_dependents();

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1u;        // rank within the CTA pair
  const uint32_t pid = crank >> 1;         // pair index within the cluster
  const uint32_t lrank = crank & ~1u;      // cluster rank of this pair's leader
  const bool leader = rank == 0;           // pair leader: issues the pair's MMAs
  const uint16_t pair_mask = (uint16_t)(0x3u << (2 * pid));

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NP);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);
      mbar_init(&lfull[a], 1);
      mbar_init(&lmasked[a], 2 * kEpiWarps);
      mbar_init(&lnext[a], 2 * kEpiWarps);
    }
    for (int i = 0; i < kSeqDepth; ++i) {
      mbar_init(&seq.full[i], 1);
      mbar_init(&seq.empty[i], TileSeq<CL>::kReaders);
    }
    fence_barrier_init();
    const int nmaps = GRP ? args.nseg : 1;
    for (int j = 0; j < nmaps; ++j) {
      tma_prefetch_desc(&maps.a[GRP && B_MN ? j : 0]);
      tma_prefetch_desc(&maps.b[j]);
      if (args.routes || GRP) {
        tma_prefetch_desc(&maps.a2[j]);
        tma_prefetch_desc(&maps.b2[j]);
      }
    }
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
  // everything above overlaps the predecessor's tail (PDL); global memory only from here
  pdl_wait();
  if (args.routes) {
    const int nr = min((args.M + 127) / 128, kSmemRoutes);
    for (int i = (int)threadIdx.x; i < nr; i += (int)blockDim.x) s_routes[i] = args.routes[i];
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int tiles = args.tiles_m * args.tiles_n;
  seq.cluster = blockIdx.x / CL;
  seq.nclusters = gridDim.x / CL;
  seq.tiles = tiles;
  seq.dynamic = args.dynamic != 0;
  const int nkb = (args.K + Cfg::BK - 1) / Cfg::BK;
  // MASKED: where the next tile's LoRA block is interleaved (debug 256: after the main loop,
  // 512: a quarter in, 1024: three quarters in)
  const int jmid = (args.segs.debug & 256) ? nkb : (args.segs.debug & 512) ? nkb / 4
                   : (args.segs.debug & 1024) ? (3 * nkb) / 4 : nkb / 2;
  // GRP: J projections (1 otherwise); the masked dgrad issues partial j of the next tile at
  // k-block split(j) of the current one (J = 1: jmid)
  const int J = GRP ? args.nseg : 1;
  auto split_at = [&](int j) { return min(nkb, jmid + (j * (nkb - jmid)) / J); };
  // GRP input gradient: K segment of k-block kb (projection j, its first k-block)
  auto kseg = [&](int kb, int& j, int& kb0) {
    j = 0;
    kb0 = 0;
    if constexpr (GRP && B_MN) {
      while (j + 1 < args.nseg && kb * Cfg::BK >= args.send[j]) {
        kb0 = args.send[j] / Cfg::BK;
        ++j;
      }
    }
  };
  auto tinfo = [&](int t) {
    TileInfo ti = tile_info<NP>(args, s_routes, t);
    ti.proj = 0;
    ti.noff = 0;
    if constexpr (GRP) {
      if constexpr (!B_MN) {
        const int n0 = ti.nb * BN;
        while (ti.proj + 1 < args.nseg && n0 >= args.send[ti.proj]) ++ti.proj;
        ti.noff = ti.proj ? args.send[ti.proj - 1] : 0;
      }
      ti.col_lo = 0;
      ti.col_hi = args.lcols[ti.proj];
    }
    return ti;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int row_half = (int)rank * Cfg::BM;  // this CTA's rows of its pair's 256-row tile
      // B (the operand every pair of the cluster shares): loaded by the pair-0 CTAs only, into
      // the same-rank CTA of every pair
      const bool loads_b = pid == 0;
      const uint16_t b_mask = (uint16_t)(((1u << CL) - 1u) & (0x5555u << rank));
      auto load_b = [&](void* dst, const CUtensorMap* map, int c0, int c1) {
        if constexpr (CL == 2) {
          tma_load_2d_pair(dst, map, &full[stage], c0, c1);
        } else {
          if (loads_b) tma_load_2d_pair_mc(dst, map, &full[stage], c0, c1, b_mask);
        }
      };
      auto begin_stage = [&](uint32_t bytes) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (leader) mbar_arrive_expect_tx(&full[stage], 2 * bytes);
      };
      auto load_main = [&](const TileInfo& ti, int kb) {
        begin_stage(Cfg::STAGE_BYTES);
        uint8_t* sA = smem + stage * Cfg::STAGE_BYTES;
        uint8_t* sB = sA + Cfg::A_BYTES;
        int j, kb0;
        kseg(kb, j, kb0);  // GRP dgrad: dY_j / W_j hold k-blocks [kb0, ...) of the concatenated K
        const int kl = (kb - kb0) * Cfg::BK;
        tma_load_2d_pair(sA, &maps.a[j], &full[stage], kl, (ti.mb * NP + (int)pid) * 256 + row_half);
        if constexpr (!B_MN) {
          // N piece h of this CTA: rows h*256 + rank*128 of the pair tile's columns (GRP: of W_proj)
          const CUtensorMap* mb = &maps.b[ti.proj];
#pragma unroll
          for (int h = 0; h < NH; ++h)
            load_b(sB + h * 16384, mb, kl, ti.nb * BN - ti.noff + h * 256 + (int)rank * 128);
        } else {
#pragma unroll
          for (int h = 0; h < NH; ++h)
#pragma unroll
            for (int i = 0; i < 2; ++i)  // 128 MN-major columns = two 64-column SW128 boxes
              load_b(sB + h * 16384 + i * 8192, &maps.b[j], ti.nb * BN + h * 256 + (int)rank * 128 + 64 * i, kl);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      };
      // LoRA K-blocks [c_lo, c_hi) of operand pair j (Ŝ_j / B_j forward, dŜ_j / A_j dgrad)
      auto load_lora_j = [&](const TileInfo& ti, int j, int c_lo, int c_hi) {
        for (int c = c_lo; c < c_hi; c += 64) {
          const int nsub = min(4, (c_hi - c) >> 4);
          begin_stage(nsub * (Cfg::BM * 32 + HBN * 32));
          uint8_t* sA = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sB = sA + Cfg::A_BYTES;
          for (int u = 0; u < nsub; ++u) {
            tma_load_2d_pair(sA + u * (Cfg::BM * 32), &maps.a2[j], &full[stage], c + 16 * u,
                             (ti.mb * NP + (int)pid) * 256 + row_half);
            if constexpr (!B_MN) {
#pragma unroll
              for (int h = 0; h < NH; ++h)
                load_b(sB + (u * NH + h) * 4096, &maps.b2[j], c + 16 * u,
                       ti.nb * BN - ti.noff + h * 256 + (int)rank * 128);
            } else {
#pragma unroll
              for (int h = 0; h < NH; ++h)
#pragma unroll
                for (int i = 0; i < 2; ++i)
                  load_b(sB + (u * NH + h) * 4096 + i * 2048, &maps.b2[j],
                         ti.nb * BN + h * 256 + (int)rank * 128 + 64 * i, c + 16 * u);
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      };
      auto load_lora = [&](const TileInfo& ti) {
        if constexpr (GRP && B_MN) {  // every projection's block (p = 0: they all accumulate)
          for (int j = 0; j < J; ++j) load_lora_j(ti, j, 0, args.lcols[j]);
        } else {
          load_lora_j(ti, ti.proj, ti.col_lo, ti.col_hi);
        }
      };
      int t = seq.first();
      if (crank == 0 && t >= 0) seq.request(1);
      for (int i = 0; t >= 0; ++i) {
        const TileInfo ti = tinfo(t);
        int tn;
        if constexpr (MASKED && WIDE) {
          // one accumulator: each tile's own LoRA block first, then its main loop
          if (ti.lora()) load_lora(ti);
          for (int kb = 0; kb < nkb; ++kb) load_main(ti, kb);
          tn = seq.read(i + 1, true);
          if (crank == 0 && tn >= 0) seq.request(i + 2);
        } else if constexpr (MASKED) {
          // partial j of the next tile's LoRA term goes in at k-block split_at(j) of this
          // tile's main loop (J = 1: half-way); GRP: projection j's dŜ_j / A_j
          auto lora_part = [&](const TileInfo& tx, int j) {
            if constexpr (GRP) load_lora_j(tx, j, 0, args.lcols[j]);
            else load_lora(tx);
          };
          if (i == 0 && ti.lora())
            for (int j = 0; j < J; ++j) lora_part(ti, j);
          int kb = 0;
          tn = -1;
          TileInfo tni;
          for (int j = 0; j < J; ++j) {
            for (const int split = split_at(j); kb < split; ++kb) load_main(ti, kb);
            if (j == 0) {
              tn = seq.read(i + 1, true);
              if (crank == 0 && tn >= 0) seq.request(i + 2);
              if (tn >= 0) tni = tinfo(tn);
            }
            if (tn >= 0 && tni.lora()) lora_part(tni, j);
          }
          for (; kb < nkb; ++kb) load_main(ti, kb);
        } else {
          for (int kb = 0; kb < nkb; ++kb) load_main(ti, kb);
          if (ti.lora()) load_lora(ti);
          tn = seq.read(i + 1, true);
          if (crank == 0 && tn >= 0) seq.request(i + 2);
        }
        t = tn;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA, whole warp; one elected lane issues)
    if (leader) {
      const uint32_t idesc = make_idesc_bf16(256, 256, false, B_MN);  // N = 256 per instruction
      int stage = 0;
      uint32_t phase = 0;
      uint32_t lora_uses0 = 0, lora_uses1 = 0;  // MASKED: LoRA partials produced per accumulator buffer
      auto mma_main_block = [&](uint32_t d, int kb, bool acc_any) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t sA = smem_u32(smem + stage * Cfg::STAGE_BYTES);
        const uint32_t sB = sA + Cfg::A_BYTES;
        const uint64_t ad0 = make_sdesc(sA, 16, 1024, kLayoutSW128);
        const uint64_t bd0 = B_MN ? make_sdesc(sB, 8192, 1024, kLayoutSW128) : make_sdesc(sB, 16, 1024, kLayoutSW128);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int h = 0; h < NH; ++h)
            umma_bf16_pair_warp(d + h * 256, sdesc_add(ad0, kk * 32),
                                sdesc_add(bd0, (B_MN ? kk * 2048 : kk * 32) + h * 16384), idesc,
                                (acc_any || (kb | kk) != 0) ? 1u : 0u);
        umma_commit_pair_warp_mask(&empty[stage], kAllCtas);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      };
      auto mma_lora_cols = [&](int c_lo, int c_hi, uint32_t d, bool acc_any) {
        uint32_t accum = acc_any ? 1u : 0u;
        for (int c = c_lo; c < c_hi; c += 64) {
          const int nsub = min(4, (c_hi - c) >> 4);
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sA = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sB = sA + Cfg::A_BYTES;
          for (int j = 0; j < nsub; ++j) {
            const uint64_t ad = make_sdesc(sA + j * (Cfg::BM * 32), 16, 256, kLayoutSW32);
            for (int h = 0; h < NH; ++h) {
              const uint64_t bd = B_MN ? make_sdesc(sB + (j * NH + h) * 4096, 2048, 1024, kLayoutSW128)
                                       : make_sdesc(sB + (j * NH + h) * 4096, 16, 256, kLayoutSW32);
              umma_bf16_pair_warp(d + h * 256, ad, bd, idesc, accum);
            }
            accum = 1u;
          }
          umma_commit_pair_warp_mask(&empty[stage], kAllCtas);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      };
      auto mma_lora = [&](const TileInfo& ti, uint32_t d, bool acc_any) {
        if constexpr (GRP && B_MN) {
          for (int j = 0; j < J; ++j) mma_lora_cols(0, args.lcols[j], d, acc_any || j > 0);
        } else {
          mma_lora_cols(ti.col_lo, ti.col_hi, d, acc_any);
        }
      };
      uint32_t next_uses0 = 0, next_uses1 = 0;  // MASKED GRP: partials handed over per buffer
      // MASKED: LoRA partial j of local tile `it` into its (drained) buffer, then signal the
      // mask pass (GRP: partial j > 0 waits until the epilogue has read partial j - 1)
      auto issue_lora_first = [&](const TileInfo& ti, int it, int j) {
        const int acc = it % NACC;
        if (j == 0) {
          mbar_wait(&tempty[acc], ((it / NACC) & 1) ^ 1);
        } else {
          uint32_t& nu = acc ? next_uses1 : next_uses0;
          mbar_wait(&lnext[acc], nu & 1);
          ++nu;
        }
        tc_fence_after();
        if constexpr (GRP) mma_lora_cols(0, args.lcols[j], tmem_base + acc * Cfg::ACC_COLS, false);
        else mma_lora(ti, tmem_base + acc * Cfg::ACC_COLS, false);
        umma_commit_pair_warp_mask(&lfull[acc], pair_mask);
      };
      int t = seq.first();
      for (int it = 0; t >= 0; ++it) {
        const TileInfo ti = tinfo(t);
        const int acc = it % NACC;
        const uint32_t d = tmem_base + acc * Cfg::ACC_COLS;
        int tn = -1;
        bool have_tn = false;
        if constexpr (MASKED && WIDE) {
          // sequential: drained accumulator -> this tile's LoRA partial -> mask pass -> main loop
          mbar_wait(&tempty[acc], ((it / NACC) & 1) ^ 1);
          tc_fence_after();
          if (ti.lora()) {
            mma_lora(ti, d, false);
            umma_commit_pair_warp_mask(&lfull[acc], pair_mask);
            uint32_t& lu = lora_uses0;
            mbar_wait(&lmasked[acc], lu & 1);
            ++lu;
            tc_fence_after();
          }
          for (int kb = 0; kb < nkb; ++kb) mma_main_block(d, kb, ti.lora());
        } else if constexpr (MASKED) {
          if (it == 0 && ti.lora())
            for (int j = 0; j < J; ++j) issue_lora_first(ti, 0, j);
          if (ti.lora()) {
            uint32_t& lu = acc ? lora_uses1 : lora_uses0;
            mbar_wait(&lmasked[acc], lu & 1);
            ++lu;
          } else {
            mbar_wait(&tempty[acc], ((it / NACC) & 1) ^ 1);
          }
          tc_fence_after();
          const bool acc_any = ti.lora();
          int kb = 0;
          TileInfo tni;
          for (int j = 0; j < J; ++j) {
            for (const int split = split_at(j); kb < split; ++kb) mma_main_block(d, kb, acc_any);
            if (j == 0) {
              tn = seq.read(it + 1, lane_id() == 0);
              have_tn = true;
              if (tn >= 0) tni = tinfo(tn);
            }
            if (tn >= 0 && tni.lora()) issue_lora_first(tni, it + 1, j);
          }
          for (; kb < nkb; ++kb) mma_main_block(d, kb, acc_any);
        } else {
          mbar_wait(&tempty[acc], ((it / NACC) & 1) ^ 1);
          tc_fence_after();
          for (int kb = 0; kb < nkb; ++kb) mma_main_block(d, kb, false);
          if (ti.lora()) mma_lora(ti, d, true);
        }
        umma_commit_pair_warp_mask(&tfull[acc], pair_mask);
        if (!have_tn) tn = seq.read(it + 1, lane_id() == 0);
        t = tn;
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..9, both CTAs)
    // two warps per TMEM lane quadrant, each owning half of the tile's columns: the drain and
    // the ⑤ mask pass run at twice the width (short-K tiles were bound by them)
    const uint32_t q = warp & 3u;  // TMEM lane quadrant this warp may access
    const int c_lo = (warp >= 6 ? 1 : 0) * (BN / 2), c_hi = c_lo + BN / 2;
    const uint32_t tempty_leader[2] = {mapa_shared(smem_u32(&tempty[0]), lrank),
                                       mapa_shared(smem_u32(&tempty[1]), lrank)};
    const uint32_t lmasked_leader[2] = {mapa_shared(smem_u32(&lmasked[0]), lrank),
                                        mapa_shared(smem_u32(&lmasked[1]), lrank)};
    // first row of this CTA's 128 rows of cluster tile `ti`
    auto cta_row0 = [&](const TileInfo& ti) { return (ti.mb * NP + (int)pid) * 256 + (int)rank * Cfg::BM; };
    uint32_t lora_uses0 = 0, lora_uses1 = 0;
    // MASKED: zero the dropped elements of tile `it`'s LoRA partial in place
    // keep bits of this thread's row over its columns [c_lo, c_hi) of tile `ti` (global
    // loads, issued ahead of the LoRA partial); `active` false = nothing to mask
    struct RowKeep {
      bool active;
      uint32_t bits[BN / 64];
    };
    auto fetch_keep = [&](const TileInfo& ti) {
      RowKeep rk;
      const int row = cta_row0(ti) + (int)(q * 32 + lane);
      int seg = -1;
      if (row < args.M) {
        const LfRoute rt = route_at(args, s_routes, 2 * (ti.mb * NP + (int)pid) + (int)rank);
        seg = find_segment(args.segs, rt.seg_lo, rt.seg_hi, row);
      }
      rk.active = seg >= 0 && (args.segs.mask_mode == 2 || args.segs.seg[seg].thr != 0);
#pragma unroll
      for (int j = 0; j < BN / 64; ++j)
        rk.bits[j] = !rk.active ? 0xFFFFFFFFu
                     : (args.segs.debug & 128) ? 0x7FFFFFFFu  // profiling: skip the bit loads, keep the TMEM pass
                                               : dgrad_keep32(args.segs, seg, row, ti.nb * BN + c_lo + 32 * j, args.N);
      if (args.segs.debug & 64) rk.active = false;
      return rk;
    };
    // MASKED: zero the dropped elements of tile `it`'s LoRA partial in place
    auto mask_apply = [&](int it, const RowKeep& rk) {
      const int acc = it % NACC;
      uint32_t& lu = acc ? lora_uses1 : lora_uses0;
      mbar_wait(&lfull[acc], lu & 1);
      ++lu;
      tc_fence_after();
      // tcgen05.ld/st are warp-collective (.sync.aligned): every branch around them is warp-uniform
      if (__any_sync(0xFFFFFFFFu, rk.active)) {
        const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * Cfg::ACC_COLS;
#pragma unroll
        for (int j = 0; j < BN / 64; ++j) {
          const int c = c_lo + 32 * j;
          const uint32_t kp = rk.bits[j];
          if (__all_sync(0xFFFFFFFFu, kp == 0xFFFFFFFFu)) continue;
          uint32_t v[32];
          tmem_ld32(taddr + c, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (!((kp >> i) & 1u)) v[i] = 0u;
          tmem_st32(taddr + c, v);
        }
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(lmasked_leader[acc]);
    };
    const uint32_t lnext_leader[2] = {mapa_shared(smem_u32(&lnext[0]), lrank), mapa_shared(smem_u32(&lnext[1]), lrank)};
    // GRP: the J masked LoRA partials of tile `it` arrive one after another in its drained
    // buffer; each is read, masked with its projection's keep bits and added to a running sum
    // in registers, and the sum goes back to TMEM for the main loop to accumulate on top. The
    // running sum of a thread's 128 columns is held as bf16 pairs between partials (fp32
    // would not fit next to the rest of the kernel in 168 registers: 3 warps share an SMSP's
    // register file): each partial is added in fp32 and the sum rounded once per partial —
    // the per-projection path rounds each projection's whole dX_j to bf16 before summing.
    auto mask_pass_grp = [&](const TileInfo& ti, int it) {
      const int acc = it % NACC;
      uint32_t& lu = acc ? lora_uses1 : lora_uses0;
      const int row = cta_row0(ti) + (int)(q * 32 + lane);
      const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * Cfg::ACC_COLS;
      const int nbytes = (int)args.ld_gbits;
      const int b0 = (ti.nb * BN + c_lo) >> 3;
      uint32_t r[BN / 4];  // 128 columns as bf16 pairs
#pragma unroll
      for (int j = 0; j < kMaxGroup; ++j) {
        if (j >= J) break;
        uint32_t kb4[BN / 64];
        const uint8_t* gb = args.gbits[j];
#pragma unroll
        for (int c = 0; c < BN / 64; ++c) {
          kb4[c] = 0xFFFFFFFFu;
          if (gb && row < args.M) {
            const uint8_t* rb = gb + (int64_t)row * nbytes;
            const int bb = b0 + 4 * c;
            if (bb + 4 <= nbytes && ((reinterpret_cast<uintptr_t>(rb + bb) & 3u) == 0)) {
              kb4[c] = *reinterpret_cast<const uint32_t*>(rb + bb);
            } else {
              uint32_t w = 0;
              for (int i = 0; i < 4; ++i)
                if (bb + i < nbytes) w |= (uint32_t)rb[bb + i] << (8 * i);
              kb4[c] = w;
            }
          }
        }
        mbar_wait(&lfull[acc], lu & 1);
        ++lu;
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {  // 16 columns per TMEM load (register pressure)
          uint32_t v[16];
          tmem_ld16(taddr + c_lo + 16 * c, v);
          tmem_ld_wait();
          const uint32_t kp = kb4[c >> 1] >> (16 * (c & 1));
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            float x0 = ((kp >> e) & 1u) ? __uint_as_float(v[e]) : 0.f;
            float x1 = ((kp >> (e + 1)) & 1u) ? __uint_as_float(v[e + 1]) : 0.f;
            uint32_t& w = r[8 * c + e / 2];
            if (j > 0) {
              x0 += __uint_as_float(w << 16);
              x1 += __uint_as_float(w & 0xFFFF0000u);
            }
            w = pack_bf16x2(x0, x1);
          }
        }
        if (j + 1 < J) {  // the MMA may overwrite the buffer with partial j + 1
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(lnext_leader[acc]);
        }
      }
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[16];
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const uint32_t w = r[8 * c + e / 2];
          v[e] = w << 16;
          v[e + 1] = w & 0xFFFF0000u;
        }
        tmem_st16(taddr + c_lo + 16 * c, v);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(lmasked_leader[acc]);
    };
    auto mask_pass = [&](const TileInfo& ti, int it) {
      if constexpr (GRP) mask_pass_grp(ti, it);
      else mask_apply(it, fetch_keep(ti));
    };
    // output of tile `ti`: base, row pitch, first column and column limit (GRP forward: the
    // projection's own Y_j)
    auto out_base = [&](const TileInfo& ti, int row, int& col0, int& lim) {
      if constexpr (GRP && !B_MN) {
        col0 = ti.nb * BN - ti.noff;
        lim = args.send[ti.proj] - ti.noff;
        return reinterpret_cast<__nv_bfloat16*>(args.Cs[ti.proj]) + (int64_t)row * args.ldcs[ti.proj];
      } else {
        col0 = ti.nb * BN;
        lim = args.N;
        return reinterpret_cast<__nv_bfloat16*>(args.C) + (int64_t)row * args.ldc;
      }
    };
    if constexpr (MASKED && WIDE) {
      // One accumulator, so tile i+1's LoRA partial and its mask pass sit between tile i's
      // main loop and tile i+1's: keep that gap short — tile i+1's keep bits are loaded
      // before tile i's drain, the drain only moves TMEM into registers, and tile i's
      // stores wait until tile i+1's mask pass has released the MMA.
      int t = seq.first();
      if (t >= 0) {
        const TileInfo t0 = tinfo(t);
        if (t0.lora()) mask_pass(t0, 0);
      }
      for (int it = 0; t >= 0; ++it) {
        const TileInfo ti = tinfo(t);
        const int tn = seq.read(it + 1, lane == 0);
        const bool next_lora = tn >= 0 && tinfo(tn).lora();
        RowKeep nk;
        if (next_lora) nk = fetch_keep(tinfo(tn));
        const int row = cta_row0(ti) + (int)(q * 32 + lane);
        mbar_wait(&tfull[0], (uint32_t)it & 1u);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((q * 32u) << 16);
        uint32_t pk[(BN / 2) / 2];
#pragma unroll
        for (int c = 0; c < BN / 2; c += 32) {
          uint32_t v[32];
          tmem_ld32(taddr + c_lo + c, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[c / 2 + j] = pack_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader[0]);
        if (next_lora) mask_apply(it + 1, nk);
        if (row < args.M) {
          __nv_bfloat16* crow = reinterpret_cast<__nv_bfloat16*>(args.C) + (int64_t)row * args.ldc;
#pragma unroll
          for (int c = 0; c < BN / 2; c += 8) {
            const int col = ti.nb * BN + c_lo + c;
            if (col < args.N)
              store_c8(crow + col, make_uint4(pk[c / 2], pk[c / 2 + 1], pk[c / 2 + 2], pk[c / 2 + 3]), ACC);
          }
        }
        t = tn;
      }
    } else {
    int t = seq.first();
    for (int it = 0; t >= 0; ++it) {
      const TileInfo ti = tinfo(t);
      const int acc = it % NACC;
      const uint32_t aph = (it / NACC) & 1;
      int tn = -1;
      if constexpr (MASKED) {
        if (it == 0 && ti.lora()) mask_pass(ti, 0);
        tn = seq.read(it + 1, lane == 0);
        if (tn >= 0) {
          const TileInfo tni = tinfo(tn);
          if (tni.lora()) mask_pass(tni, it + 1);
        }
      }
      const int row = cta_row0(ti) + (int)(q * 32 + lane);
      int n0, nlim;
      __nv_bfloat16* crow = out_base(ti, row, n0, nlim);
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * Cfg::ACC_COLS;
      if constexpr (NACC == 1) {
        // single accumulator: the next tile's MMAs wait for it, so hand TMEM back as soon as
        // this warp's 256 columns sit in registers as bf16 (128 regs), then store them while
        // the next tile's main loop runs
        uint32_t pk[(BN / 2) / 2];
#pragma unroll
        for (int c = 0; c < BN / 2; c += 32) {
          uint32_t v[32];
          tmem_ld32(taddr + c_lo + c, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[c / 2 + j] = pack_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader[acc]);
        if (row < args.M) {
#pragma unroll
          for (int c = 0; c < BN / 2; c += 8) {
            const int col = n0 + c_lo + c;
            if (col < nlim)
              store_c8(crow + col, make_uint4(pk[c / 2], pk[c / 2 + 1], pk[c / 2 + 2], pk[c / 2 + 3]), ACC);
          }
        }
        if constexpr (!MASKED) tn = seq.read(it + 1, lane == 0);
        t = tn;
        continue;
      } else {
#pragma unroll 1
      for (int c = c_lo; c < c_hi; c += 32) {
        const int col0 = n0 + c;
        uint32_t v[32];
        tmem_ld32(taddr + c, v);
        tmem_ld_wait();
        if (row < args.M) {
          uint4 pk[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            pk[j] = make_uint4(pack_bf16x2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1])),
                               pack_bf16x2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                               pack_bf16x2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                               pack_bf16x2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (col0 + 8 * j < nlim) store_c8(crow + col0 + 8 * j, pk[j], ACC);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader[acc]);
      if constexpr (!MASKED) tn = seq.read(it + 1, lane == 0);
      t = tn;
      }  // NACC == 2
    }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
  }
}

template <bool B_MN, bool MASKED, int STAGES, bool WIDE, int CL, bool ACC = false, bool GRP = false>
static int launch_one(const GemmMaps& maps, const GemmArgs& args, int num_sms, cudaStream_t stream) {
  using Cfg = GemmCfg<B_MN, STAGES, WIDE>;
  auto kern = lf_gemm_kernel<B_MN, MASKED, STAGES, WIDE, CL, ACC, GRP>;
  static std::atomic<uint64_t> attr_done{0};  // per instantiation, per device
  if (ensure_smem_attr(kern, Cfg::SMEM_BYTES, attr_done)) return -1;
  const int tiles = args.tiles_m * args.tiles_n;
  // dynamic: one cluster per tile (the resident clusters take over the rest through CLC);
  // static: one persistent cluster per CL SMs, round-robin tiles
  const int clusters = args.dynamic ? tiles : (tiles < num_sms / CL ? tiles : num_sms / CL);
  if (launch_k(kern, dim3(CL * clusters), dim3(kGemmThreads), Cfg::SMEM_BYTES, stream, maps, args))
    return -1;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

static int env_int_or(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// tile width, tile schedule and raster of one launch (see gemm_launch); returns `wide`
static bool gemm_schedule(GemmKind kind, GemmArgs& args, int num_sms, bool cl4, bool allow_wide) {
  static const int wide_env = [] { const char* e = getenv("LF_WIDE"); return e ? atoi(e) : -1; }();
  const int min_k = kind == kGemmDgradMasked ? 8192 : 4096;
  const bool wide_fit = (int64_t)((args.M + 255) / 256) * ((args.N + 511) / 512) >= 4 * (num_sms / 2) &&
                        args.K >= min_k;
  const bool wide = allow_wide && (wide_env >= 0 ? wide_env == 1 : wide_fit);
  static const int sched_env = [] { const char* e = getenv("LF_SCHED"); return e ? atoi(e) : 0; }();
  const double operand_bytes = 2.0 * ((double)args.M + (double)args.N) * (double)args.K;
  args.dynamic = sched_env == 1 ? 0 : sched_env == 2 ? 1 : (operand_bytes > 128.0 * (1 << 20) ? 1 : 0);
  args.tiles_m = cl4 ? (args.M + 511) / 512 : (args.M + 255) / 256;
  args.tiles_n = wide ? (args.N + 511) / 512 : (args.N + 255) / 256;
  if (args.group <= 0) args.group = cl4 ? 4 : 8;
  return wide;
}

// Shared-input group in one launch: the forward concatenates the projections' output
// columns (q/k/v: N = 4096 + 1024 + 1024 as one 10-wave GEMM instead of a 7-wave one and two
// 1.7-wave ones), the input gradient their reduction dims (K = n_q + n_k + n_v: dX written
// once, no accumulation launches). Segments must be whole tiles (forward: multiples of the
// tile width; dgrad: of 64). The masked dgrad runs on 256 x 256 tiles (its J partials take
// turns in the second accumulator buffer).
int gemm_launch_group(GemmKind kind, const GemmMaps& maps, const GemmArgs& a, int num_sms, cudaStream_t stream) {
  GemmArgs args = a;
  if (args.nseg < 2 || args.nseg > kMaxGroup || args.accumulate) return kGemmUnsupported;
  // The input gradient's concatenated K widens every tile's operand footprint: a wave of
  // 8 x 9 tiles streams ~8.8 K bytes of dY / W, which must stay in L2 for the grouped raster to
  // reuse it — measured: q/k/v at K = 6144 one launch 314.6 vs 327.1 µs for three; gate/up at
  // K = 28672 1346 vs 1250 µs (C2) and 11.3 vs 10.0 ms (C4). LF_GROUP_DGRAD_K overrides.
  static const int kmax = env_int_or("LF_GROUP_DGRAD_K", 12288);
  if (kind != kGemmFwd && args.K > kmax) return kGemmUnsupported;
  // forward: 256 x 512 tiles only with >= 8 waves of them (q/k/v at C2: 5.2 waves of wide
  // tiles, 294 µs, vs 10.4 of 256 x 256)
  const bool allow_wide = kind == kGemmFwd &&
                          (int64_t)((args.M + 255) / 256) * ((args.N + 511) / 512) >= 8 * (num_sms / 2);
  const bool wide = gemm_schedule(kind, args, num_sms, false, allow_wide || kind == kGemmDgrad);
  const int unit = kind == kGemmFwd ? (wide ? 512 : 256) : 64;
  for (int j = 0; j < args.nseg; ++j) {
    const int lo = j ? args.send[j - 1] : 0;
    if (args.send[j] <= lo || (args.send[j] - lo) % unit != 0 || args.lcols[j] <= 0 || args.lcols[j] % 16 != 0)
      return kGemmUnsupported;
  }
  switch (kind) {
    case kGemmFwd:
      return wide ? launch_one<false, false, 4, true, 2, false, true>(maps, args, num_sms, stream)
                  : launch_one<false, false, 6, false, 2, false, true>(maps, args, num_sms, stream);
    case kGemmDgrad:
      return wide ? launch_one<true, false, 4, true, 2, false, true>(maps, args, num_sms, stream)
                  : launch_one<true, false, 6, false, 2, false, true>(maps, args, num_sms, stream);
    case kGemmDgradMasked:
      return launch_one<true, true, 6, false, 2, false, true>(maps, args, num_sms, stream);
  }
  return -1;
}

int gemm_launch(GemmKind kind, const GemmMaps& maps, const GemmArgs& a, int num_sms, cudaStream_t stream) {
  GemmArgs args = a;
  // 256 x 512 tiles for the forward GEMM when they still fill >= 4 waves (LF_WIDE=0|1 forces):
  // 25% fewer L2 sectors per FLOP buys clock under the power cap — C4 q/gate/down 6/5.5/12.6%
  // faster, C2 gate 3.8%; with fewer than ~4 waves the coarser tiles quantise badly (C2 q,
  // down: 4–14% slower). ncu, profiles/r01_wide_tiles_ab.txt
  // The masked dgrad runs wide tiles sequentially (drain to registers -> LoRA partial -> TMEM
  // mask pass -> main loop; next tile's keep bits prefetched, stores deferred), which pays off
  // from K = 8192: C4 q/o 1.45 -> 1.40, gate/up 5.24 -> 4.91, down 5.05 -> 4.91 ms; at K = 4096
  // (C2 down) 2% slower.
  // Tile schedule. While both operands fit in L2 together, the static persistent
  // round-robin is ~5% faster (C2 q/kv, C1: no per-tile CLC round trip and the pairs'
  // drift costs nothing); beyond that, drifting pairs re-read their operands from DRAM
  // and the in-order CLC schedule wins (C4 q 1.49 -> 1.43 ms, gate 5.5 -> 5.08 ms; ncu,
  // profiles/r01_sched_shapes.txt). LF_SCHED=1 forces static, 2 dynamic (A/B runs).
  // Two CTA pairs per cluster sharing B by TMA multicast (LF_CL=4; parity-green, off by
  // default): it cuts the power drawn per FLOP (C4 gate: 1.37 -> 1.47 GHz under the cap) but
  // a B200 holds only 33 four-CTA clusters at one CTA per SM — 132 of 148 SMs; pairs use
  // all 148 (tools/cluster_occupancy.cu) — so every shape measured slower end to end
  // (C4 step 42.0 -> 46.4 ms, C2 5.67 -> 6.56 ms; profiles/r02_cluster_multicast_ab.txt)
  static const int cl_env = [] { const char* e = getenv("LF_CL"); return e ? atoi(e) : 0; }();
  const bool cl4 = cl_env == 4;
  const bool wide = gemm_schedule(kind, args, num_sms, cl4, true);
#define LF_GEMM_LAUNCH(BMN, MSK, ST, WD)                                                        \
  (cl4 ? launch_one<BMN, MSK, ST, WD, 4>(maps, args, num_sms, stream)                          \
       : launch_one<BMN, MSK, ST, WD, 2>(maps, args, num_sms, stream))
  // accumulating dgrads (lf_grad_input_accum) are their own instantiations (pairs only)
  if (args.accumulate) {
    if (kind == kGemmFwd) return -1;
    if (kind == kGemmDgradMasked)
      return wide ? launch_one<true, true, 4, true, 2, true>(maps, args, num_sms, stream)
                  : launch_one<true, true, 6, false, 2, true>(maps, args, num_sms, stream);
    return wide ? launch_one<true, false, 4, true, 2, true>(maps, args, num_sms, stream)
                : launch_one<true, false, 6, false, 2, true>(maps, args, num_sms, stream);
  }
  switch (kind) {
    case kGemmFwd:
      return wide ? LF_GEMM_LAUNCH(false, false, 4, true) : LF_GEMM_LAUNCH(false, false, 6, false);
    case kGemmDgrad:
      return wide ? LF_GEMM_LAUNCH(true, false, 4, true) : LF_GEMM_LAUNCH(true, false, 6, false);
    case kGemmDgradMasked:
      return wide ? LF_GEMM_LAUNCH(true, true, 4, true) : LF_GEMM_LAUNCH(true, true, 6, false);
  }
#undef LF_GEMM_LAUNCH_ACC
#undef LF_GEMM_LAUNCH
  return -1;
}

}  // namespace lf
