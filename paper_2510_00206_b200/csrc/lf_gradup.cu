// lf_gradup.cu — ③ grad_up_fused: one read of dY serves both rank-R gradients.
//
// Reference contract: ls/costmodel.py:268-269 (R (mn + mr + rn), W (mr + rn)).
//   dŜ     = bf16( s_seg · dY·B_cat )   (m x R; off-segment columns zero)
//   dB_cat += dYᵀ·Ŝ                     (n x R, fp32)
//
// Each CTA owns a block of 128-row m-tiles x 128-column n-subtiles. Every dY tile is
// TMA-loaded once into shared memory and consumed by two tcgen05 MMAs through two
// descriptors over the same bytes: K-major (rows = tokens) for dŜ += dY·B_cat, and
// MN-major (rows = out features) for dBᵀ += dYᵀ·Ŝ. Both accumulators live in TMEM:
// dŜ double-buffered per m-tile, dB per n-subtile for the CTA's whole m-range.
// dŜ partials over n-subtiles meet in an fp32 workspace (red.global.add); the split-K
// epilogue kernel (lf_finalize_kernel, lf_lowrank.cu) then scales, masks off-segment
// columns, converts to bf16 and re-zeroes the workspace.
#include "lf_device.cuh"
#include <cstring>

#include "lf_kernels.h"

namespace lf {

namespace gup {
constexpr int DY_BYTES = 2 * 128 * 64 * 2;  // 32 KB: two 64-column SW128 boxes of 128 rows
constexpr int MAX_SMEM = 200 * 1024;
}  // namespace gup

// one CTA's share of ③: n-subtiles [bx·tiles_n/n_split, ...) x m-tiles [by·tiles_m/m_split, ...)
__device__ __forceinline__ void gradup_cta(const CUtensorMap& tmDy, const CUtensorMap& tmB, const CUtensorMap& tmS,
                                           const GradUpArgs& args, int stages, int stage_bytes, int bx, int by) {
  using namespace gup;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const int rtot = args.rtot;
  const int sh_bytes = (args.segs.wmax / 16) * 4096;  // Ŝ / B_cat columns of the widest routing hull
  uint8_t* sSh0 = smem + stages * stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sSh0 + 2 * sh_bytes);
  uint64_t* empty = full + stages;
  uint64_t* sh_full = empty + stages;   // [2]
  uint64_t* sh_empty = sh_full + 2;     // [2]
  uint64_t* ds_full = sh_empty + 2;     // [2]
  uint64_t* ds_empty = ds_full + 2;     // [2]
  uint64_t* db_full = ds_empty + 2;     // [1]
  uint64_t* tzero = db_full + 1;        // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tzero + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int tiles_m = (args.m + 127) / 128;
  const int tiles_n = (args.n + 127) / 128;
  const int nt0 = (int)((int64_t)bx * tiles_n / args.n_split);
  const int nt1 = (int)((int64_t)(bx + 1) * tiles_n / args.n_split);
  const int mt0 = (int)((int64_t)by * tiles_m / args.m_split);
  const int mt1 = (int)((int64_t)(by + 1) * tiles_m / args.m_split);
  const int nsub = nt1 - nt0;
  // NA independent accumulators per chain (consecutive K-steps rotate through them): small-N
  // MMAs into a single accumulator serialise on its latency
  const int NA = args.nacc;
  // dŜ accumulators hold one m-tile's routing hull (≤ wmax columns, tile-relative); the dB
  // accumulators of an n-subtile collect every adapter's block (rtot columns)
  const int wmax = args.segs.wmax;
  const int AWs = NA * wmax;  // TMEM columns of one dŜ (multi-)accumulator
  const int AW = NA * rtot;   // TMEM columns of one dB (multi-)accumulator
  const uint32_t tmem_need = (uint32_t)(2 * AWs + nsub * AW);
  uint32_t tmem_cols = 32;
  while (tmem_cols < tmem_need) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&sh_full[a], 1);
      mbar_init(&sh_empty[a], 1);
      mbar_init(&ds_full[a], 1);
      mbar_init(&ds_empty[a], 4);
    }
    mbar_init(db_full, 1);
    mbar_init(tzero, 4);
    fence_barrier_init();
    tma_prefetch_desc(&tmDy);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmS);
  }
  pdl_launch_dependents();
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();  // the prologue above overlaps the predecessor's tail; global memory only from here
  const uint32_t tmem = *tmem_slot;
  const uint32_t tm_ds = tmem;            // 2 buffers x AWs columns
  const uint32_t tm_db = tmem + 2 * AWs;  // nsub x AW columns

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && nsub > 0) {
      int stage = 0;
      uint32_t phase = 0;
      int lm = 0;
      for (int mt = mt0; mt < mt1; ++mt) {
        const LfRoute rt = args.routes[mt];
        const int N = rt.col_hi - rt.col_lo;
        if (N <= 0) continue;
        const int b = lm & 1;
        const uint32_t bph = (lm >> 1) & 1;
        ++lm;
        mbar_wait(&sh_empty[b], bph ^ 1);
        uint8_t* sSh = sSh0 + b * sh_bytes;
        mbar_arrive_expect_tx(&sh_full[b], (N / 16) * 4096);
        for (int j = 0; j < N / 16; ++j) tma_load_2d(sSh + j * 4096, &tmS, &sh_full[b], rt.col_lo + 16 * j, mt * 128);
        for (int nt = nt0; nt < nt1; ++nt) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sDy = smem + stage * stage_bytes;
          uint8_t* sB = sDy + DY_BYTES;
          mbar_arrive_expect_tx(&full[stage], DY_BYTES + (N / 16) * 4096);
          tma_load_2d(sDy, &tmDy, &full[stage], nt * 128, mt * 128);
          tma_load_2d(sDy + 16384, &tmDy, &full[stage], nt * 128 + 64, mt * 128);
          for (int j = 0; j < N / 16; ++j) tma_load_2d(sB + j * 4096, &tmB, &full[stage], rt.col_lo + 16 * j, nt * 128);
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (whole warp, one lane issues)
    if (nsub > 0) {
      mbar_wait(tzero, 0);
      tc_fence_after();
      int stage = 0;
      uint32_t phase = 0;
      int lm = 0;
      for (int mt = mt0; mt < mt1; ++mt) {
        const LfRoute rt = args.routes[mt];
        const int N = rt.col_hi - rt.col_lo;
        if (N <= 0) continue;
        const int b = lm & 1;
        const uint32_t bph = (lm >> 1) & 1;
        ++lm;
        mbar_wait(&ds_empty[b], bph ^ 1);
        mbar_wait(&sh_full[b], bph);
        tc_fence_after();
        const uint32_t sSh = smem_u32(sSh0 + b * sh_bytes);
        const uint32_t d_ds = tm_ds + b * AWs;  // tile-relative: column c <-> rank-concat col_lo + c
        const uint32_t idesc_ds = make_idesc_bf16(128, (uint32_t)N, false, true);
        const uint32_t idesc_db = make_idesc_bf16(128, (uint32_t)N, true, true);
        for (int nt = nt0; nt < nt1; ++nt) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sDy = smem_u32(smem + stage * stage_bytes);
          const uint32_t sB = sDy + DY_BYTES;
          const uint32_t d_db = tm_db + (nt - nt0) * AW + rt.col_lo;
          // the two chains share each dY K-step and are issued interleaved:
          //   dŜ[m-tile]        += dY[m-tile, n-sub]  · B_cat[n-sub, cols]   (K = 128 out features)
          //   dB_cat[n-sub, ..] += dY[m-tile, n-sub]ᵀ · Ŝ[m-tile, cols]      (K = 128 tokens)
          const uint64_t a_ds = make_sdesc(sDy, 16, 1024, kLayoutSW128);
          const uint64_t b_ds = make_sdesc(sB, 4096, 256, kLayoutSW32);
          const uint64_t a_db = make_sdesc(sDy, 16384, 1024, kLayoutSW128);
          const uint64_t b_db = make_sdesc(sSh, 4096, 256, kLayoutSW32);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t a = (uint32_t)(kk % NA) * rtot;
            if (!(args.segs.debug & 1))
              umma_bf16_warp(d_ds + (uint32_t)(kk % NA) * wmax, sdesc_add(a_ds, (kk >> 2) * 16384 + (kk & 3) * 32), sdesc_add(b_ds, kk * 512),
                             idesc_ds, (nt > nt0 || kk >= NA) ? 1u : 0u);
            if (!(args.segs.debug & 32))
              umma_bf16_warp(d_db + a, sdesc_add(a_db, kk * 2048), sdesc_add(b_db, kk * 512), idesc_db, 1u);
          }
          umma_commit_warp(&empty[stage]);
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
        umma_commit_warp(&ds_full[b]);
        umma_commit_warp(&sh_empty[b]);
      }
      umma_commit_warp(db_full);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const uint32_t q = warp & 3u;
    const uint32_t lane_off = (q * 32u) << 16;
    if (nsub > 0) {
      uint32_t z[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) z[i] = 0u;
      for (int c = 0; c < nsub * AW; c += 16) tmem_st16(tm_db + lane_off + c, z);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tzero);
    }
    const int rit = (int)(q * 32 + lane);
    int lm = 0;
    uint32_t touched = 0;
    for (int mt = mt0; mt < mt1; ++mt) {
      const LfRoute rt = args.routes[mt];
      const int N = rt.col_hi - rt.col_lo;
      const int row = mt * 128 + rit;
      if (N > 0 && nsub > 0) {
        for (int c = rt.col_lo; c < rt.col_hi; c += 16) touched |= 1u << (c >> 4);
        const int b = lm & 1;
        const uint32_t bph = (lm >> 1) & 1;
        ++lm;
        mbar_wait(&ds_full[b], bph);
        tc_fence_after();
        float* wrow = args.ws + (int64_t)row * rtot + rt.col_lo;
        for (int c = 0; c < N; c += 16) {
          float s[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) s[j] = 0.f;
          for (int a = 0; a < NA; ++a) {
            uint32_t v[16];
            tmem_ld16(tm_ds + lane_off + b * AWs + a * wmax + c, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) s[j] += __uint_as_float(v[j]);
          }
          if (row < args.m && !(args.segs.debug & 2)) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) red_add_v4(wrow + c + j, s[j], s[j + 1], s[j + 2], s[j + 3]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ds_empty[b]);
      }
    }
    if (touched && nsub > 0) {
      mbar_wait(db_full, 0);
      tc_fence_after();
      for (int i = 0; i < nsub; ++i) {
        const int ncol = (nt0 + i) * 128 + rit;
        float* drow = args.db + (int64_t)ncol * rtot;
        for (int g = 0; g < rtot / 16; ++g) {
          if (!((touched >> g) & 1u)) continue;
          float s[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) s[j] = 0.f;
          for (int a = 0; a < NA; ++a) {
            uint32_t v[16];
            tmem_ld16(tm_db + lane_off + i * AW + a * rtot + g * 16, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) s[j] += __uint_as_float(v[j]);
          }
          if (ncol < args.n && !(args.segs.debug & 2)) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) red_add_v4(drow + g * 16 + j, s[j], s[j + 1], s[j + 2], s[j + 3]);
          }
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

__global__ void __launch_bounds__(192, 2)
    lf_gradup_kernel(const __grid_constant__ CUtensorMap tmDy, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmS, const __grid_constant__ GradUpArgs args, int stages,
                     int stage_bytes) {
  gradup_cta(tmDy, tmB, tmS, args, stages, stage_bytes, (int)blockIdx.x, (int)blockIdx.y);
}

// ③ for a shared-input group in one launch: CTAs [cta_end[j-1], cta_end[j]) run projection j's
// grid (n_split_j x m_split_j, its own stage ring); one launch pays the fixed costs once
__global__ void __launch_bounds__(192, 2)
    lf_gradup_group_kernel(const __grid_constant__ GroupUpMaps maps, const __grid_constant__ GroupUpArgs g) {
  int j = 0;
  while (j + 1 < g.J && (int)blockIdx.x >= g.cta_end[j]) ++j;
  const int local = (int)blockIdx.x - (j ? g.cta_end[j - 1] : 0);
  const GradUpArgs& a = g.p[j];
  gradup_cta(maps.dy[j], maps.b[j], maps.s[j], a, g.stages[j], g.stage_bytes[j], local % a.n_split, local / a.n_split);
}

// CTA grid: n_split x m_split blocks of (n-subtiles x m-tiles). The dB accumulators of a
// CTA's n-range must fit TMEM next to the two dŜ buffers: (2 + nsub) * R <= 512.
// Among admissible splits pick the smallest critical path (waves x max units of one 32 KB
// dY tile per CTA), then the least partial-sum traffic R * (m_split * n + n_split * m).
void grad_up_grid(int m, int n, int rtot, int wmax, int sms, int per_sm, int* n_split, int* m_split, int* nacc) {
  const int tiles_m = (m + 127) / 128, tiles_n = (n + 127) / 128;
  // measured on B200: rotating K-steps over several accumulators does not speed the
  // small-N chains up (the pipelines are TMA-bound), so one accumulator keeps TMEM free
  *nacc = 1;
  // per_sm CTAs share an SM's 512 TMEM columns (and its shared memory)
  // at most 8 n-subtiles per CTA: each CTA flushes its dB partials (nsub x 128 x R fp32
  // red.adds) at its very end, where nothing overlaps them — measured at n = 28672, R = 16:
  // 25 subtiles per CTA 36.9 / 53.2 / 86.1 µs at m = 2048 / 4096 / 8192, <= 8 subtiles
  // 26.8 / ~47 / 81.9 µs (profiles/r01_gradup_split_sweep.txt)
  int max_nsub = ((512 / per_sm) - 2 * *nacc * wmax) / (*nacc * rtot);
  if (max_nsub > 8) max_nsub = 8;
  sms *= per_sm;
  *n_split = 0;
  *m_split = 0;
  if (max_nsub < 1) return;
  long best_units = -1;
  double best_traffic = 0;
  for (int ns = (tiles_n + max_nsub - 1) / max_nsub; ns <= tiles_n; ++ns) {
    int ms = sms / ns;
    if (ms < 1) ms = 1;
    if (ms > tiles_m) ms = tiles_m;
    // critical path in 32 KB units; a grid wider than the resident CTAs (ns > SMs leaves
    // ms = 1) runs in several waves: C4 gate/up (n = 28672) picked ns = 224 on 148 SMs
    // without the wave factor — 275 µs instead of 154 at ns = 9
    const long waves = ((long)ns * ms + sms - 1) / sms;
    const long units = waves * ((tiles_m + ms - 1) / ms) * ((tiles_n + ns - 1) / ns);
    const double traffic = (double)rtot * ((double)ms * n + (double)ns * m);
    if (best_units < 0 || units < best_units || (units == best_units && traffic < best_traffic)) {
      best_units = units;
      best_traffic = traffic;
      *n_split = ns;
      *m_split = ms;
    }
  }
}

// stage ring of one ③ problem: (stages, stage_bytes, dynamic smem bytes), or -1
static int gradup_ring(const GradUpArgs& args, int per_sm, int* stages_out, int* stage_bytes_out) {
  const int sh_bytes = (args.segs.wmax / 16) * 4096;
  const int stage_bytes = gup::DY_BYTES + sh_bytes;
  int stages = (gup::MAX_SMEM / per_sm - 2 * sh_bytes) / stage_bytes;
  if (stages > 6) stages = 6;  // deep ring: ~180 KB of dY in flight per SM
  if (stages < 2) return -1;
  *stages_out = stages;
  *stage_bytes_out = stage_bytes;
  return stages * stage_bytes + 2 * sh_bytes + 1024 + 1024;
}

int grad_up_group_launch(const GroupUpMaps& maps, GroupUpArgs& g, cudaStream_t stream) {
  int smem = 0, ctas = 0;
  for (int j = 0; j < g.J; ++j) {
    const int sm_j = gradup_ring(g.p[j], 1, &g.stages[j], &g.stage_bytes[j]);
    if (sm_j < 0 || g.p[j].n_split <= 0) return -1;
    if (sm_j > smem) smem = sm_j;
    ctas += g.p[j].n_split * g.p[j].m_split;
    g.cta_end[j] = ctas;
  }
  static std::atomic<uint64_t> attr_done{0};
  if (ensure_smem_attr(lf_gradup_group_kernel, gup::MAX_SMEM + 2048, attr_done)) return -1;
  if (launch_k(lf_gradup_group_kernel, dim3(ctas), dim3(192), smem, stream, maps, g)) return -1;
  GroupFinArgs f;
  memset(&f, 0, sizeof(f));
  f.J = g.J;
  int64_t chunks = 0;
  for (int j = 0; j < g.J; ++j) {
    chunks += (int64_t)g.p[j].segs.m * (g.p[j].segs.rtot / 8);
    f.chunk_end[j] = chunks;
    f.segs[j] = g.p[j].segs;
    f.routes[j] = g.p[j].routes;
    f.ws[j] = g.p[j].ws;
    f.out[j] = reinterpret_cast<__nv_bfloat16*>(g.p[j].ds);
  }
  return launch_k(lf_finalize_group_kernel, dim3((unsigned)((chunks + 127) / 128)), dim3(128), 0, stream, f);
}

int grad_up_launch(const CUtensorMap& tm_dy, const CUtensorMap& tm_b, const CUtensorMap& tm_s,
                   const GradUpArgs& args, int num_sms, int per_sm, cudaStream_t stream) {
  (void)num_sms;
  int stages = 0, stage_bytes = 0;
  const int smem = gradup_ring(args, per_sm, &stages, &stage_bytes);
  if (smem < 0) return -1;
  static std::atomic<uint64_t> attr_done{0};
  if (ensure_smem_attr(lf_gradup_kernel, gup::MAX_SMEM + 2048, attr_done)) return -1;
  dim3 grid(args.n_split, args.m_split);
  if (launch_k(lf_gradup_kernel, grid, dim3(192), smem, stream, tm_dy, tm_b, tm_s, args, stages, stage_bytes))
    return -1;
  // a separate, fully parallel finalize: in-kernel "last contributor finalizes" leaves the
  // finalize of a whole m-range on the tail of one CTA here (up to 13 tiles at gate/up)
  return finalize_launch(args.segs, args.routes, args.ws, args.ds, stream);
}

}  // namespace lf
