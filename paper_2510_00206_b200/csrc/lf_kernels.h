// lf_kernels.h — host-visible launch entry points of the sm_100a kernels (internal).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <atomic>
#include <utility>

#include "lf_params.h"

namespace lf {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): a function
// attribute is per-device state, and one process may drive several GPUs from several host
// threads. `done` is the caller's static per-kernel bitmask of configured device ordinals
// (devices >= 64 are set on every launch); the set is idempotent, so a race between two
// threads only repeats it.
template <typename Kern>
inline int ensure_smem_attr(Kern kern, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return -1;
  if (bit) done.fetch_or(bit, std::memory_order_acq_rel);
  return 0;
}

// Programmatic dependent launch for every lf kernel (see pdl_wait in lf_device.cuh); set
// LF_PDL=0 in the environment to launch with plain stream ordering instead.
bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline int launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                    Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...) == cudaSuccess ? 0 : -1;
}

// ② / ⑤: persistent warp-specialised tcgen05 GEMM  C[M,N] = A[M,K]·B (+ LoRA K-chunk).
//  kind FWD       : B is K-major  (N x K, nn.Linear.weight), LoRA B2 = B_cat (N x R) K-major
//  kind DGRAD     : B is MN-major (K x N, W as stored),      LoRA B2 = A_cat (R x N) MN-major,
//                   LoRA term concatenated into the main accumulator (no dropout)
//  kind DGRAD_MASK: as DGRAD but the LoRA K-block of a tile is issued first into its empty
//                   accumulator, the epilogue warps zero its dropped elements in TMEM, and
//                   the dY·W main loop accumulates on top (dropout p > 0)
enum GemmKind { kGemmFwd = 0, kGemmDgrad = 1, kGemmDgradMasked = 2 };
constexpr int kMaxGroup = 3;  // projections of one shared-input group (q/k/v)
constexpr int kGemmUnsupported = -3;  // gemm_launch: valid request this build does not run (nothing launched)

struct GemmArgs {
  int32_t M, N, K;
  int32_t tiles_m, tiles_n;
  int32_t group;          // raster: m-tiles sharing each n sweep (set by gemm_launch)
  int32_t dynamic;        // 1: CLC tile sequence (one cluster per tile), 0: static persistent
  int64_t ldc;
  void* C;                // bf16 output, row-major M x N (ldc elements)
  int32_t accumulate;     // 1: C += result (bf16 read-modify-write in the epilogue)
  const LfRoute* routes;  // nullptr = no LoRA chunk
  LfSegTable segs;        // keep-mask source for kGemmDgradMasked
  // shared-input groups (gemm_launch_group, nseg = J > 1 projections in one launch):
  //   kGemmFwd    N-concat: projection j owns output columns [send[j-1], send[j]) and writes
  //               them to Cs[j] (row pitch ldcs[j]); its LoRA K-block reads Ŝ_j / B_j
  //   kGemmDgrad* K-concat: projection j owns reduction rows [send[j-1], send[j]) (dY_j, W_j);
  //               its LoRA term reads dŜ_j / A_j, masked with the packed keep bits gbits[j]
  int32_t nseg;                     // 0: single problem
  int32_t send[kMaxGroup];          // cumulative segment ends (N forward, K dgrad)
  int32_t lcols[kMaxGroup];         // padded rank of projection j
  void* Cs[kMaxGroup];
  int64_t ldcs[kMaxGroup];
  const uint8_t* gbits[kMaxGroup];  // null: projection j keeps everything
  int64_t ld_gbits;
};

// operand tensor maps: [0] for a single problem; per projection j for a group (forward:
// a[0] = X, b[j] = W_j; dgrad: a[j] = dY_j, b[j] = W_j; LoRA a2[j] / b2[j])
struct GemmMaps {
  CUtensorMap a[kMaxGroup], b[kMaxGroup], a2[kMaxGroup], b2[kMaxGroup];
};

int gemm_launch(GemmKind kind, const GemmMaps& maps, const GemmArgs& args, int num_sms, cudaStream_t stream);
// one GEMM for a shared-input group (args.nseg = J >= 2; see GemmArgs); kGemmUnsupported when
// the group's shape has no group variant (nothing launched: run the projections one by one)
int gemm_launch_group(GemmKind kind, const GemmMaps& maps, const GemmArgs& args, int num_sms, cudaStream_t stream);

// ① dropout + down projection
struct DownArgs {
  int32_t m, k, rtot;
  int32_t ctas;           // persistent CTAs sharing the (row tile, k-block) units
  void* s_hat;            // bf16 m x rtot
  float* ws;              // fp32 m x rtot partials (zero on entry and exit)
  int32_t* counters;      // per 128-row tile (zero on entry and exit)
  const LfRoute* routes;
  LfSegTable segs;
};
void down_config(int wmax, int* stages, int* stage_bytes);
int down_extra_smem(int mask_mode);  // ①'s keep-bit ring (LF_DOWN_SPLIT), bytes
int down_launch(const CUtensorMap& tm_x, const CUtensorMap& tm_a, const DownArgs& args, int num_sms,
                cudaStream_t stream);

// ③ fused dS / dB
struct GradUpArgs {
  int32_t m, n, rtot;
  int32_t n_split, m_split;  // CTA grid
  int32_t nacc;              // independent accumulators per MMA chain
  void* ds;                  // bf16 m x rtot
  float* db;                 // fp32 n x rtot accumulator
  float* ws;                 // fp32 m x rtot partials (zero on entry and exit)
  int32_t* counters;         // per 128-row tile
  const LfRoute* routes;
  LfSegTable segs;
};
void grad_up_grid(int m, int n, int rtot, int wmax, int sms, int per_sm, int* n_split, int* m_split, int* nacc);
// ③ for a shared-input group: one launch for the J projections (each its own grid, ring and
// split-K workspace), then one dŜ finalize launch for all of them
struct GroupUpMaps {
  CUtensorMap dy[kMaxGroup], b[kMaxGroup], s[kMaxGroup];
};
struct GroupUpArgs {
  int32_t J;
  int32_t cta_end[kMaxGroup];     // cumulative CTA counts (set by grad_up_group_launch)
  int32_t stages[kMaxGroup], stage_bytes[kMaxGroup];
  GradUpArgs p[kMaxGroup];
};
struct GroupFinArgs {
  int32_t J;
  int64_t chunk_end[kMaxGroup];   // cumulative 8-column chunk counts
  LfSegTable segs[kMaxGroup];
  const LfRoute* routes[kMaxGroup];
  float* ws[kMaxGroup];
  __nv_bfloat16* out[kMaxGroup];
};
int grad_up_group_launch(const GroupUpMaps& maps, GroupUpArgs& args, cudaStream_t stream);
__global__ void lf_finalize_group_kernel(const __grid_constant__ GroupFinArgs f);
int grad_up_launch(const CUtensorMap& tm_dy, const CUtensorMap& tm_b, const CUtensorMap& tm_s,
                   const GradUpArgs& args, int num_sms, int per_sm, cudaStream_t stream);

// ④ dA
struct GradDownArgs {
  int32_t m, k, rtot;
  int32_t ctas;      // persistent CTAs sharing the (k-tile, row tile) units
  int32_t bits_tma;  // keep bits arrive in each stage by TMA (tmK valid)
  float* da;  // fp32 rtot x k accumulator
  const LfRoute* routes;
  LfSegTable segs;
};
// ④ for a shared-input group: dA_j += dŜ_jᵀ·(M_j⊙X) for the J projections
// that read the same X (q/k/v, gate/up), one launch. Each unit loads the X tile once per
// projection, back to back, so only the first load of a tile comes from DRAM (the
// projection-major layout of separate launches reads X J times from DRAM); each projection
// has its own keep bits (TMA'd per stage), dŜ and accumulators.
struct GroupDownArgs {
  int32_t m, k, J;
  int32_t ctas;
  int32_t rsum;                   // Σ_j R_j: one TMEM accumulator buffer
  int32_t rmax;                   // widest R_j: sizes the dŜ part of a stage
  int32_t R[kMaxGroup];           // padded rank of projection j
  int32_t off[kMaxGroup];         // its accumulator's first TMEM column in a buffer
  int32_t masked[kMaxGroup];      // its keep bits ride in each stage (p > 0)
  int32_t debug;
  float* da[kMaxGroup];           // fp32 R_j x k accumulators
};
struct GroupDownMaps {
  CUtensorMap x, d[kMaxGroup], bits[kMaxGroup];
};
void grad_down_group_config(int rmax, int* stages, int* stage_bytes);
int grad_down_group_launch(const GroupDownMaps& maps, const GroupDownArgs& args, cudaStream_t stream);

// split-K epilogue of ③: fp32 partials (ws) -> scaled bf16 m x R, workspace re-zeroed
int finalize_launch(const LfSegTable& segs, const LfRoute* routes, float* ws, void* out, cudaStream_t stream);
void grad_down_config(int wmax, bool bits_tma, int* stages, int* stage_bytes);
int grad_down_launch(const CUtensorMap& tm_x, const CUtensorMap& tm_ds, const CUtensorMap& tm_bits,
                     const GradDownArgs& args, int num_sms, cudaStream_t stream);


// routing table + explicit mask materialisation
int routes_launch(const LfSegTable& segs, int32_t* routes, int ntiles, cudaStream_t stream);
int mask_launch(const LfSegTable& segs, int32_t k, uint8_t* keep, cudaStream_t stream);
int keep_bits_launch(const LfSegTable& segs, int32_t k, uint8_t* bits, int64_t ld, int num_sms, cudaStream_t stream);

// lf_copy_column_blocks: dst (rows x width, contiguous) = src[:, col : col + width] of a rows x ld matrix
constexpr int kMaxCopyBlocks = 64;
struct CopyBlock {
  const float* src;
  float* dst;
  int32_t rows, ld, col, width;
};
struct CopyBlocksArgs {
  int32_t n;
  CopyBlock blk[kMaxCopyBlocks];
};
int copy_blocks_launch(const CopyBlocksArgs& a, int num_sms, cudaStream_t stream);

}  // namespace lf
