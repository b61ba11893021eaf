/*
 * lorafusion_b200.h — C ABI of the B200-native FusedLoRA / FusedMultiLoRA layer.
 *
 * Plain pointers, sizes and a plain stream handle; no torch or CUDA types in any
 * signature. Every entry point is stream-ordered (no host synchronisation), returns
 * LF_OK (0) or a negative LF_E_* code, and leaves a thread-local message for
 * lf_last_error(). All device buffers are owned and allocated by the caller.
 *
 * The reference (lorasched, /root/reference/pkg) defines this hot path only as an
 * analytic contract. Each launcher below replaces one kernel of that contract:
 *
 *   lf_dropout_down_fwd  ①  `dropout_down_proj_fused`   ls/costmodel.py:258-261
 *   lf_base_fwd          ②  `base_gemm_epilogue_fused`  ls/costmodel.py:262-264
 *   lf_grad_up           ③  `grad_up_fused`             ls/costmodel.py:268-269
 *   lf_grad_down         ④  `grad_down_fused`           ls/costmodel.py:270-272
 *   lf_grad_input        ⑤  `grad_base_accum_fused`     ls/costmodel.py:273-277
 *   lf_build_routes         `adapter_routing_table`     ls/costmodel.py:279-281
 *                           (ROUTING_TILE_ROWS=128, ROUTING_ENTRY_BYTES=16, :23-26)
 *
 * Semantics (Eq. 1; full statement in SPEC.md):
 *   Y  = X·Wᵀ + Ŝ·B_catᵀ            Ŝ  = bf16( s_i · (M⊙X)·A_catᵀ )  on segment i's columns
 *   dŜ = bf16( s_i · dY·B_cat )      (s_i = scaling_i / (1 - p_i))
 *   dB_cat += dYᵀ·Ŝ                  dA_cat += dŜᵀ·(M⊙X)
 *   dX = dY·W + M ⊙ (dŜ·A_cat)
 * with X (m×k), W (n×k) = nn.Linear.weight, A_cat (R×k) = stacked lora_A.weight,
 * B_cat (n×R) = stacked lora_B.weight, all row-major bf16 (uint16_t storage);
 * dA/dB accumulators are fp32. M is the keep mask of SPEC.md §3 (Philox4x32-10)
 * or an explicit uint8 keep mask.
 *
 * Segments mirror lorasched's MicrobatchSegment (ls/packing.py:41-60): one
 * (adapter, global batch) group of token rows, with that adapter's AdapterSpec
 * hyper-parameters (ls/workload.py:25-48). Segments are sorted by row and disjoint;
 * each owns a 16-aligned column block of the concatenated rank dimension, either its
 * own (disjoint from the others) or shared with segments of the same adapter (SPEC.md §1).
 */
#ifndef LORAFUSION_B200_H
#define LORAFUSION_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define LF_API __attribute__((visibility("default")))
#else
#define LF_API
#endif

#define LF_ABI_VERSION 6
#define LF_MAX_SEGMENTS 32
#define LF_MAX_RANK_TOTAL 128
#define LF_MAX_COPY_BLOCKS 64 /* lf_copy_column_blocks blocks per call */
#define LF_ROUTE_TILE_ROWS 128 /* ls/costmodel.py:25 ROUTING_TILE_ROWS */
#define LF_ROUTE_ENTRY_BYTES 16 /* ls/costmodel.py:26 ROUTING_ENTRY_BYTES */

enum {
  LF_OK = 0,
  LF_E_INVALID = -1,     /* bad argument: maps to ValueError (ls/errors.py:12) */
  LF_E_CUDA = -2,        /* CUDA runtime / driver failure: maps to RuntimeError */
  LF_E_UNSUPPORTED = -3, /* device is not sm_100, or a variant this build does not provide */
};

/* One (adapter, global batch) segment of token rows. */
typedef struct LfSegment {
  int32_t row_start; /* first token row */
  int32_t row_end;   /* one past the last token row */
  int32_t col_start; /* first column of this segment's block in the rank-concat dim (multiple of 16) */
  int32_t rank;      /* width of the block: adapter rank padded to a multiple of 16 */
  float scaling;     /* Eq. 1 alpha (PEFT: lora_alpha / r) */
  float dropout_p;   /* in [0, 1) */
  uint64_t seed;     /* Philox4x32-10 key */
  uint64_t offset;   /* Philox counter words 2..3 (per training step) */
} LfSegment;

/* Problem description shared by all launchers of one layer call. */
typedef struct LfProblem {
  int32_t m, k, n;          /* tokens, in_features, out_features */
  int32_t rank_total;       /* R: width of the rank-concat dim (multiple of 16, <= 128) */
  int32_t num_segments;     /* 0 .. LF_MAX_SEGMENTS (0 = frozen linear, no adapter) */
  int32_t row_base;         /* added to every row index of the Philox counter (SPEC.md §3): a microbatch
                               split over several calls keeps its masks; 0 otherwise */
  LfSegment segments[LF_MAX_SEGMENTS];
  const int32_t* routes;    /* device: ceil(m/128) x 4 int32, from lf_build_routes */
  const uint8_t* keep_mask; /* device, optional explicit m x k keep mask (1 keep, 0 drop); NULL = Philox */
  void* workspace;          /* device scratch, zero-filled once, >= lf_workspace_bytes(); kernels leave it zeroed */
  size_t workspace_bytes;
  /* device, optional m x (k/8) bytes: the Philox keep mask bit-packed (bit e of byte
   * [row][col/8] = column col/8*8+e). lf_dropout_down_fwd writes it for rows of segments
   * with p > 0; lf_grad_down / lf_grad_input read it instead of re-running Philox.
   * NULL: every kernel regenerates the mask. Ignored when keep_mask is set. */
  uint8_t* keep_bits;
  /* device, optional: a uint64 step counter added to every segment's Philox offset,
   * read by the kernels when they run — so a captured CUDA graph that advances it on
   * the device draws a fresh mask on every replay. NULL: offsets are the host values. */
  const uint64_t* offset_dev;
} LfProblem;

/* Bytes of zero-initialised scratch one problem needs (split-K partials + tile counters). */
LF_API size_t lf_workspace_bytes(int32_t m, int32_t rank_total);

/* Host-only introspection (no device work, no CUDA context): the CTA grid lf_grad_up would
   launch for an m x n problem of width rank_total on `sms` SMs — n_split CTAs along n, each
   owning at most 8 128-column subtiles, times m_split along m, in one resident wave
   (n_split * m_split <= sms). LF_E_INVALID for non-positive sizes or a rank_total whose
   accumulators do not fit TMEM. */
LF_API int lf_grad_up_grid(int32_t m, int32_t n, int32_t rank_total, int32_t sms, int32_t* n_split, int32_t* m_split);

/* Routing table: per 128-row tile {seg_lo, seg_hi, col_lo, col_hi} (16 B). */
LF_API int lf_build_routes(const LfProblem* p, int32_t* routes_out, void* stream);

/* ① dropout + down-projection: s_hat (m x R, bf16) = scaled (M⊙X)·A_catᵀ, zero off-segment. */
LF_API int lf_dropout_down_fwd(const LfProblem* p, const uint16_t* x, const uint16_t* a_cat, uint16_t* s_hat,
                        void* stream);

/* ② base GEMM with the up-projection fused as one extra K-chunk: y = X·Wᵀ + Ŝ·B_catᵀ. */
LF_API int lf_base_fwd(const LfProblem* p, const uint16_t* x, const uint16_t* w, const uint16_t* s_hat,
                const uint16_t* b_cat, uint16_t* y, void* stream);

/* ③ one read of dY: ds (m x R, bf16) = scaled dY·B_cat; db_accum (n x R, fp32) += dYᵀ·Ŝ. */
LF_API int lf_grad_up(const LfProblem* p, const uint16_t* dy, const uint16_t* b_cat, const uint16_t* s_hat, uint16_t* ds,
               float* db_accum, void* stream);

/* ③ for projections that read the same input (q/k/v, gate/up): lf_grad_up for j < nproj
 * (<= 3) as one launch plus one dŜ finalize launch (the per-launch fixed cost paid once).
 * Each problem needs its own workspace (one launch holds all their split-K partials); falls
 * back to per-projection lf_grad_up when workspaces are shared. ABI 5. */
LF_API int lf_grad_up_group(const LfProblem* const* probs, int32_t nproj, const uint16_t* const* dy,
                            const uint16_t* const* b_cat, const uint16_t* const* s_hat, uint16_t* const* ds,
                            float* const* db_accum, void* stream);

/* ④ da_accum (R x k, fp32) += dŜᵀ·(M⊙X). */
LF_API int lf_grad_down(const LfProblem* p, const uint16_t* x, const uint16_t* ds, float* da_accum, void* stream);

/* ④ for projections that read the same input X (q/k/v, gate/up):
 * da_accum[j] (R_j x k, fp32) += dŜ_jᵀ·(M_j⊙X) for j < nproj (<= 3), one launch that reads
 * each X tile from DRAM once (projection j's copy is masked with its own keep bits).
 * probs[j] is projection j's problem (same m, k; any segment table since ABI 5). Falls back
 * to per-projection lf_grad_down when the accumulators do not fit one launch. ABI 4. */
LF_API int lf_grad_down_group(const LfProblem* const* probs, int32_t nproj, const uint16_t* x,
                              const uint16_t* const* ds, float* const* da_accum, void* stream);

/* ② for a shared-input group (q/k/v): y[j] = X·W_jᵀ + Ŝ_j·B_jᵀ for j < nproj (<= 3) as ONE
 * GEMM over the concatenated output columns (k/v's narrow N no longer runs as its own
 * under-filled launch). probs[j]: projection j's problem (same m, k; any segment table);
 * w / s_hat / b_cat / y: per-projection arrays as for lf_base_fwd. Falls back to
 * per-projection lf_base_fwd for other shapes. ABI 5. */
LF_API int lf_base_fwd_group(const LfProblem* const* probs, int32_t nproj, const uint16_t* x,
                             const uint16_t* const* w, const uint16_t* const* s_hat, const uint16_t* const* b_cat,
                             uint16_t* const* y, void* stream);

/* ⑤ for a shared-input group: dx = Σ_j dY_j·W_j + M_j ⊙ (dŜ_j·A_cat_j) as ONE GEMM over the
 * concatenated reduction dims, written once (each projection's masked LoRA term enters the
 * accumulator before the main loop; masks from the packed keep bits ① wrote). Falls back to
 * lf_grad_input + lf_grad_input_accum per projection for other shapes. ABI 5. */
LF_API int lf_grad_input_group(const LfProblem* const* probs, int32_t nproj, const uint16_t* const* dy,
                               const uint16_t* const* w, const uint16_t* const* ds, const uint16_t* const* a_cat,
                               uint16_t* dx, void* stream);

/* ⑤ dx = dY·W + M ⊙ (dŜ·A_cat), written once. */
LF_API int lf_grad_input(const LfProblem* p, const uint16_t* dy, const uint16_t* w, const uint16_t* ds,
                  const uint16_t* a_cat, uint16_t* dx, void* stream);

/* ⑤ accumulating: dx += dY·W + M ⊙ (dŜ·A_cat) — the GEMM epilogue adds its bf16 result into
 * dx (bf16, m x k) in L2 (red.add of bf16 pairs, one rounding per element; each element is
 * added once per call, so the sum is deterministic). Several projections that read the
 * same input (q/k/v, gate/up: SURVEY §8(f)#4) sum their input gradients this way instead of
 * through separate elementwise adds. Every tile shape is supported (LF_E_UNSUPPORTED is
 * kept for ABI 4 callers). ABI 4. */
LF_API int lf_grad_input_accum(const LfProblem* p, const uint16_t* dy, const uint16_t* w, const uint16_t* ds,
                        const uint16_t* a_cat, uint16_t* dx, void* stream);

/* Materialise the keep mask (m x k uint8) of SPEC.md §3 — for explicit-mask callers and parity tests. */
LF_API int lf_dropout_mask(const LfProblem* p, uint8_t* keep_out, void* stream);

/* Packed keep bits of the same mask (m x k/8 bytes, 16-byte aligned; bit c of byte j of a
 * row = column 8j + c). Input-free, so callers may run it on a side stream ahead of ①. */
LF_API int lf_keep_bits(const LfProblem* p, uint8_t* bits_out, void* stream);

/* Column blocks of fp32 row-major matrices copied out contiguously, all in one launch: for
 * block i, dst[i] (rows[i] x width[i], row-major) = src[i][:, col[i] : col[i] + width[i]] of a
 * rows[i] x ld[i] matrix. Turns dB_cat's per-adapter column blocks (n x R) into the
 * contiguous n x r gradients an optimizer expects (a multi-adapter call's lora_B grads);
 * no reference counterpart (the reference has no gradient layout). 0 <= nblocks <=
 * LF_MAX_COPY_BLOCKS. ABI 6. */
LF_API int lf_copy_column_blocks(int32_t nblocks, const float* const* src, const int32_t* rows, const int32_t* ld,
                                 const int32_t* col, const int32_t* width, float* const* dst, void* stream);

/* Thread-local message describing the last failure (never NULL). */
LF_API const char* lf_last_error(void);

LF_API int lf_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LORAFUSION_B200_H */
