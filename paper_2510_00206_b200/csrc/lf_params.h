// lf_params.h — kernel parameter structs shared by the host launchers and the kernels.
// Passed by value (kernel parameter space), so a launch needs no H2D copy of the
// segment table: the per-segment data rides in the constant bank of every CTA.
#pragma once

#include <stdint.h>

#define LF_MAX_SEGS 32
#define LF_TILE_M 128
#define LF_MAX_RANK 128

namespace lf {

// Device-side view of one LfSegment (include/lorafusion_b200.h) with the derived
// quantities precomputed on the host: scale = scaling / (1 - p) as fp32 and the
// integer dropout threshold thr = 2 * floor(p * 32768), even (SPEC.md §3).
struct LfSegDev {
  int32_t row0, row1;  // token rows [row0, row1)
  int32_t col0, ncol;  // rank-concat columns [col0, col0 + ncol)
  float scale;         // scaling / (1 - p)
  uint32_t thr;        // keep iff u16 >= thr
  uint32_t key0, key1; // Philox key (seed)
  uint32_t off0, off1; // Philox counter words 2,3 (offset)
};

struct LfSegTable {
  int32_t nseg;
  int32_t m;
  int32_t rtot;         // rank-concat width R
  int32_t wmax;         // widest routing hull (col_hi - col_lo) of any 128-row tile: sizes the
                        // per-stage R-column operand buffers of ①③④ (≤ rtot; C3: 64 of 128)
  int32_t mask_mode;    // 0 = no dropout anywhere, 1 = Philox, 2 = explicit uint8 mask
  const uint8_t* mask;  // explicit keep mask (m x ld_mask) when mask_mode == 2
  int64_t ld_mask;
  uint8_t* bits;        // bit-packed Philox keep mask (m x ld_bits bytes) when mask_mode == 1, or null
  int64_t ld_bits;      // = k / 8
  int32_t debug;        // profiling knobs (env LF_DEBUG, default 0): skip pipeline pieces, results invalid
  int32_t row_base;     // added to the row word of every Philox counter (LfProblem::row_base)
  const uint64_t* off_dev;  // device step counter added to every segment's Philox offset, or null
  LfSegDev seg[LF_MAX_SEGS];
};

// per-128-row routing entry (16 B): segments [seg_lo, seg_hi], columns [col_lo, col_hi)
struct LfRoute {
  int32_t seg_lo, seg_hi, col_lo, col_hi;
};

}  // namespace lf
