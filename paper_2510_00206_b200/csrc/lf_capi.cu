// lf_capi.cu — the extern "C" boundary (include/lorafusion_b200.h).
//
// Host side only: argument validation (ValueError-class failures → LF_E_INVALID, the
// reference's ValidationError convention, ls/errors.py:12), conversion of the segment
// table into kernel-parameter form, TMA tensor-map encoding, grid heuristics and the
// launches. No allocation, no host synchronisation, no global device state beyond a
// per-device cache of the SM count.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "lf_kernels.h"
#include "lorafusion_b200.h"

namespace lf {
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("LF_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
}  // namespace lf

namespace {

thread_local std::string g_err = "no error";

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(const char* what) {
  const cudaError_t e = cudaGetLastError();
  return fail(LF_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D bf16 row-major tensor [rows, cols] (row stride ld elements), box [box_rows, box_cols]
bool make_map(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_cols,
              uint32_t box_rows, CUtensorMapSwizzle sw) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D map over a row-major uint8 array (the packed keep bits); ld in bytes, multiple of 16
bool make_map_u8(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_cols,
                 uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// tuning override from the environment (profiling sweeps), read once per name
int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

struct Dev {
  int id = -1;
  int sms = 0;
  int major = 0;
  int minor = 0;
};

int current_device(Dev* d) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_fail("cudaGetDevice");
  static Dev cache[64];
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64) return fail(LF_E_CUDA, "device ordinal %d out of range", dev);
  if (cache[dev].id != dev) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return cuda_fail("cudaGetDeviceProperties");
    cache[dev].id = dev;
    cache[dev].sms = prop.multiProcessorCount;
    cache[dev].major = prop.major;
    cache[dev].minor = prop.minor;
  }
  *d = cache[dev];
  if (d->major != 10 || d->minor != 0)
    return fail(LF_E_UNSUPPORTED, "lorafusion_b200 kernels are built for sm_100a (B200); device is sm_%d%d",
                d->major, d->minor);
  return LF_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// ---------------------------------------------------------------------------------
// validation + conversion of the problem into kernel-parameter form
// ---------------------------------------------------------------------------------
int validate(const LfProblem* p, bool need_routes, lf::LfSegTable* t) {
  if (!p) return fail(LF_E_INVALID, "problem is NULL");
  if (p->m < 1 || p->k < 1 || p->n < 1) return fail(LF_E_INVALID, "m, k, n must all be >= 1, got (%d, %d, %d)", p->m, p->k, p->n);
  if (p->k % 8 || p->n % 8)
    return fail(LF_E_INVALID, "k and n must be multiples of 8 (16-byte TMA row pitch), got k=%d n=%d", p->k, p->n);
  if (p->num_segments < 0 || p->num_segments > LF_MAX_SEGMENTS)
    return fail(LF_E_INVALID, "num_segments must be in [0, %d], got %d", LF_MAX_SEGMENTS, p->num_segments);
  if (p->rank_total < 0 || p->rank_total > LF_MAX_RANK_TOTAL || p->rank_total % 16)
    return fail(LF_E_INVALID, "rank_total must be a multiple of 16 in [0, %d], got %d", LF_MAX_RANK_TOTAL,
                p->rank_total);
  if (p->num_segments > 0 && p->rank_total < 16)
    return fail(LF_E_INVALID, "rank_total must be >= 16 when segments are present");
  memset(t, 0, sizeof(*t));
  static const int debug_flags = [] {
    const char* e = getenv("LF_DEBUG");
    return e ? atoi(e) : 0;
  }();
  t->debug = debug_flags;
  t->nseg = p->num_segments;
  t->m = p->m;
  t->rtot = p->rank_total;
  if (p->row_base < 0) return fail(LF_E_INVALID, "row_base must be >= 0, got %d", p->row_base);
  t->row_base = p->row_base;
  bool any_dropout = false;
  int prev_row = 0;
  for (int i = 0; i < p->num_segments; ++i) {
    const LfSegment& s = p->segments[i];
    if (s.row_start < prev_row || s.row_end < s.row_start || s.row_end > p->m)
      return fail(LF_E_INVALID,
                  "segment %d rows [%d, %d) must be sorted, disjoint and inside [0, m=%d)", i, s.row_start, s.row_end,
                  p->m);
    if (s.rank < 16 || s.rank % 16 || s.col_start % 16 || s.col_start < 0 || s.col_start + s.rank > p->rank_total)
      return fail(LF_E_INVALID, "segment %d columns [%d, %d) must be 16-aligned and inside rank_total=%d", i,
                  s.col_start, s.col_start + s.rank, p->rank_total);
    // column blocks are shared (segments of one adapter, SPEC.md §1) or disjoint
    for (int j = 0; j < i; ++j) {
      const LfSegment& o = p->segments[j];
      const bool same = o.col_start == s.col_start && o.rank == s.rank;
      const bool disjoint = o.col_start + o.rank <= s.col_start || s.col_start + s.rank <= o.col_start;
      if (!same && !disjoint)
        return fail(LF_E_INVALID, "segment %d columns [%d, %d) partially overlap segment %d's [%d, %d)", i,
                    s.col_start, s.col_start + s.rank, j, o.col_start, o.col_start + o.rank);
    }
    if (!(s.dropout_p >= 0.f && s.dropout_p < 1.f))
      return fail(LF_E_INVALID, "segment %d dropout_p must be in [0, 1), got %g", i, (double)s.dropout_p);
    if (!std::isfinite(s.scaling)) return fail(LF_E_INVALID, "segment %d scaling must be finite", i);
    prev_row = s.row_end;
    lf::LfSegDev& d = t->seg[i];
    d.row0 = s.row_start;
    d.row1 = s.row_end;
    d.col0 = s.col_start;
    d.ncol = s.rank;
    d.scale = (float)((double)s.scaling / (1.0 - (double)s.dropout_p));
    d.thr = 2u * (uint32_t)std::floor((double)s.dropout_p * 32768.0);  // even: SPEC.md §3
    d.key0 = (uint32_t)(s.seed & 0xFFFFFFFFull);
    d.key1 = (uint32_t)(s.seed >> 32);
    d.off0 = (uint32_t)(s.offset & 0xFFFFFFFFull);
    d.off1 = (uint32_t)(s.offset >> 32);
    if (d.thr) any_dropout = true;
  }
  // widest per-tile hull, as lf_routes_kernel forms it: segments are sorted and disjoint, so
  // only a segment's first and last 128-row tiles can be shared with neighbours
  {
    int cur = -1, c0 = 0, c1 = 0, wmax = 0;
    for (int i = 0; i < p->num_segments; ++i) {
      const lf::LfSegDev& d = t->seg[i];
      if (d.row0 >= d.row1) continue;
      const int t0 = d.row0 / 128, t1 = (d.row1 - 1) / 128;
      if (t0 == cur) {
        c0 = c0 < d.col0 ? c0 : d.col0;
        c1 = c1 > d.col0 + d.ncol ? c1 : d.col0 + d.ncol;
      } else {
        if (cur >= 0 && c1 - c0 > wmax) wmax = c1 - c0;
        cur = t0;
        c0 = d.col0;
        c1 = d.col0 + d.ncol;
      }
      if (t1 > t0) {  // t0 is complete; interior tiles carry this block alone
        if (c1 - c0 > wmax) wmax = c1 - c0;
        cur = t1;
        c0 = d.col0;
        c1 = d.col0 + d.ncol;
      }
    }
    if (cur >= 0 && c1 - c0 > wmax) wmax = c1 - c0;
    t->wmax = wmax > 0 ? wmax : 16;
  }
  if (p->keep_mask) {
    t->mask_mode = 2;
    t->mask = p->keep_mask;
    t->ld_mask = p->k;
  } else {
    t->mask_mode = any_dropout ? 1 : 0;
    if (any_dropout && p->keep_bits) {
      if (!aligned16(p->keep_bits)) return fail(LF_E_INVALID, "keep_bits must be 16-byte aligned");
      t->bits = p->keep_bits;
      t->ld_bits = p->k / 8;
    }
  }
  if (need_routes && p->num_segments > 0 && !p->routes) return fail(LF_E_INVALID, "routes is NULL (call lf_build_routes)");
  if (p->offset_dev && (reinterpret_cast<uintptr_t>(p->offset_dev) & 7u))
    return fail(LF_E_INVALID, "offset_dev must be 8-byte aligned");
  t->off_dev = p->offset_dev;
  return LF_OK;
}

int check_ptr(const void* ptr, const char* name) {
  if (!ptr) return fail(LF_E_INVALID, "%s is NULL", name);
  if (!aligned16(ptr)) return fail(LF_E_INVALID, "%s must be 16-byte aligned", name);
  return LF_OK;
}

int check_workspace(const LfProblem* p) {
  if (!p->workspace) return fail(LF_E_INVALID, "workspace is NULL");
  if (p->workspace_bytes < lf_workspace_bytes(p->m, p->rank_total))
    return fail(LF_E_INVALID, "workspace too small: %zu < %zu bytes", p->workspace_bytes,
                lf_workspace_bytes(p->m, p->rank_total));
  if (!aligned16(p->workspace)) return fail(LF_E_INVALID, "workspace must be 16-byte aligned");
  return LF_OK;
}

void split_workspace(const LfProblem* p, float** ws, int32_t** counters) {
  *ws = reinterpret_cast<float*>(p->workspace);
  *counters = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(p->workspace) +
                                         align_up((size_t)p->m * p->rank_total * 4, 256));
}

int occupancy_for_smem(int smem_bytes) {
  const int per_sm = 228 * 1024;
  int c = per_sm / (smem_bytes + 1024);
  return c < 1 ? 1 : c;
}

#define LF_TRY(expr)             \
  do {                           \
    const int _rc = (expr);      \
    if (_rc != LF_OK) return _rc; \
  } while (0)

}  // namespace

// =================================================================================
extern "C" {

int lf_abi_version(void) { return LF_ABI_VERSION; }

const char* lf_last_error(void) { return g_err.c_str(); }

size_t lf_workspace_bytes(int32_t m, int32_t rank_total) {
  if (m < 0 || rank_total < 0) return 0;
  const size_t tiles = ((size_t)m + 127) / 128;
  return align_up((size_t)m * rank_total * 4, 256) + align_up(tiles * 4, 256);
}

int lf_grad_up_grid(int32_t m, int32_t n, int32_t rank_total, int32_t sms, int32_t* n_split, int32_t* m_split) {
  if (!n_split || !m_split) return fail(LF_E_INVALID, "n_split / m_split is NULL");
  if (m < 1 || n < 1 || sms < 1 || rank_total < 16 || rank_total % 16 || rank_total > LF_MAX_RANK_TOTAL)
    return fail(LF_E_INVALID, "bad grad_up grid query (m=%d n=%d rank_total=%d sms=%d)", m, n, rank_total, sms);
  int ns = 0, ms = 0, nacc = 0;
  lf::grad_up_grid(m, n, rank_total, rank_total, sms, 1, &ns, &ms, &nacc);
  if (ns <= 0) return fail(LF_E_INVALID, "rank_total=%d too large for grad_up TMEM budget", rank_total);
  *n_split = ns;
  *m_split = ms;
  return LF_OK;
}

int lf_build_routes(const LfProblem* p, int32_t* routes_out, void* stream) {
  lf::LfSegTable t;
  LF_TRY(validate(p, false, &t));
  LF_TRY(check_ptr(routes_out, "routes_out"));
  Dev d;
  LF_TRY(current_device(&d));
  if (lf::routes_launch(t, routes_out, (p->m + 127) / 128, (cudaStream_t)stream)) return cuda_fail("routes launch");
  return LF_OK;
}

int lf_dropout_mask(const LfProblem* p, uint8_t* keep_out, void* stream) {
  lf::LfSegTable t;
  LF_TRY(validate(p, false, &t));
  if (!keep_out) return fail(LF_E_INVALID, "keep_out is NULL");
  Dev d;
  LF_TRY(current_device(&d));
  if (lf::mask_launch(t, p->k, keep_out, (cudaStream_t)stream)) return cuda_fail("mask launch");
  return LF_OK;
}

int lf_keep_bits(const LfProblem* p, uint8_t* bits_out, void* stream) {
  lf::LfSegTable t;
  LF_TRY(validate(p, false, &t));
  LF_TRY(check_ptr(bits_out, "bits_out"));
  Dev d;
  LF_TRY(current_device(&d));
  if (lf::keep_bits_launch(t, p->k, bits_out, p->k / 8, d.sms, (cudaStream_t)stream))
    return cuda_fail("keep_bits launch");
  return LF_OK;
}

// Per-adapter dB gradients out of dB_cat's column blocks in one launch (see the header)
int lf_copy_column_blocks(int32_t nblocks, const float* const* src, const int32_t* rows, const int32_t* ld,
                          const int32_t* col, const int32_t* width, float* const* dst, void* stream) {
  if (nblocks < 0 || nblocks > LF_MAX_COPY_BLOCKS)
    return fail(LF_E_INVALID, "lf_copy_column_blocks: nblocks %d outside [0, %d]", nblocks, LF_MAX_COPY_BLOCKS);
  if (nblocks == 0) return LF_OK;
  if (!src || !rows || !ld || !col || !width || !dst)
    return fail(LF_E_INVALID, "lf_copy_column_blocks: NULL argument array");
  lf::CopyBlocksArgs a;
  a.n = nblocks;
  for (int i = 0; i < nblocks; ++i) {
    if (!src[i] || !dst[i]) return fail(LF_E_INVALID, "lf_copy_column_blocks: block %d has a NULL pointer", i);
    if (rows[i] <= 0 || width[i] <= 0 || col[i] < 0 || (int64_t)col[i] + width[i] > ld[i])
      return fail(LF_E_INVALID, "lf_copy_column_blocks: block %d: rows %d, columns [%d, %d) of a row of %d", i,
                  rows[i], col[i], col[i] + width[i], ld[i]);
    a.blk[i] = lf::CopyBlock{src[i], dst[i], rows[i], ld[i], col[i], width[i]};
  }
  Dev d;
  LF_TRY(current_device(&d));
  if (lf::copy_blocks_launch(a, d.sms, (cudaStream_t)stream)) return cuda_fail("copy_column_blocks launch");
  return LF_OK;
}

int lf_dropout_down_fwd(const LfProblem* p, const uint16_t* x, const uint16_t* a_cat, uint16_t* s_hat,
                        void* stream) {
  lf::LfSegTable t;
  LF_TRY(validate(p, true, &t));
  if (p->num_segments == 0) return fail(LF_E_INVALID, "lf_dropout_down_fwd needs at least one segment");
  LF_TRY(check_ptr(x, "x"));
  LF_TRY(check_ptr(a_cat, "a_cat"));
  LF_TRY(check_ptr(s_hat, "s_hat"));
  LF_TRY(check_workspace(p));
  Dev d;
  LF_TRY(current_device(&d));
  CUtensorMap tx, ta;
  if (!make_map(&tx, x, p->m, p->k, p->k, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&ta, a_cat, p->rank_total, p->k, p->k, 64, 16, CU_TENSOR_MAP_SWIZZLE_128B))
    return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (x / a_cat)");
  lf::DownArgs a;
  memset(&a, 0, sizeof(a));
  a.m = p->m;
  a.k = p->k;
  a.rtot = p->rank_total;
  a.s_hat = s_hat;
  split_workspace(p, &a.ws, &a.counters);
  a.routes = reinterpret_cast<const lf::LfRoute*>(p->routes);
  a.segs = t;
  const int tiles_m = (p->m + 127) / 128;
  const int nkb = (p->k + 63) / 64;
  int stages = 0, stage_bytes = 0;
  lf::down_config(t.wmax, &stages, &stage_bytes);
  const int occ = occupancy_for_smem(stages * stage_bytes + 2048 + lf::down_extra_smem(t.mask_mode));
  // one resident wave sharing the units evenly (stream-K); at least 4 k-blocks per CTA so
  // the split-K partial traffic stays small next to the X stream
  const long units = (long)tiles_m * nkb;
  long ctas = (long)occ * d.sms;
  if (ctas > units / 4) ctas = units / 4;
  if (ctas < 1) ctas = 1;
  a.ctas = (int)ctas;
  if (lf::down_launch(tx, ta, a, d.sms, (cudaStream_t)stream)) return cuda_fail("dropout_down launch");
  return LF_OK;
}

int lf_base_fwd(const LfProblem* p, const uint16_t* x, const uint16_t* w, const uint16_t* s_hat,
                const uint16_t* b_cat, uint16_t* y, void* stream) {
  lf::LfSegTable t;
  LF_TRY(validate(p, true, &t));
  LF_TRY(check_ptr(x, "x"));
  LF_TRY(check_ptr(w, "w"));
  LF_TRY(check_ptr(y, "y"));
  const bool lora = p->num_segments > 0;
  if (lora) {
    LF_TRY(check_ptr(s_hat, "s_hat"));
    LF_TRY(check_ptr(b_cat, "b_cat"));
  }
  Dev d;
  LF_TRY(current_device(&d));
  lf::GemmMaps maps;
  memset(&maps, 0, sizeof(maps));
  if (!make_map(&maps.a[0], x, p->m, p->k, p->k, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&maps.b[0], w, p->n, p->k, p->k, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))
    return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (x / w)");
  if (lora) {
    if (!make_map(&maps.a2[0], s_hat, p->m, p->rank_total, p->rank_total, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B) ||
        !make_map(&maps.b2[0], b_cat, p->n, p->rank_total, p->rank_total, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B))
      return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (s_hat / b_cat)");
  } else {
    maps.a2[0] = maps.a[0];
    maps.b2[0] = maps.b[0];
  }
  lf::GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = p->m;
  a.N = p->n;
  a.K = p->k;
  a.ldc = p->n;
  a.C = y;
  a.routes = lora ? reinterpret_cast<const lf::LfRoute*>(p->routes) : nullptr;
  a.segs = t;
  a.group = env_int("LF_GROUP", 0);
  if (lf::gemm_launch(lf::kGemmFwd, maps, a, d.sms, (cudaStream_t)stream)) return cuda_fail("base_fwd launch");
  return LF_OK;
}

int lf_grad_up(const LfProblem* p, const uint16_t* dy, const uint16_t* b_cat, const uint16_t* s_hat, uint16_t* ds,
               float* db_accum, void* stream) {
  lf::LfSegTable t;
  LF_TRY(validate(p, true, &t));
  if (p->num_segments == 0) return fail(LF_E_INVALID, "lf_grad_up needs at least one segment");
  LF_TRY(check_ptr(dy, "dy"));
  LF_TRY(check_ptr(b_cat, "b_cat"));
  LF_TRY(check_ptr(s_hat, "s_hat"));
  LF_TRY(check_ptr(ds, "ds"));
  LF_TRY(check_ptr(db_accum, "db_accum"));
  LF_TRY(check_workspace(p));
  Dev d;
  LF_TRY(current_device(&d));
  CUtensorMap tdy, tb, ts;
  if (!make_map(&tdy, dy, p->m, p->n, p->n, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&tb, b_cat, p->n, p->rank_total, p->rank_total, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B) ||
      !make_map(&ts, s_hat, p->m, p->rank_total, p->rank_total, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B))
    return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (dy / b_cat / s_hat)");
  lf::GradUpArgs a;
  memset(&a, 0, sizeof(a));
  a.m = p->m;
  a.n = p->n;
  a.rtot = p->rank_total;
  a.ds = ds;
  a.db = db_accum;
  split_workspace(p, &a.ws, &a.counters);
  a.routes = reinterpret_cast<const lf::LfRoute*>(p->routes);
  a.segs = t;
  static const int gu_per_sm_env = env_int("LF_GU_PER_SM", 0);
  const int per_sm = gu_per_sm_env > 0 ? gu_per_sm_env : 1;
  lf::grad_up_grid(p->m, p->n, p->rank_total, t.wmax, d.sms, per_sm, &a.n_split, &a.m_split, &a.nacc);
  static const int gu_ns_env = env_int("LF_GU_NSPLIT", 0);  // profiling: force the n-split
  if (gu_ns_env > 0 && a.n_split > 0) {
    const int tiles_n = (p->n + 127) / 128, tiles_m = (p->m + 127) / 128;
    const int max_nsub = (512 / per_sm - 2 * t.wmax) / p->rank_total;
    int ns = gu_ns_env < tiles_n ? gu_ns_env : tiles_n;
    if ((tiles_n + ns - 1) / ns <= max_nsub) {
      int ms = d.sms * per_sm / ns;
      a.n_split = ns;
      a.m_split = ms < 1 ? 1 : (ms > tiles_m ? tiles_m : ms);
    }
  }
  if (a.n_split <= 0) return fail(LF_E_INVALID, "rank_total=%d too large for grad_up TMEM budget", p->rank_total);
  if (lf::grad_up_launch(tdy, tb, ts, a, d.sms, per_sm, (cudaStream_t)stream)) return cuda_fail("grad_up launch");
  return LF_OK;
}

int lf_grad_down(const LfProblem* p, const uint16_t* x, const uint16_t* ds, float* da_accum, void* stream) {
  lf::LfSegTable t;
  LF_TRY(validate(p, true, &t));
  if (p->num_segments == 0) return fail(LF_E_INVALID, "lf_grad_down needs at least one segment");
  LF_TRY(check_ptr(x, "x"));
  LF_TRY(check_ptr(ds, "ds"));
  LF_TRY(check_ptr(da_accum, "da_accum"));
  Dev d;
  LF_TRY(current_device(&d));
  CUtensorMap tx, td, tk;
  if (!make_map(&tx, x, p->m, p->k, p->k, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&td, ds, p->m, p->rank_total, p->rank_total, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B))
    return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (x / ds)");
  lf::GradDownArgs a;
  memset(&a, 0, sizeof(a));
  // ①'s packed keep bits ride in each stage by TMA (16 B x 128 rows per unit) when the
  // bit rows are 16-byte pitched; otherwise the mask warps read them from global memory
  tk = tx;
  if (t.mask_mode == 1 && t.bits && t.ld_bits % 16 == 0) {
    if (!make_map_u8(&tk, t.bits, p->m, t.ld_bits, t.ld_bits, 16, 128))
      return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (keep bits)");
    a.bits_tma = 1;
  }
  a.m = p->m;
  a.k = p->k;
  a.rtot = p->rank_total;
  a.da = da_accum;
  a.routes = reinterpret_cast<const lf::LfRoute*>(p->routes);
  a.segs = t;
  int stages = 0, stage_bytes = 0;
  lf::grad_down_config(t.wmax, a.bits_tma != 0, &stages, &stage_bytes);
  const int occ = occupancy_for_smem(stages * stage_bytes + 2048);
  const int tiles_k = (p->k + 127) / 128;
  const int tiles_m = (p->m + 127) / 128;
  // one resident wave sharing the units evenly (stream-K)
  long ctas = (long)occ * d.sms;
  if (ctas > (long)tiles_m * tiles_k) ctas = (long)tiles_m * tiles_k;
  a.ctas = (int)ctas;
  if (lf::grad_down_launch(tx, td, tk, a, d.sms, (cudaStream_t)stream)) return cuda_fail("grad_down launch");
  return LF_OK;
}

// ③ over a shared-input group: one ③ launch and one dŜ finalize launch for the J projections
// (each its own grid, sized by its share of the dY bytes, and its own split-K workspace —
// the problems must not share one); otherwise (J = 1, LF_GROUP_UP=0) per projection.
int lf_grad_up_group(const LfProblem* const* probs, int32_t nproj, const uint16_t* const* dy,
                     const uint16_t* const* b_cat, const uint16_t* const* s_hat, uint16_t* const* ds,
                     float* const* db_accum, void* stream) {
  if (!probs || nproj < 1 || nproj > lf::kMaxGroup || !dy || !b_cat || !s_hat || !ds || !db_accum)
    return fail(LF_E_INVALID, "lf_grad_up_group: 1..%d projections with dy / b_cat / s_hat / ds / db arrays",
                lf::kMaxGroup);
  static const int group_env = env_int("LF_GROUP_UP", 1);
  bool fused = nproj > 1 && group_env;
  lf::LfSegTable t[lf::kMaxGroup];
  double bytes[lf::kMaxGroup], total = 0;
  for (int j = 0; j < nproj; ++j) {
    const LfProblem* p = probs[j];
    if (!p) return fail(LF_E_INVALID, "lf_grad_up_group: projection %d has no problem", j);
    LF_TRY(validate(p, true, &t[j]));
    if (p->num_segments == 0) return fail(LF_E_INVALID, "lf_grad_up_group needs at least one segment");
    LF_TRY(check_ptr(dy[j], "dy"));
    LF_TRY(check_ptr(b_cat[j], "b_cat"));
    LF_TRY(check_ptr(s_hat[j], "s_hat"));
    LF_TRY(check_ptr(ds[j], "ds"));
    LF_TRY(check_ptr(db_accum[j], "db_accum"));
    LF_TRY(check_workspace(p));
    for (int i = 0; i < j; ++i)
      if (probs[i]->workspace == p->workspace) fused = false;  // one launch needs disjoint workspaces
    bytes[j] = (double)p->m * p->n;
    total += bytes[j];
  }
  if (!fused) {
    for (int j = 0; j < nproj; ++j) LF_TRY(lf_grad_up(probs[j], dy[j], b_cat[j], s_hat[j], ds[j], db_accum[j], stream));
    return LF_OK;
  }
  Dev d;
  LF_TRY(current_device(&d));
  lf::GroupUpMaps maps;
  memset(&maps, 0, sizeof(maps));
  lf::GroupUpArgs g;
  memset(&g, 0, sizeof(g));
  g.J = nproj;
  for (int j = 0; j < nproj; ++j) {
    const LfProblem* p = probs[j];
    if (!make_map(&maps.dy[j], dy[j], p->m, p->n, p->n, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_map(&maps.b[j], b_cat[j], p->n, p->rank_total, p->rank_total, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B) ||
        !make_map(&maps.s[j], s_hat[j], p->m, p->rank_total, p->rank_total, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B))
      return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (dy / b_cat / s_hat)");
    lf::GradUpArgs& a = g.p[j];
    a.m = p->m;
    a.n = p->n;
    a.rtot = p->rank_total;
    a.ds = ds[j];
    a.db = db_accum[j];
    split_workspace(p, &a.ws, &a.counters);
    a.routes = reinterpret_cast<const lf::LfRoute*>(p->routes);
    a.segs = t[j];
    // this projection's share of the SMs, by its dY bytes (one resident wave for the group)
    int sms_j = (int)(d.sms * bytes[j] / total);
    if (sms_j < 1) sms_j = 1;
    lf::grad_up_grid(p->m, p->n, p->rank_total, t[j].wmax, sms_j, 1, &a.n_split, &a.m_split, &a.nacc);
    if (a.n_split <= 0) return fail(LF_E_INVALID, "rank_total=%d too large for grad_up TMEM budget", p->rank_total);
  }
  if (lf::grad_up_group_launch(maps, g, (cudaStream_t)stream)) return cuda_fail("grad_up_group launch");
  return LF_OK;
}

// ④ over a shared-input group: one launch when every projection's keep bits (if any) ①'s
// launch left 16-byte pitched and the J accumulators fit TMEM; otherwise (and for J = 1) the
// per-projection lf_grad_down. Any segment table: dŜ_j is zero off each row's segment.
int lf_grad_down_group(const LfProblem* const* probs, int32_t nproj, const uint16_t* x, const uint16_t* const* ds,
                       float* const* da_accum, void* stream) {
  if (!probs || nproj < 1 || nproj > lf::kMaxGroup || !ds || !da_accum)
    return fail(LF_E_INVALID, "lf_grad_down_group: 1..%d projections with ds / da_accum arrays", lf::kMaxGroup);
  LF_TRY(check_ptr(x, "x"));
  bool fused = nproj > 1;
  lf::LfSegTable t[lf::kMaxGroup];
  int rsum = 0, rmax = 0;
  for (int j = 0; j < nproj; ++j) {
    const LfProblem* p = probs[j];
    if (!p) return fail(LF_E_INVALID, "lf_grad_down_group: projection %d has no problem", j);
    LF_TRY(validate(p, true, &t[j]));
    LF_TRY(check_ptr(ds[j], "ds"));
    LF_TRY(check_ptr(da_accum[j], "da_accum"));
    if (p->m != probs[0]->m || p->k != probs[0]->k)
      return fail(LF_E_INVALID, "lf_grad_down_group: projections must share the input (m, k)");
    // any segment table (dŜ_j is zero off each row's segment; ① leaves all-ones keep bits
    // on rows of p = 0 segments)
    const bool bits_ok = t[j].mask_mode == 0 || (t[j].mask_mode == 1 && t[j].bits && t[j].ld_bits % 16 == 0);
    if (p->row_base != 0 || !bits_ok) fused = false;
    rsum += p->rank_total;
    if (p->rank_total > rmax) rmax = p->rank_total;
  }
  static const int group_env = env_int("LF_GROUP_DOWN", 1);
  if (2 * rsum > 512 || !group_env) fused = false;
  if (!fused) {
    for (int j = 0; j < nproj; ++j) LF_TRY(lf_grad_down(probs[j], x, ds[j], da_accum[j], stream));
    return LF_OK;
  }
  Dev d;
  LF_TRY(current_device(&d));
  lf::GroupDownMaps maps;
  memset(&maps, 0, sizeof(maps));
  lf::GroupDownArgs a;
  memset(&a, 0, sizeof(a));
  const LfProblem* p0 = probs[0];
  if (!make_map(&maps.x, x, p0->m, p0->k, p0->k, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))
    return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (x)");
  int off = 0;
  for (int j = 0; j < nproj; ++j) {
    const LfProblem* p = probs[j];
    if (!make_map(&maps.d[j], ds[j], p->m, p->rank_total, p->rank_total, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B))
      return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (ds)");
    a.masked[j] = t[j].mask_mode == 1;
    if (a.masked[j] && !make_map_u8(&maps.bits[j], t[j].bits, p->m, t[j].ld_bits, t[j].ld_bits, 16, 128))
      return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (keep bits)");
    a.R[j] = p->rank_total;
    a.off[j] = off;
    off += p->rank_total;
    a.da[j] = da_accum[j];
  }
  a.m = p0->m;
  a.k = p0->k;
  a.J = nproj;
  a.rsum = rsum;
  a.rmax = rmax;
  a.debug = t[0].debug;
  int stages = 0, stage_bytes = 0;
  lf::grad_down_group_config(rmax, &stages, &stage_bytes);
  const int occ = occupancy_for_smem(stages * stage_bytes + 2048);
  const long units = (long)((p0->k + 127) / 128) * ((p0->m + 127) / 128) * nproj;
  long ctas = (long)occ * d.sms;
  if (ctas > units) ctas = units;
  a.ctas = (int)ctas;
  if (lf::grad_down_group_launch(maps, a, (cudaStream_t)stream)) return cuda_fail("grad_down_group launch");
  return LF_OK;
}

static int grad_input_impl(const LfProblem* p, const uint16_t* dy, const uint16_t* w, const uint16_t* ds,
                           const uint16_t* a_cat, uint16_t* dx, int accumulate, void* stream) {
  lf::LfSegTable t;
  LF_TRY(validate(p, true, &t));
  LF_TRY(check_ptr(dy, "dy"));
  LF_TRY(check_ptr(w, "w"));
  LF_TRY(check_ptr(dx, "dx"));
  const bool lora = p->num_segments > 0;
  if (lora) {
    LF_TRY(check_ptr(ds, "ds"));
    LF_TRY(check_ptr(a_cat, "a_cat"));
  }
  Dev d;
  LF_TRY(current_device(&d));
  const bool masked = lora && t.mask_mode != 0;
  lf::GemmMaps maps;
  memset(&maps, 0, sizeof(maps));
  // dX[m, k] = dY[m, n] · W[n, k]: A = dY (K-major), B = W (MN-major), K = n
  if (!make_map(&maps.a[0], dy, p->m, p->n, p->n, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&maps.b[0], w, p->n, p->k, p->k, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B))
    return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (dy / w)");
  if (lora) {
    if (!make_map(&maps.a2[0], ds, p->m, p->rank_total, p->rank_total, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B) ||
        !make_map(&maps.b2[0], a_cat, p->rank_total, p->k, p->k, 64, 16, CU_TENSOR_MAP_SWIZZLE_128B))
      return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (ds / a_cat)");
  } else {
    maps.a2[0] = maps.a[0];
    maps.b2[0] = maps.b[0];
  }
  lf::GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = p->m;
  a.N = p->k;
  a.K = p->n;
  a.ldc = p->k;
  a.C = dx;
  a.accumulate = accumulate;
  a.routes = lora ? reinterpret_cast<const lf::LfRoute*>(p->routes) : nullptr;
  a.segs = t;
  a.group = env_int("LF_GROUP", 0);
  const int rc = lf::gemm_launch(masked ? lf::kGemmDgradMasked : lf::kGemmDgrad, maps, a, d.sms, (cudaStream_t)stream);
  if (rc == lf::kGemmUnsupported)
    return fail(LF_E_UNSUPPORTED, "grad_input: accumulation is not built for the 256x512 tiles this shape uses");
  if (rc) return cuda_fail("grad_input launch");
  return LF_OK;
}

// shared-input groups (② / ⑤ over J projections that read the same input): one GEMM when
// the group's widths fit the group tiling; otherwise the projections run one by one (⑤: the
// first writes dX, the others add into it). LF_GROUP_GEMM=0 forces the per-projection path.
// The group kernels take each projection's whole rank-concat width as its LoRA K-range
// (no routing table): Ŝ_j / dŜ_j are zero off each row's segment, and ① leaves all-ones
// keep bits on rows of p = 0 segments, so any segment table works.
static bool group_ok(const LfProblem* p) { return p->row_base == 0 && p->rank_total >= 16; }

int lf_base_fwd_group(const LfProblem* const* probs, int32_t nproj, const uint16_t* x, const uint16_t* const* w,
                      const uint16_t* const* s_hat, const uint16_t* const* b_cat, uint16_t* const* y, void* stream) {
  if (!probs || nproj < 1 || nproj > lf::kMaxGroup || !w || !s_hat || !b_cat || !y)
    return fail(LF_E_INVALID, "lf_base_fwd_group: 1..%d projections with w / s_hat / b_cat / y arrays", lf::kMaxGroup);
  LF_TRY(check_ptr(x, "x"));
  bool fused = nproj > 1;
  lf::LfSegTable t[lf::kMaxGroup];
  for (int j = 0; j < nproj; ++j) {
    const LfProblem* p = probs[j];
    if (!p) return fail(LF_E_INVALID, "lf_base_fwd_group: projection %d has no problem", j);
    LF_TRY(validate(p, true, &t[j]));
    if (p->m != probs[0]->m || p->k != probs[0]->k)
      return fail(LF_E_INVALID, "lf_base_fwd_group: projections must share the input (m, k)");
    LF_TRY(check_ptr(w[j], "w"));
    LF_TRY(check_ptr(y[j], "y"));
    if (!group_ok(p)) fused = false;
  }
  static const int group_env = env_int("LF_GROUP_GEMM", 1);
  if (fused && group_env) {
    Dev d;
    LF_TRY(current_device(&d));
    lf::GemmMaps maps;
    memset(&maps, 0, sizeof(maps));
    lf::GemmArgs a;
    memset(&a, 0, sizeof(a));
    const LfProblem* p0 = probs[0];
    if (!make_map(&maps.a[0], x, p0->m, p0->k, p0->k, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))
      return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (x)");
    int n = 0;
    for (int j = 0; j < nproj; ++j) {
      const LfProblem* p = probs[j];
      LF_TRY(check_ptr(s_hat[j], "s_hat"));
      LF_TRY(check_ptr(b_cat[j], "b_cat"));
      if (!make_map(&maps.b[j], w[j], p->n, p->k, p->k, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
          !make_map(&maps.a2[j], s_hat[j], p->m, p->rank_total, p->rank_total, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B) ||
          !make_map(&maps.b2[j], b_cat[j], p->n, p->rank_total, p->rank_total, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B))
        return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (w / s_hat / b_cat)");
      n += p->n;
      a.send[j] = n;
      a.lcols[j] = p->rank_total;
      a.Cs[j] = y[j];
      a.ldcs[j] = p->n;
    }
    a.nseg = nproj;
    a.M = p0->m;
    a.N = n;
    a.K = p0->k;
    a.segs = t[0];
    a.group = env_int("LF_GROUP", 0);
    const int rc = lf::gemm_launch_group(lf::kGemmFwd, maps, a, d.sms, (cudaStream_t)stream);
    if (rc == 0) return LF_OK;
    if (rc != lf::kGemmUnsupported) return cuda_fail("base_fwd_group launch");
  }
  for (int j = 0; j < nproj; ++j) LF_TRY(lf_base_fwd(probs[j], x, w[j], s_hat[j], b_cat[j], y[j], stream));
  return LF_OK;
}

int lf_grad_input_group(const LfProblem* const* probs, int32_t nproj, const uint16_t* const* dy,
                        const uint16_t* const* w, const uint16_t* const* ds, const uint16_t* const* a_cat, uint16_t* dx,
                        void* stream) {
  if (!probs || nproj < 1 || nproj > lf::kMaxGroup || !dy || !w || !ds || !a_cat)
    return fail(LF_E_INVALID, "lf_grad_input_group: 1..%d projections with dy / w / ds / a_cat arrays", lf::kMaxGroup);
  LF_TRY(check_ptr(dx, "dx"));
  bool fused = nproj > 1;
  bool masked = false;
  lf::LfSegTable t[lf::kMaxGroup];
  for (int j = 0; j < nproj; ++j) {
    const LfProblem* p = probs[j];
    if (!p) return fail(LF_E_INVALID, "lf_grad_input_group: projection %d has no problem", j);
    LF_TRY(validate(p, true, &t[j]));
    if (p->m != probs[0]->m || p->k != probs[0]->k)
      return fail(LF_E_INVALID, "lf_grad_input_group: projections must share the input (m, k)");
    LF_TRY(check_ptr(dy[j], "dy"));
    LF_TRY(check_ptr(w[j], "w"));
    // the J masked LoRA partials take turns in the accumulator over each projection's whole
    // rank-concat width: wide multi-adapter widths (C3: R = 128, routing hulls of 64) make the
    // turns longer than the per-projection launches' hull-sized partials (C3 ⑤ 2.33 -> 2.40 ms)
    if (!group_ok(p) || p->rank_total > 32) fused = false;
    const bool m_j = t[j].mask_mode != 0;  // some segment drops (Philox) or an explicit mask
    if (m_j && !(t[j].mask_mode == 1 && t[j].bits)) fused = false;  // packed bits from ① only
    masked = masked || m_j;
  }
  static const int group_env = env_int("LF_GROUP_GEMM", 1);
  if (fused && group_env) {
    Dev d;
    LF_TRY(current_device(&d));
    lf::GemmMaps maps;
    memset(&maps, 0, sizeof(maps));
    lf::GemmArgs a;
    memset(&a, 0, sizeof(a));
    const LfProblem* p0 = probs[0];
    int kk = 0;
    for (int j = 0; j < nproj; ++j) {
      const LfProblem* p = probs[j];
      LF_TRY(check_ptr(ds[j], "ds"));
      LF_TRY(check_ptr(a_cat[j], "a_cat"));
      // dX[m, k] = Σ_j dY_j[m, n_j] · W_j[n_j, k]: A = dY_j (K-major), B = W_j (MN-major)
      if (!make_map(&maps.a[j], dy[j], p->m, p->n, p->n, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
          !make_map(&maps.b[j], w[j], p->n, p->k, p->k, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B) ||
          !make_map(&maps.a2[j], ds[j], p->m, p->rank_total, p->rank_total, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B) ||
          !make_map(&maps.b2[j], a_cat[j], p->rank_total, p->k, p->k, 64, 16, CU_TENSOR_MAP_SWIZZLE_128B))
        return fail(LF_E_CUDA, "cuTensorMapEncodeTiled failed (dy / w / ds / a_cat)");
      kk += p->n;
      a.send[j] = kk;
      a.lcols[j] = p->rank_total;
      a.gbits[j] = t[j].mask_mode == 1 ? t[j].bits : nullptr;
    }
    a.ld_gbits = t[0].ld_bits;
    a.nseg = nproj;
    a.M = p0->m;
    a.N = p0->k;
    a.K = kk;
    a.ldc = p0->k;
    a.C = dx;
    a.segs = t[0];
    a.group = env_int("LF_GROUP", 0);
    const int rc = lf::gemm_launch_group(masked ? lf::kGemmDgradMasked : lf::kGemmDgrad, maps, a, d.sms,
                                         (cudaStream_t)stream);
    if (rc == 0) return LF_OK;
    if (rc != lf::kGemmUnsupported) return cuda_fail("grad_input_group launch");
  }
  for (int j = 0; j < nproj; ++j)
    LF_TRY(grad_input_impl(probs[j], dy[j], w[j], ds[j], a_cat[j], dx, j > 0 ? 1 : 0, stream));
  return LF_OK;
}

int lf_grad_input(const LfProblem* p, const uint16_t* dy, const uint16_t* w, const uint16_t* ds,
                  const uint16_t* a_cat, uint16_t* dx, void* stream) {
  return grad_input_impl(p, dy, w, ds, a_cat, dx, 0, stream);
}

int lf_grad_input_accum(const LfProblem* p, const uint16_t* dy, const uint16_t* w, const uint16_t* ds,
                        const uint16_t* a_cat, uint16_t* dx, void* stream) {
  return grad_input_impl(p, dy, w, ds, a_cat, dx, 1, stream);
}

}  // extern "C"
