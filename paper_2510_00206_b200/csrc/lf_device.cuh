// lf_device.cuh — sm_100a building blocks shared by every LoRAFusion-B200 kernel:
// mbarriers, TMA (cp.async.bulk.tensor), tcgen05 (UMMA issue, TMEM alloc/ld/st),
// UMMA shared-memory / instruction descriptors and the Philox4x32-10 mask generator.
//
// Everything is inline PTX written for `-gencode arch=compute_100a,code=sm_100a`.
// Descriptor encodings follow the PTX ISA "tcgen05 matrix descriptors" layout
// (start>>4 @0, LBO>>4 @16, SBO>>4 @32, version=1 @46, layout @61).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "lf_params.h"

namespace lf {

// ---------------------------------------------------------------------------------
// generic helpers
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 1024-byte aligned view of dynamic shared memory (SW128 atoms). Pointer arithmetic on the
// __shared__ array keeps the shared address space visible to the compiler (an integer
// round-trip would turn every access into a generic LD.E/ST.E).
__device__ __forceinline__ uint8_t* align_smem_1024(uint8_t* raw) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(raw));
  return raw + ((1024u - (a & 1023u)) & 1023u);
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint64_t lds64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t addr, uint64_t v) {
  asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t warp_id() { return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0); }
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Programmatic dependent launch (all lf kernels are launched with programmatic stream
// serialization, lf_kernels.h launch_k): a kernel may start while its predecessor in the
// stream drains, runs its prologue (mbarrier init, TMEM alloc, tensor-map prefetch), and
// must pass pdl_wait() — full completion and memory visibility of the predecessor — before
// its first global-memory access, read or write. No-ops without the launch attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// named barrier among a subset of warps (ids 1..15; 0 is __syncthreads)
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------------------------
// mbarrier
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok;
}
// try_wait with a suspend-time hint: a thread whose phase is still open sleeps in the
// barrier unit until the phase completes (or the hint, in ns, runs out) instead of
// re-issuing try_wait — spinning waiters otherwise steal issue slots from the ALU-bound
// mask warps sharing their scheduler.
#ifndef LF_SUSPEND_NS
#define LF_SUSPEND_NS 0x100000u
#endif
__device__ __forceinline__ uint32_t mbar_try_wait_sleep(uint32_t addr, uint32_t parity) {
  if (LF_SUSPEND_NS == 0u) return mbar_try_wait(addr, parity);
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"(LF_SUSPEND_NS)
      : "memory");
  return ok;
}
// Wait for the phase with the given parity to complete. A wait that has not
// completed after ~4e9 SM cycles traps instead of hanging the device: a protocol
// bug becomes a launch failure the host reports, never a wedged GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait_sleep(addr, parity)) {
    if (clock64() - t0 > 4000000000LL) __trap();
  }
}

// ---------------------------------------------------------------------------------
// TMA
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// generic-proxy smem writes (mask pass) -> visible to the async proxy (UMMA operand reads)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------------
// tcgen05 / TMEM
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] · B[smem], bf16 inputs, fp32 accumulate, cta_group::1
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on an mbarrier once every tcgen05 op previously issued by this thread completes
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// Whole-warp forms: called by all 32 lanes of a converged warp with warp-uniform operands;
// one elected lane (always the same, the lowest) issues. Keeping the issuing loop warp-wide
// lets ptxas hold descriptors in uniform registers instead of a per-MMA R2UR waterfall.
__device__ __forceinline__ void umma_bf16_warp(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------------------------
// thread-block clusters / CTA pairs (cta_group::2)
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// arrive (one count) + expect `bytes` of transactions on an mbarrier of CTA `rank`'s smem
__device__ __forceinline__ void mbar_arrive_expect_tx_cluster(uint32_t cluster_addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr),
               "r"(bytes)
               : "memory");
}

// ---------------------------------------------------------------------------------
// cluster launch control (dynamic persistent scheduling, sm_100)
// ---------------------------------------------------------------------------------
// Ask the hardware to cancel the launch of a not-yet-running cluster of this grid; the
// 16-byte response is multicast to the same smem offset in every CTA of the cluster and
// completes 16 transaction bytes on the mbarrier at the same offset in each of them.
__device__ __forceinline__ void clc_try_cancel_multicast(uint32_t resp_addr, uint32_t bar_addr) {
  asm volatile(
      "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.multicast::cluster::all.b128 "
      "[%0], [%1];" ::"r"(resp_addr),
      "r"(bar_addr)
      : "memory");
}
// Decode a response: the canceled cluster's first CTA x-coordinate, or -1 if none was left.
__device__ __forceinline__ int clc_first_ctaid_x(uint32_t resp_addr) {
  uint32_t x = 0, ok = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b128 r;\n\t"
      "ld.shared.b128 r, [%2];\n\t"
      "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\n\t"
      "selp.u32 %1, 1, 0, p;\n\t"
      "@p clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %0, r;\n\t}"
      : "=r"(x), "=r"(ok)
      : "r"(resp_addr)
      : "memory");
  return ok ? (int)x : -1;
}

// TMA load whose completion bytes are counted on the pair leader's mbarrier (same smem
// offset, peer bit cleared): each CTA of a pair fills its own half of a 2-CTA MMA operand
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                 int32_t c1) {
  const uint32_t leader_bar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
// The same pair load multicast to every CTA in `mask` (cluster ranks): the tile lands at the
// same smem offset in each destination, and each destination's bytes complete on its own
// pair leader's mbarrier (peer bit cleared) — one L2 read feeds several CTA pairs
__device__ __forceinline__ void tma_load_2d_pair_mc(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                                    int32_t c1, uint16_t mask) {
  const uint32_t leader_bar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%4, %5}], [%2], %3;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "h"(mask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// D[tmem, both CTAs] (+)= A[smem, both CTAs] · B[smem, both CTAs] — issued by the pair leader
__device__ __forceinline__ void umma_bf16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the mbarrier at this smem offset in both CTAs of the pair once the leader's MMAs finish
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
// whole-warp forms (see umma_bf16_warp)
__device__ __forceinline__ void umma_bf16_pair_warp(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                    uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

// arrive on the mbarrier at this smem offset in every CTA of `mask` once the leader's MMAs finish
__device__ __forceinline__ void umma_commit_pair_warp_mask(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// ---------------------------------------------------------------------------------
// UMMA descriptors
// ---------------------------------------------------------------------------------
enum : uint32_t { kLayoutNone = 0, kLayoutSW128 = 2, kLayoutSW64 = 4, kLayoutSW32 = 6 };

// Shared-memory matrix descriptor. For K-major swizzled operands LBO is unused
// (encoded 16 B); SBO = byte stride between 8-row groups. For MN-major swizzled
// operands LBO = byte stride between swizzle atoms along MN, SBO = byte stride
// between 8-row groups along K.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;  // descriptor version (sm_100)
  d |= (uint64_t)layout << 61;
  return d;
}

// descriptor of the same layout `bytes` further on (start-address field = addr >> 4 in bits
// 0..13; shared-window addresses stay below 256 KB, so the field never carries)
__device__ __forceinline__ uint64_t sdesc_add(uint64_t d, uint32_t bytes) { return d + (uint64_t)(bytes >> 4); }

// Instruction descriptor, kind::f16 with bf16 A/B and fp32 D.
__host__ __device__ constexpr uint32_t make_idesc_bf16(uint32_t M, uint32_t N, bool a_mn_major, bool b_mn_major) {
  return (1u << 4)                          // D format: f32
         | (1u << 7)                        // A format: bf16
         | (1u << 10)                       // B format: bf16
         | ((a_mn_major ? 1u : 0u) << 15)   // A major
         | ((b_mn_major ? 1u : 0u) << 16)   // B major
         | ((N >> 3) << 17)                 // N / 8
         | ((M >> 4) << 24);                // M / 16
}

// ---------------------------------------------------------------------------------
// numeric helpers
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void red_add_v4(float* gptr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(gptr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ void red_add_f32(float* gptr, float a) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(gptr), "f"(a) : "memory");
}
__device__ __forceinline__ float4 ld_cg_f4(const float* gptr) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(gptr)
               : "memory");
  return v;
}

// ---------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11; Random123) — SPEC.md §3
// ---------------------------------------------------------------------------------
struct U4 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
#if defined(__CUDA_ARCH__)
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
#else
    const uint64_t p0 = (uint64_t)M0 * c.x, p1 = (uint64_t)M1 * c.z;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += W0;
    k1 += W1;
  }
  return c;
}

// Philox counter words 2..3 of a segment: its host offset plus the device step counter
// (LfSegTable::off_dev, 0 when absent) — read once per thread after pdl_wait()
__device__ __forceinline__ uint64_t table_offset(const LfSegTable& t) { return t.off_dev ? *t.off_dev : 0ull; }
__device__ __forceinline__ void seg_offset_words(const LfSegDev& s, uint64_t extra, uint32_t& o0, uint32_t& o1) {
  const uint64_t o = ((((uint64_t)s.off1) << 32) | (uint64_t)s.off0) + extra;
  o0 = (uint32_t)o;
  o1 = (uint32_t)(o >> 32);
}

// keep bits (bit e = column col8*8+e kept) for 8 consecutive columns of one row
__device__ __forceinline__ uint32_t philox_keep8(uint32_t col8, uint32_t row, const LfSegDev& s,
                                                 uint64_t extra_offset = 0) {
  uint32_t o0, o1;
  seg_offset_words(s, extra_offset, o0, o1);
  const U4 r = philox4x32_10(U4{col8, row, o0, o1}, s.key0, s.key1);
  const uint32_t thr = s.thr;
  uint32_t bits = 0;
  bits |= ((r.x & 0xFFFFu) >= thr) ? 0x01u : 0u;
  bits |= ((r.x >> 16) >= thr) ? 0x02u : 0u;
  bits |= ((r.y & 0xFFFFu) >= thr) ? 0x04u : 0u;
  bits |= ((r.y >> 16) >= thr) ? 0x08u : 0u;
  bits |= ((r.z & 0xFFFFu) >= thr) ? 0x10u : 0u;
  bits |= ((r.z >> 16) >= thr) ? 0x20u : 0u;
  bits |= ((r.w & 0xFFFFu) >= thr) ? 0x40u : 0u;
  bits |= ((r.w >> 16) >= thr) ? 0x80u : 0u;
  return bits;
}

// Per-(segment, row) Philox state hoisted out of the column loop: the round keys, the
// constant counter words (row, offset) and the packed 16-bit threshold. One call then
// costs 10 x (2 IMAD.WIDE + 2 LOP3) plus a SIMD compare of the eight 16-bit lanes.
#ifndef LF_PHILOX_KEYS_INLINE
#define LF_PHILOX_KEYS_INLINE 0  // 1: philox_masks adds the Weyl constants per round instead of reading k0[]/k1[]
#endif
struct PhiloxRow {
  uint32_t k0[10], k1[10];
  uint32_t c1, c2, c3;
  uint32_t thr2;   // thr in both 16-bit halves
  uint32_t hthr2;  // thr / 2 in both 16-bit halves (SWAR keep test)
};

__device__ __forceinline__ PhiloxRow philox_row(const LfSegDev& s, uint32_t row, uint64_t extra_offset = 0) {
  PhiloxRow pr;
  uint32_t a = s.key0, b = s.key1;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    pr.k0[i] = a;
    pr.k1[i] = b;
    a += 0x9E3779B9u;
    b += 0xBB67AE85u;
  }
  pr.c1 = row;
  seg_offset_words(s, extra_offset, pr.c2, pr.c3);
  pr.thr2 = s.thr | (s.thr << 16);
  // opaque to the compiler: otherwise it folds the keep test's subtraction of hthr2 into an
  // IMAD on the FMA-heavy pipe (next to the Philox IMAD.WIDEs) instead of an ALU IADD
  uint32_t h = (s.thr >> 1) * 0x00010001u;
  asm volatile("prmt.b32 %0, %0, 0, 0x3210;" : "+r"(h));
  pr.hthr2 = h;
  return pr;
}

// 0x00/0x01 per byte (4 lanes) -> 4 bits
__device__ __forceinline__ uint32_t gather_lsb4(uint32_t x) { return ((x & 0x01010101u) * 0x01020408u) >> 24; }

__device__ __forceinline__ uint32_t philox_row_keep8(const PhiloxRow& pr, uint32_t col8) {
  uint32_t c0 = col8, c1 = pr.c1, c2 = pr.c2, c3 = pr.c3;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ pr.k0[i];
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ pr.k1[i];
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
  }
  // per 16-bit lane: 0xFFFF where lane >= thr; gather one byte per lane, then one bit per byte
  const uint32_t r0 = __vcmpgeu2(c0, pr.thr2), r1 = __vcmpgeu2(c1, pr.thr2);
  const uint32_t r2 = __vcmpgeu2(c2, pr.thr2), r3 = __vcmpgeu2(c3, pr.thr2);
  const uint32_t lo = __byte_perm(r0, r1, 0x6420);  // lanes 0..3
  const uint32_t hi = __byte_perm(r2, r3, 0x6420);  // lanes 4..7
  return gather_lsb4(lo) | (gather_lsb4(hi) << 4);
}

// keep bits for 8 consecutive columns from an explicit uint8 mask row (col multiple of 8)
__device__ __forceinline__ uint32_t explicit_keep8(const uint8_t* mask_row, uint32_t col, uint32_t ncols) {
  uint32_t bits = 0;
  if (col + 8 <= ncols && ((reinterpret_cast<uintptr_t>(mask_row + col) & 7u) == 0)) {
    const uint2 v = *reinterpret_cast<const uint2*>(mask_row + col);
#pragma unroll
    for (int e = 0; e < 4; ++e) bits |= (((v.x >> (8 * e)) & 0xFFu) ? 1u : 0u) << e;
#pragma unroll
    for (int e = 0; e < 4; ++e) bits |= (((v.y >> (8 * e)) & 0xFFu) ? 1u : 0u) << (4 + e);
  } else {
    for (int e = 0; e < 8; ++e)
      if (col + e < ncols && mask_row[col + e]) bits |= 1u << e;
  }
  return bits;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// zero the bf16 lanes of a 16-byte chunk whose keep bit is clear. The 8 bits are spread to
// the sign bits of 8 bytes (byte j of p/q: 0x80-ish iff bit j / j+4 is set), then prmt's
// sign-replicate selectors (nibble bit 3) expand them to 0xFFFF / 0x0000 bf16 lanes.
__device__ __forceinline__ uint4 apply_keep8(uint4 v, uint32_t bits) {
  const uint32_t t = bits * 0x01010101u;
  const uint32_t p = (t & 0x08040201u) + 0x7F7F7F7Fu;
  const uint32_t q = (t & 0x80402010u) + 0x7F7F7F7Fu;
  return make_uint4(v.x & prmt(p, 0, 0x9988u), v.y & prmt(p, 0, 0xBBAAu), v.z & prmt(q, 0, 0x9988u),
                    v.w & prmt(q, 0, 0xBBAAu));
}

// keep bits of CH*8 consecutive columns [col, col + 8*CH) of one row: byte c = chunk c.
// The CH Philox streams (counters col/8 .. col/8+CH-1) advance round by round in lockstep,
// so every round exposes CH independent IMAD.WIDE/LOP3 chains to the scheduler.
template <int CH>
__device__ __forceinline__ uint64_t keep_bits_philox(const PhiloxRow& pr, int col) {
  uint32_t c0[CH], c1[CH], c2[CH], c3[CH];
  const uint32_t base = (uint32_t)col >> 3;
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    c0[j] = base + j;
    c1[j] = pr.c1;
    c2[j] = pr.c2;
    c3[j] = pr.c3;
  }
#pragma unroll
  for (int i = 0; i < 10; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const uint64_t p0 = (uint64_t)0xD2511F53u * c0[j];
      const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2[j];
      const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1[j] ^ pr.k0[i];
      const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3[j] ^ pr.k1[i];
      c1[j] = (uint32_t)p1;
      c3[j] = (uint32_t)p0;
      c0[j] = n0;
      c2[j] = n2;
    }
  }
  uint64_t bits = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const uint32_t r0 = __vcmpgeu2(c0[j], pr.thr2), r1 = __vcmpgeu2(c1[j], pr.thr2);
    const uint32_t r2 = __vcmpgeu2(c2[j], pr.thr2), r3 = __vcmpgeu2(c3[j], pr.thr2);
    const uint32_t b = gather_lsb4(__byte_perm(r0, r1, 0x6420)) | (gather_lsb4(__byte_perm(r2, r3, 0x6420)) << 4);
    bits |= (uint64_t)b << (8 * j);
  }
  return bits;
}
__device__ __forceinline__ uint64_t keep_bits64_philox(const PhiloxRow& pr, int col) {
  return keep_bits_philox<8>(pr, col);
}

// SPEC.md §3 keep test of both 16-bit lanes of a Philox word at once (even threshold, so
// u16 >= thr <=> (u16 >> 1) >= thr/2): the 15-bit halves biased by 0x8000 never borrow
// across lanes, and lane j's verdict lands in bit 16j + 15.
__device__ __forceinline__ uint32_t keep_sign2(uint32_t w, uint32_t hthr2) {
  return (((w >> 1) & 0x7FFF7FFFu) | 0x80008000u) - hthr2;
}
// byte MSBs -> 4 bits (byte j -> bit j)
__device__ __forceinline__ uint32_t gather_msb4(uint32_t x) { return (((x >> 7) & 0x01010101u) * 0x01020408u) >> 24; }

// ① hot path: the CH Philox streams of keep_bits_philox, but the verdicts become bf16 lane
// masks (0xFFFF per kept element, word i of chunk j in msk[j][i]) applied with a plain AND,
// plus the packed keep bits (byte j = chunk j) that ④ and ⑤ read.
template <int CH>
__device__ __forceinline__ uint64_t philox_masks(const PhiloxRow& pr, int col, uint32_t (&msk)[CH][4]) {
  uint32_t c0[CH], c1[CH], c2[CH], c3[CH];
  const uint32_t base = (uint32_t)col >> 3;
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    c0[j] = base + j;
    c1[j] = pr.c1;
    c2[j] = pr.c2;
    c3[j] = pr.c3;
  }
#if LF_PHILOX_KEYS_INLINE
  uint32_t ka = pr.k0[0], kb = pr.k1[0];
#endif
#pragma unroll
  for (int i = 0; i < 10; ++i) {
#if LF_PHILOX_KEYS_INLINE
    const uint32_t ki0 = ka, ki1 = kb;
    ka += 0x9E3779B9u;
    kb += 0xBB67AE85u;
#else
    const uint32_t ki0 = pr.k0[i], ki1 = pr.k1[i];
#endif
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const uint64_t p0 = (uint64_t)0xD2511F53u * c0[j];
      const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2[j];
      const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1[j] ^ ki0;
      const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3[j] ^ ki1;
      c1[j] = (uint32_t)p1;
      c3[j] = (uint32_t)p0;
      c0[j] = n0;
      c2[j] = n2;
    }
  }
  // packed keep bits: chunk j's verdicts (byte MSBs of y = columns 0..3, z = 4..7) are
  // folded to bit positions 3 + 8i (y) and 7 + 8i (z) of one word, and one multiply by
  // 2^21 + 2^14 + 2^7 + 1 gathers them into its top byte (all partial products land on
  // distinct bits: no carries); the top bytes of the CH products are then byte-permuted
  // into place — 6 instructions per chunk instead of two multiply-gathers and the shifts
  uint32_t p[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const uint32_t d0 = keep_sign2(c0[j], pr.hthr2), d1 = keep_sign2(c1[j], pr.hthr2);
    const uint32_t d2 = keep_sign2(c2[j], pr.hthr2), d3 = keep_sign2(c3[j], pr.hthr2);
    msk[j][0] = prmt(d0, 0, 0xBB99u);
    msk[j][1] = prmt(d1, 0, 0xBB99u);
    msk[j][2] = prmt(d2, 0, 0xBB99u);
    msk[j][3] = prmt(d3, 0, 0xBB99u);
    const uint32_t y = prmt(d0, d1, 0x7531u), z = prmt(d2, d3, 0x7531u);
    p[j] = ((z & 0x80808080u) | ((y & 0x80808080u) >> 4)) * 0x00204081u;
  }
  uint64_t bits = 0;
#pragma unroll
  for (int j = 0; j < CH; j += 4) {
    const uint32_t lo = prmt(p[j], j + 1 < CH ? p[j + 1] : 0u, 0x0073u);
    const uint32_t hi = j + 2 < CH ? prmt(p[j + 2], j + 3 < CH ? p[j + 3] : 0u, 0x0073u) : 0u;
    bits |= (uint64_t)prmt(lo, hi, 0x5410u) << (8 * j);
  }
  return bits;
}

// AND lane masks into chunks [c0, c0 + CH) of one 128-byte SW128 tile row
template <int CH>
__device__ __forceinline__ void apply_masks_sw128(uint8_t* tile, int rit, int c0, const uint32_t (&msk)[CH][4]) {
  const uint32_t rowa = smem_u32(tile) + (uint32_t)rit * 128u;
  uint4 v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = lds128(rowa + (uint32_t)(((c0 + c) ^ (rit & 7)) << 4));
#pragma unroll
  for (int c = 0; c < CH; ++c)
    sts128(rowa + (uint32_t)(((c0 + c) ^ (rit & 7)) << 4),
           make_uint4(v[c].x & msk[c][0], v[c].y & msk[c][1], v[c].z & msk[c][2], v[c].w & msk[c][3]));
}

// zero the dropped bf16 elements of chunks [c0, c0 + CH) of one 128-byte SW128 tile row
template <int CH>
__device__ __forceinline__ void apply_chunks_sw128(uint8_t* tile, int rit, int c0, uint32_t bits) {
  const uint32_t rowa = smem_u32(tile) + (uint32_t)rit * 128u;
  uint4 v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = lds128(rowa + (uint32_t)(((c0 + c) ^ (rit & 7)) << 4));
#pragma unroll
  for (int c = 0; c < CH; ++c) sts128(rowa + (uint32_t)(((c0 + c) ^ (rit & 7)) << 4), apply_keep8(v[c], (bits >> (8 * c)) & 0xFFu));
}
__device__ __forceinline__ uint64_t keep_bits64_explicit(const LfSegTable& t, int row, int col, int ncols) {
  uint64_t bits = 0;
  const uint8_t* mrow = t.mask + (int64_t)row * t.ld_mask;
#pragma unroll
  for (int c = 0; c < 8; ++c) bits |= (uint64_t)explicit_keep8(mrow, col + 8 * c, ncols) << (8 * c);
  return bits;
}

// 8 bytes of a bit-packed mask row starting at byte b0 (bounded by the row length)
__device__ __forceinline__ uint64_t load_bits64(const uint8_t* row_bits, int b0, int row_bytes) {
  const uint8_t* p = row_bits + b0;
  if (b0 + 8 <= row_bytes && ((reinterpret_cast<uintptr_t>(p) & 7u) == 0))
    return *reinterpret_cast<const uint64_t*>(p);
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i)
    if (b0 + i < row_bytes) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

__device__ __forceinline__ void store_bits64(uint8_t* row_bits, int b0, int row_bytes, uint64_t v) {
  uint8_t* p = row_bits + b0;
  if (b0 + 8 <= row_bytes && ((reinterpret_cast<uintptr_t>(p) & 7u) == 0)) {
    *reinterpret_cast<uint64_t*>(p) = v;
    return;
  }
  for (int i = 0; i < 8; ++i)
    if (b0 + i < row_bytes) p[i] = (uint8_t)(v >> (8 * i));
}

// zero the dropped bf16 elements of one 128-byte row of an SW128 tile (64 columns):
// all eight 16-byte chunks are loaded first (ld.shared), masked, then stored back
__device__ __forceinline__ void apply_row_sw128(uint8_t* tile, int rit, uint64_t bits) {
  if (bits == ~0ull) return;
  const uint32_t rowa = smem_u32(tile) + (uint32_t)rit * 128u;
  uint4 v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = lds128(rowa + (uint32_t)((c ^ (rit & 7)) << 4));
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint32_t b = (uint32_t)(bits >> (8 * c)) & 0xFFu;
    sts128(rowa + (uint32_t)((c ^ (rit & 7)) << 4), apply_keep8(v[c], b));
  }
}

// index of the segment holding `row` among [lo, hi] (sorted, disjoint), or -1
__device__ __forceinline__ int find_segment(const LfSegTable& t, int lo, int hi, int row) {
  for (int i = lo; i <= hi; ++i) {
    if (row >= t.seg[i].row0 && row < t.seg[i].row1) return i;
  }
  return -1;
}

// finalize one row of a split-K reduced m x R result: scale own-segment columns, zero the
// rest, write bf16, and return the partial-sum workspace to zero. The loads of up to four
// 8-column chunks are issued before any store (the stores alias the loaded workspace, so a
// load-store-load loop would pay one L2 round trip per chunk: 16 at R = 128).
__device__ __forceinline__ void finalize_row(const LfSegTable& t, const LfRoute& rt, int row, float* ws,
                                             __nv_bfloat16* out) {
  const int rtot = t.rtot;
  const int seg = find_segment(t, rt.seg_lo, rt.seg_hi, row);
  const int own0 = seg >= 0 ? t.seg[seg].col0 : 0;
  const int own1 = seg >= 0 ? t.seg[seg].col0 + t.seg[seg].ncol : 0;
  const float scale = seg >= 0 ? t.seg[seg].scale : 0.f;
  float* wrow = ws + (int64_t)row * rtot;
  __nv_bfloat16* orow = out + (int64_t)row * rtot;
  for (int g = 0; g < rtot; g += 32) {
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = g + 8 * i;
      const bool in_range = c < rtot && c >= rt.col_lo && c < rt.col_hi;
      v[2 * i] = in_range ? ld_cg_f4(wrow + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      v[2 * i + 1] = in_range ? ld_cg_f4(wrow + c + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = g + 8 * i;
      if (c >= rtot) break;
      if (c >= rt.col_lo && c < rt.col_hi) {
        *reinterpret_cast<float4*>(wrow + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4*>(wrow + c + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      const float sc = (c >= own0 && c < own1) ? scale : 0.f;
      const float4 a = v[2 * i], b = v[2 * i + 1];
      *reinterpret_cast<uint4*>(orow + c) = make_uint4(pack_bf16x2(a.x * sc, a.y * sc), pack_bf16x2(a.z * sc, a.w * sc),
                                                       pack_bf16x2(b.x * sc, b.y * sc), pack_bf16x2(b.z * sc, b.w * sc));
    }
  }
}

// one 8-column chunk of finalize_row (the separate finalize launch: one thread per chunk)
__device__ __forceinline__ void finalize_chunk(const LfSegTable& t, const LfRoute& rt, int row, int c, float* ws,
                                               __nv_bfloat16* out) {
  const int seg = find_segment(t, rt.seg_lo, rt.seg_hi, row);
  const bool own = seg >= 0 && c >= t.seg[seg].col0 && c < t.seg[seg].col0 + t.seg[seg].ncol;
  const float sc = own ? t.seg[seg].scale : 0.f;
  float* w = ws + (int64_t)row * t.rtot + c;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
  if (c >= rt.col_lo && c < rt.col_hi) {
    a = ld_cg_f4(w);
    b = ld_cg_f4(w + 4);
    *reinterpret_cast<float4*>(w) = make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(w + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  *reinterpret_cast<uint4*>(out + (int64_t)row * t.rtot + c) =
      make_uint4(pack_bf16x2(a.x * sc, a.y * sc), pack_bf16x2(a.z * sc, a.w * sc), pack_bf16x2(b.x * sc, b.y * sc),
                 pack_bf16x2(b.z * sc, b.w * sc));
}

// zero one row of an m x R bf16 result (row tiles no adapter touches)
__device__ __forceinline__ void zero_row(int rtot, int row, __nv_bfloat16* out) {
  __nv_bfloat16* orow = out + (int64_t)row * rtot;
  for (int c = 0; c < rtot; c += 8) *reinterpret_cast<uint4*>(orow + c) = make_uint4(0u, 0u, 0u, 0u);
}

// Split-K completion of one 128-row tile, run by 128 epilogue threads (one row each, named
// barrier `bar_id`) after their red.adds of this tile's partial: the partial counts `units`
// towards `total`, and the CTA that completes the tile finalizes it (finalize_row) and
// re-arms the counter — no separate finalize launch. Ordering: the first barrier puts every
// thread's red.adds before thread 0's acq_rel atomic (release is cumulative over what the
// barrier ordered before it); the second puts the atomic's acquire before all the reads.
__device__ __forceinline__ int atom_add_acq_rel_gpu(int32_t* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void tile_contribute(const LfSegTable& segs, const LfRoute& rt, int tile, int rit,
                                                int units, int total, int32_t* counters, float* ws,
                                                __nv_bfloat16* out, uint32_t bar_id, int* s_last) {
  named_bar_sync(bar_id, 128);
  if (rit == 0) *s_last = atom_add_acq_rel_gpu(&counters[tile], units) + units == total;
  named_bar_sync(bar_id, 128);
  const bool last = *s_last != 0;
  named_bar_sync(bar_id, 128);  // s_last is reused by the next call
  if (!last) return;
  const int row = tile * 128 + rit;
  if (row < segs.m && !(segs.debug & 16)) finalize_row(segs, rt, row, ws, out);
  if (rit == 0) counters[tile] = 0;
}

}  // namespace lf
