// Thin inline-PTX helpers for sm_100a: mbarrier, bulk/TMA copies, tcgen05 (TMEM + UMMA).
//
// Everything here is a one-instruction wrapper; the kernels in this directory compose them.
// Compile only with -gencode arch=compute_100a,code=sm_100a.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

#define W4_DEV __device__ __forceinline__

namespace w4 {

W4_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

W4_DEV uint32_t lane_id() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

// warp-uniform warp index
W4_DEV uint32_t warp_idx() { return __shfl_sync(0xffffffffu, threadIdx.x / 32, 0); }

W4_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- mbarrier
W4_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

W4_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

W4_DEV void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

W4_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

W4_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// How waits poll an mbarrier phase (-DW4A16_WAIT=...): 0 = try_wait (the thread may be suspended
// until the phase completes or a system time limit), 1 = test_wait spin (never suspends),
// 2 = try_wait with a short suspend-time hint.
#ifndef W4A16_WAIT
#define W4A16_WAIT 0
#endif
#if W4A16_WAIT == 1
#define W4_WAIT_OP "mbarrier.test_wait.parity"
#define W4_WAIT_HINT ""
#elif W4A16_WAIT == 2
#define W4_WAIT_OP "mbarrier.try_wait.parity"
#define W4_WAIT_HINT ", 0x20"
#else
#define W4_WAIT_OP "mbarrier.try_wait.parity"
#define W4_WAIT_HINT ""
#endif

W4_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "W4_WAIT_%=:\n\t"
      W4_WAIT_OP ".shared::cta.b64 P, [%0], %1" W4_WAIT_HINT ";\n\t"
      "@!P bra W4_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- clusters (CTA pairs)
W4_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
W4_DEV uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
W4_DEV uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// shared::cluster address of `bar` in CTA `rank` of this cluster
W4_DEV uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
W4_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Acquire scope of the waits below: .cluster when CTA peers arrive on the barrier (cta_group::2 pairs);
// .cta otherwise -- an acquire at cluster scope invalidates L1 (CCTL.IVALL), which ncu showed as the
// most stall-sampled instruction of the decode GEMMs.
#define W4_WAIT_BODY1(LABEL, SCOPE)                                                        \
  "{\n\t.reg .pred P;\n\t" LABEL ":\n\t" W4_WAIT_OP ".acquire." SCOPE ".shared::cta.b64 P, [%0], %1" \
  W4_WAIT_HINT ";\n\t@!P bra " LABEL ";\n\t}"
template <bool kCluster = true>
W4_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  if constexpr (kCluster)
    asm volatile(W4_WAIT_BODY1("W4_WAITC_%=", "cluster") ::"r"(smem_u32(bar)), "r"(parity) : "memory");
  else
    asm volatile(W4_WAIT_BODY1("W4_WAITA_%=", "cta") ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// Wait for two barrier phases at once: both try_waits are in flight together, so a ready barrier
// costs its latency once instead of once per barrier (a completed phase stays completed until the
// waiter consumes it, so re-testing is safe).
W4_DEV void mbar_wait2_cluster(uint64_t* b0, uint32_t ph0, uint64_t* b1, uint32_t ph1) {
  asm volatile(
      "{\n\t.reg .pred P0, P1;\n\t"
      "W4_WAIT2_%=:\n\t"
      W4_WAIT_OP ".acquire.cluster.shared::cta.b64 P0, [%0], %1" W4_WAIT_HINT ";\n\t"
      W4_WAIT_OP ".acquire.cluster.shared::cta.b64 P1, [%2], %3" W4_WAIT_HINT ";\n\t"
      "@!P0 bra W4_WAIT2_%=;\n\t"
      "@!P1 bra W4_WAIT2_%=;\n\t}" ::"r"(smem_u32(b0)),
      "r"(ph0), "r"(smem_u32(b1)), "r"(ph1)
      : "memory");
}

// Warp-wide forms: the whole (converged) warp waits and branches on a vote, so ptxas sees uniform
// control flow afterwards and keeps warp-uniform values in uniform registers (MMA operands).
#define W4_WAIT_BODYW(LABEL, SCOPE)                                                               \
  "{\n\t.reg .pred P, Q;\n\t" LABEL ":\n\t" W4_WAIT_OP ".acquire." SCOPE ".shared::cta.b64 P, [%0], %1"   \
  W4_WAIT_HINT ";\n\tvote.sync.all.pred Q, P, 0xffffffff;\n\t@!Q bra.uni " LABEL ";\n\t}"
#define W4_WAIT_BODY2W(LABEL, SCOPE)                                                                      \
  "{\n\t.reg .pred P0, P1, P, Q;\n\t" LABEL ":\n\t" W4_WAIT_OP ".acquire." SCOPE                     \
  ".shared::cta.b64 P0, [%0], %1" W4_WAIT_HINT ";\n\t" W4_WAIT_OP ".acquire." SCOPE                      \
  ".shared::cta.b64 P1, [%2], %3" W4_WAIT_HINT ";\n\tand.pred P, P0, P1;\n\t"                          \
  "vote.sync.all.pred Q, P, 0xffffffff;\n\t@!Q bra.uni " LABEL ";\n\t}"
template <bool kCluster = true>
W4_DEV void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  if constexpr (kCluster)
    asm volatile(W4_WAIT_BODYW("W4_WAITW_%=", "cluster") ::"r"(smem_u32(bar)), "r"(parity) : "memory");
  else
    asm volatile(W4_WAIT_BODYW("W4_WAITWA_%=", "cta") ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
template <bool kCluster = true>
W4_DEV void mbar_wait2_warp(uint64_t* b0, uint32_t ph0, uint64_t* b1, uint32_t ph1) {
  if constexpr (kCluster)
    asm volatile(W4_WAIT_BODY2W("W4_WAIT2W_%=", "cluster") ::"r"(smem_u32(b0)), "r"(ph0), "r"(smem_u32(b1)),
                 "r"(ph1) : "memory");
  else
    asm volatile(W4_WAIT_BODY2W("W4_WAIT2WA_%=", "cta") ::"r"(smem_u32(b0)), "r"(ph0), "r"(smem_u32(b1)),
                 "r"(ph1) : "memory");
}

W4_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- bulk copies (async proxy)
// 1-D bulk copy global -> shared, completion counted on an mbarrier (bytes % 16 == 0).
W4_DEV void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Same, with an L2 eviction-priority hint (weights are streamed exactly once per tile).
W4_DEV void bulk_g2s_hint(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

W4_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

W4_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 8-byte cp.async global -> shared (LDGSTS), and an mbarrier arrival once all of this thread's prior
// cp.async complete (.noinc: the barrier's expected count includes this arrival).
W4_DEV void cp_async_8(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
}
W4_DEV void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 2-D TMA tile load (tensor map in param/const/global space), coordinates innermost first.
W4_DEV void tma_load_2d(void* dst_smem, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst_smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

W4_DEV void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---------------------------------------------------------------- tcgen05: TMEM
template <uint32_t kCols>
W4_DEV void tmem_alloc(uint32_t* dst_smem) {
  static_assert(kCols >= 32 && kCols <= 512 && (kCols & (kCols - 1)) == 0, "TMEM alloc: pow2 in [32,512]");
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

template <uint32_t kCols>
W4_DEV void tmem_alloc_pair(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <uint32_t kCols>
W4_DEV void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}

template <uint32_t kCols>
W4_DEV void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}

W4_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
W4_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
W4_DEV void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
W4_DEV void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// tcgen05.st 32 lanes x 32 bit, 16 consecutive columns per thread (thread i -> lane base+i)
W4_DEV void tmem_st_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// tcgen05.ld 32 lanes x 32 bit, 16 consecutive columns
W4_DEV void tmem_ld_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

// Orders later uses of tcgen05.ld destination registers after the tcgen05.wait::ld that precedes this
// call: the (volatile) empty asm "rewrites" them, so the compiler cannot hoist their consumers above it.
W4_DEV void reg_fence16(uint32_t (&r)[16]) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]));
}

// tcgen05.ld 32 lanes x 32 bit, 4 consecutive columns
W4_DEV void tmem_ld_x4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr)
               : "memory");
}

// ---------------------------------------------------------------- tcgen05: UMMA
// D[tmem] (+)= A[tmem] * B[smem desc]; kind::f16 (fp16 or bf16 inputs, fp32 accumulate).
W4_DEV void umma_ts_f16(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D[tmem] (+)= A[smem desc] * B[smem desc]; kind::f16.
W4_DEV void umma_ss_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Warp-collective forms: the whole (converged) warp executes them with warp-uniform operands and one
// elected lane issues -- the operands stay in uniform registers, so back-to-back MMAs issue without
// the per-instruction waterfall the compiler emits for a lane-0-only region.
W4_DEV void umma_ts_f16_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// single-thread commit for a CTA pair (caller elected)
W4_DEV void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

// commit for a CTA pair: arrive on the barrier at the same smem offset in both CTAs (mask 0b11)
W4_DEV void umma_commit_pair_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::
          "r"(smem_u32(bar)), "h"(static_cast<uint16_t>(3))
      : "memory");
}

W4_DEV void umma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05 async ops of this thread complete.
W4_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Instruction descriptor, kind::f16: fp32 accumulate, K-major A and B, M=128.
//   bits [4,6) c_format (1 = f32), [7,10) a_format, [10,13) b_format (0 f16, 1 bf16),
//   [15] a_major, [16] b_major (0 = K), [17,23) N>>3, [24,29) M>>4.
__host__ __device__ constexpr uint32_t make_idesc_f16(uint32_t m, uint32_t n, bool bf16) {
  return (1u << 4) | ((bf16 ? 1u : 0u) << 7) | ((bf16 ? 1u : 0u) << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

// Shared-memory matrix descriptor for a K-major operand stored in 128-byte swizzled atoms
// (8 rows x 128 B, rows contiguous, atoms stacked every 1024 B along M/N).
// sbo = byte stride between consecutive 8-row groups; sbo = 0 makes every 8-row group read the same
// atom (a row-periodic operand stored once).
W4_DEV uint64_t make_sdesc_sw128(uint32_t smem_addr, uint32_t sbo = 1024u) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);       // start address  [0,14)
  d |= static_cast<uint64_t>(1u) << 16;                           // LBO (unused for SW128 K-major)
  d |= static_cast<uint64_t>(sbo >> 4) << 32;                     // SBO            [32,46)
  d |= static_cast<uint64_t>(1u) << 46;                           // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2u) << 61;                           // SWIZZLE_128B
  return d;
}

// ---------------------------------------------------------------- misc
W4_DEV uint32_t lop3_and_or(uint32_t a, uint32_t mask, uint32_t orv) {
  uint32_t r;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(mask), "r"(orv));  // (a & b) | c
  return r;
}

W4_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
W4_DEV void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace w4
