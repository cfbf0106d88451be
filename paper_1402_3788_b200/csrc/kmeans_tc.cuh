// kmeans_tc.cuh — tcgen05 (5th-gen tensor core) fused Lloyd pass for sm_100a.
//
// ASSIGN on the tensor cores (kind::f16, fp32 accumulation in TMEM).  Per
// 128-point tile, with every operand prescaled by 2^s (|x·2^s| < 1, exact):
//   A row p   = [ xh_p | xl_p ]   xh = fp16(x'), xl = fp16(x' − xh); feature m = 1
//   B row c   = [ wh_c | wh_c ],  B row KP+c = [ wl_c | 0 ]
//               w_c = 2^s·(−2·fl32(c)), feature m = 2^2s·‖fl32(c)‖²
//   D = A·Bᵀ  →  D[p][c] + D[p][KP+c] = x·wh + xh·wl ≈ ‖c‖² − 2x·c  (dropped xl·wl ≈ 2⁻²² rel.)
// The packed [hi|lo] row (64 halfs = one 128-byte SW128 row) keeps the
// operand at 128 B/point, written once and read once by the MMA.  The
// epilogue (thread = point = TMEM lane) certifies the argmin with the bound
// E = coef·(‖x'‖+max‖c'‖)² and re-decides uncertified points with the
// reference's exact fp64 recurrence (see kmeans_kernels.cuh).
//
// UPDATE by exact integer deltas: cluster sums are int64 fixed point, so
//   S(L_t) = S(L_{t-1}) + Σ_{i: L_t(i) ≠ L_{t-1}(i)} (x_i → L_t(i)) − (x_i → L_{t-1}(i))
// is bit-identical to recomputing them.  Changed points add/subtract their
// fixed-point coordinates into per-CTA shared-memory accumulators (one flush
// per CTA); the finish kernel folds Δ into the running totals.  The first
// pass (no previous labels) adds every point.
//
// Points whose label the filter cannot certify are re-decided in the epilogue
// with the reference's exact fp64 recurrence over the candidate centres (those
// whose filter score lies within 2E of the best; every other centre is strictly
// farther), which the HBM-bound pipeline absorbs.
//
// Warp roles (persistent CTA, one per SM), pipelined over 128-point tiles:
//   warps 0-7  : transform   two groups, alternate tiles: raw tile → fp16 [hi|lo] A operand
//   warps 8-19 : epilogue    three groups, round-robin tiles (two when the TMEM score ring is
//                            shallower than 6 buffers, KP > 32): TMEM scores → top-2 →
//                            certify → Δ update (thread = point = TMEM lane)
//   warp 20    : TMA producer (cp.async.bulk 1-D copies of raw 4·m-byte rows)
//   warps 21-22: TMEM allocator + MMA issuers (alternate tiles); warp 23: recheck
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>

#include "kmeans_tc.h"

namespace km {
namespace tc {

constexpr int kQueueCap = 768;                     // per-CTA staging of uncertified points (smem)
// queue capacity (candidate masks grow with KP: KP/32 words per queued point)
template <int KP>
__host__ __device__ constexpr int tc_qcap() { return KP <= 128 ? kQueueCap : 128; }
// 64-bit add into the shared-memory Δ accumulator (two 32-bit atomics with carry)
__device__ __forceinline__ void acc_add64(unsigned long long* p, unsigned long long v) { smem_add64(p, v); }
constexpr long long kQueueFlag = 1ll << 62;
// a queue entry of a point whose label CHANGED (not a recheck): flag | change | row << 16 |
// (old + 1) << 8 | new.  The recheck warp applies its exact Δ off the epilogue's critical path.
constexpr long long kChangeFlag = 1ll << 61;
#ifndef KM_HEAVY_PASSES
#define KM_HEAVY_PASSES 1
#endif
#ifndef KM_HEAVY_DIV
#define KM_HEAVY_DIV 256  // a pass is heavy when its predecessor changed more than 1/KM_HEAVY_DIV of the CTA's points
#endif
#ifndef KM_QUEUE_CHANGES
#define KM_QUEUE_CHANGES 0
#endif
constexpr int kTileRows = 128;
#ifndef KM_TRANSFORM_GROUPS
#define KM_TRANSFORM_GROUPS 2
#endif
constexpr int kTransformGroups = KM_TRANSFORM_GROUPS;  // transform warpgroups (tile g → group g mod groups)
constexpr int kTransformWarps = 4 * kTransformGroups;
#ifndef KM_EPI_GROUPS
#define KM_EPI_GROUPS 3
#endif
constexpr int kEpiGroups = KM_EPI_GROUPS;          // epilogue warpgroups (tile g → group g mod kEpiGroups)
constexpr int kEpiWarps = 4 * kEpiGroups;
constexpr int kProducerWarp = kTransformWarps + kEpiWarps;  // TMA producer
constexpr int kMmaWarp = kProducerWarp + 1;                 // TMEM allocator + MMA issuer (even tiles)
constexpr int kMmaWarps = 2;                                // issuers: tile g → warp kMmaWarp + g % 2
constexpr int kRecheckWarp = kMmaWarp + kMmaWarps;          // exact re-decision of queued points, during the pass
constexpr int kThreadsTC = (kRecheckWarp + 1) * 32;
// tail of a run-ahead pass boundary: every warp but the transform groups and the producer
constexpr int kTailThreads = kThreadsTC - (kTransformWarps + 1) * 32;
constexpr int kTailBar = 14;  // named barrier of those warps
#ifndef KM_RUN_AHEAD
#define KM_RUN_AHEAD 1
#endif
// Ring depths and tile height.  The pass is HBM bound: the raw ring (TMA → transform) gets the
// shared memory the other sections leave (~64 KB in flight per SM covers the loaded DRAM
// latency).  Tiles of 256 points (two M=128 MMA blocks) halve every per-tile handshake per
// point where they fit; the A ring (transform → MMA) then holds one tile per transform group.
#ifndef KM_A_IN_TMEM
#define KM_A_IN_TMEM 1
#endif
// A operand in TMEM (transform → tcgen05.st, MMA reads it from TMEM) when its columns fit next
// to the score ring; otherwise the A tile is staged in shared memory (SW128)
template <int KP, int TR>
__host__ __device__ constexpr bool tc_a_in_tmem() { return KM_A_IN_TMEM && KP <= 32 && TR == 128; }

// Per-epilogue-warp private Δ accumulators (plain shared-memory adds, no atomics: the shared atomic
// unit takes ~5 lane-ops per clock per SM, which bounded the change-heavy passes) where the 12
// copies fit in 56 KB; the recheck warp and the tail keep the CTA-shared atomic accumulator.
#ifndef KM_PRIV_DELTA
#define KM_PRIV_DELTA 1
#endif
template <int MP, int KP>
__host__ __device__ constexpr int tc_pdelta_stride() { return KP * (MP + 1) + KP; }  // int64 entries per copy
template <int MP, int KP>
__host__ __device__ constexpr bool tc_pdelta() {
  return KM_PRIV_DELTA && kEpiWarps * tc_pdelta_stride<MP, KP>() * 8 <= 56 * 1024;
}
template <int MP, int KP>
__host__ __device__ constexpr int tc_pdelta_bytes() {
  return tc_pdelta<MP, KP>() ? (kEpiWarps * tc_pdelta_stride<MP, KP>() * 8 + 1023) / 1024 * 1024 : 0;
}

template <int MP, int KP, int TR>
struct TcBudget {
// A buffers per transform group with A in TMEM: 6 at KP = 16 (12 × 32 + 8 score buffers × 16 = 512
// TMEM columns; deeper run-ahead in the tail: 42.8 → 42.1 µs per steady pass at cfg3), 4 at KP = 32
// (so the score ring keeps 8 buffers and three epilogue groups)
#ifndef KM_TS_ABUF
#define KM_TS_ABUF (KP <= 16 ? 6 : 4)
#endif
  // A buffers: per transform group (a group owns buffers g mod a); in TMEM they are cheap
  static constexpr int a = (tc_a_in_tmem<KP, TR>() ? KM_TS_ABUF : 2) * kTransformGroups;
  static constexpr int mw = (KP + 31) / 32;
  static constexpr int raw_stride_max = ((TR * MP * 4 + 256 + 1023) / 1024) * 1024;
  static constexpr int fixed = (tc_a_in_tmem<KP, TR>() ? 0 : a * TR * 128) + 2 * KP * 128 +  // A ring, B tile
                               ((KP * (MP + 1) + KP) * 8 + 1023) / 1024 * 1024 +       // Δ accumulators
                               tc_qcap<KP>() * (8 + 4 * mw) + 1024 +                   // recheck queue
                               2048 + 1024 + 8192 +                                    // barriers, align, static
                               tc_pdelta_bytes<MP, KP>();                              // per-warp private Δ
  static constexpr int cres = ((3 * KP * MP + KP) * 8 + 1023) / 1024 * 1024;          // resident centres + totals
  // keep room for the resident loop's centres unless that would starve the raw ring
  // (the widest shapes then run launch-per-iteration)
  static constexpr int fit_res = (227 * 1024 - fixed - cres) / raw_stride_max;
  static constexpr int fit = fit_res >= 4 ? fit_res : (227 * 1024 - fixed) / raw_stride_max;
  static constexpr int raw = fit > 12 ? 12 : fit;
};
template <int MP, int KP>
struct TcStages {
#ifndef KM_TALL_TILES
#define KM_TALL_TILES 0
#endif
  // 256-point tiles (two M=128 MMA blocks per tile: half the handshakes per point) when at least
  // two 256-row raw slots (≥ 50 KB in flight) fit beside the doubled A ring and the resident state
  static constexpr bool tall = KM_TALL_TILES && KP <= 32 &&
                               (227 * 1024 - TcBudget<MP, KP, 256>::fixed - TcBudget<MP, KP, 256>::cres) /
                                       TcBudget<MP, KP, 256>::raw_stride_max >= 2;
  static constexpr int TR = tall ? 256 : 128;  // points per tile
  static constexpr int raw_fit = tall ? (227 * 1024 - TcBudget<MP, KP, 256>::fixed - TcBudget<MP, KP, 256>::cres) /
                                            TcBudget<MP, KP, 256>::raw_stride_max
                                      : TcBudget<MP, KP, 128>::raw;
  static constexpr int raw = raw_fit > 12 ? 12 : raw_fit;
  static constexpr int a = TcBudget<MP, KP, TR>::a;
  static_assert(raw >= 2, "shared-memory budget");
};

// ---- PTX helpers -----------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// Wait strategy (build-time tuning knob):
//   KM_WAIT_MODE 1: mbarrier.test_wait polling
//   otherwise     : mbarrier.try_wait with a short suspend-time hint (bounded)
// Tuning instrumentation (per-tile clock stamps, timing experiments) is compiled in only for
// the KM_TC_TUNING=1 library variant (tools/); the product kernel carries none of it.
#ifndef KM_TC_TUNING
#define KM_TC_TUNING 0
#endif
#define KM_DBG_FLAGS (KM_TC_TUNING ? a.dbg_flags : 0)
#ifndef KM_TRY_HINT
#define KM_TRY_HINT 0x100000  // try_wait suspend-time hint (ns)
#endif
#ifndef KM_WAIT_MODE
#define KM_WAIT_MODE 2
#endif
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a long suspend-time hint (10 ms, as CUTLASS's ClusterBarrier::wait): a waiting
// thread sleeps until the phase completes instead of spinning, so waiting warps take no
// issue slots from the warps doing the work (spinning waits were ~1/3 of all instructions)
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(KM_TRY_HINT)
      : "memory");
  return ok != 0;
}
// bounded: a wait that cannot complete (a bug) traps instead of hanging the device
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if KM_WAIT_MODE == 1
  while (!mbar_test(bar, parity)) {
  }
#elif KM_WAIT_MODE >= 3  // tuning: poll + fixed sleep (no wake-ups on unrelated barrier events)
  uint32_t n = 0;
  while (!mbar_test(bar, parity)) {
    __nanosleep(KM_WAIT_MODE);
    if (++n == (1u << 26)) __trap();
  }
#else
  // bounded in TIME (a failed try_wait may sleep up to its suspend hint): a deadlocked pipeline
  // traps after ~4 s instead of hanging the device
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(bar, parity)) {
    if (clock64() - t0 > (1ll << 33)) __trap();
  }
#endif
}
// Wait of a role that is normally ahead of its producer (the epilogue on the MMA): a failed
// try_wait returns on any barrier event of the CTA, so with 12 epilogue warps waiting the retry
// loop would take a quarter of the SM's issue slots away from the transform; back off instead.
// Group waits (tuning knob: bit 0 epilogue groups, bit 1 transform groups; both on measured slower —
// 44.6 vs 43.6 µs per steady pass, the bar.sync hand-off adds latency): in each 4-warp group only one warp polls the mbarrier (a
// failed try_wait wakes on every barrier event of the CTA — with 20 waiting warps the retry loops
// were ~25% of all issued instructions); the others park in a named barrier (bar.sync issues
// nothing while blocked) and proceed after tcgen05.fence::after_thread_sync.
#ifndef KM_GROUP_WAIT
#define KM_GROUP_WAIT 0
#endif
#ifndef KM_EPI_SLEEP
#define KM_EPI_SLEEP 0
#endif
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
#if KM_EPI_SLEEP > 0
  uint32_t n = 0;
  while (!mbar_try(bar, parity)) {
    __nanosleep(KM_EPI_SLEEP);
    if (++n == (1u << 26)) __trap();
  }
#else
  mbar_wait(bar, parity);
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// streaming copy: the points are read once per pass, so they should not push the labels,
// the totals and the rows queued for re-decision out of L2
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void prefetch_l2_keep(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "selp.b32 %0, 1, 0, px;\n"
      "}\n"
      : "+r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// D[tmem] (+)= A[smem] · B[smem]
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// A operand from TMEM ("TS"): a_tmem = column address of the 128-lane × K tile (2 halfs per column)
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
      : "memory");
}
// 32 lanes × 8 / 16 / 32 columns of 32-bit from registers: thread i of the warp → lane (base + i)
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3])
               : "memory");
}
// n (multiple of 4, compile-time) consecutive columns
template <int N>
__device__ __forceinline__ void tmem_st_row(uint32_t taddr, const uint32_t* r) {
#pragma unroll
  for (int c = 0; c + 8 <= N; c += 8) tmem_st8(taddr + c, r + c);
  if constexpr (N % 8 == 4) tmem_st4(taddr + (N - 4), r + (N - 4));
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// 32 lanes × 16 columns of 32-bit: thread i of the warp gets row (lane base + i), 16 consecutive columns.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, SWIZZLE_128B (layout type 2), sm100 version bit.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// Instruction descriptors (cute/arch/mma_sm100_desc.hpp InstrDescriptor bit layout).
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kTile >> 4) << 24);
}
// kind::f16, A = B = F16 (format 0), D = F32, both K-major
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
  return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kTile >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_u8_amn(int n) {
  return (2u << 4) | (0u << 7) | (0u << 10) | (1u << 15) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(kTile >> 4) << 24);
}

// byte offset of 16-B chunk q of row r inside a SW128 region (8-row atoms of 1 KiB)
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t sw128(int r, int q) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + (((q ^ (r & 7)) & 7) << 4));
}


template <int MP>
struct TcLayout {
  static constexpr int HW = 8 * ((MP + 1 + 7) / 8);  // halfs per part (features incl. the ones column)
  static constexpr int KSTEPS = (2 * HW) / 16;       // kind::f16 MMA k-steps (16 halfs = 32 B each)
};

#ifndef KM_K3_SMEM
#define KM_K3_SMEM 1
#endif
#ifndef KM_NS_MAX
#define KM_NS_MAX 8
#endif
// K3: the MMA accumulates all three products (xh·wh + xl·wh + xh·wl) into ONE column per centre
// (A row [xh | xl | xh], B rows [wh | wh] and [wl]), otherwise hi and lo parts land in two
// columns that the epilogue adds.
template <int KP, int MB, int HW = 32, int AS = 0, bool K3 = false>
struct TcTmem {
  static constexpr int per = MB * (K3 ? 1 : 2) * KP;                       // score columns per tile
  static constexpr int ktail = (HW + 15) / 16;                             // K3: k-steps of the xh·wl tail
  // A columns per row (TS): [xh | xl] — the K3 tail MMA re-reads the xh columns (A at a column
  // offset), so no third copy is stored
  static constexpr int arow = HW;
  static constexpr int acols = AS * MB * arow;                             // TS: A buffers
  static constexpr int NS0 = (512 - acols) / per;
  static constexpr int NS = NS0 >= KM_NS_MAX ? KM_NS_MAX : NS0;            // TMEM score buffers
  static constexpr uint32_t a_base = NS * per;                             // first A column (TS)
  static constexpr uint32_t cols = NS * per + acols;
  static constexpr uint32_t alloc = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
};

// smem carve-up (1 KiB aligned sections; the raw ring depends on the runtime m)
template <int MP, int KP>
struct TcSmem {
  static constexpr int RS = TcStages<MP, KP>::raw, AS = TcStages<MP, KP>::a;
  uint32_t raw_stride, off_raw, off_a, off_w, off_acc, off_pacc, off_q, off_c, off_bar, total;
  // kres = k for the resident loop (two fp64 centre sets stay in shared memory), else 0
  __host__ __device__ TcSmem(int m, int kres) {
    // fixed-size sections first (compile-time offsets: no per-use address arithmetic in the
    // hot loops), then the raw ring (row stride depends on m) and the resident centres (on k)
    off_bar = 0;                              // mbarriers + TMEM address (1 KiB)
    off_w = 1024;                             // [2KP rows × 128 B] B operand (SW128)
    off_a = off_w + 2 * KP * 128;             // [AS][TR rows × 128 B]
    off_acc = off_a + (tc_a_in_tmem<KP, TcStages<MP, KP>::TR>() ? 0 : AS * TcStages<MP, KP>::TR * 128);                    // [KP·(MP+1) + KP] int64 Δ
    off_pacc = off_acc + ((KP * (MP + 1) + KP) * 8 + 1023) / 1024 * 1024;  // [kEpiWarps][stride] private Δ
    off_q = off_pacc + tc_pdelta_bytes<MP, KP>();                            // recheck queue: rows, masks, scalars
    off_raw = off_q + ((tc_qcap<KP>() * (8 + 4 * ((KP + 31) / 32)) + 1024) + 1023) / 1024 * 1024;
    // + 256 B slack: the transform reads MP ≥ m floats per row without bounds branches
    raw_stride = ((uint32_t)TcStages<MP, KP>::TR * m * 4 + 256 + 1023) & ~1023u;
    off_c = off_raw + RS * raw_stride;        // resident: [2][kres·m] fp64 centres, then [kres·m + kres] int64 totals
    total = off_c + ((uint32_t)((2 * kres * m + kres * m + kres) * 8) + 1023) / 1024 * 1024 + 1024;  // + 1 KiB slack
  }
};

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin until *p ≥ target (one thread).  Bounded: a grid that is not co-resident (or a
// bug) traps with an error after ~4 s instead of hanging the device.
__device__ __forceinline__ void grid_spin(const unsigned int* p, unsigned int target) {
  const long long t0 = clock64();
  while (ld_acquire_u32(p) < target) {
    if (clock64() - t0 > (1ll << 33)) __trap();
  }
}

// Per-CTA filter prep for the resident loop: ‖fl32(c)‖², max ‖fl32(c)‖ and the fp16 hi/lo
// B operand written straight into the CTA's SW128 tile — the same values block_prep_filter
// (kmeans_finish.cuh) writes to global memory for the launch-per-iteration path.
__device__ __forceinline__ void cta_prep_operand(const double* __restrict__ C, int k, int m, int kp, float pre,
                                                 unsigned char* s_w, float* s_cmax) {
  __shared__ double s_cn2[512];  // tensor-core operand rows (kp ≤ 512)
  __shared__ float s_red[32];
  float local_max = 0.f;
  for (int cc = threadIdx.x; cc < k; cc += blockDim.x) {
    double s = 0.0;
    for (int f = 0; f < m; ++f) {
      const double v = (double)__double2float_rn(C[(size_t)cc * m + f]);
      s = __fma_rn(v, v, s);
    }
    s_cn2[cc] = s;
    local_max = fmaxf(local_max, __double2float_ru(sqrt(s) * (1.0 + 1e-12)));
  }
  for (int o = 16; o > 0; o >>= 1) local_max = fmaxf(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = local_max;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) mx = fmaxf(mx, s_red[i]);
    s_cmax[0] = mx;
  }
  const int hw = 8 * ((m + 1 + 7) / 8);
  for (int i = threadIdx.x; i < kp * 64; i += blockDim.x) {
    const int cc = i >> 6, col = i & 63;
    const int f = col < hw ? col : col - hw;
    float v = 0.f;
    if (cc < k && col < 2 * hw) {
      if (f < m) v = -2.0f * __double2float_rn(C[(size_t)cc * m + f]) * pre;
      else if (f == m) v = __double2float_rn(s_cn2[cc] * (double)pre * (double)pre);
    } else if (cc >= k && col < 2 * hw && f == m) {
      v = 65504.f;
    }
    const __half h = __float2half_rn(v);
    const __half l = __float2half_rn(v - __half2float(h));
    const uint32_t off = sw128(0, col >> 3) + (col & 7) * 2;
    *reinterpret_cast<unsigned short*>(s_w + sw128(cc, col >> 3) + (col & 7) * 2) =
        (col < 2 * hw) ? __half_as_ushort(h) : (unsigned short)0;
    *reinterpret_cast<unsigned short*>(s_w + sw128(kp + cc, col >> 3) + (col & 7) * 2) =
        (col < hw) ? __half_as_ushort(l) : (unsigned short)0;
    (void)off;
  }
  fence_proxy_async();  // generic-proxy writes of the B tile → visible to the tensor core
  __syncthreads();
}

// Exact label of one point by one thread over its candidate centres (bit set in mk):
// the reference recurrence (features ascending, no FMA) per centre, centres ascending,
// strict '<' (lowest index on ties).  Non-candidates are strictly farther than the best
// candidate (filter bound), so the result equals the reference's argmin over all k.
template <int MP, int MW, typename T>
__device__ __forceinline__ int exact_candidates(const T* __restrict__ gx, int m, const double* __restrict__ C,
                                                const uint32_t (&mk)[MW], T (&xr)[MP],
                                                long long* ts = nullptr) {
#pragma unroll
  for (int f = 0; f < MP; ++f) xr[f] = (f < m) ? __ldg(gx + f) : (T)0;
  if (ts) {
    T sx = 0;
#pragma unroll
    for (int f = 0; f < MP; ++f) sx += xr[f];
    ts[0] = clock64() + (sx == 12345.f);
  }
  double bd = 0.0;
  int bl = -1;
#pragma unroll 1
  for (int w = 0; w < MW; ++w) {
    uint32_t bits = mk[w];
#pragma unroll 1
    while (bits) {
      const int c = w * 32 + __ffs(bits) - 1;
      bits &= bits - 1;
      // the candidate's row first (all loads in flight together), then the dependent chain
      const double* cr = C + (size_t)c * m;
      double cv[MP];
#pragma unroll
      for (int f = 0; f < MP; ++f) cv[f] = (f < m) ? cr[f] : 0.0;
      double acc = 0.0;
#pragma unroll
      for (int f = 0; f < MP; ++f) {
        if (f < m) {
          const double d = __dsub_rn((double)xr[f], cv[f]);
          acc = __dadd_rn(acc, __dmul_rn(d, d));
        }
      }
      if (bl < 0 || acc < bd) { bd = acc; bl = c; }
    }
  }
  return bl;
}

// MT > 0: exact feature count m = MT (compile-time); MT < 0: runtime m ≤ −MT.
// PRE: multiply x by the power-of-two prescale (off when the data range is fp16-safe as is).
//
// a.resident == 0: one pass (+ the finish in the last CTA to arrive when a.fuse_finish).
// a.resident == 1: the Lloyd loop runs inside ONE cooperative launch (single GPU):
//   pass t → flush the CTA's Δ into the running totals → grid barrier → every CTA
//   computes C_{t+1} = S/N, the empty count, the congruence test and its own copy of
//   the B operand (bit-identical in every CTA) → pass t+1.  The TMA producer streams
//   the first tiles of pass t+1, and the transform groups convert them (run-ahead), while
//   the other warps run the tail, the barrier and the finish.  Stops
//   on convergence, after the final assign pass of an exhausted run, or on empty
//   clusters (the host repairs them and relaunches).
// Exact incremental update of the per-cluster fixed-point sums for the changed points of one warp
// (`pend`: lanes whose label changed; lane l holds point wrow0 + l, new label bi, old label old).
// Out of line so its registers do not weigh on the steady-state epilogue, where changes are rare.
//  * sparse (steady state): warp-cooperative, four changed points at a time: lane f loads
//    feature f of each (one coalesced L2 round trip per batch, the rows were just streamed) and
//    adds it to the new cluster / subtracts it from the old one; lane m moves the counts;
//  * the first pass (every point adds its row): thread per point, loads batched ahead of the
//    atomics.
// Δ of up to two changed points into a warp's accumulator row of this lane (slot(c): label c's
// word).  Read-modify-writes through possibly equal addresses would serialise on the shared-memory
// load latency, so updates whose addresses are known to differ — new ≠ old of one point; the four
// labels of two points when distinct — load together, then store together.  !priv: the CTA-shared
// accumulator, 32-bit atomic pairs (order-free).
template <typename Slot>
__device__ __forceinline__ void acc_apply2(Slot slot, bool priv, bool two, int n0, int o0, long long q0, int n1, int o1,
                                           long long q1) {
  if (!priv) {
    acc_add64(slot(n0), (unsigned long long)q0);
    if (o0 >= 0) acc_add64(slot(o0), (unsigned long long)(-q0));
    if (two) {
      acc_add64(slot(n1), (unsigned long long)q1);
      if (o1 >= 0) acc_add64(slot(o1), (unsigned long long)(-q1));
    }
    return;
  }
  const bool distinct = two && n0 != n1 && n0 != o1 && o0 != n1 && (o0 != o1 || o0 < 0);
  if (distinct) {
    unsigned long long* pa = slot(n0);
    unsigned long long* pc = slot(n1);
    unsigned long long* pb = o0 >= 0 ? slot(o0) : nullptr;
    unsigned long long* pd = o1 >= 0 ? slot(o1) : nullptr;
    const unsigned long long a = *pa, c = *pc, b = pb ? *pb : 0ull, d = pd ? *pd : 0ull;
    *pa = a + (unsigned long long)q0;
    *pc = c + (unsigned long long)q1;
    if (pb) *pb = b - (unsigned long long)q0;
    if (pd) *pd = d - (unsigned long long)q1;
    return;
  }
  for (int u = 0; u < (two ? 2 : 1); ++u) {  // per point (its two addresses differ), in order
    const int nn = u ? n1 : n0, oo = u ? o1 : o0;
    const long long qq = u ? q1 : q0;
    unsigned long long* pa = slot(nn);
    if (oo >= 0) {
      unsigned long long* pb = slot(oo);
      const unsigned long long a = *pa, b = *pb;
      *pa = a + (unsigned long long)qq;
      *pb = b - (unsigned long long)qq;
    } else {
      *pa += (unsigned long long)qq;
    }
  }
}

template <bool X64>
static __device__ __noinline__ void delta_rows(const float* __restrict__ x, const double* __restrict__ x64, int m,
                                        int64_t wrow0, int lane, int bi, int old,
                                        unsigned int pend, bool full, unsigned long long* s_acc, int km,
                                        float scale_f, double scale_d, bool use_dscale, bool priv) {
  // fixed-point value of coordinate f of row r: from the exact fp64 row for fp64 points (x64)
  auto ldq = [&](int64_t r, int f) -> long long {
    if (X64) return __double2ll_rn(__dmul_rn(__ldg(x64 + r * m + f), scale_d));
    const float v = __ldg(x + r * m + f);
    return use_dscale ? __double2ll_rn(__dmul_rn((double)v, scale_d)) : __float2ll_rn(__fmul_rn(v, scale_f));
  };
  // priv: s_acc is this warp's private accumulator — the lane-per-feature path adds without atomics
  if (full) {
    if (!((pend >> lane) & 1u)) return;
    constexpr int CH = 8;
    for (int f0 = 0; f0 < m; f0 += CH) {
      long long qv[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) qv[j] = (f0 + j < m) ? ldq(wrow0 + lane, f0 + j) : 0ll;
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        if (f0 + j < m) {
          const long long v = qv[j];
          acc_add64(s_acc + (size_t)bi * m + f0 + j, (unsigned long long)v);
          if (old >= 0) acc_add64(s_acc + (size_t)old * m + f0 + j, (unsigned long long)(-v));
        }
      }
    }
    acc_add64(s_acc + (size_t)km + bi, 1ull);
    if (old >= 0) acc_add64(s_acc + (size_t)km + old, ~0ull);
    return;
  }
  // sparse: two changed points per step; lane f loads feature f of both rows (L2), lane m counts
  auto slot = [&](int c) -> unsigned long long* { return lane < m ? s_acc + (size_t)c * m + lane : s_acc + (size_t)km + c; };
  while (pend) {
    const int j0 = __ffs(pend) - 1;
    pend &= pend - 1;
    const bool two = pend != 0;
    const int j1 = two ? __ffs(pend) - 1 : j0;
    if (two) pend &= pend - 1;
    const int n0 = __shfl_sync(0xffffffffu, bi, j0), o0 = __shfl_sync(0xffffffffu, old, j0);
    const int n1 = __shfl_sync(0xffffffffu, bi, j1), o1 = __shfl_sync(0xffffffffu, old, j1);
    const long long q0 = lane < m ? ldq(wrow0 + j0, lane) : 1ll;
    const long long q1 = lane < m && two ? ldq(wrow0 + j1, lane) : 1ll;
    if (lane <= m) acc_apply2(slot, priv, two, n0, o0, q0, n1, o1, q1);
  }
}

// Heavy-pass Δ (many labels change): the changed points of one warp read their rows from the
// pass's raw shared-memory tile, which the epilogue (not the transform) releases in heavy passes —
// lane f takes feature f of each changed point (a short LDS instead of an L2/DRAM round trip).
// `prow0`: row in the tile of lane 0's point; rows past the tile's 16-byte bulk come from global.
static __device__ __forceinline__ void delta_rows_smem(const float* __restrict__ rs, uint32_t bulk_elems,
                                                       const float* __restrict__ gx_tile, int m, int prow0, int lane,
                                                       int bi, int old, unsigned int pend,
                                                       unsigned long long* __restrict__ s_acc, int km, float scale_f,
                                                       double scale_d, bool use_dscale, bool priv) {
  // Two changed points per step: rows loaded and converted first, then acc_apply2.
  const int col = lane < m ? lane : 0;
  auto value = [&](int j) -> long long {
    const uint32_t e = (uint32_t)(prow0 + j) * m + col;
    const float v = e < bulk_elems ? rs[e] : __ldg(gx_tile + e);
    return use_dscale ? __double2ll_rn(__dmul_rn((double)v, scale_d)) : __float2ll_rn(__fmul_rn(v, scale_f));
  };
  // address of label c's accumulator for this lane (lane m: the counts)
  auto slot = [&](int c) -> unsigned long long* { return lane < m ? s_acc + (size_t)c * m + lane : s_acc + (size_t)km + c; };
  const bool act = lane <= m;
  while (pend) {
    const int j0 = __ffs(pend) - 1;
    pend &= pend - 1;
    const bool two = pend != 0;
    const int j1 = two ? __ffs(pend) - 1 : j0;
    if (two) pend &= pend - 1;
    const int n0 = __shfl_sync(0xffffffffu, bi, j0), o0 = __shfl_sync(0xffffffffu, old, j0);
    const int n1 = __shfl_sync(0xffffffffu, bi, j1), o1 = __shfl_sync(0xffffffffu, old, j1);
    const long long v0 = value(j0), v1 = value(j1);
    const long long q0 = lane < m ? v0 : 1ll, q1 = lane < m ? v1 : 1ll;
    if (act) acc_apply2(slot, priv, two, n0, o0, q0, n1, o1, q1);
  }
}

// Epilogue warpgroups of an instantiation: four for the cfg5 shape (m = 25, K = 64, fp32 points),
// whose 64-score epilogue bounds the pass (69.6 → 68.4 µs per 2M-point pass; 28 warps at 72
// registers: that instantiation spills ~0.2 KB, the m-bucket ones would spill ~1 KB), three elsewhere.
template <int MT, int KP, bool X64>
__host__ __device__ constexpr int tc_epi_groups() { return (MT == 25 && KP == 64 && !X64) ? 4 : kEpiGroups; }
template <int MT, int KP, bool X64>
__host__ __device__ constexpr int tc_threads() { return (kTransformWarps + 4 * tc_epi_groups<MT, KP, X64>() + 4) * 32; }

// X64: fp64 points — the pass streams their fp32 shadow (a.x), the exact rows (a.x64) feed the
// recheck and the Δ; a separate instantiation so the fp32 kernels carry none of it
template <int MT, int KP, bool PRE, bool X64>
__global__ void __launch_bounds__(tc_threads<MT, KP, X64>(), 1) lloyd_pass_tc_kernel(TcArgs a) {
  // this instantiation's warp roles (they shadow the defaults above)
  constexpr int kEpiGroups = tc_epi_groups<MT, KP, X64>();
  constexpr int kEpiWarps = 4 * kEpiGroups;
  constexpr int kProducerWarp = kTransformWarps + kEpiWarps;
  constexpr int kMmaWarp = kProducerWarp + 1;
  constexpr int kRecheckWarp = kMmaWarp + kMmaWarps;
  constexpr int kThreadsTC = (kRecheckWarp + 1) * 32;
  constexpr int kTailThreads = kThreadsTC - (kTransformWarps + 1) * 32;
  static_assert(kThreadsTC == (kTransformWarps + kEpiWarps + 4) * 32, "warp-role layout");
  static_assert(kThreadsTC == tc_threads<MT, KP, X64>(), "launch bounds");
  const double* __restrict__ x64p = X64 ? a.x64 : nullptr;
  constexpr int MP = MT > 0 ? MT : -MT;
  static_assert(!tc_pdelta<MP, KP>() || kEpiWarps == tc::kEpiWarps, "private Δ is sized for the default roles");
  if (a.gate && (a.st->done || a.st->need_host)) return;
  using L = TcLayout<MP>;
  constexpr int TR = TcStages<MP, KP>::TR;  // points per tile
  constexpr int MB = TR / 128;              // M=128 MMA blocks per tile
  // A operand in TMEM (written by the transform with tcgen05.st, read by the MMA): takes the A
  // tile off shared memory (its stores and the MMA's operand reads) where the columns fit
  constexpr bool TS = tc_a_in_tmem<KP, TR>();
  // one score column per centre (see TcTmem): the tail MMA xh·wl re-reads the xh k-steps of A —
  // from TMEM (TS) or from the SW128 shared-memory tile — into the same accumulator
  constexpr bool K3 = KM_K3_SMEM || TS;
  using TM = TcTmem<KP, MB, TcLayout<MP>::HW, TS ? TcStages<MP, KP>::a : 0, K3>;
  constexpr int SC = K3 ? KP : 2 * KP;  // score columns per M block
  // Active epilogue groups.  A group waiting on tile g must know that the previous fill of the
  // score buffer (tile g − NS) has completed, or the parity wait aliases: it has consumed tiles
  // g − EG, g − 2·EG, …, and a consumed tile issued by the same MMA warp as g (same parity) at or
  // after g − NS implies it (tcgen05.commit covers every earlier MMA of that thread).  So NS must
  // reach the first even multiple of EG; narrower score rings (KP > 32) run two groups and the
  // third idles.
  constexpr int EG = TM::NS < 2 ? 1
                     : TM::NS % 2 == 0 && TM::NS >= (kEpiGroups % 2 ? 2 * kEpiGroups : kEpiGroups) ? kEpiGroups : 2;
  const bool resident = a.resident != 0;
  const TcSmem<MP, KP> S(MT > 0 ? MT : a.m, resident ? a.k : 0);
  constexpr int RS = TcStages<MP, KP>::raw, AS = TcStages<MP, KP>::a;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1 KiB align the carve-up (SW128 atoms must be 1 KiB aligned); pointer arithmetic on the
  // __shared__ array keeps the shared address space (LDS/STS, not generic LD/ST)
  unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* raw = reinterpret_cast<float*>(sm + S.off_raw);
  unsigned char* s_w = sm + S.off_w;
  unsigned long long* s_acc = reinterpret_cast<unsigned long long*>(sm + S.off_acc);
  constexpr bool PD = tc_pdelta<MP, KP>();
  constexpr int PST = tc_pdelta_stride<MP, KP>();
  unsigned long long* s_pacc = reinterpret_cast<unsigned long long*>(sm + S.off_pacc);
  constexpr int MW = (KP + 31) / 32;                                          // candidate mask words
  long long* s_q = reinterpret_cast<long long*>(sm + S.off_q);                 // [cap] row << 8 | old + 1
  constexpr int QCAP = tc_qcap<KP>();
  uint32_t* s_qm = reinterpret_cast<uint32_t*>(sm + S.off_q + QCAP * 8);  // [cap][MW] candidate masks
  unsigned int* s_qn = s_qm + QCAP * MW;                                  // [0] queue length
  float* s_cmax = reinterpret_cast<float*>(s_qn + 4);                          // resident: max ‖c‖
  double* s_cbuf = reinterpret_cast<double*>(sm + S.off_c);                            // resident: [2][k·m]
  unsigned long long* s_tot = reinterpret_cast<unsigned long long*>(s_cbuf + 2 * (size_t)a.k * (MT > 0 ? MT : a.m));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + S.off_bar);
  uint64_t* full_raw = bars;                 // [RS] TMA → transform
  uint64_t* empty_raw = full_raw + RS;       // [RS] transform → TMA
  uint64_t* a_full = empty_raw + RS;         // [AS] transform → MMA
  uint64_t* a_empty = a_full + AS;           // [AS] MMA commit → transform
  uint64_t* s_full = a_empty + AS;           // [NS] MMA commit → epilogue
  uint64_t* s_empty = s_full + TM::NS;       // [NS] epilogue → MMA
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_empty + TM::NS);

  const int m = MT > 0 ? MT : a.m;
  const int k = a.k;
  const int km = k * m;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (a.n + TR - 1) / TR;
  // contiguous tile range per CTA: [t_lo, t_lo + my_tiles) (TLB- and DRAM-page-friendly streams)
  const int64_t t_lo = ntiles * blockIdx.x / gridDim.x;
  const int my_tiles = (int)(ntiles * (blockIdx.x + 1) / gridDim.x - t_lo);
  const int nacc = km + k;
  const int npre = resident ? min(RS, my_tiles) : 0;  // next-pass tiles streamed during the tail

  // ---- setup ----
  if (tid == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(full_raw + s, 1);
      mbar_init(empty_raw + s, 4);  // the 4 warps of the transform group that consumed it
    }
    for (int s = 0; s < AS; ++s) {
      mbar_init(a_full + s, 4);
      mbar_init(a_empty + s, 1);
    }
    for (int s = 0; s < TM::NS; ++s) {
      mbar_init(s_full + s, 1);
      mbar_init(s_empty + s, 4);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_holder, TM::alloc);
  if (warp < kTransformWarps + kEpiWarps) {
    const int nthr = (kTransformWarps + kEpiWarps) * 32;
    // B operand rows (already fp16-split and packed by the prep kernel) → SW128 K-major smem
    for (int i = tid; i < 2 * KP * 8; i += nthr) {
      const int r = i >> 3, q = i & 7;
      *reinterpret_cast<uint4*>(s_w + sw128(r, q)) = *reinterpret_cast<const uint4*>(a.wop + (size_t)r * 64 + q * 8);
    }
    // A operand buffers zeroed once (chunks beyond the used width stay zero)
    if (!TS)
      for (int i = tid; i < AS * TR * 8; i += nthr)
      *reinterpret_cast<uint4*>(sm + S.off_a + i * 16) = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < nacc; i += nthr) s_acc[i] = 0ull;
    if (PD)
      for (int i = tid; i < kEpiWarps * PST; i += nthr) s_pacc[i] = 0ull;
    for (int i = tid; i < QCAP; i += nthr) s_q[i] = 0;
    if (resident) {
      for (int i = tid; i < km; i += nthr) s_cbuf[i] = a.c64[i];
      // totals of the current labels (peer loop after a separate first pass: the local sums in
      // fin.tot are this rank's first contribution to the exchange, the totals start at zero)
      const bool tot0 = a.xch_peers != nullptr && a.skip_first;
      for (int i = tid; i < nacc; i += nthr) s_tot[i] = tot0 ? 0ull : a.fin.tot[i];
    }
    if (tid == 0) {
      s_qn[0] = s_qn[1] = s_qn[2] = 0u;
      s_cmax[0] = a.cmax[0];
    }
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const float pre = a.pre;

  // loop state: every CTA derives the same decisions from the same totals
  DevState* st = a.st;
  int t_upd = st->t;
  bool exhausted = st->exhausted != 0;
  const int max_iters = st->max_iters;
  const double tol = st->tol;
  bool full = a.full != 0;
  const bool no_sums = a.no_sums != 0;
  // Heavy passes (many label changes): the raw tile stays until the epilogue, which takes the
  // changed points' rows from shared memory.  Decided per CTA from its previous pass's changes
  // (the first pass after a separate L0 pass, and full first passes, are heavy).
  __shared__ int s_tail[5];  // run-ahead: loop state published by the tail for the warps that skipped it
  __shared__ int s_heavy;
  __shared__ unsigned int s_pass_changes;
  if (tid == 0) {
    // (fp64 points: the raw tiles hold the fp32 shadow, not the exact rows — no heavy passes)
    s_heavy = KM_HEAVY_PASSES && !no_sums && !x64p && (a.full || (resident && a.skip_first)) ? 1 : 0;
    s_pass_changes = 0u;
  }
  __syncthreads();
  int cb = 0;      // resident: s_cbuf half holding C_t
  int g0 = 0;      // tiles of earlier passes (ring positions continue across passes)
  int issued = 0;  // producer: tiles of the current pass already in flight
  int pre_done = 0;  // transform: tiles of the current pass transformed ahead (in the last tail)
  int last_pass_tiles = my_tiles;

  // tuning only: per-pass phase ends (globaltimer, max over CTAs) of the resident loop
  unsigned long long* pst = (KM_TC_TUNING && a.dbg_times != nullptr && resident && tid == kTransformWarps * 32)
                                ? reinterpret_cast<unsigned long long*>(a.dbg_times + 4096) : nullptr;
  for (int it = 0;; ++it) {
    // tiles of this pass (resident skip_first: the labels and their sums come from a separate
    // first pass + cluster-sums launch, so iteration 0 starts at the tail with Δ = 0)
    const int pass_tiles = (resident && it == 0 && a.skip_first) ? 0 : my_tiles;
    last_pass_tiles = pass_tiles;
    const bool heavy = s_heavy != 0;
    const double* C = resident ? s_cbuf + cb * km : a.c64;
    if (pst && it < 256 && blockIdx.x == 0) pst[it * 8 + 0] = globaltimer();
    if (pst && (it == 100 || it == 101 || it == 150))
      a.dbg_times[6144 + (it == 100 ? 0 : it == 101 ? 300 : 600) + blockIdx.x * 2] = (long long)globaltimer();
    // exact re-decision of queue entry q (thread per point, candidate centres only); Δ into s_acc
    // Δ of a changed point (queued by the epilogue): its row from global memory (L2: streamed
    // moments ago), + to the new cluster, − from the old one
    auto apply_change = [&](unsigned int q, long long ent) {
      const long long row = (ent >> 16) & ((1ll << 44) - 1);
      const int old = (int)((ent >> 8) & 0xff) - 1, nw = (int)(ent & 0xff);
      const float* xr = a.x + row * m;
      float xq[MP];
#pragma unroll
      for (int f = 0; f < MP; ++f) xq[f] = (f < m && !x64p) ? __ldg(xr + f) : 0.f;
#pragma unroll
      for (int f = 0; f < MP; ++f) {
        if (f < m) {
          const long long v = x64p ? __double2ll_rn(__dmul_rn(__ldg(x64p + row * m + f), a.scale_d))
                              : a.use_dscale ? __double2ll_rn(__dmul_rn((double)xq[f], a.scale_d))
                                             : __float2ll_rn(__fmul_rn(xq[f], a.scale_f));
          acc_add64(s_acc + (size_t)nw * m + f, (unsigned long long)v);
          if (old >= 0) acc_add64(s_acc + (size_t)old * m + f, (unsigned long long)(-v));
        }
      }
      acc_add64(s_acc + (size_t)km + nw, 1ull);
      if (old >= 0) acc_add64(s_acc + (size_t)km + old, ~0ull);
      s_q[q] = 0;  // free for the next pass
    };
    auto redecide = [&](unsigned int q, long long ent) {
      if (ent & kChangeFlag) { apply_change(q, ent); return; }
      const long long row = (ent >> 8) & ((1ll << 54) - 1);
      const int old = (int)(ent & 0xff) - 1;
      uint32_t mk[MW];
#pragma unroll
      for (int w = 0; w < MW; ++w) mk[w] = s_qm[q * MW + w];
      // exact label and fixed-point row (fp64 points: from the exact fp64 coordinates)
      long long qv[MP];
      int bl;
      if (x64p) {
        double xq[MP];
        bl = resident ? exact_candidates<MP, MW>(x64p + row * m, m, s_cbuf + cb * km, mk, xq)
                      : exact_candidates<MP, MW>(x64p + row * m, m, a.c64, mk, xq);
#pragma unroll
        for (int f = 0; f < MP; ++f) qv[f] = __double2ll_rn(__dmul_rn(xq[f], a.scale_d));
      } else {
        float xq[MP];
        bl = resident ? exact_candidates<MP, MW>(a.x + row * m, m, s_cbuf + cb * km, mk, xq)
                      : exact_candidates<MP, MW>(a.x + row * m, m, a.c64, mk, xq);
#pragma unroll
        for (int f = 0; f < MP; ++f)
          qv[f] = a.use_dscale ? __double2ll_rn(__dmul_rn((double)xq[f], a.scale_d))
                               : __float2ll_rn(__fmul_rn(xq[f], a.scale_f));
      }
      if (bl != old) {
        a.labels[row] = bl;
        if (!full) atomicAdd(&st->changed, 1ull);
        if (no_sums) { s_q[q] = 0; return; }
#pragma unroll
        for (int f = 0; f < MP; ++f) {
          if (f < m) {
            const long long v = qv[f];
            acc_add64(s_acc + (size_t)bl * m + f, (unsigned long long)v);
            if (old >= 0) acc_add64(s_acc + (size_t)old * m + f, (unsigned long long)(-v));
          }
        }
        acc_add64(s_acc + (size_t)km + bl, 1ull);
        if (old >= 0) acc_add64(s_acc + (size_t)km + old, ~0ull);
      }
      s_q[q] = 0;  // free for the next pass
    };
    // TMA producer: tile g (index i of its pass) → raw slot g % RS (one thread); also issued ahead in the tail
    const uint64_t pol = l2_policy_evict_first();
    auto issue = [&](int g, int i) {
      const int s = g % RS;
      if (g >= RS) mbar_wait(empty_raw + s, ((g / RS) - 1) & 1);
      const int64_t row0 = (t_lo + i) * TR;
      const int64_t rem = a.n - row0;
      const int rows = rem < TR ? (int)rem : TR;
      const uint32_t bytes = ((uint32_t)rows * m * 4u) & ~15u;
      mbar_arrive_expect_tx(full_raw + s, bytes);
      if (bytes)
        bulk_g2s_hint(reinterpret_cast<unsigned char*>(raw) + s * S.raw_stride, a.x + row0 * m, bytes, full_raw + s, pol);
    };
    // transform of tile g (index i of its pass): raw rows → the A operand; hv: heavy pass (the
    // epilogue, not the transform, releases the raw slot).  Also run ahead in the tail (below).
    const int tg = warp >> 2;
    const int p_t = tid & 127;
    auto transform_tile = [&](const int g, const int i, const bool hv) {
      const int p = p_t;
      const uint32_t row_off = (uint32_t)((p >> 3) * 1024 + (p & 7) * 128);  // SW128 geometry of row p
      const int key = p & 7;
      const float* __restrict__ gx = a.x;
        const int s = g % RS, sa = g % AS;
        const int64_t row0 = (t_lo + i) * TR;
        const int64_t rem = a.n - row0;
        const int rows = rem < TR ? (int)rem : TR;
        const bool stamp = KM_TC_TUNING && a.dbg_times != nullptr && blockIdx.x == 0 && p == 0 && i < 64 && it == (resident ? 100 : 0);
        long long* ts = stamp ? a.dbg_times + (size_t)i * 8 : nullptr;
        if (stamp) ts[0] = clock64();
        if (KM_GROUP_WAIT & 2) {  // one warp of the group polls both barriers, the other three park in bar.sync
          if ((warp & 3) == 0) {
            mbar_wait(full_raw + s, (g / RS) & 1);
            if (g >= AS) mbar_wait(a_empty + sa, ((g / AS) - 1) & 1);  // this group's A buffer is free
          }
          named_bar_sync(1 + kEpiGroups + tg, 128);
          tc_fence_after();
        } else {
          mbar_wait(full_raw + s, (g / RS) & 1);
        }
        if (stamp) ts[1] = clock64();
        if (KM_DBG_FLAGS & 4) {  // tuning only: measure the TMA stream alone
          __syncwarp();
          if (lane == 0) mbar_arrive(empty_raw + s);
          return;
        }
        const float* rs = raw + s * (S.raw_stride / 4);
        if (!(KM_GROUP_WAIT & 2) && g >= AS) mbar_wait(a_empty + sa, ((g / AS) - 1) & 1);  // this group's A buffer is free
        if (stamp) ts[7] = clock64();
        unsigned char* s_a = sm + S.off_a + sa * (TR * 128);
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {  // thread = points p and p + 128 (tall tiles)
          const int pp = p + 128 * mb;
          const bool active = pp < rows;
          float xs[L::HW];
          if (KM_DBG_FLAGS & 512) {  // timing experiment only: no raw-tile loads
#pragma unroll
            for (int f = 0; f < L::HW; ++f) xs[f] = 0.f;
          } else if (rows == TR) {  // full tile: branch-free loads (over-reads stay inside the padded slot)
            const float* xr = rs + pp * m;
#pragma unroll
            for (int f = 0; f < L::HW; ++f) {
              const float v = (f < MP) ? xr[f] : 0.f;
              xs[f] = (f < m) ? (PRE ? v * pre : v) : 0.f;
            }
          } else {  // ragged last tile: bulk part + ≤ 3 trailing floats from global
            const uint32_t bulk_elems = (((uint32_t)rows * m * 4u) & ~15u) >> 2;
            for (int f = 0; f < L::HW; ++f) {
              float v = 0.f;
              if (f < MP && f < m && active) {
                const uint32_t e = (uint32_t)pp * m + f;
                v = ((e < bulk_elems) ? rs[e] : __ldg(gx + row0 * m + e));
                if (PRE) v *= pre;
              }
              xs[f] = v;
            }
          }
#pragma unroll
          for (int f = 0; f < L::HW; ++f)
            if (f == m) xs[f] = active ? 1.f : 0.f;  // ones column picks up ‖c‖²
          uint32_t hw[L::HW / 2], lw[L::HW / 2];
#pragma unroll
          for (int q = 0; q < L::HW / 2; ++q) {
            if (KM_DBG_FLAGS & 512) {  // timing experiment only: no transform arithmetic
              hw[q] = lw[q] = 0u;
              continue;
            }
            const __half2 h2 = __floats2half2_rn(xs[2 * q], xs[2 * q + 1]);
            const float2 hf = __half22float2(h2);
            // x − fl(xh) for both lanes in one packed FADD2
            const float2 d = __fadd2_rn(make_float2(xs[2 * q], xs[2 * q + 1]), make_float2(-hf.x, -hf.y));
            const __half2 l2 = __floats2half2_rn(d.x, d.y);
            hw[q] = *reinterpret_cast<const uint32_t*>(&h2);
            lw[q] = *reinterpret_cast<const uint32_t*>(&l2);
          }
          if constexpr (TS) {
            // the point's A row [xh | xl] (HW 32-bit columns) → TMEM lane p of this tile's A buffer
            const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + TM::a_base + (uint32_t)(sa * TM::arow);
            tmem_st_row<L::HW / 2>(ta, hw);             // [xh | xl]
            tmem_st_row<L::HW / 2>(ta + L::HW / 2, lw);
          } else {
            unsigned char* s_ab = s_a + mb * (128 * 128);
#pragma unroll
            for (int q = 0; q < L::HW / 8; ++q) {
              *reinterpret_cast<uint4*>(s_ab + row_off + ((uint32_t)(q ^ key) << 4)) =
                  make_uint4(hw[4 * q], hw[4 * q + 1], hw[4 * q + 2], hw[4 * q + 3]);
              *reinterpret_cast<uint4*>(s_ab + row_off + ((uint32_t)((q + L::HW / 8) ^ key) << 4)) =
                  make_uint4(lw[4 * q], lw[4 * q + 1], lw[4 * q + 2], lw[4 * q + 3]);
            }
          }
        }
        // raw slot consumed (every loaded value has been used, so no LDS is still in flight):
        // the TMA producer may refill it (heavy passes: the epilogue releases it)
        __syncwarp();
        if (lane == 0 && !hv) mbar_arrive(empty_raw + s);
        if (stamp) ts[2] = clock64();
        if constexpr (TS) {
          tmem_st_wait();      // the A row is in TMEM
          tc_fence_before();   // ordered before the hand-off to the MMA issuer
        } else {
          fence_proxy_async();  // generic-proxy A stores → visible to the tensor core
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full + sa);
        if (stamp) ts[3] = clock64();
    };
    if (warp == kRecheckWarp) {
      // ===================== recheck warp: re-decides queued points while the pass streams =====================
      unsigned int done = 0;
      for (;;) {
        const unsigned int avail = __shfl_sync(0xffffffffu, min(*reinterpret_cast<volatile unsigned int*>(s_qn), (unsigned int)QCAP), 0);
        if (done < avail) {
          const unsigned int q = done + lane;
          if (q < avail) {
            long long ent;
            while ((ent = *reinterpret_cast<volatile long long*>(s_q + q)) == 0) {
            }
            __threadfence_block();
            redecide(q, ent);
          }
          done = min(done + 32u, avail);
        } else {
          const unsigned int fin = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile unsigned int*>(s_qn + 1), 0);
          if (fin >= (unsigned int)kEpiWarps) {
            __threadfence_block();
            const unsigned int av2 = __shfl_sync(0xffffffffu, min(*reinterpret_cast<volatile unsigned int*>(s_qn), (unsigned int)QCAP), 0);
            if (av2 == done) break;
          } else {
            __nanosleep(256);
          }
        }
      }
      if (lane == 0) s_qn[2] = done;
    } else if (warp == kProducerWarp) {
      // ===================== TMA producer: tile g → raw slot g % RS =====================
      if (lane == 0) {
        for (int i = issued; i < pass_tiles; ++i) issue(g0 + i, i);
        for (int j = 0; j < npre; ++j) issue(g0 + pass_tiles + j, j);  // next pass (resident)
      }
      issued = npre;
    } else if (warp >= kMmaWarp) {
      // ===================== MMA issuers: warp kMmaWarp + j takes tiles g ≡ j (mod 2); the whole warp
      // runs the (uniform) loop, one elected lane issues (per-tile issue cost halves per warp) =====================
      const int mj = warp - kMmaWarp;
      const uint32_t a0 = smem_u32(sm + S.off_a), w0 = smem_u32(s_w);
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);  // warp-uniform → uniform registers
      // N ≤ 256 per MMA: the large-K pass issues SC / 256 column blocks (B rows h·NN.. of each half)
      constexpr int NSUB = SC > 256 ? SC / 256 : 1;
      constexpr int NN = SC / NSUB;
      constexpr uint32_t idesc = idesc_f16(NN);
      const uint64_t bdescL = make_desc(w0 + KP * 128, 16, 1024);  // B rows KP.. ([wl | 0]) for the K3 tail
      const uint64_t bdesc0 = make_desc(w0, 16, 1024);
      // Two issuers alternate tiles only when the score ring has an even depth: a buffer is then
      // always reused by the same warp, whose own earlier wait orders the parity check.  With one
      // score buffer (the K = 512 pass) consecutive tiles share it, and an issuer could pass the
      // parity wait of a phase two behind — a single issuer takes every tile.
      constexpr int NI = TM::NS % 2 == 0 ? kMmaWarps : 1;
      for (int i = NI == 1 ? (mj == 0 ? 0 : pass_tiles) : (mj - (g0 & 1)) & 1; i < pass_tiles && !(KM_DBG_FLAGS & 4);
           i += NI) {
        const int g = g0 + i;
        const int sa = g % AS, ss = g % TM::NS;
        long long* ms = (KM_TC_TUNING && a.dbg_times != nullptr && blockIdx.x == 0 && i < 64 && lane == 0 && it == (resident ? 100 : 0))
                            ? a.dbg_times + 3072 + i * 4 : nullptr;
        if (ms) ms[0] = clock64();
        mbar_wait(a_full + sa, (g / AS) & 1);
        if (ms) ms[1] = clock64();
        if (g >= TM::NS) mbar_wait(s_empty + ss, ((g / TM::NS) - 1) & 1);
        if (ms) ms[2] = clock64();
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int mb = 0; mb < MB; ++mb) {  // block mb: points 128·mb.. of the tile → columns mb·2KP..
            const uint32_t dcol = tm + ss * TM::per + mb * SC;
            if constexpr (TS) {  // A from TMEM: 16 halfs = 8 columns per k-step
              const uint32_t at = tm + TM::a_base + (uint32_t)(sa * TM::arow);
#pragma unroll
              for (int ks = 0; ks < L::KSTEPS; ++ks)  // [xh | xl] · [wh | wh]
                mma_f16_ts(dcol, at + 8 * ks, bdesc0 + 2 * ks, idesc, ks > 0 ? 1u : 0u);
              if constexpr (K3) {
#pragma unroll
                for (int ks = 0; ks < TM::ktail; ++ks)  // + xh · wl (the xh columns again), same accumulator
                  mma_f16_ts(dcol, at + 8 * ks, bdescL + 2 * ks, idesc, 1u);
              }
            } else {
              const uint64_t adesc0 = make_desc(a0 + sa * (TR * 128) + mb * (128 * 128), 16, 1024);
#pragma unroll
              for (int h = 0; h < NSUB; ++h) {
                const uint32_t dc = dcol + h * NN;
                const uint64_t bo = (uint64_t)(h * NN * 128 / 16);  // B rows h·NN.. (address field, 16-B units)
#pragma unroll
                for (int ks = 0; ks < L::KSTEPS; ++ks)  // +32 B per k-step = +2 in the descriptor's address field
                  mma_f16(dc, adesc0 + 2 * ks, bdesc0 + bo + 2 * ks, idesc, ks > 0 ? 1u : 0u);
                if constexpr (K3) {
#pragma unroll
                  for (int ks = 0; ks < TM::ktail; ++ks)  // + xh · wl (the xh k-steps again), same accumulator
                    mma_f16(dc, adesc0 + 2 * ks, bdescL + bo + 2 * ks, idesc, 1u);
                }
              }
            }
          }
          mma_commit(s_full + ss);   // scores ready
          mma_commit(a_empty + sa);  // A buffer consumed
        }
        __syncwarp();
        if (ms) ms[3] = clock64();
      }
    } else if (warp < kTransformWarps) {
      // ===================== transform: thread = point; group tg takes tiles g ≡ tg (mod 2) =====================
      // (tiles below pre_done were transformed during the previous pass's tail)
      for (int i = ((tg - g0) % kTransformGroups + kTransformGroups) % kTransformGroups; i < pass_tiles;
           i += kTransformGroups)
        if (i >= pre_done) transform_tile(g0 + i, i, heavy);
    } else {
      // ===================== epilogue groups: thread = point = TMEM lane; group e takes tiles g ≡ e (mod 2) =====================
      const int ew = warp - kTransformWarps;  // 0..7
      const int e = ew >> 2;
      const int p = ((ew & 3) << 5) | lane;  // TMEM lane of this thread
      const uint32_t lane_base = (uint32_t)((ew & 3) * 32) << 16;
      const float scale_f = a.scale_f;
      // certified bound with the dataset's max ‖x‖ (per pass constant, prescaled units)
      const float tt = (a.xnorm_max + (resident ? s_cmax[0] : a.cmax[0])) * pre;
      const float E2 = 2.f * __fmaf_rn(a.err_coef * tt, tt, a.err_floor);
      const float inv_pre2 = 1.0f / (pre * pre);
      const double scale_d = a.scale_d;
      const bool use_dscale = a.use_dscale != 0, exact_only = a.exact_only != 0;
      unsigned int my_changed = 0, my_rechecked = 0;
      auto prev_label = [&](int i, int mb) -> int {  // previous label of point p + 128·mb of tile i (or -1)
        if (full || i >= pass_tiles) return -1;
        if (KM_DBG_FLAGS & 128) return 0;  // timing experiment only: no label loads
        const int64_t r = (t_lo + i) * TR + 128 * mb + p;
        return r < a.n ? __ldcg(a.labels + r) : -1;  // written by this CTA in the previous pass
      };
      const int i0 = e < EG ? ((e - g0) % EG + EG) % EG : pass_tiles;  // groups ≥ EG idle
      // previous labels prefetched two tiles of this group ahead (an L2 or DRAM round trip
      // must not stall the epilogue)
      int old_n1[MB], old_n2[MB];
#pragma unroll
      for (int mb = 0; mb < MB; ++mb) {
        old_n1[mb] = prev_label(i0, mb);
        old_n2[mb] = prev_label(i0 + EG, mb);
      }
      for (int i = i0; i < pass_tiles && !(KM_DBG_FLAGS & 4); i += EG) {
        const int g = g0 + i;
        const int ss = g % TM::NS;
        const int64_t row0 = (t_lo + i) * TR;
        const int64_t rem = a.n - row0;
        const int rows = rem < TR ? (int)rem : TR;
        int olds[MB];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
          olds[mb] = old_n1[mb];
          old_n1[mb] = old_n2[mb];
          old_n2[mb] = prev_label(i + 2 * EG, mb);
        }
        const bool stamp = KM_TC_TUNING && a.dbg_times != nullptr && blockIdx.x == 0 && p == 0 && i < 64 && it == (resident ? 100 : 0);
        long long* ts = stamp ? a.dbg_times + (size_t)i * 8 : nullptr;
        if (stamp) ts[4] = clock64();
        if (KM_GROUP_WAIT & 1) {  // one warp of the group polls the barrier, the other three park in bar.sync
          if ((ew & 3) == 0) mbar_wait_backoff(s_full + ss, (g / TM::NS) & 1);
          named_bar_sync(1 + e, 128);
        } else {
          mbar_wait_backoff(s_full + ss, (g / TM::NS) & 1);
        }
        if (stamp) ts[5] = clock64();
        tc_fence_after();
        if (KM_DBG_FLAGS & 32) {  // timing experiment only: no epilogue work (labels unchanged)
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_empty + ss);
          continue;
        }
        int bis[MB];
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
          const int pp = p + 128 * mb;
          const bool active = pp < rows;
          const int old = olds[mb];
          const uint32_t tcol = tmem + lane_base + ss * TM::per + mb * SC;
          // Certification: best = min score, candidates = {c : score ≤ best + E2}; the point is
          // certified iff the best is the only candidate (then it is the reference's argmin).
          // The candidate mask is built with one compare + select per centre (no serial counter
          // chain); count = popcount, argmin = the lowest set bit.  KP ≤ 32: the scores stay in
          // registers between the min and the mask.
          constexpr int NCH = KP / 16;
          constexpr bool KEEP = KP <= 32;
          float vk[KEEP ? KP : 16];
          float best = __int_as_float(0x7f800000);
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            uint32_t r0[16], r1[16];
            tmem_ld16(tcol + ch * 16, r0);
            if constexpr (!K3) tmem_ld16(tcol + KP + ch * 16, r1);
            tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {  // padded centres (c ≥ k) score +65504: never a candidate
              const float v = K3 ? __uint_as_float(r0[jj]) : __uint_as_float(r0[jj]) + __uint_as_float(r1[jj]);
              vk[KEEP ? ch * 16 + jj : jj] = v;
            }
            if (a.dbg_scores != nullptr && active) {
#pragma unroll
              for (int jj = 0; jj < 16; ++jj)
                if (ch * 16 + jj < k) a.dbg_scores[(row0 + pp) * k + ch * 16 + jj] = vk[KEEP ? ch * 16 + jj : jj] * inv_pre2;
            }
            float m4[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              m4[q] = fminf(fminf(vk[(KEEP ? ch * 16 : 0) + 4 * q], vk[(KEEP ? ch * 16 : 0) + 4 * q + 1]),
                            fminf(vk[(KEEP ? ch * 16 : 0) + 4 * q + 2], vk[(KEEP ? ch * 16 : 0) + 4 * q + 3]));
            best = fminf(best, fminf(fminf(m4[0], m4[1]), fminf(m4[2], m4[3])));
          }
          const float thr = exact_only ? __int_as_float(0x7f800000) : best + E2;
          uint32_t mk[MW];
#pragma unroll
          for (int w = 0; w < MW; ++w) mk[w] = 0u;
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            if (!KEEP) {
              uint32_t r0[16], r1[16];
              tmem_ld16(tcol + ch * 16, r0);
              if constexpr (!K3) tmem_ld16(tcol + KP + ch * 16, r1);
              tmem_ld_wait();
#pragma unroll
              for (int jj = 0; jj < 16; ++jj)
                vk[jj] = K3 ? __uint_as_float(r0[jj]) : __uint_as_float(r0[jj]) + __uint_as_float(r1[jj]);
            }
            // 16 bits as a sum of disjoint selected powers of two (adds pair up into IADD3 trees)
            uint32_t b[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int jj = 0; jj < 16; ++jj)
              b[jj & 3] += vk[KEEP ? ch * 16 + jj : jj] <= thr ? (1u << jj) : 0u;
            mk[(ch * 16) >> 5] += ((b[0] + b[1]) + (b[2] + b[3])) << ((ch * 16) & 31);
          }
          uint32_t ncand = 0;
          int first = -1;
#pragma unroll
          for (int w = MW - 1; w >= 0; --w) {
            ncand += __popc(mk[w]);
            if (mk[w]) first = 32 * w + __ffs(mk[w]) - 1;
          }
          int bi = (KM_DBG_FLAGS & 512) ? old : first;  // (dbg 512: timing only, labels frozen)
          const bool unc = active && ncand != 1u && !(KM_DBG_FLAGS & (256 | 512));  // (dbg 256: timing only)
          if (__any_sync(0xffffffffu, unc)) {
            if (unc) {
              // padded centres (c ≥ k) are never candidates, whatever the threshold (exact_only
              // sets it to +inf): the recheck only ever reads real centre rows
#pragma unroll
              for (int w = 0; w < MW; ++w) {
                const int lim = k - 32 * w;
                mk[w] &= lim >= 32 ? 0xffffffffu : lim <= 0 ? 0u : ((1u << lim) - 1u);
              }
              // uncertified: only the candidates can be the reference's argmin (every other
              // centre is strictly farther) — queue the point with its candidate mask
              ++my_rechecked;
              const unsigned int slot = atomicAdd(s_qn, 1u);
              if (slot < QCAP) {
                // keep the row in L2 until it is re-decided
                if (x64p) {
                  prefetch_l2_keep(x64p + (row0 + pp) * m);
                  prefetch_l2_keep(x64p + (row0 + pp) * m + m - 1);
                } else {
                  prefetch_l2_keep(a.x + (row0 + pp) * m);
                  prefetch_l2_keep(a.x + (row0 + pp) * m + m - 1);
                }
#pragma unroll
                for (int w = 0; w < MW; ++w) s_qm[slot * MW + w] = mk[w];
                __threadfence_block();  // masks before the entry that publishes them
                // flag | row | previous label + 1 (0 = none); an entry of 0 = not yet written
                *reinterpret_cast<volatile long long*>(s_q + slot) =
                    kQueueFlag | ((row0 + pp) << 8) | (long long)(old + 1);
                bi = old;  // decided by the recheck warp (or the tail)
              } else {     // staging full (rare): decide here
                if (x64p) {
                  double xq[MP];
                  bi = exact_candidates<MP, MW>(x64p + (row0 + pp) * m, m, C, mk, xq);
                } else {
                  float xq[MP];
                  bi = exact_candidates<MP, MW>(a.x + (row0 + pp) * m, m, C, mk, xq);
                }
              }
            }
          }
          bis[mb] = active ? bi : old;
        }
        tc_fence_before();  // TMEM reads ordered before the MMA reuses this buffer
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty + ss);
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
          const int bi = bis[mb], old = olds[mb];
          // --- exact incremental update of the per-cluster fixed-point sums (delta_rows)
          bool chg = bi != old;
          if (chg) {
            ++my_changed;
            a.labels[row0 + 128 * mb + p] = bi;
          }
          if (KM_QUEUE_CHANGES && !full && chg && !no_sums) {
            // hand the Δ to the recheck warp (its loads and atomics leave the epilogue's critical
            // path); a full queue (rare) keeps it here
            const unsigned int slot = atomicAdd(s_qn, 1u);
            if (slot < QCAP) {
              *reinterpret_cast<volatile long long*>(s_q + slot) =
                  kQueueFlag | kChangeFlag | ((row0 + 128 * mb + p) << 16) | ((long long)(old + 1) << 8) | bi;
              chg = false;
            }
          }
          const unsigned int pend = __ballot_sync(0xffffffffu, chg && !no_sums);
          if (pend) {
            unsigned long long* my_acc = PD ? s_pacc + ew * PST : s_acc;  // this warp's (private) Δ
            if (heavy)
              delta_rows_smem(raw + (g % RS) * (S.raw_stride / 4), (((uint32_t)rows * m * 4u) & ~15u) >> 2,
                              a.x + row0 * m, m, 128 * mb + (p & ~31), lane, bi, old, pend, my_acc, km, scale_f,
                              scale_d, use_dscale, PD);
            else
              delta_rows<X64>(a.x, x64p, m, row0 + 128 * mb + (p & ~31), lane, bi, old, pend, full, my_acc, km, scale_f, scale_d,
                         use_dscale, PD);
          }
        }
        if (heavy) {  // the raw tile's rows are no longer needed: the TMA producer may refill it
          __syncwarp();
          if (lane == 0) mbar_arrive(empty_raw + g % RS);
        }
        if (stamp) ts[6] = clock64();
      }
      unsigned int my_changed_all = my_changed;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) my_changed_all += __shfl_xor_sync(0xffffffffu, my_changed_all, o);
      unsigned int w2 = full ? 0u : my_changed, w3 = my_rechecked;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        w2 += __shfl_xor_sync(0xffffffffu, w2, o);
        w3 += __shfl_xor_sync(0xffffffffu, w3, o);
      }
      if (lane == 0 && w2) atomicAdd(&st->changed, (unsigned long long)w2);
      if (lane == 0 && my_changed_all) atomicAdd(&s_pass_changes, my_changed_all);
      if (lane == 0 && w3) atomicAdd(&st->rechecked, (unsigned long long)w3);
      __threadfence_block();
      __syncwarp();
      if (lane == 0) atomicAdd(s_qn + 1, 1u);  // this epilogue warp has queued everything of the pass
    }
    // ===================== tail =====================
    tc_fence_before();
    __syncthreads();  // every role done with this pass: the CTA's Δ is complete in s_acc
    if (tid == 0 && pass_tiles > 0) {  // the next pass is heavy if this one changed > 1/256 of the CTA's points
      s_heavy = KM_HEAVY_PASSES && !no_sums && !x64p && s_pass_changes * (unsigned int)KM_HEAVY_DIV > (unsigned int)pass_tiles * kTileRows ? 1 : 0;
      s_pass_changes = 0u;
    }
    if (pst && it < 256) atomicMax(pst + it * 8 + 1, globaltimer());
    if (pst && (it == 100 || it == 101 || it == 150))
      a.dbg_times[6144 + (it == 100 ? 0 : it == 101 ? 300 : 600) + blockIdx.x * 2 + 1] = (long long)globaltimer();
    // Run-ahead (resident, not the final pass of an exhausted run): while the other warps run the
    // tail below (Δ flush, grid barrier, finish, next B operand), the transform groups convert the
    // next pass's first AS tiles (already prefetched) into the A buffers and — unless the next pass
    // is heavy (its epilogue, not the transform, releases the raw slots) — the producer streams
    // the next tiles into the slots this frees: the HBM stream and the transform no longer stop
    // for the tail.  Only tile data moves ahead; nothing depends on C.
    __syncthreads();  // s_heavy of the next pass, visible to every role
    const bool ra = KM_RUN_AHEAD && resident && !exhausted && my_tiles > 0;
    const bool hv_next = s_heavy != 0;
    const bool ra_role = ra && (warp < kTransformWarps || warp == kProducerWarp);
    // tail threads: all of them, or (run-ahead) every warp but the transform groups and the producer
    const int ttid = !ra ? tid : warp < kProducerWarp ? tid - kTransformWarps * 32 : tid - (kTransformWarps + 1) * 32;
    const int tthr = ra ? kTailThreads : kThreadsTC;
    const int twarp = ttid >> 5;
    auto tsync = [&]() {
      if (ra) named_bar_sync(kTailBar, kTailThreads);
      else __syncthreads();
    };
    bool stop = false;
    pre_done = 0;
    if (ra_role) {
      const int gn = g0 + pass_tiles;        // first tile of the next pass
      // transformed ahead: tiles the producer has issued or issues now (heavy next pass: no slot is
      // released before its epilogue, so only the npre prefetched tiles)
      const int pre_n = min(AS, hv_next ? npre : my_tiles);
      if (warp == kProducerWarp) {
        if (lane == 0 && !hv_next) {  // refill the slots the run-ahead transform releases
          const int upto = min(npre + pre_n, my_tiles);
          for (int j = issued; j < upto; ++j) issue(gn + j, j);
          issued = max(issued, upto);
        }
      } else {
        for (int j = ((tg - gn) % kTransformGroups + kTransformGroups) % kTransformGroups; j < pre_n;
             j += kTransformGroups)
          transform_tile(gn + j, j, hv_next);
      }
      pre_done = pre_n;
    } else {
      double* s_stage = reinterpret_cast<double*>(sm + S.off_raw);
      const int stage_cap = (int)(RS * S.raw_stride / 8);
      {
        // queue entries the recheck warp had not reached when the pass ended: thread per point
        const unsigned int qn = min(s_qn[0], (unsigned int)QCAP);
        for (unsigned int q = s_qn[2] + ttid; q < qn; q += tthr) redecide(q, s_q[q]);
        tsync();
        if (PD) {  // the epilogue warps' private Δ into the CTA's accumulator (and cleared for the next pass)
          for (int i = ttid; i < nacc; i += tthr) {
            unsigned long long v = 0ull;
  #pragma unroll 4
            for (int w = 0; w < kEpiWarps; ++w) {
              v += s_pacc[w * PST + i];
              s_pacc[w * PST + i] = 0ull;
            }
            s_acc[i] += v;
          }
          tsync();
        }
        if (ttid == 0) {
          s_qn[0] = 0u;
          s_qn[1] = 0u;
          s_qn[2] = 0u;
        }
        if (pst && it < 256) atomicMax(pst + it * 8 + 2, globaltimer());
      }
      if (!resident) {
        for (int i = ttid; i < nacc; i += tthr) {  // one flush of the CTA's Δ
          const unsigned long long v = s_acc[i];
          if (v) atomicAdd(a.part + i, v);
        }
        if (a.fuse_finish) {
          // the last CTA to arrive runs the finish of this iteration (no separate launch)
          __shared__ int s_last;
          __threadfence();
          tsync();
          if (ttid == 0) s_last = atomicAdd(a.cta_done, 1u) == gridDim.x - 1;
          tsync();
          if (s_last) {
            __threadfence();
            finish_block(a.fin, s_stage, stage_cap);
            if (ttid == 0) *a.cta_done = 0u;
          }
        }
        break;
      }
      // ---- resident: Δ → the pass's global delta buffer, grid barrier ----
      // Three delta buffers rotate: pass it accumulates into dlt[it % 3]; before arriving, CTA 0
      // clears dlt[(it + 1) % 3] — last read in the finish of pass it − 2, which every CTA completed
      // before it arrived at barrier it − 1 — so no CTA ever waits for the others to finish reading.
      unsigned long long* dlt = a.dlt + (size_t)(it % 3) * nacc;
      for (int i = ttid; i < nacc; i += tthr) {
        const unsigned long long v = s_acc[i];
        if (v) atomicAdd(dlt + i, v);
        s_acc[i] = 0ull;
      }
      if (blockIdx.x == 0) {
        unsigned long long* nxt = a.dlt + (size_t)((it + 1) % 3) * nacc;
        for (int i = ttid; i < nacc; i += tthr) nxt[i] = 0ull;
      }
      // grid barrier (the cooperative-groups pattern): the CTA's writes are ordered before thread
      // 0's gpu-scope fence by the CTA barrier, so one fence per CTA (not one per thread) releases them
      tsync();
      if (pst && it < 256) atomicMax(pst + it * 8 + 3, globaltimer());
      if (ttid == 0) {
        __threadfence();
        atomicAdd(a.grid_sync, 1u);
        grid_spin(a.grid_sync, (unsigned int)(it + 1) * gridDim.x);
      }
      tsync();
      if (pst && it < 256) atomicMax(pst + it * 8 + 4, globaltimer());  // (tuning: barrier passed)
      if (a.xch_peers != nullptr) {
        // ---- row-sharded multi-GPU: exchange this iteration's Δ with every rank over NVLink ----
        // CTA 0 pushes the rank's complete Δ (the local grid barrier has passed) into slot
        // t_upd & 1, row `rank`, of every rank's buffer, then releases a sequence flag there; every
        // CTA of every rank waits for all `world` flags and adds the world rows (exact integers, the
        // same sum on every rank).  Slots alternate: a rank can be at most one exchange ahead (it
        // needs this rank's next flag to pass the next exchange), so a slot is never overwritten
        // while it is being read.
        const int W = a.world;
        const size_t slot_words = (size_t)W * nacc;
        const int slot = t_upd & 1;
        const unsigned long long seq = ((unsigned long long)a.epoch << 32) | (unsigned long long)(unsigned)(t_upd + 1);
        if (blockIdx.x == 0) {
          const bool add_local_sums = it == 0 && a.skip_first;
          for (int pr = 0; pr < W; ++pr) {
            unsigned long long* dst = a.xch_peers[pr] + slot * slot_words + (size_t)a.rank * nacc;
            for (int i = ttid; i < nacc; i += tthr)
              dst[i] = __ldcg(dlt + i) + (add_local_sums ? a.fin.tot[i] : 0ull);
          }
          __threadfence_system();
          tsync();
          if (ttid < W) {
            unsigned long long* flag = a.xch_peers[ttid] + 2 * slot_words + slot * W + a.rank;
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(seq) : "memory");
          }
        }
        if (ttid < W) {  // bounded wait (a rank that never arrives traps instead of hanging the GPU)
          const unsigned long long* flag = a.xch_local + 2 * slot_words + slot * W + ttid;
          const long long t0 = clock64();
          for (;;) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
            if (v >= seq) break;
            if (clock64() - t0 > (1ll << 35)) __trap();
          }
        }
        tsync();
        const unsigned long long* rows = a.xch_local + slot * slot_words;
        for (int i = ttid; i < nacc; i += tthr) {
          unsigned long long d = 0;
          for (int r = 0; r < W; ++r) d += __ldcg(rows + (size_t)r * nacc + i);
          const unsigned long long v = s_tot[i] + d;
          s_tot[i] = v;
          if (blockIdx.x == 0) a.fin.tot[i] = v;  // published for the host (repair, counts)
        }
      } else {
        // running totals of the current labels, per CTA: S_t = S_{t−1} + Δ_t (exact int64)
        for (int i = ttid; i < nacc; i += tthr) {
          const unsigned long long v = s_tot[i] + __ldcg(dlt + i);
          s_tot[i] = v;
          if (blockIdx.x == 0) a.fin.tot[i] = v;  // published for the host (repair, counts)
        }
      }
      tsync();
      const unsigned long long* tot = s_tot;
      // ---- resident finish (every CTA; CTA 0 publishes) — engine._finish_update / converged ----
      const bool pub = blockIdx.x == 0;
      if (pub && ttid == 0 && pass_tiles > 0) st->passes += 1;
      if (exhausted) {
        // the final assign pass of an exhausted run: counts = bincount(L_T), C_T unchanged
        if (pub) {
          for (int cc = ttid; cc < k; cc += tthr) a.fin.model_counts[cc] = (long long)tot[km + cc];
          if (ttid == 0) st->done = 1;
        }
        stop = true;
      } else {
        double* Cn = s_cbuf + (cb ^ 1) * km;
        // warp per centre, lane per feature: C_{t+1} = S/N, the congruence terms, ‖fl32(c)‖² and the
        // centre's two B-operand rows in one pass (no per-centre serial loops on the critical path)
        __shared__ float s_wmax[32];
        __shared__ int s_wflags[32];  // bit 0: some cluster empty, bit 1: some centre moved
        const int hw = 8 * ((m + 1 + 7) / 8);
        float wmax = 0.f;
        int wflags = 0;
        for (int c = twarp; c < k; c += tthr / 32) {
          const long long nc = (long long)tot[km + c];
          const bool fv = lane < m;
          const long long sv = fv ? (long long)tot[(size_t)c * m + lane] : 0ll;
          // empty clusters get a placeholder; every one is re-seeded by the host repair
          const double v = (fv && nc > 0) ? __ddiv_rn(__dmul_rn((double)sv, a.fin.inv_scale), (double)nc) : 0.0;
          const double vo = fv ? C[(size_t)c * m + lane] : 0.0;
          if (fv) Cn[(size_t)c * m + lane] = v;
          if (pub) {
            if (fv) {
              a.fin.prev[(size_t)c * m + lane] = vo;
              a.fin.cur[(size_t)c * m + lane] = v;
            }
            if (lane == 0) a.fin.model_counts[c] = nc;
          }
          // congruence (engine.converged): sqrt(Σ_f (prev − next)², features ascending) ≤ tol
          const double dd = fv ? __dmul_rn(__dsub_rn(vo, v), __dsub_rn(vo, v)) : 0.0;
          bool moved;
          if (tol == 0.0) {
            moved = __any_sync(0xffffffffu, dd != 0.0);  // a sum of non-negative terms is 0 iff every term is
          } else {
            double acc = 0.0;
            for (int f = 0; f < m; ++f) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, dd, f));
            moved = !(sqrt(acc) <= tol);
          }
          wflags |= (nc == 0 ? 1 : 0) | (moved ? 2 : 0);
          // filter operand: ‖fl32(c)‖² (fp64, exact squares, fixed tree order), max ‖c‖ rounded up
          const double q = fv ? (double)__double2float_rn(v) : 0.0;
          double cn2 = q * q;
  #pragma unroll
          for (int o = 16; o > 0; o >>= 1) cn2 += __shfl_xor_sync(0xffffffffu, cn2, o);
          wmax = fmaxf(wmax, __double2float_ru(sqrt(cn2) * (1.0 + 1e-12)));
  #pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = lane + 32 * h;
            const int f = col < hw ? col : col - hw;
            const double vf = __shfl_sync(0xffffffffu, v, f < 32 ? f : 0);
            float w = 0.f;
            if (col < 2 * hw) {
              if (f < m) w = -2.0f * __double2float_rn(vf) * pre;
              else if (f == m) w = __double2float_rn(cn2 * (double)pre * (double)pre);
            }
            const __half wh = __float2half_rn(w);
            const __half wl = __float2half_rn(w - __half2float(wh));
            *reinterpret_cast<unsigned short*>(s_w + sw128(c, col >> 3) + (col & 7) * 2) =
                (col < 2 * hw) ? __half_as_ushort(wh) : (unsigned short)0;
            *reinterpret_cast<unsigned short*>(s_w + sw128(KP + c, col >> 3) + (col & 7) * 2) =
                (col < hw) ? __half_as_ushort(wl) : (unsigned short)0;
          }
        }
        fence_proxy_async();  // B-operand rows → visible to the tensor core after the barrier
        if (lane == 0) {
          s_wmax[twarp] = wmax;
          s_wflags[twarp] = wflags;
        }
        tsync();
        if (pst && it < 256) atomicMax(pst + it * 8 + 5, globaltimer());
        int flags = 0;
        float cmx = 0.f;
        for (int w = 0; w < tthr / 32; ++w) {
          flags |= s_wflags[w];
          cmx = fmaxf(cmx, s_wmax[w]);
        }
        ++t_upd;
        if (pub && ttid == 0) st->t = t_upd;
        if (flags & 1) {
          if (pub && ttid == 0) {
            int ne = 0;
            for (int c = 0; c < k; ++c) ne += (tot[km + c] == 0ull);
            st->n_empty = ne;
            st->need_host = 1;
          }
          stop = true;
        } else if (!(flags & 2) && !(KM_DBG_FLAGS & 64)) {  // (dbg 64: timing experiments never converge)
          if (pub && ttid == 0) {
            st->n_empty = 0;
            st->converged = 1;
            st->done = 1;
          }
          stop = true;
        } else {
          if (t_upd >= max_iters) {  // reference: one more assign pass, then return
            exhausted = true;
            if (pub && ttid == 0) st->exhausted = 1;
          }
          if (ttid == 0) s_cmax[0] = cmx;
          cb ^= 1;
          full = false;
        }
        if (pst && it < 256) atomicMax(pst + it * 8 + 6, globaltimer());
      }
      if (ra && ttid == 0) {  // the loop state for the run-ahead warps (they skipped the finish)
        s_tail[0] = stop ? 1 : 0;
        s_tail[1] = exhausted ? 1 : 0;
        s_tail[2] = t_upd;
        s_tail[3] = cb;
        s_tail[4] = full ? 1 : 0;
      }
    }
    __syncthreads();
    if (ra_role) {
      stop = s_tail[0] != 0;
      exhausted = s_tail[1] != 0;
      t_upd = s_tail[2];
      cb = s_tail[3];
      full = s_tail[4] != 0;
    }
    if (pst && it < 256) atomicMax(pst + it * 8 + 7, globaltimer());
    if (stop) break;
    g0 += pass_tiles;
  }
  // ---- teardown ----
  if (resident && warp == kProducerWarp && lane == 0) {
    // the prefetched tiles of the pass that does not run: let their copies land before exit
    // (npre, plus the tiles issued ahead in the last tail: only each slot's latest tile — an earlier
    // occupant's phase completed before its slot was reused, and its parity would alias)
    for (int j = max(0, issued - RS); j < issued; ++j) {
      const int g = g0 + last_pass_tiles + j;
      mbar_wait(full_raw + g % RS, (g / RS) & 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, TM::alloc);
  }
}

template <int MT, int KP, bool PRE, bool X64>
inline int launch_t(const TcArgs& a, int num_sms, size_t smem_optin, cudaStream_t stream, cudaError_t* ce, char* msg,
                    size_t len) {
  auto kern = lloyd_pass_tc_kernel<MT, KP, PRE, X64>;
  constexpr int MP = MT > 0 ? MT : -MT;
  // per-instantiation launch facts, queried once (a launch is otherwise one cudaLaunchKernelEx):
  // static smem, and the largest dynamic smem size already granted to the function
  static size_t static_smem = SIZE_MAX, granted = 0;
  cudaError_t c;
  if (static_smem == SIZE_MAX) {
    cudaFuncAttributes fa{};
    c = cudaFuncGetAttributes(&fa, kern);
    if (c != cudaSuccess) { *ce = c; snprintf(msg, len, "cudaFuncGetAttributes(tc)"); return 1; }
    c = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (c != cudaSuccess) { *ce = c; snprintf(msg, len, "cudaFuncSetAttribute(tc carveout)"); return 1; }
    static_smem = fa.sharedSizeBytes;
  }
  const size_t smem = TcSmem<MP, KP>(a.m, a.resident ? a.k : 0).total;
  if (smem + static_smem > smem_optin) {
    snprintf(msg, len, "tensor-core pass needs %zu B of shared memory (max %zu)", smem + static_smem, smem_optin);
    return a.resident ? 3 : 2;
  }
  if (smem > granted) {
    c = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (c != cudaSuccess) { *ce = c; snprintf(msg, len, "cudaFuncSetAttribute(tc smem)"); return 1; }
    granted = smem;
  }
  // one CTA of kThreadsTC threads with ≤ 227 KB of shared memory per SM: fits whenever the
  // shared-memory check above passes (the register budget is fixed by __launch_bounds__)
  const int64_t ntiles = (a.n + TcStages<MP, KP>::TR - 1) / TcStages<MP, KP>::TR;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms));  // one persistent CTA/SM
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(tc_threads<MT, KP, X64>());
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // resident loop: grid barrier needs every CTA co-resident
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.resident ? 1 : 0;
  c = cudaLaunchKernelEx(&cfg, kern, a);
  if (c != cudaSuccess) { *ce = c; snprintf(msg, len, "lloyd_pass_tc_kernel launch"); return 1; }
  return 0;
}

}  // namespace tc
}  // namespace km
