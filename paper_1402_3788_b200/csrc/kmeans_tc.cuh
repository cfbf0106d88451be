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
// Points whose label the filter cannot certify are queued and re-decided by
// recheck_kernel (the reference's exact fp64 recurrence over all centres), so
// the rare slow path never stalls the pipelined hot loop.
//
// Warp roles (persistent CTA, one per SM), pipelined over 128-point tiles:
//   warps 0-7  : transform   two groups, alternate tiles: raw tile → fp16 [hi|lo] A operand
//   warps 8-15 : epilogue    two groups, alternate tiles: TMEM scores → top-2 →
//                            certify → Δ update (thread = point = TMEM lane)
//   warp 16    : TMA producer (cp.async.bulk 1-D copies of raw 4·m-byte rows)
//   warp 17    : TMEM allocator + single-thread MMA issuer
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>

#include "kmeans_tc.h"

namespace km {
namespace tc {

constexpr int kTransformGroups = 2;                // transform warpgroups (alternate tiles)
constexpr int kTransformWarps = 4 * kTransformGroups;
constexpr int kEpiGroups = 2;                      // epilogue warpgroups (alternate tiles)
constexpr int kEpiWarps = 4 * kEpiGroups;
constexpr int kProducerWarp = kTransformWarps + kEpiWarps;  // TMA producer
constexpr int kMmaWarp = kProducerWarp + 1;                 // TMEM allocator + MMA issuer
constexpr int kThreadsTC = (kMmaWarp + 1) * 32;
constexpr int kQueueCap = 1024;                    // per-CTA staging of uncertified points (smem)
// ring depths: raw tiles in flight (TMA → transform) and A operand buffers (transform → MMA);
// shallower for the widest shapes so the CTA fits in 227 KB of shared memory
template <int MP, int KP>
struct TcStages {
  static constexpr int raw = (MP <= 23 && KP <= 32) ? 6 : 4;
  static constexpr int a = (MP <= 23 && KP <= 32) ? 6 : 4;
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
//   KM_WAIT_MODE 0: mbarrier.try_wait (HW suspend, default time limit)
//   KM_WAIT_MODE 1: mbarrier.test_wait polling
//   KM_WAIT_MODE 2: mbarrier.try_wait with a short suspend-time hint
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if KM_WAIT_MODE == 1
  while (!mbar_test(bar, parity)) {
  }
#elif KM_WAIT_MODE == 2
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(64)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
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

template <int KP>
struct TcTmem {
  static constexpr int NS = KP <= 32 ? 8 : KP <= 64 ? 4 : 2;  // TMEM score buffers (2KP columns each)
  static constexpr uint32_t cols = NS * 2 * KP;
  static constexpr uint32_t alloc = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
};

// smem carve-up (1 KiB aligned sections; the raw ring depends on the runtime m)
template <int MP, int KP>
struct TcSmem {
  static constexpr int RS = TcStages<MP, KP>::raw, AS = TcStages<MP, KP>::a;
  uint32_t raw_stride, off_raw = 0, off_a, off_w, off_acc, off_q, off_bar, total;
  __host__ __device__ explicit TcSmem(int m) {
    // + 256 B slack: the transform reads MP ≥ m floats per row without bounds branches
    raw_stride = ((uint32_t)kTile * m * 4 + 256 + 1023) & ~1023u;
    off_a = RS * raw_stride;                 // [AS][128 rows × 128 B]
    off_w = off_a + AS * kTile * 128;          // [2KP rows × 128 B]
    off_acc = off_w + 2 * KP * 128;                  // [KP·(MP+1) + KP] int64 Δ accumulators
    off_q = off_acc + ((KP * (MP + 1) + KP) * 8 + 1023) / 1024 * 1024;  // [kQueueCap] int64 rows + counter
    off_bar = off_q + kQueueCap * 8 + 1024;
    total = off_bar + 1024 + 1024;                   // barriers + 1 KiB alignment slack
  }
};

// MT > 0: exact feature count m = MT (compile-time); MT < 0: runtime m ≤ −MT.
// PRE: multiply x by the power-of-two prescale (off when the data range is fp16-safe as is).
template <int MT, int KP, bool PRE>
__global__ void __launch_bounds__(kThreadsTC, 1) lloyd_pass_tc_kernel(TcArgs a) {
  static_assert(kThreadsTC == 576, "warp-role layout");
  constexpr int MP = MT > 0 ? MT : -MT;
  if (a.gate && (a.st->done || a.st->need_host)) return;
  using L = TcLayout<MP>;
  using TM = TcTmem<KP>;
  const TcSmem<MP, KP> S(MT > 0 ? MT : a.m);
  constexpr int RS = TcStages<MP, KP>::raw, AS = TcStages<MP, KP>::a;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1 KiB align the carve-up (SW128 atoms must be 1 KiB aligned); pointer arithmetic on the
  // __shared__ array keeps the shared address space (LDS/STS, not generic LD/ST)
  unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* raw = reinterpret_cast<float*>(sm + S.off_raw);
  unsigned char* s_w = sm + S.off_w;
  unsigned long long* s_acc = reinterpret_cast<unsigned long long*>(sm + S.off_acc);
  long long* s_q = reinterpret_cast<long long*>(sm + S.off_q);
  unsigned int* s_qn = reinterpret_cast<unsigned int*>(sm + S.off_q + kQueueCap * 8);  // [0] count, [1] global base
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + S.off_bar);
  uint64_t* full_raw = bars;                        // [RS] TMA → transform
  uint64_t* empty_raw = full_raw + RS;      // [RS] transform → TMA
  uint64_t* a_full = empty_raw + RS;        // [AS]   transform → MMA
  uint64_t* a_empty = a_full + AS;            // [AS]   MMA commit → transform
  uint64_t* s_full = a_empty + AS;            // [NS]         MMA commit → epilogue
  uint64_t* s_empty = s_full + TM::NS;              // [NS]         epilogue → MMA
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_empty + TM::NS);

  const int m = MT > 0 ? MT : a.m;
  const int k = a.k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  const int my_tiles = (int)((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
  const int nacc = k * m + k;
  if (a.dbg_times != nullptr && tid == 0) {
    a.dbg_times[64 * 8 + (blockIdx.x % 64) * 8 + 7] = clock64();
    a.dbg_times[4096 + blockIdx.x * 4] = (long long)globaltimer();
  }

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
    for (int i = tid; i < AS * kTile * 8; i += nthr)
      *reinterpret_cast<uint4*>(sm + S.off_a + i * 16) = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < nacc; i += nthr) s_acc[i] = 0ull;
    if (tid == 0) s_qn[0] = 0u;
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const float pre = a.pre;

  if (warp == kProducerWarp) {
    // ===================== TMA producer: tile i → raw slot i % RS =====================
    if (lane == 0) {
      for (int i = 0; i < my_tiles; ++i) {
        const int s = i % RS;
        const int u = i / RS;
        if (u > 0) mbar_wait(empty_raw + s, (u - 1) & 1);
        const int64_t t = blockIdx.x + (int64_t)i * gridDim.x;
        const int64_t row0 = t * kTile;
        const int64_t rem = a.n - row0;
        const int rows = rem < kTile ? (int)rem : kTile;
        const uint32_t bytes = ((uint32_t)rows * m * 4u) & ~15u;
        mbar_arrive_expect_tx(full_raw + s, bytes);
        if (bytes) bulk_g2s(reinterpret_cast<unsigned char*>(raw) + s * S.raw_stride, a.x + row0 * m, bytes,
                            full_raw + s);
      }
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      const uint32_t a0 = smem_u32(sm + S.off_a), w0 = smem_u32(s_w);
      constexpr uint32_t idesc = idesc_f16(2 * KP);
      for (int i = 0; i < my_tiles; ++i) {
        const int sa = i % AS, ss = i % TM::NS;
        mbar_wait(a_full + sa, (i / AS) & 1);
        if (i >= TM::NS) mbar_wait(s_empty + ss, ((i / TM::NS) - 1) & 1);
        tc_fence_after();
        const uint32_t ag = a0 + sa * (kTile * 128);
        const uint32_t dcol = tmem + ss * 2 * KP;
#pragma unroll
        for (int ks = 0; ks < L::KSTEPS; ++ks) {
          if (a.dbg_flags & 2) break;
          mma_f16(dcol, make_desc(ag + ks * 32, 16, 1024), make_desc(w0 + ks * 32, 16, 1024), idesc,
                  ks > 0 ? 1u : 0u);
        }
        mma_commit(s_full + ss);   // scores ready
        mma_commit(a_empty + sa);  // A buffer consumed
      }
    }
  } else if (warp < kTransformWarps) {
    // ===================== transform: thread = point; group tg takes tiles i ≡ tg (mod 2) =====================
    const int tg = warp >> 2;
    const int p = tid & 127;
    const uint32_t row_off = (uint32_t)((p >> 3) * 1024 + (p & 7) * 128);  // SW128 geometry of row p
    const int key = p & 7;
    const float* __restrict__ gx = a.x;
    for (int i = tg; i < my_tiles; i += kTransformGroups) {
      const int s = i % RS, sa = i % AS;
      const int64_t t = blockIdx.x + (int64_t)i * gridDim.x;
      const int64_t row0 = t * kTile;
      const int64_t rem = a.n - row0;
      const int rows = rem < kTile ? (int)rem : kTile;
      const bool active = p < rows;
      const bool stamp = a.dbg_times != nullptr && blockIdx.x == 0 && p == 0 && i < 64;
      long long* ts = stamp ? a.dbg_times + (size_t)i * 8 : nullptr;
      if (stamp) ts[0] = clock64();
      mbar_wait(full_raw + s, (i / RS) & 1);
      if (stamp) ts[1] = clock64();
      const float* rs = raw + s * (S.raw_stride / 4);
      float xs[L::HW];
      if (rows == kTile) {  // full tile: branch-free loads (over-reads stay inside the padded slot)
        const float* xr = rs + p * m;
#pragma unroll
        for (int f = 0; f < L::HW; ++f) {
          const float v = (f < MP) ? xr[f] : 0.f;
          xs[f] = (f < m) ? (PRE ? v * pre : v) : 0.f;
        }
      } else {              // ragged last tile: bulk part + ≤ 3 trailing floats from global
        const uint32_t bulk_elems = (((uint32_t)rows * m * 4u) & ~15u) >> 2;
        for (int f = 0; f < L::HW; ++f) {
          float v = 0.f;
          if (f < MP && f < m && active) {
            const uint32_t e = (uint32_t)p * m + f;
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
        const __half2 h2 = __floats2half2_rn(xs[2 * q], xs[2 * q + 1]);
        const float2 hf = __half22float2(h2);
        const __half2 l2 = __floats2half2_rn(xs[2 * q] - hf.x, xs[2 * q + 1] - hf.y);
        hw[q] = *reinterpret_cast<const uint32_t*>(&h2);
        lw[q] = *reinterpret_cast<const uint32_t*>(&l2);
      }
      // raw slot consumed (every loaded value has been used, so no LDS is still in flight):
      // the TMA producer may refill it
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_raw + s);
      if (stamp) ts[7] = clock64();
      if (i >= AS) mbar_wait(a_empty + sa, ((i / AS) - 1) & 1);
      if (stamp) ts[2] = clock64();
      unsigned char* s_a = sm + S.off_a + sa * (kTile * 128);
#pragma unroll
      for (int q = 0; q < L::HW / 8; ++q) {
        *reinterpret_cast<uint4*>(s_a + row_off + ((uint32_t)(q ^ key) << 4)) =
            make_uint4(hw[4 * q], hw[4 * q + 1], hw[4 * q + 2], hw[4 * q + 3]);
        *reinterpret_cast<uint4*>(s_a + row_off + ((uint32_t)((q + L::HW / 8) ^ key) << 4)) =
            make_uint4(lw[4 * q], lw[4 * q + 1], lw[4 * q + 2], lw[4 * q + 3]);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full + sa);
      if (stamp) ts[3] = clock64();
    }
  } else {
    // ===================== epilogue groups: thread = point = TMEM lane; group e takes tiles i ≡ e (mod 2) =====================
    const int ew = warp - kTransformWarps;          // 0..7
    const int e = ew >> 2;
    const int p = ((ew & 3) << 5) | lane;          // TMEM lane of this thread
    const uint32_t lane_base = (uint32_t)((ew & 3) * 32) << 16;
    const float scale_f = a.scale_f;
    // certified bound with the dataset's max ‖x‖ (per launch constant, prescaled units)
    const float tt = (a.xnorm_max + a.cmax[0]) * pre;
    const float E2 = 2.f * __fmaf_rn(a.err_coef * tt, tt, a.err_floor);
    const float inv_pre2 = 1.0f / (pre * pre);
    const double scale_d = a.scale_d;
    const bool use_dscale = a.use_dscale != 0, exact_only = a.exact_only != 0, full = a.full != 0;
    unsigned int my_changed = 0;
    auto prev_label = [&](int i) -> int {  // previous label of this thread's point in tile i (or -1)
      if (full || i >= my_tiles) return -1;
      const int64_t r = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + p;
      return r < a.n ? __ldg(a.labels + r) : -1;
    };
    int old_next = prev_label(e);
    for (int i = e; i < my_tiles; i += kEpiGroups) {
      const int ss = i % TM::NS;
      const int64_t t = blockIdx.x + (int64_t)i * gridDim.x;
      const int64_t row0 = t * kTile;
      const int64_t rem = a.n - row0;
      const int rows = rem < kTile ? (int)rem : kTile;
      const bool active = p < rows;
      const int old = old_next;
      old_next = prev_label(i + kEpiGroups);  // prefetch one tile ahead (global latency off the critical path)
      const bool stamp = a.dbg_times != nullptr && blockIdx.x == 0 && p == 0 && i < 64;
      long long* ts = stamp ? a.dbg_times + (size_t)i * 8 : nullptr;
      if (stamp) ts[4] = clock64();
      mbar_wait(s_full + ss, (i / TM::NS) & 1);
      if (stamp) ts[5] = clock64();
      tc_fence_after();
      // top-2 over the scores: per 16-column chunk a 4-level tree, then a running merge.
      // (The filter's argmin tie order is irrelevant: a tie is never certified.)
      float best = __int_as_float(0x7f800000), min2 = best;
      int bi = 0;
#pragma unroll
      for (int c0 = 0; c0 < KP; c0 += 16) {
        uint32_t r0[16], r1[16];
        tmem_ld16(tmem + lane_base + ss * 2 * KP + c0, r0);
        tmem_ld16(tmem + lane_base + ss * 2 * KP + KP + c0, r1);
        tmem_ld_wait();
        float v[16], s2[16];
        int ix[16];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {  // padded centres (c ≥ k) score +65504: never best or runner-up
          v[jj] = __uint_as_float(r0[jj]) + __uint_as_float(r1[jj]);
          s2[jj] = __int_as_float(0x7f800000);
          ix[jj] = c0 + jj;
        }
        if (a.dbg_scores != nullptr && active) {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            if (c0 + jj < k) a.dbg_scores[(row0 + p) * k + c0 + jj] = v[jj] * inv_pre2;
        }
#pragma unroll
        for (int w = 1; w < 16; w <<= 1) {
#pragma unroll
          for (int jj = 0; jj < 16; jj += 2 * w) {
            const bool rb = v[jj + w] < v[jj];
            const float lo = rb ? v[jj + w] : v[jj], hi = rb ? v[jj] : v[jj + w];
            s2[jj] = fminf(hi, fminf(s2[jj], s2[jj + w]));
            ix[jj] = rb ? ix[jj + w] : ix[jj];
            v[jj] = lo;
          }
        }
        const bool rb = v[0] < best;
        min2 = fminf(rb ? best : v[0], fminf(min2, s2[0]));
        bi = rb ? ix[0] : bi;
        best = rb ? v[0] : best;
      }
      tc_fence_before();  // TMEM reads ordered before the MMA reuses this buffer
      __syncwarp();
      if (lane == 0) mbar_arrive(s_empty + ss);
      const bool certified = !exact_only && (min2 > best + E2);
      if (active && !certified) {
        // defer: recheck_kernel re-decides this point exactly and applies its update
        const unsigned int slot = atomicAdd(s_qn, 1u);
        if (slot < kQueueCap) {
          s_q[slot] = ((row0 + p) << 24) | (long long)(old + 1);  // row | previous label (+1; 0 = none)
        } else {  // CTA staging full: straight to the global queue
          a.recheck_rows[atomicAdd(a.recheck_count, 1u)] = row0 + p;
        }
      } else if (active && bi != old) {
        // --- exact incremental update of the per-cluster fixed-point sums
        ++my_changed;
        a.labels[row0 + p] = bi;
        const float* xr = a.x + (row0 + p) * m;  // just streamed: L2 hit
        for (int f = 0; f < m; ++f) {
          const float xv = __ldg(xr + f);
          const long long v = use_dscale ? __double2ll_rn(__dmul_rn((double)xv, scale_d))
                                         : __float2ll_rn(__fmul_rn(xv, scale_f));
          smem_add64(s_acc + (size_t)bi * m + f, (unsigned long long)v);
          if (old >= 0) smem_add64(s_acc + (size_t)old * m + f, (unsigned long long)(-v));
        }
        smem_add64(s_acc + (size_t)k * m + bi, 1ull);
        if (old >= 0) smem_add64(s_acc + (size_t)k * m + old, ~0ull);
      }
      if (stamp) ts[6] = clock64();
    }
    unsigned int w2 = my_changed;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w2 += __shfl_xor_sync(0xffffffffu, w2, o);
    if (lane == 0 && w2) atomicAdd(&a.st->changed, (unsigned long long)w2);
  }
  // ===================== tail (all warps) =====================
  long long* tstamp = (a.dbg_times != nullptr && tid == 0) ? a.dbg_times + 64 * 8 + (blockIdx.x % 64) * 8 : nullptr;
  if (tstamp) tstamp[0] = clock64();
  if (a.dbg_times != nullptr && tid == 0) a.dbg_times[4096 + blockIdx.x * 4 + 1] = (long long)globaltimer();
  tc_fence_before();
  __syncthreads();  // every role done: Δ atomics and the CTA's recheck queue are complete
  if (tstamp) tstamp[1] = clock64();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, TM::alloc);
  }
  // the raw ring is free now: stage the fp64 centres there for the recheck (and the finish)
  double* s_stage = reinterpret_cast<double*>(sm + S.off_raw);
  const int stage_cap = (int)(RS * S.raw_stride / 8);
  const unsigned int qn = min(s_qn[0], (unsigned int)kQueueCap);
  const bool c_staged = k * m <= stage_cap;
  if (qn && c_staged) {
    for (int i = tid; i < k * m; i += kThreadsTC) s_stage[i] = a.c64[i];
    __syncthreads();
  }
  long long* rst = (a.dbg_times != nullptr && lane == 0 && warp == 0) ? a.dbg_times + 2048 + (blockIdx.x % 64) * 8 : nullptr;
  if (rst) rst[0] = clock64();
  {
    // exact re-decision of this CTA's uncertified points (warp per point), Δ into s_acc
    const bool full = a.full != 0;
    const double* C = c_staged ? s_stage : a.c64;
    // batches of 4 points per warp: their x rows (one feature per lane) are fetched together
    for (unsigned int q0 = warp * 4; q0 < qn; q0 += (kThreadsTC / 32) * 4) {
      long long ent[4];
      float xb[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        ent[j] = (q0 + j < qn) ? s_q[q0 + j] : -1;
        xb[j] = (ent[j] >= 0 && lane < m) ? __ldg(a.x + (ent[j] >> 24) * m + lane) : 0.f;
      }
      if (rst && q0 == 0) { rst[1] = clock64() + (long long)(xb[0] + xb[1] + xb[2] + xb[3] == 12345.f); }
      int lb[4];
      exact_label_warp_batch<MP, 4>(xb, m, k, C, lb);
      if (rst && q0 == 0) { rst[2] = clock64() + (lb[0] + lb[1] + lb[2] + lb[3] == 12345); }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (ent[j] < 0) continue;
        const long long row = ent[j] >> 24;
        const float xl = xb[j];
        const int bl = lb[j];
        const int old = full ? -1 : (int)(ent[j] & 0xffffff) - 1;
        if (bl != old) {
          if (lane == 0) {
            a.labels[row] = bl;
            smem_add64(s_acc + (size_t)k * m + bl, 1ull);
            if (old >= 0) smem_add64(s_acc + (size_t)k * m + old, ~0ull);
            if (!full) atomicAdd(&a.st->changed, 1ull);
          }
          if (lane < m) {
            const long long v = a.use_dscale ? __double2ll_rn(__dmul_rn((double)xl, a.scale_d))
                                             : __float2ll_rn(__fmul_rn(xl, a.scale_f));
            smem_add64(s_acc + (size_t)bl * m + lane, (unsigned long long)v);
            if (old >= 0) smem_add64(s_acc + (size_t)old * m + lane, (unsigned long long)(-v));
          }
        }
      }
    }
    if (rst) rst[3] = clock64();
    if (tid == 0 && qn) atomicAdd(&a.st->rechecked, (unsigned long long)qn);
    if (tstamp) tstamp[5] = qn;
  }
  __syncthreads();
  if (tstamp) tstamp[2] = clock64();
  if (a.dbg_times != nullptr && tid == 0) a.dbg_times[4096 + blockIdx.x * 4 + 2] = (long long)globaltimer();
  for (int i = tid; i < nacc; i += kThreadsTC) {  // one flush of the CTA's Δ
    const unsigned long long v = s_acc[i];
    if (v) atomicAdd(a.part + i, v);
  }
  if (a.fuse_finish) {
    // the last CTA to arrive runs the finish of this iteration (no separate launch)
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(a.cta_done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (tstamp) tstamp[3] = clock64();
    if (s_last) {
      __threadfence();
      finish_block(a.fin, s_stage, stage_cap, tstamp ? tstamp + 8 * 64 : nullptr);
      if (tid == 0) *a.cta_done = 0u;
      if (tstamp) { tstamp[4] = clock64(); tstamp[6] = 1; }
    }
  }
  if (a.dbg_times != nullptr && tid == 0) a.dbg_times[4096 + blockIdx.x * 4 + 3] = (long long)globaltimer();
}

template <int MT, int KP, bool PRE>
inline int launch_t(const TcArgs& a, int num_sms, size_t smem_optin, cudaStream_t stream, cudaError_t* ce, char* msg,
             size_t len) {
  auto kern = lloyd_pass_tc_kernel<MT, KP, PRE>;
  constexpr int MP = MT > 0 ? MT : -MT;
  const size_t smem = TcSmem<MP, KP>(a.m).total;
  if (smem > smem_optin) {
    snprintf(msg, len, "tensor-core pass needs %zu B of shared memory (max %zu)", smem, smem_optin);
    return 2;
  }
  cudaError_t c = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (c != cudaSuccess) { *ce = c; snprintf(msg, len, "cudaFuncSetAttribute(tc smem)"); return 1; }
  c = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (c != cudaSuccess) { *ce = c; snprintf(msg, len, "cudaFuncSetAttribute(tc carveout)"); return 1; }
  int per_sm = 0;
  c = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreadsTC, smem);
  if (c != cudaSuccess) { *ce = c; snprintf(msg, len, "occupancy(tc)"); return 1; }
  if (per_sm < 1) { snprintf(msg, len, "tensor-core pass does not fit on an SM"); return 2; }
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms));  // one persistent CTA/SM
  kern<<<(unsigned)grid, kThreadsTC, smem, stream>>>(a);
  c = cudaGetLastError();
  if (c != cudaSuccess) { *ce = c; snprintf(msg, len, "lloyd_pass_tc_kernel launch"); return 1; }
  return 0;
}

}  // namespace tc
}  // namespace km
