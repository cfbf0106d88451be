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
// Warp roles (persistent CTA, one per SM):
//   warps 0-7 : two compute warpgroups, ping-pong over tiles; thread = point
//   warp 8    : TMA producer (cp.async.bulk 1-D copies of raw 4·m-byte rows)
//   warp 9    : TMEM allocator + single-thread MMA issuer
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "kmeans_tc.h"

namespace km {
namespace tc {

constexpr int kGroups = 2;                         // compute warpgroups (ping-pong over tiles)
constexpr int kComputeWarps = 4 * kGroups;
constexpr int kProducerWarp = kComputeWarps;       // TMA producer
constexpr int kMmaWarp = kComputeWarps + 1;        // TMEM allocator + MMA issuer
constexpr int kThreadsTC = (kComputeWarps + 2) * 32;
constexpr int kRawStages = 4;

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
__device__ __forceinline__ uint32_t sw128(int r, int q) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + (((q ^ (r & 7)) & 7) << 4));
}


template <int MP>
struct TcLayout {
  static constexpr int HW = 8 * ((MP + 1 + 7) / 8);  // halfs per part (features incl. the ones column)
  static constexpr int KSTEPS = (2 * HW) / 16;       // kind::f16 MMA k-steps (16 halfs = 32 B each)
};

// smem carve-up (1 KiB aligned sections; the raw ring depends on the runtime m)
template <int MP, int KP>
struct TcSmem {
  uint32_t raw_stride, off_raw = 0, off_a, off_w, off_acc, off_bar, total;
  __host__ __device__ explicit TcSmem(int m) {
    raw_stride = ((uint32_t)kTile * m * 4 + 1023) & ~1023u;
    off_a = kRawStages * raw_stride;                 // [kGroups][128 rows × 128 B]
    off_w = off_a + kGroups * kTile * 128;           // [2KP rows × 128 B]
    off_acc = off_w + 2 * KP * 128;                  // [KP·(MP+1) + KP] int64 Δ accumulators
    off_bar = off_acc + ((KP * (MP + 1) + KP) * 8 + 1023) / 1024 * 1024;
    total = off_bar + 512 + 1024;                    // barriers + 1 KiB alignment slack
  }
};

template <int MP, int KP>
__global__ void __launch_bounds__(kThreadsTC, 1) lloyd_pass_tc_kernel(TcArgs a) {
  if (a.gate && (a.st->done || a.st->need_host)) return;
  using L = TcLayout<MP>;
  const TcSmem<MP, KP> S(a.m);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1 KiB align the carve-up (SW128 atoms must be 1 KiB aligned); pointer arithmetic on the
  // __shared__ array keeps the shared address space (LDS/STS, not generic LD/ST)
  unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* raw = reinterpret_cast<float*>(sm + S.off_raw);
  unsigned char* s_w = sm + S.off_w;
  unsigned long long* s_acc = reinterpret_cast<unsigned long long*>(sm + S.off_acc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + S.off_bar);
  uint64_t* full_raw = bars;                      // [kRawStages]  TMA → compute
  uint64_t* empty_raw = bars + kRawStages;        // [kRawStages]  compute → TMA
  uint64_t* op_full = bars + 2 * kRawStages;      // [kGroups] A operand written (compute → MMA)
  uint64_t* s_full = op_full + kGroups;           // [kGroups] scores in TMEM   (MMA → compute)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_full + kGroups);

  const int m = a.m, k = a.k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  const int my_tiles = (int)((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
  constexpr uint32_t kCols = kGroups * 2 * KP;  // S[g] = columns [2KP·g, 2KP·(g+1))
  constexpr uint32_t kTmemCols = kCols <= 32 ? 32 : kCols <= 64 ? 64 : kCols <= 128 ? 128 : kCols <= 256 ? 256 : 512;
  const int nacc = k * m + k;

  // ---- setup ----
  if (tid == 0) {
    for (int s = 0; s < kRawStages; ++s) {
      mbar_init(full_raw + s, 1);
      mbar_init(empty_raw + s, 4);
    }
    for (int g = 0; g < kGroups; ++g) {
      mbar_init(op_full + g, 128);
      mbar_init(s_full + g, 1);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_holder, kTmemCols);
  if (warp < kComputeWarps) {
    // B operand rows (already fp16-split and packed by the prep kernel) → SW128 K-major smem
    for (int i = tid; i < 2 * KP * 8; i += kComputeWarps * 32) {
      const int r = i >> 3, q = i & 7;
      *reinterpret_cast<uint4*>(s_w + sw128(r, q)) = *reinterpret_cast<const uint4*>(a.wop + (size_t)r * 64 + q * 8);
    }
    // A operand planes zeroed once (chunks beyond the used width stay zero)
    for (int i = tid; i < kGroups * kTile * 8; i += kComputeWarps * 32)
      *reinterpret_cast<uint4*>(sm + S.off_a + i * 16) = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < nacc; i += kComputeWarps * 32) s_acc[i] = 0ull;
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == kProducerWarp) {
    // ===================== TMA producer: tile i → raw slot i % kRawStages =====================
    if (lane == 0) {
      for (int i = 0; i < my_tiles; ++i) {
        const int s = i % kRawStages;
        const int u = i / kRawStages;
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
    // ===================== MMA issuer (one thread): assign MMAs for whichever group is ready =====================
    if (lane == 0) {
      const uint32_t a0 = smem_u32(sm + S.off_a), w0 = smem_u32(s_w);
      constexpr uint32_t idesc = idesc_f16(2 * KP);
      int next[kGroups];
#pragma unroll
      for (int g = 0; g < kGroups; ++g) next[g] = g;
      int issued = 0;
      while (issued < my_tiles) {
#pragma unroll
        for (int g = 0; g < kGroups; ++g) {
          const int i = next[g];
          if (i < my_tiles && mbar_test(op_full + g, (i / kGroups) & 1)) {
            tc_fence_after();
            const uint32_t ag = a0 + g * (kTile * 128);
#pragma unroll
            for (int ks = 0; ks < L::KSTEPS; ++ks) {
              if (a.dbg_flags & 2) break;
              mma_f16(tmem + g * 2 * KP, make_desc(ag + ks * 32, 16, 1024), make_desc(w0 + ks * 32, 16, 1024),
                      idesc, ks > 0 ? 1u : 0u);
            }
            mma_commit(s_full + g);
            next[g] += kGroups;
            ++issued;
          }
        }
      }
    }
  } else {
    // ===================== compute warpgroups: thread = point; group g takes tiles i ≡ g (mod 2) =====================
    const int g = warp >> 2;
    const int p = tid & 127;                      // row in tile = TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    unsigned char* s_a = sm + S.off_a + g * (kTile * 128);
    const float pre = a.pre;
    const float cmaxp = a.cmax[0] * pre;
    const float scale_f = a.scale_f, err_coef = a.err_coef, err_floor = a.err_floor, nx_inflate = a.nx_inflate;
    const float inv_pre2 = 1.0f / (pre * pre);
    const double scale_d = a.scale_d;
    const bool use_dscale = a.use_dscale != 0, exact_only = a.exact_only != 0, full = a.full != 0;
    const float* __restrict__ gx = a.x;
    const uint32_t row_off = (uint32_t)((p >> 3) * 1024 + (p & 7) * 128);  // SW128 geometry of row p
    const int key = p & 7;
    unsigned int my_rechecks = 0, my_changed = 0;
    for (int i = g; i < my_tiles; i += kGroups) {
      const int j = i / kGroups;
      const int s = i % kRawStages;
      const int u = i / kRawStages;
      const int64_t t = blockIdx.x + (int64_t)i * gridDim.x;
      const int64_t row0 = t * kTile;
      const int64_t rem = a.n - row0;
      const int rows = rem < kTile ? (int)rem : kTile;
      const bool active = p < rows;
      const bool stamp = a.dbg_times != nullptr && blockIdx.x == 0 && (tid & 127) == 0 && i < 64;
      long long* ts = stamp ? a.dbg_times + (size_t)i * 8 : nullptr;
      if (stamp) ts[0] = clock64();
      // previous label (incremental update); issued early to hide its latency
      const int old = (active && !full) ? __ldg(a.labels + row0 + p) : -1;
      mbar_wait(full_raw + s, u & 1);
      if (stamp) ts[1] = clock64();
      const float* rs = raw + s * (S.raw_stride / 4);
      float x[MP];
      if (rows == kTile) {  // full tile: whole rows inside the bulk copy (12800 B is a multiple of 16)
#pragma unroll
        for (int f = 0; f < MP; ++f) x[f] = (f < m) ? rs[p * m + f] : 0.f;
      } else {              // ragged last tile: bulk part + ≤ 3 trailing floats from global
        const uint32_t bulk_elems = (((uint32_t)rows * m * 4u) & ~15u) >> 2;
#pragma unroll
        for (int f = 0; f < MP; ++f) {
          float v = 0.f;
          if (f < m && active) {
            const uint32_t e = (uint32_t)p * m + f;
            v = (e < bulk_elems) ? rs[e] : __ldg(gx + row0 * m + e);
          }
          x[f] = v;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_raw + s);
      if (stamp) ts[2] = clock64();
      // --- A row: [xh | xl] fp16, prescaled; feature m carries the ‖c‖² term
      float xs[L::HW];
      float nx2 = 0.f;
#pragma unroll
      for (int f = 0; f < L::HW; ++f) {
        float v = (f < MP) ? x[f] * pre : 0.f;
        if (f == m) v = active ? 1.f : 0.f;
        xs[f] = v;
        if (f < MP) nx2 = __fmaf_rn(v, (f == m) ? 0.f : v, nx2);
      }
      uint32_t hw[L::HW / 2], lw[L::HW / 2];
#pragma unroll
      for (int q = 0; q < L::HW / 2; ++q) {
        const __half2 h2 = __floats2half2_rn(xs[2 * q], xs[2 * q + 1]);
        const float2 hf = __half22float2(h2);
        const __half2 l2 = __floats2half2_rn(xs[2 * q] - hf.x, xs[2 * q + 1] - hf.y);
        hw[q] = *reinterpret_cast<const uint32_t*>(&h2);
        lw[q] = *reinterpret_cast<const uint32_t*>(&l2);
      }
      // row layout (halfs): [0, HW) = xh, [HW, 2HW) = xl; 16-byte chunks of 8 halfs
#pragma unroll
      for (int q = 0; q < L::HW / 8; ++q) {
        *reinterpret_cast<uint4*>(s_a + row_off + ((uint32_t)(q ^ key) << 4)) =
            make_uint4(hw[4 * q], hw[4 * q + 1], hw[4 * q + 2], hw[4 * q + 3]);
        *reinterpret_cast<uint4*>(s_a + row_off + ((uint32_t)((q + L::HW / 8) ^ key) << 4)) =
            make_uint4(lw[4 * q], lw[4 * q + 1], lw[4 * q + 2], lw[4 * q + 3]);
      }
      fence_proxy_async();
      mbar_arrive(op_full + g);
      if (stamp) ts[3] = clock64();
      // --- epilogue: scores from TMEM
      mbar_wait(s_full + g, j & 1);
      if (stamp) ts[4] = clock64();
      tc_fence_after();
      float sc[KP];
#pragma unroll
      for (int c0 = 0; c0 < KP; c0 += 16) {
        uint32_t r0[16], r1[16];
        tmem_ld16(tmem + lane_base + g * 2 * KP + c0, r0);
        tmem_ld16(tmem + lane_base + g * 2 * KP + KP + c0, r1);
        tmem_ld_wait();
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) sc[c0 + jj] = __uint_as_float(r0[jj]) + __uint_as_float(r1[jj]);
      }
      tc_fence_before();  // TMEM reads ordered before the next MMA into S[g]
      float best = __int_as_float(0x7f800000), min2 = best;
      int bi = 0;
#pragma unroll
      for (int c = 0; c < KP; ++c) {
        if (c < k) {
          if (a.dbg_scores && active) a.dbg_scores[(row0 + p) * k + c] = sc[c] * inv_pre2;
          const bool lt = sc[c] < best;
          min2 = lt ? best : fminf(min2, sc[c]);
          bi = lt ? c : bi;
          best = lt ? sc[c] : best;
        }
      }
      const float tt = __fmaf_rn(sqrtf(nx2), nx_inflate, cmaxp);
      const float E = __fmaf_rn(err_coef * tt, tt, err_floor);
      const float thr = best + 2.f * E;
      int lab = bi;
      if (active && (exact_only || !(min2 > thr))) {
        // exact re-decision among the candidates (reference recurrence, ascending c, strict <)
        ++my_rechecks;
        double bd = 0.0;
        int bl = -1;
#pragma unroll
        for (int c = 0; c < KP; ++c) {
          if (c < k && (exact_only || sc[c] <= thr)) {
            const double* cc = a.c64 + (size_t)c * m;
            double acc = 0.0;
#pragma unroll
            for (int f = 0; f < MP; ++f) {
              if (f < m) {
                const double d = __dsub_rn((double)x[f], cc[f]);
                acc = __dadd_rn(acc, __dmul_rn(d, d));
              }
            }
            if (bl < 0 || acc < bd) { bd = acc; bl = c; }
          }
        }
        lab = bl;
      }
      // --- exact incremental update of the per-cluster fixed-point sums
      if (active && lab != old) {
        ++my_changed;
        a.labels[row0 + p] = lab;
#pragma unroll
        for (int f = 0; f < MP; ++f) {
          if (f < m) {
            const long long v = use_dscale ? __double2ll_rn(__dmul_rn((double)x[f], scale_d))
                                           : __float2ll_rn(__fmul_rn(x[f], scale_f));
            smem_add64(s_acc + (size_t)lab * m + f, (unsigned long long)v);
            if (old >= 0) smem_add64(s_acc + (size_t)old * m + f, (unsigned long long)(-v));
          }
        }
        smem_add64(s_acc + (size_t)k * m + lab, 1ull);
        if (old >= 0) smem_add64(s_acc + (size_t)k * m + old, ~0ull);
      }
      if (stamp) ts[5] = clock64();
    }
    unsigned int w1 = my_rechecks, w2 = my_changed;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      w1 += __shfl_xor_sync(0xffffffffu, w1, o);
      w2 += __shfl_xor_sync(0xffffffffu, w2, o);
    }
    if (lane == 0 && w1) atomicAdd(&a.st->rechecked, (unsigned long long)w1);
    if (lane == 0 && w2) atomicAdd(&a.st->changed, (unsigned long long)w2);
    // all compute warps done with their atomics → flush the Δ accumulators (one pass per CTA)
    asm volatile("bar.sync 1, %0;" ::"r"(kComputeWarps * 32) : "memory");
    for (int i = tid; i < nacc; i += kComputeWarps * 32) {
      const unsigned long long v = s_acc[i];
      if (v) atomicAdd(a.part + i, v);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

}  // namespace tc
}  // namespace km
