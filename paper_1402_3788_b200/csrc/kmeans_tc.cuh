// kmeans_tc.cuh — tcgen05 (5th-gen tensor core) fused Lloyd pass for sm_100a.
//
// Per 128-point tile, one CTA runs two tensor-core GEMMs whose results never
// leave the SM until the end of the kernel:
//
//  (1) ASSIGN  (kind::tf32, 3×TF32 split, accumulators in TMEM)
//        S[128 × K] = X~[128 × 32] · W~ᵀ[32 × K]
//      X~ row p = (x_p0 … x_p,M−1, 1, 0…)      split into tf32 hi + lo
//      W~ row c = (−2c_0 … −2c_M−1, ‖c‖², 0…)  split into tf32 hi + lo
//      S = Xh·Wh + Xh·Wl + Xl·Wh  (the dropped Xl·Wl term is ≤ 2⁻²² relative)
//      so S_c = ‖c‖² − 2x·c, the argmin key.  The epilogue (thread = point,
//      TMEM lane = point) takes argmin / runner-up, certifies the label with
//      an error bound E_tc·(‖x‖+max‖c‖)² and re-decides uncertified points
//      with the reference's exact fp64 recurrence (see kmeans_kernels.cuh).
//
//  (2) UPDATE  (kind::i8, exact int32 accumulation in TMEM across all tiles)
//        U[8(M+1) × K] += Bytesᵀ[8(M+1) × 128] · Onehot[128 × K]
//      Bytes row p = the 8 little-endian bytes of every int64 fixed-point
//      coordinate round(x_pf·2^F) plus a pseudo-feature f = M with value 1;
//      Onehot[p][c] = (label_p == c).  Unsigned byte sums are exact in int32,
//      and Σ_b U[8f+b][c]·256^b (mod 2^64) is exactly the two's-complement
//      fixed-point sum of feature f over cluster c; the pseudo-feature gives
//      the counts.  The Bytes operand is MN-major (each thread writes its own
//      point's row) and the Onehot operand is K-major (one byte per point).
//      No atomics in the tile loop; one flush per CTA at the end.
//
// Warp roles (persistent CTA, 6 warps):
//   warps 0-3 : transform + epilogue, thread = point of the 128-point tile
//   warp 4    : TMA producer (cp.async.bulk 1-D copies of raw 100-byte rows)
//   warp 5    : TMEM allocator + single-thread MMA issuer
#pragma once
#include <cuda_runtime.h>
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
  static constexpr int KS = ((MP + 1) + 7) / 8;           // tf32 k-steps (8 features each) incl. the ones column
  static constexpr int NB = (8 * (MP + 1) + 127) / 128;   // 128-row M-blocks of the byte operand
};

// smem carve-up (1 KiB aligned sections); the raw ring depends on the runtime m.
// Per compute warpgroup g: X~ hi, X~ lo (K-major SW128), fixed-point bytes
// (MN-major SW128, NB blocks), one-hot (K-major SW128, KP rows).
template <int MP, int KP>
struct TcSmem {
  uint32_t raw_stride, off_raw = 0, off_grp, grp_stride, off_xh, off_xl, off_dig, off_oh, off_wh, off_wl, off_bar,
      total;
  __host__ __device__ explicit TcSmem(int m) {
    raw_stride = ((uint32_t)kTile * m * 4 + 1023) & ~1023u;
    off_grp = kRawStages * raw_stride;
    off_xh = 0;
    off_xl = off_xh + kTile * 128;
    off_dig = off_xl + kTile * 128;
    off_oh = off_dig + TcLayout<MP>::NB * kTile * 128;
    grp_stride = off_oh + ((KP * 128 + 1023) & ~1023u);
    off_wh = off_grp + kGroups * grp_stride;
    off_wl = off_wh + ((KP * 128 + 1023) & ~1023u);
    off_bar = off_wl + ((KP * 128 + 1023) & ~1023u);
    total = off_bar + 512 + 1024;  // barriers + 1 KiB alignment slack
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
  unsigned char* s_wh = sm + S.off_wh;
  unsigned char* s_wl = sm + S.off_wl;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + S.off_bar);
  uint64_t* full_raw = bars;                      // [kRawStages]  TMA → compute
  uint64_t* empty_raw = bars + kRawStages;        // [kRawStages]  compute → TMA
  uint64_t* op_full = bars + 2 * kRawStages;      // [kGroups] operands written   (compute → MMA)
  uint64_t* s_full = op_full + kGroups;           // [kGroups] assign MMAs done   (MMA → compute)
  uint64_t* ob_full = s_full + kGroups;           // [kGroups] one-hot written    (compute → MMA)
  uint64_t* op_free = ob_full + kGroups;          // [kGroups] update MMAs done   (MMA → compute)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(op_free + kGroups);

  const int m = a.m, k = a.k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  const int my_tiles = (int)((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
  // TMEM columns: S[g] at [g*KP, (g+1)*KP); U block b at [kGroups*KP + b*KP, ...)
  constexpr uint32_t kCols = (kGroups + TcLayout<MP>::NB) * KP;
  constexpr uint32_t kTmemCols = kCols <= 32 ? 32 : kCols <= 64 ? 64 : kCols <= 128 ? 128 : kCols <= 256 ? 256 : 512;
  constexpr uint32_t colU = kGroups * KP;

  // ---- setup ----
  if (tid == 0) {
    for (int s = 0; s < kRawStages; ++s) {
      mbar_init(full_raw + s, 1);
      mbar_init(empty_raw + s, 4);
    }
    for (int g = 0; g < kGroups; ++g) {
      mbar_init(op_full + g, 128);
      mbar_init(s_full + g, 1);
      mbar_init(ob_full + g, 128);
      mbar_init(op_free + g, 1);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_holder, kTmemCols);
  if (warp < kComputeWarps) {
    // W~ hi/lo → SW128 K-major smem (row c, chunk q = features 4q..4q+3); one-hot planes cleared
    for (int i = tid; i < KP * 8; i += kComputeWarps * 32) {
      const int c = i >> 3, q = i & 7;
      const float4 h = *reinterpret_cast<const float4*>(a.wsplit + (size_t)c * 32 + q * 4);
      const float4 l = *reinterpret_cast<const float4*>(a.wsplit + (size_t)(KP + c) * 32 + q * 4);
      *reinterpret_cast<float4*>(s_wh + sw128(c, q)) = h;
      *reinterpret_cast<float4*>(s_wl + sw128(c, q)) = l;
    }
    for (int g = 0; g < kGroups; ++g)
      for (int i = tid; i < KP * 8; i += kComputeWarps * 32)
        *reinterpret_cast<uint4*>(sm + S.off_grp + g * S.grp_stride + S.off_oh + i * 16) = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == kProducerWarp) {
    // ===================== TMA producer: raw 4·m-byte rows, tile i → slot i % kRawStages =====================
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
    // ===================== MMA issuer (one thread): event loop over ready barriers =====================
    // assign(i) needs op_full of tile i; update(i) needs ob_full of tile i.  Issue whichever is
    // ready (polling), so neither warpgroup waits on the other.  U sums are integers: any order.
    if (lane == 0) {
      const uint32_t grp0 = smem_u32(sm + S.off_grp);
      const uint32_t wh0 = smem_u32(s_wh), wl0 = smem_u32(s_wl);
      constexpr uint32_t id_tf32 = idesc_tf32(KP);
      constexpr uint32_t id_u8 = idesc_u8_amn(KP);
      int na = 0, nu = 0;  // next tile to assign / to update
      bool first_update = true;
      while (nu < my_tiles) {
        if (na < my_tiles) {
          const int g = na % kGroups, j = na / kGroups;
          if (mbar_test(op_full + g, j & 1)) {
            tc_fence_after();
            const uint32_t xh0 = grp0 + g * S.grp_stride + S.off_xh, xl0 = grp0 + g * S.grp_stride + S.off_xl;
#pragma unroll
            for (int ks = 0; ks < ((a.dbg_flags & 2) ? 0 : L::KS); ++ks) {
              const uint64_t dxh = make_desc(xh0 + ks * 32, 16, 1024), dxl = make_desc(xl0 + ks * 32, 16, 1024);
              const uint64_t dwh = make_desc(wh0 + ks * 32, 16, 1024), dwl = make_desc(wl0 + ks * 32, 16, 1024);
              mma_tf32(tmem + g * KP, dxh, dwh, id_tf32, ks > 0 ? 1u : 0u);
              mma_tf32(tmem + g * KP, dxh, dwl, id_tf32, 1u);
              mma_tf32(tmem + g * KP, dxl, dwh, id_tf32, 1u);
            }
            mma_commit(s_full + g);
            ++na;
          }
        }
        if (nu < na) {
          const int g = nu % kGroups, j = nu / kGroups;
          if (mbar_test(ob_full + g, j & 1)) {
            tc_fence_after();
            const uint32_t dig0 = grp0 + g * S.grp_stride + S.off_dig, oh0 = grp0 + g * S.grp_stride + S.off_oh;
#pragma unroll
            for (int b = 0; b < ((a.dbg_flags & 1) ? 0 : L::NB); ++b) {
#pragma unroll
              for (int ks = 0; ks < kTile / 32; ++ks) {
                const uint64_t da = make_desc(dig0 + b * (kTile * 128) + ks * 4096, 128 * 8, 1024);
                const uint64_t db = make_desc(oh0 + ks * 32, 16, 1024);
                mma_i8(tmem + colU + b * KP, da, db, id_u8, (!first_update || ks > 0) ? 1u : 0u);
              }
            }
            first_update = false;
            mma_commit(op_free + g);
            ++nu;
          }
        }
      }
    }
  } else {
    // ===================== compute warpgroups: thread = point, group g takes tiles i ≡ g (mod 2) =====================
    const int g = warp >> 2;
    const int p = tid & 127;                      // row in tile = TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    unsigned char* grp = sm + S.off_grp + g * S.grp_stride;
    unsigned char* s_xh = grp + S.off_xh;
    unsigned char* s_xl = grp + S.off_xl;
    unsigned char* s_dig = grp + S.off_dig;
    unsigned char* s_oh = grp + S.off_oh;
    const float cmax = a.cmax[0];
    const float scale_f = a.scale_f, err_coef = a.err_coef, err_floor = a.err_floor, nx_inflate = a.nx_inflate;
    const double scale_d = a.scale_d;
    const bool use_dscale = a.use_dscale != 0, exact_only = a.exact_only != 0;
    const float* __restrict__ gx = a.x;
    // per-thread SW128 geometry: row p → 8-row atom, row-in-atom, XOR key
    const uint32_t row_off = (uint32_t)((p >> 3) * 1024 + (p & 7) * 128);
    const int key = p & 7;
    int prev_lab = -1;
    unsigned int my_rechecks = 0;
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
      mbar_wait(full_raw + s, u & 1);
      if (stamp) ts[1] = clock64();
      const float* rs = raw + s * (S.raw_stride / 4);
      float x[MP];
      if (rows == kTile && ((kTile * m) & 3) == 0) {  // full tile, whole rows in the bulk copy
#pragma unroll
        for (int f = 0; f < MP; ++f) x[f] = (f < m) ? rs[p * m + f] : 0.f;
      } else {                                        // ragged last tile: bulk part + ≤ 3 trailing floats
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
      if (j > 0) mbar_wait(op_free + g, (j - 1) & 1);  // this group's previous tile: MMAs done with the operands
      if (stamp) ts[3] = clock64();
      if (prev_lab >= 0) s_oh[sw128(prev_lab, p >> 4) + (p & 15)] = 0;
      // --- operands: X~ hi/lo rows (K-major SW128) and fixed-point bytes (MN-major SW128)
#pragma unroll
      for (int q = 0; q < 2 * L::KS; ++q) {
        float h[4], l[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int f = q * 4 + jj;
          float v = (f < MP) ? x[f] : 0.f;
          if (f == m) v = active ? 1.f : 0.f;
          const float hv = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
          h[jj] = hv;
          l[jj] = v - hv;
        }
        const uint32_t o = row_off + ((uint32_t)(q ^ key) << 4);
        *reinterpret_cast<float4*>(s_xh + o) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(s_xl + o) = make_float4(l[0], l[1], l[2], l[3]);
      }
      long long fx[MP + 1];
      if (!use_dscale) {
#pragma unroll
        for (int f = 0; f < MP; ++f) fx[f] = __float2ll_rn(__fmul_rn(x[f], scale_f));
      } else {
#pragma unroll
        for (int f = 0; f < MP; ++f) fx[f] = __double2ll_rn(__dmul_rn((double)x[f], scale_d));
      }
      fx[MP] = 0;
#pragma unroll
      for (int f = 0; f <= MP; ++f) {
        if (f >= m) fx[f] = 0;
        if (f == m) fx[f] = active ? 1 : 0;   // pseudo-feature m: the counts
      }
#pragma unroll
      for (int b = 0; b < L::NB; ++b) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int f0 = b * 16 + q * 2;
          const long long v0 = (f0 <= MP) ? fx[f0] : 0, v1 = (f0 + 1 <= MP) ? fx[f0 + 1] : 0;
          *reinterpret_cast<longlong2*>(s_dig + b * (kTile * 128) + row_off + ((uint32_t)(q ^ key) << 4)) =
              make_longlong2(v0, v1);
        }
      }
      fence_proxy_async();
      mbar_arrive(op_full + g);
      float nx2 = 0.f;
#pragma unroll
      for (int f = 0; f < MP; ++f) nx2 = __fmaf_rn(x[f], x[f], nx2);
      // --- epilogue: scores from TMEM
      if (stamp) ts[4] = clock64();
      mbar_wait(s_full + g, j & 1);
      if (stamp) ts[5] = clock64();
      tc_fence_after();
      float sc[KP];
#pragma unroll
      for (int c0 = 0; c0 < KP; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tmem + lane_base + g * KP + c0, r);
        tmem_ld_wait();
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) sc[c0 + jj] = __uint_as_float(r[jj]);
      }
      tc_fence_before();  // TMEM reads ordered before the MMA thread reuses S[g]
      float best = __int_as_float(0x7f800000), min2 = best;
      int bi = 0;
#pragma unroll
      for (int c = 0; c < KP; ++c) {
        if (c < k) {
          if (a.dbg_scores && active) a.dbg_scores[(row0 + p) * k + c] = sc[c];
          const bool lt = sc[c] < best;
          min2 = lt ? best : fminf(min2, sc[c]);
          bi = lt ? c : bi;
          best = lt ? sc[c] : best;
        }
      }
      const float tt = __fmaf_rn(sqrtf(nx2), nx_inflate, cmax);
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
      if (active) {
        a.labels[row0 + p] = lab;
        s_oh[sw128(lab, p >> 4) + (p & 15)] = 1;
        prev_lab = lab;
      } else {
        prev_lab = -1;
      }
      fence_proxy_async();
      mbar_arrive(ob_full + g);
      if (stamp) ts[6] = clock64();
    }
    // ---- group 0 flushes the exact update accumulators: U[8f+b][c] (row = TMEM lane) ----
    if (g == 0 && my_tiles > 0) {
      const int last = my_tiles - 1;
      mbar_wait(op_free + (last % kGroups), (last / kGroups) & 1);  // commits are cumulative: all MMAs done
      tc_fence_after();
#pragma unroll
      for (int b = 0; b < L::NB; ++b) {
        const int R = b * 128 + p;  // byte row
        const int f = R >> 3, byte = R & 7;
#pragma unroll
        for (int c0 = 0; c0 < KP; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(tmem + lane_base + colU + b * KP + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            unsigned long long v = (unsigned long long)r[jj] << (8 * byte);
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            const int c = c0 + jj;
            if (byte == 0 && c < k && v != 0ull) {
              if (f < m) {
                if (a.do_sums) atomicAdd(a.part + (size_t)c * m + f, v);
              } else if (f == m) {
                atomicAdd(a.part + (size_t)k * m + c, v);
              }
            }
          }
        }
      }
    }
    unsigned int wsum = my_rechecks;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
    if (lane == 0 && wsum) atomicAdd(&a.st->rechecked, (unsigned long long)wsum);
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
