// kmeans_sums.cuh — exact per-cluster fixed-point sums of a whole labelled point set.
//
// The reference's update reduction (`_kernels.cluster_sums_block`, _kernels.py:97-113, folded
// over accumulation blocks by `model.fold_blocks`, model.py:163-173) for ALL n points at once,
// used where the fused pass cannot update the sums incrementally: the first pass of a Lloyd run
// (no previous labels — every point would have to be added through shared-memory atomics
// inside the tensor-core epilogue, ~6× a steady pass).  Instead the first pass only writes the
// labels L0 = A(C0) and this kernel adds the points to their clusters in one HBM stream.
//
// Arithmetic: each coordinate becomes the int64 fixed-point value round(x·2^F) — the SAME
// conversion the tensor-core pass uses for its per-point deltas (to_fixed) — so the running
// totals S(L_t) = S(L0) + Σ Δ stay bit-identical to a from-scratch recomputation, for any grid.
//
// Streaming: each CTA owns a contiguous range of 128-row tiles; one elected thread keeps a ring
// of bulk copies (cp.async.bulk, the rows and their labels, L2 evict-first) in flight, so the
// loads need no registers and are fully coalesced.  Consumption: lane f of a warp owns feature f
// (lane m counts); a row's label is warp-uniform, so one warp instruction adds a whole row into
// accumulator row `label` with distinct addresses per lane.  PRIV: every warp owns a private
// [k][m+1] int64 accumulator (plain LDS/IADD/STS); otherwise (large k·m) the CTA shares one copy
// updated with 32-bit atomic pairs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kmeans_kernels.cuh"
#include "kmeans_tc.cuh"

namespace km {

constexpr int kSumsWarps = 16;                      // consumer warps (+ one producer warp)
constexpr int kSumsThreads = (kSumsWarps + 1) * 32;
constexpr int kSumsTile = 128;                      // rows per bulk tile (kSumsWarps × 8)
constexpr int kSumsStages = 4;                      // tiles in flight per CTA

// shared memory: [stages] × (row tile + labels) ring, then the accumulators
__host__ __device__ inline size_t sums_stage_bytes(int m, int esz = 4) {
  return (((size_t)kSumsTile * m * esz + 15) & ~(size_t)15) + kSumsTile * 4;
}
__host__ __device__ inline size_t sums_smem_bytes(int m, int k, bool priv, int esz = 4) {
  return 1024 + kSumsStages * sums_stage_bytes(m, esz) + (size_t)(priv ? kSumsWarps : 1) * k * (m + 1) * 8;
}

// One tile's rows of this warp into its accumulator (lane f ≤ m; lane m counts).
template <typename T, bool PRIV, bool USE_D>
__device__ __forceinline__ void sums_rows(const T* __restrict__ sx, const int32_t* __restrict__ sl, int r0, int r1,
                                          int m, int lane, unsigned long long* acc, int row_len, float scale_f,
                                          double scale_d) {
#pragma unroll 4
  for (int r = r0; r < r1; ++r) {
    const int L = sl[r];                                      // warp-uniform (broadcast)
    unsigned long long q = 1ull;                              // lane m: the count
    if (lane < m) {
      q = (unsigned long long)to_fixed<T>(sx[r * m + lane], scale_f, scale_d, USE_D);
    }
    unsigned long long* dst = acc + L * row_len + lane;
    if (PRIV) *dst += q; else smem_add64(dst, q);
  }
}

// Full 128-row tile, compile-time m (MT): the warp's RPW rows at immediate offsets.  The count
// lane (lane MT) converts cnt_v = 2^-F, which the fixed-point conversion maps to exactly 1, so
// every lane runs the same instruction stream: ~10 warp instructions per row.
template <typename T, int MT, int RPW, bool PRIV>
__device__ __forceinline__ void sums_rows_full(const T* __restrict__ sxw, const int32_t* __restrict__ slw,
                                               int lane, unsigned long long* acc_lane, float scale_f, double scale_d,
                                               T cnt_v) {
  const bool feat = lane < MT;
  if (PRIV) {
    // rows in pairs: the read-modify-writes of two different labels load together, then store
    // together (one dependent chain per pair instead of per row); equal labels add in registers
#pragma unroll
    for (int j = 0; j < RPW; j += 2) {
      const int L0 = slw[j], L1 = slw[j + 1];
      const unsigned long long q0 = (unsigned long long)to_fixed<T>(feat ? sxw[j * MT] : cnt_v, scale_f, scale_d, 0);
      const unsigned long long q1 = (unsigned long long)to_fixed<T>(feat ? sxw[(j + 1) * MT] : cnt_v, scale_f, scale_d, 0);
      unsigned long long* d0 = acc_lane + L0 * (MT + 1);
      if (L0 != L1) {
        unsigned long long* d1 = acc_lane + L1 * (MT + 1);
        const unsigned long long a0 = *d0, a1 = *d1;
        *d0 = a0 + q0;
        *d1 = a1 + q1;
      } else {
        *d0 += q0 + q1;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < RPW; ++j) {
      const int L = slw[j];
      const T v = feat ? sxw[j * MT] : cnt_v;
      smem_add64(acc_lane + L * (MT + 1), (unsigned long long)to_fixed<T>(v, scale_f, scale_d, 0));
    }
  }
}

// MT > 0: compile-time feature count (the full-tile fast path); MT = 0: runtime m
// T = float, or double for fp64 points (the fp64 coordinates are what every Δ of those points uses)
template <typename T, int MT, bool PRIV, bool USE_D>
__global__ void __launch_bounds__(kSumsThreads) cluster_sums_f32_kernel(
    const T* __restrict__ x, const int32_t* __restrict__ labels, int64_t n, int m, int k, float scale_f,
    double scale_d, unsigned long long* __restrict__ out /* [k·m sums][k counts] */) {
  extern __shared__ __align__(1024) unsigned char s_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(s_raw);      // [stages]
  uint64_t* empty = full + kSumsStages;                      // [stages]
  unsigned char* ring = s_raw + 1024;
  constexpr uint32_t ESZ = sizeof(T);
  const size_t stage = sums_stage_bytes(m, ESZ);
  const size_t xbytes_max = stage - kSumsTile * 4;
  unsigned long long* s_acc = reinterpret_cast<unsigned long long*>(ring + kSumsStages * stage);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row_len = m + 1, per = k * row_len, copies = PRIV ? kSumsWarps : 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSumsStages; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(empty + s, kSumsWarps);
    }
    tc::fence_barrier_init();
  }
  for (int i = threadIdx.x; i < per * copies; i += kSumsThreads) s_acc[i] = 0ull;
  __syncthreads();
  unsigned long long* acc = s_acc + (PRIV ? (size_t)warp * per : 0);

  const int64_t ntiles = (n + kSumsTile - 1) / kSumsTile;
  const int64_t t_lo = ntiles * blockIdx.x / gridDim.x, t_hi = ntiles * (blockIdx.x + 1) / gridDim.x;
  const int my = (int)(t_hi - t_lo);
  // the last tile of the array may be ragged: its tail (≤ 3 floats / labels past the 16-byte
  // bulk granule) is patched in from global memory by the CTA that owns it
  auto issue = [&](int i) {  // tile i of this CTA → stage i % S (one thread)
    const int s = i % kSumsStages;
    if (i >= kSumsStages) tc::mbar_wait(empty + s, ((i / kSumsStages) - 1) & 1);
    const int64_t row0 = (t_lo + i) * kSumsTile;
    const int rows = (int)(n - row0 < kSumsTile ? n - row0 : kSumsTile);
    const uint32_t xb = ((uint32_t)rows * m * ESZ) & ~15u, lb = ((uint32_t)rows * 4u) & ~15u;
    tc::mbar_arrive_expect_tx(full + s, xb + lb);
    unsigned char* dst = ring + s * stage;
    const uint64_t pol = tc::l2_policy_evict_first();
    if (xb) tc::bulk_g2s_hint(dst, x + row0 * m, xb, full + s, pol);
    if (lb) tc::bulk_g2s_hint(dst + xbytes_max, labels + row0, lb, full + s, pol);
  };
  constexpr int RPW = kSumsTile / kSumsWarps;  // rows per warp and tile
  // 2^-F: converts to exactly 1 (the count lane)
  const T cnt_v = sizeof(T) == 8 ? (T)(1.0 / scale_d) : (T)(1.0f / scale_f);
  if (warp == kSumsWarps) {  // producer warp: one thread keeps the ring full
    if (lane == 0)
      for (int i = 0; i < my; ++i) issue(i);
  } else {
    const bool active = lane <= m;
    for (int i = 0; i < my; ++i) {
      const int s = i % kSumsStages;
      const int64_t row0 = (t_lo + i) * kSumsTile;
      const int rows = (int)(n - row0 < kSumsTile ? n - row0 : kSumsTile);
      // one warp polls the barrier, the others park in bar.sync (no wake-up storms)
      if (warp == 0) tc::mbar_wait(full + s, (i / kSumsStages) & 1);
      tc::named_bar_sync(1, kSumsWarps * 32);
      T* sx = reinterpret_cast<T*>(ring + s * stage);
      int32_t* sl = reinterpret_cast<int32_t*>(ring + s * stage + xbytes_max);
      if (rows < kSumsTile) {  // ragged last tile: patch the sub-granule tail from global memory
        const uint32_t xe = (((uint32_t)rows * m * ESZ) & ~15u) / ESZ, le = (((uint32_t)rows * 4u) & ~15u) / 4u;
        for (uint32_t e = xe + threadIdx.x; e < (uint32_t)rows * m; e += kSumsWarps * 32) sx[e] = __ldg(x + row0 * m + e);
        for (uint32_t e = le + threadIdx.x; e < (uint32_t)rows; e += kSumsWarps * 32) sl[e] = __ldg(labels + row0 + e);
        tc::named_bar_sync(1, kSumsWarps * 32);
      }
      if (MT > 0 && (sizeof(T) == 8 || !USE_D) && rows == kSumsTile) {
        if (active)
          sums_rows_full<T, (MT > 0 ? MT : 1), RPW, PRIV>(sx + warp * RPW * MT + (lane < m ? lane : 0), sl + warp * RPW, lane,
                                                       acc + lane, scale_f, scale_d, cnt_v);
      } else {
        const int r0 = min(warp * RPW, rows), r1 = min(r0 + RPW, rows);
        if (active) sums_rows<T, PRIV, USE_D>(sx, sl, r0, r1, m, lane, acc, row_len, scale_f, scale_d);
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(empty + s);
    }
  }
  __syncthreads();
  // one global atomic per non-zero accumulator and CTA
  for (int i = threadIdx.x; i < per; i += kSumsThreads) {
    unsigned long long v = 0;
    for (int w = 0; w < copies; ++w) v += s_acc[(size_t)w * per + i];
    if (v) {
      const int c = i / row_len, f = i - c * row_len;
      atomicAdd(out + (f < m ? (size_t)c * m + f : (size_t)k * m + c), v);
    }
  }
}

}  // namespace km
