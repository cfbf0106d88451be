// kmeans_kernels.cuh — device code of the B200 Lloyd engine.
//
// One Lloyd iteration = ONE fused pass over the resident point matrix
// (assign + per-cluster fixed-point sums) followed by a one-CTA finish kernel
// (divide, empty-cluster count, convergence flag, fp32 filter prep).
//
// Arithmetic contract (what makes labels bit-identical to the reference):
//  * Labels are decided by a certified fp32 filter.  Score
//        S~_c = fl(‖c~‖² + Σ_f x~_f·(−2c~_f))      (M FMAs, features ascending)
//    differs from the exact ‖x−c‖² − ‖x‖² by at most
//        E = coef·(‖x‖ + max_c‖c‖)²,  coef = (M+8)·2⁻²⁴·1.25
//    (FMA-chain γ_M bound + rounding of x, c, ‖c‖² to fp32 + the fp64
//    rounding of the reference's own distance).  When the
//    runner-up score exceeds best + 2E the fp32 argmin IS the reference
//    argmin.  Otherwise every centre with S~_c ≤ best + 2E is re-decided with
//    the reference's exact fp64 recurrence (_kernels.py:31-44: d = x−c,
//    acc += d*d, no FMA, ascending c, strict '<' keeps the lowest index).
//  * Cluster sums are int64 fixed point with 2^F scaling (F chosen from
//    max|x| and n so no sum can overflow): integer adds are associative, so the
//    sums — and the centres — are bit-identical for any grid size and any
//    number of GPUs (the reference gets the same property from canonical
//    blocks, model.py:18-24; we get it from exact integer arithmetic).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "kmeans_state.h"
#include "kmeans_finish.cuh"

namespace km {

constexpr int kTileRows = 256;   // rows per CTA tile == threads per CTA
constexpr int kThreads = 256;


struct PassArgs {
  const void* x;          // n × m row-major, T = float or double
  int64_t n;
  int32_t m, k;
  const float* w;         // k × MPAD: −2·fl32(c)  (zero padded)
  const float* cn;        // k: fl32(‖fl32(c)‖²)
  const float* cmax;      // [0]: max_c ‖fl32(c)‖ rounded up
  const double* c64;      // k × m reference-precision centres (for the exact recheck)
  int32_t* labels;        // n
  unsigned long long* part;  // k·m sums (fixed point, two's complement) then k counts
  float scale_f;          // 2^F as float (valid when !use_dscale)
  double scale_d;         // 2^F
  int32_t use_dscale;
  int32_t mpad;           // row pitch of w
  float err_coef;         // (M+8)·2^-24·1.25
  float err_floor;        // absolute floor for subnormal effects
  float nx_inflate;       // 1 + (M+2)·2^-24
  int32_t exact_only;     // filter disabled (extreme magnitudes): fp64 for every centre
  DevState* st;           // loop state (statistics; gating when `gate`)
  int32_t gate;           // early-exit when the loop is done / waiting for the host
};

template <typename T>
__device__ __forceinline__ float to_f32(T v) { return (float)v; }

template <typename T>
__device__ __forceinline__ double to_f64(T v) { return (double)v; }

// Reference recurrence for one squared distance (_kernels.py:33-41): no FMA.
template <typename T>
__device__ __forceinline__ double exact_d2(const T* xrow, const double* __restrict__ c, int m) {
  double acc = 0.0;
  for (int f = 0; f < m; ++f) {
    double d = __dsub_rn(to_f64(xrow[f]), c[f]);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  return acc;
}

template <typename T>
__device__ __forceinline__ long long to_fixed(T v, float sf, double sd, int use_d);

template <>
__device__ __forceinline__ long long to_fixed<float>(float v, float sf, double sd, int use_d) {
  return use_d ? __double2ll_rn(__dmul_rn((double)v, sd)) : __float2ll_rn(__fmul_rn(v, sf));
}
template <>
__device__ __forceinline__ long long to_fixed<double>(double v, float, double sd, int) {
  return __double2ll_rn(__dmul_rn(v, sd));
}

// fp32 filter score of centre c for a point held in registers.
template <int MP>
__device__ __forceinline__ float score_reg(const float (&xr)[MP], const float* __restrict__ wc, float cn) {
  float a = cn;
#pragma unroll
  for (int f = 0; f < MP; f += 4) {
    const float4 w4 = *reinterpret_cast<const float4*>(wc + f);
    a = __fmaf_rn(xr[f + 0], w4.x, a);
    a = __fmaf_rn(xr[f + 1], w4.y, a);
    a = __fmaf_rn(xr[f + 2], w4.z, a);
    a = __fmaf_rn(xr[f + 3], w4.w, a);
  }
  return a;
}

// Generic-M filter score, x read from the shared-memory tile.
template <typename T>
__device__ __forceinline__ float score_smem(const T* xrow, int m, const float* __restrict__ wc, float cn) {
  float a = cn;
  for (int f = 0; f < m; ++f) a = __fmaf_rn(to_f32(xrow[f]), wc[f], a);
  return a;
}

// Cooperative copy of `bytes` (multiple of 4) from global to shared, 16 B vectors
// where the source is 16 B aligned (it is: cudaMalloc base + tile offsets that
// are multiples of 1 KiB).
__device__ __forceinline__ void tile_copy(void* dst, const void* src, int64_t bytes) {
  const int64_t nv = bytes >> 4;
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) d4[i] = __ldg(s4 + i);
  const int64_t tail = (bytes - (nv << 4)) >> 2;
  const float* s1 = reinterpret_cast<const float*>(src) + (nv << 2);
  float* d1 = reinterpret_cast<float*>(dst) + (nv << 2);
  for (int64_t i = threadIdx.x; i < tail; i += blockDim.x) d1[i] = __ldg(s1 + i);
}

// ---------------------------------------------------------------------------
// Fused pass: labels + per-cluster fixed-point sums + counts.
//   DO_ASSIGN: compute labels (else read them and validate, update_step path)
//   DO_SUMS:   accumulate coordinate sums (counts are always accumulated)
//   MP:        padded feature count held in registers (0 = generic, from smem)
//   SMEM_ACC:  privatised per-CTA accumulators in shared memory
// ---------------------------------------------------------------------------
template <typename T, int MP, bool DO_ASSIGN, bool DO_SUMS, bool SMEM_ACC>
__global__ void __launch_bounds__(kThreads) lloyd_pass_kernel(PassArgs a) {
  if (a.gate && (a.st->done || a.st->need_host)) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int m = a.m, k = a.k, tid = threadIdx.x;
  const int mpad = a.mpad;
  // layout (16 B aligned sections): [w k*mpad f32][cn k f32][acc k*m u64][cnt k u64][tile 256*m T]
  auto align16 = [](size_t v) { return (v + 15) & ~size_t(15); };
  size_t off = 0;
  float* s_w = reinterpret_cast<float*>(smem + off);
  off = align16(off + (DO_ASSIGN ? (size_t)k * mpad * 4 : 0));
  float* s_cn = reinterpret_cast<float*>(smem + off);
  off = align16(off + (DO_ASSIGN ? (size_t)k * 4 : 0));
  unsigned long long* s_acc = reinterpret_cast<unsigned long long*>(smem + off);
  unsigned long long* s_cnt = s_acc + (SMEM_ACC ? (size_t)k * m : 0);
  off = align16(off + (SMEM_ACC ? ((size_t)k * m + k) * 8 : 0));
  T* s_tile = reinterpret_cast<T*>(smem + off);

  if (SMEM_ACC) {
    for (int i = tid; i < k * m + k; i += kThreads) s_acc[i] = 0ull;
  }
  if (DO_ASSIGN) {
    for (int i = tid; i < k * mpad; i += kThreads) s_w[i] = a.w[i];
    for (int i = tid; i < k; i += kThreads) s_cn[i] = a.cn[i];
  }
  unsigned long long* g_acc = a.part;
  unsigned long long* g_cnt = a.part + (size_t)k * m;
  unsigned long long* acc = SMEM_ACC ? s_acc : g_acc;
  unsigned long long* cnt = SMEM_ACC ? s_cnt : g_cnt;

  const float cmax = DO_ASSIGN ? a.cmax[0] : 0.f;
  const T* __restrict__ X = reinterpret_cast<const T*>(a.x);
  const int64_t ntiles = (a.n + kTileRows - 1) / kTileRows;
  unsigned int my_rechecks = 0;
  int bad = 0;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * kTileRows;
    const int64_t rem = a.n - row0;
    const int rows = rem < kTileRows ? (int)rem : kTileRows;
    __syncthreads();  // previous tile fully consumed (and smem init done)
    tile_copy(s_tile, X + row0 * m, (int64_t)rows * m * (int64_t)sizeof(T));
    __syncthreads();
    if (tid < rows) {
      const T* xrow = s_tile + (size_t)tid * m;
      int lab;
      if (DO_ASSIGN) {
        float best = __int_as_float(0x7f800000), min2 = best;
        int bi = 0;
        float nx2 = 0.f;
        if constexpr (MP > 0) {
          float xr[MP];
#pragma unroll
          for (int f = 0; f < MP; ++f) xr[f] = (f < m) ? to_f32(xrow[f]) : 0.f;
#pragma unroll
          for (int f = 0; f < MP; ++f) nx2 = __fmaf_rn(xr[f], xr[f], nx2);
          for (int c = 0; c < k; ++c) {
            const float s = score_reg<MP>(xr, s_w + (size_t)c * mpad, s_cn[c]);
            const bool lt = s < best;
            min2 = lt ? best : fminf(min2, s);
            bi = lt ? c : bi;
            best = lt ? s : best;
          }
          const float t = __fmaf_rn(sqrtf(nx2), a.nx_inflate, cmax);
          const float E = __fmaf_rn(a.err_coef * t, t, a.err_floor);
          const float thr = best + 2.f * E;
          if (a.exact_only || !(min2 > thr)) {
            ++my_rechecks;
            double bd = 0.0;
            int bl = -1;
            for (int c = 0; c < k; ++c) {
              bool cand = a.exact_only != 0;
              if (!cand) cand = score_reg<MP>(xr, s_w + (size_t)c * mpad, s_cn[c]) <= thr;
              if (cand) {
                const double d = exact_d2<T>(xrow, a.c64 + (size_t)c * m, m);
                if (bl < 0 || d < bd) { bd = d; bl = c; }
              }
            }
            bi = bl;
          }
        } else {
          for (int f = 0; f < m; ++f) { const float v = to_f32(xrow[f]); nx2 = __fmaf_rn(v, v, nx2); }
          for (int c = 0; c < k; ++c) {
            const float s = score_smem<T>(xrow, m, s_w + (size_t)c * mpad, s_cn[c]);
            const bool lt = s < best;
            min2 = lt ? best : fminf(min2, s);
            bi = lt ? c : bi;
            best = lt ? s : best;
          }
          const float t = __fmaf_rn(sqrtf(nx2), a.nx_inflate, cmax);
          const float E = __fmaf_rn(a.err_coef * t, t, a.err_floor);
          const float thr = best + 2.f * E;
          if (a.exact_only || !(min2 > thr)) {
            ++my_rechecks;
            double bd = 0.0;
            int bl = -1;
            for (int c = 0; c < k; ++c) {
              bool cand = a.exact_only != 0;
              if (!cand) cand = score_smem<T>(xrow, m, s_w + (size_t)c * mpad, s_cn[c]) <= thr;
              if (cand) {
                const double d = exact_d2<T>(xrow, a.c64 + (size_t)c * m, m);
                if (bl < 0 || d < bd) { bd = d; bl = c; }
              }
            }
            bi = bl;
          }
        }
        lab = bi;
        a.labels[row0 + tid] = lab;
      } else {
        lab = a.labels[row0 + tid];
        if (lab < 0 || lab >= k) { bad = 1; lab = -1; }
      }
      if (lab >= 0) {
        if (SMEM_ACC) {
          atomicAdd(reinterpret_cast<unsigned int*>(cnt + lab), 1u);  // counts < 2^32 per CTA
          if (DO_SUMS) {
            unsigned long long* dst = acc + (size_t)lab * m;
            for (int f = 0; f < m; ++f)
              smem_add64(dst + f, (unsigned long long)to_fixed<T>(xrow[f], a.scale_f, a.scale_d, a.use_dscale));
          }
        } else {
          atomicAdd(cnt + lab, 1ull);
          if (DO_SUMS) {
            unsigned long long* dst = acc + (size_t)lab * m;
            for (int f = 0; f < m; ++f)
              atomicAdd(dst + f, (unsigned long long)to_fixed<T>(xrow[f], a.scale_f, a.scale_d, a.use_dscale));
          }
        }
      }
    }
  }
  // statistics / validation
  if (DO_ASSIGN) {
    unsigned int wsum = my_rechecks;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
    if ((tid & 31) == 0 && wsum) atomicAdd(&a.st->rechecked, (unsigned long long)wsum);
  }
  if (!DO_ASSIGN && bad) atomicExch(&a.st->bad_label, 1);
  if (SMEM_ACC) {
    __syncthreads();
    for (int i = tid; i < k * m; i += kThreads)
      if (s_acc[i]) atomicAdd(g_acc + i, s_acc[i]);
    for (int i = tid; i < k; i += kThreads)
      if (s_cnt[i]) atomicAdd(g_cnt + i, s_cnt[i]);
  }
}

// ---------------------------------------------------------------------------
// Register-blocked fused pass for large K (fp32 points, m ≤ MP ≤ 32): the FP32-bound regime
// (BASELINE cfg4, K = 512).  Each thread owns kBlkPts points (coordinates in registers) and walks
// the centres in chunks of kBlkC: per feature f, kBlkC/4 broadcast LDS.128 of the transposed
// operand wt[f][c] feed kBlkPts·kBlkC independent FMAs (an SGEMM-style outer product), against
// 1 LDS.128 per 4 FMAs in lloyd_pass_kernel.  Every score is the same FMA chain as score_reg
// (a = ‖c‖², then a = fma(x_f, −2c_f, a) for f ascending), so the filter, its certificate and the
// exact fp64 recheck (same candidates, same lowest-index rule) decide bit-identical labels.
// The FMAs are packed fp32x2 (FFMA2, one issue slot for both points' lanes).
// Sums: the per-CTA fixed-point accumulators of lloyd_pass_kernel.
// ---------------------------------------------------------------------------
constexpr int kBlkThreads = 384;
constexpr int kBlkPts = 2;
constexpr int kBlkC = 8;
constexpr int kBlkTileRows = kBlkThreads * kBlkPts;

static_assert(kBlkPts == 2, "the blocked pass pairs its two points in fp32x2 registers");
__device__ __forceinline__ unsigned long long pack_f32x2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack_f32x2(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ float lane_f32x2(unsigned long long v, int p) {
  float lo, hi;
  unpack_f32x2(v, lo, hi);
  return p ? hi : lo;
}
// lane-wise fma.rn (no ftz): FFMA2 on sm_100a
__device__ __forceinline__ unsigned long long ffma_f32x2(unsigned long long a, unsigned long long b,
                                                         unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

__device__ __forceinline__ void blk_take(float s, int c, float& best, float& min2, int& bi) {
  min2 = fminf(min2, fmaxf(best, s));  // = (s < best ? best : min(min2, s)), best ≤ min2
  const bool lt = s < best;
  bi = lt ? c : bi;
  best = lt ? s : best;
}

template <int MP, bool DO_SUMS, bool SMEM_ACC>
__global__ void __launch_bounds__(kBlkThreads, 1) lloyd_pass_blocked_kernel(PassArgs a, int kp8) {
  if (a.gate && (a.st->done || a.st->need_host)) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int m = a.m, k = a.k, tid = threadIdx.x;
  // layout: [wt MP × kp8 f32][cn kp8 f32][acc k·m u64][cnt k u64]
  float* s_wt = reinterpret_cast<float*>(smem);
  float* s_cn = s_wt + (size_t)MP * kp8;
  unsigned long long* s_acc = reinterpret_cast<unsigned long long*>(s_cn + kp8);  // kp8·4 B keeps 16 B alignment
  unsigned long long* s_cnt = s_acc + (size_t)k * m;
  for (int i = tid; i < MP * kp8; i += kBlkThreads) {
    const int f = i / kp8, c = i - f * kp8;
    s_wt[i] = (c < k && f < m) ? a.w[(size_t)c * a.mpad + f] : 0.f;
  }
  for (int c = tid; c < kp8; c += kBlkThreads) s_cn[c] = c < k ? a.cn[c] : __int_as_float(0x7f800000);
  if (SMEM_ACC)
    for (int i = tid; i < k * m + k; i += kBlkThreads) s_acc[i] = 0ull;
  __syncthreads();
  unsigned long long* g_acc = a.part;
  unsigned long long* g_cnt = a.part + (size_t)k * m;
  unsigned long long* acc = SMEM_ACC ? s_acc : g_acc;
  unsigned long long* cnt = SMEM_ACC ? s_cnt : g_cnt;
  const float cmax = a.cmax[0];
  const float* __restrict__ X = reinterpret_cast<const float*>(a.x);
  const int64_t ntiles = (a.n + kBlkTileRows - 1) / kBlkTileRows;
  unsigned int my_rechecks = 0;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // the two points of a thread share one packed fp32x2 FMA per (feature, centre): FFMA2 with the
    // centre operand broadcast; each lane is the IEEE fma.rn of score_reg (bit-identical chains)
    unsigned long long xp2[MP];
    int64_t row[kBlkPts];
    bool live[kBlkPts];
#pragma unroll
    for (int p = 0; p < kBlkPts; ++p) {
      row[p] = tile * kBlkTileRows + p * kBlkThreads + tid;
      live[p] = row[p] < a.n;
    }
    {
      const float* x0 = X + (live[0] ? row[0] : 0) * m;
      const float* x1 = X + (live[1] ? row[1] : 0) * m;
#pragma unroll
      for (int f = 0; f < MP; ++f)
        xp2[f] = pack_f32x2((live[0] && f < m) ? __ldg(x0 + f) : 0.f, (live[1] && f < m) ? __ldg(x1 + f) : 0.f);
    }
    float best[kBlkPts], min2[kBlkPts];
    int bi[kBlkPts];
#pragma unroll
    for (int p = 0; p < kBlkPts; ++p) best[p] = min2[p] = __int_as_float(0x7f800000), bi[p] = 0;
#pragma unroll 2
    for (int c0 = 0; c0 < kp8; c0 += kBlkC) {
      unsigned long long s2[kBlkC];
      const float4 n0 = *reinterpret_cast<const float4*>(s_cn + c0);
      const float4 n1 = *reinterpret_cast<const float4*>(s_cn + c0 + 4);
      s2[0] = pack_f32x2(n0.x, n0.x), s2[1] = pack_f32x2(n0.y, n0.y);
      s2[2] = pack_f32x2(n0.z, n0.z), s2[3] = pack_f32x2(n0.w, n0.w);
      s2[4] = pack_f32x2(n1.x, n1.x), s2[5] = pack_f32x2(n1.y, n1.y);
      s2[6] = pack_f32x2(n1.z, n1.z), s2[7] = pack_f32x2(n1.w, n1.w);
#pragma unroll
      for (int f = 0; f < MP; ++f) {
        const float4 w0 = *reinterpret_cast<const float4*>(s_wt + (size_t)f * kp8 + c0);
        const float4 w1 = *reinterpret_cast<const float4*>(s_wt + (size_t)f * kp8 + c0 + 4);
        s2[0] = ffma_f32x2(xp2[f], pack_f32x2(w0.x, w0.x), s2[0]);
        s2[1] = ffma_f32x2(xp2[f], pack_f32x2(w0.y, w0.y), s2[1]);
        s2[2] = ffma_f32x2(xp2[f], pack_f32x2(w0.z, w0.z), s2[2]);
        s2[3] = ffma_f32x2(xp2[f], pack_f32x2(w0.w, w0.w), s2[3]);
        s2[4] = ffma_f32x2(xp2[f], pack_f32x2(w1.x, w1.x), s2[4]);
        s2[5] = ffma_f32x2(xp2[f], pack_f32x2(w1.y, w1.y), s2[5]);
        s2[6] = ffma_f32x2(xp2[f], pack_f32x2(w1.z, w1.z), s2[6]);
        s2[7] = ffma_f32x2(xp2[f], pack_f32x2(w1.w, w1.w), s2[7]);
      }
#pragma unroll
      for (int j = 0; j < kBlkC; ++j) {
        float lo, hi;
        unpack_f32x2(s2[j], lo, hi);
        blk_take(lo, c0 + j, best[0], min2[0], bi[0]);
        blk_take(hi, c0 + j, best[1], min2[1], bi[1]);
      }
    }
#pragma unroll
    for (int p = 0; p < kBlkPts; ++p) {
      float thr = 0.f;
      bool need = false;
      int lab = bi[p];
      if (live[p]) {
        float nx2 = 0.f;
#pragma unroll
        for (int f = 0; f < MP; ++f) nx2 = __fmaf_rn(lane_f32x2(xp2[f], p), lane_f32x2(xp2[f], p), nx2);
        const float t = __fmaf_rn(sqrtf(nx2), a.nx_inflate, cmax);
        const float E = __fmaf_rn(a.err_coef * t, t, a.err_floor);
        thr = best[p] + 2.f * E;
        need = a.exact_only || !(min2[p] > thr);
      }
      // exact recheck, warp-cooperative: for each lane whose certificate failed, the 32 lanes split
      // the centres (c ≡ lane mod 32, ascending), keep the candidates within 2E of the best filter
      // score, evaluate the reference fp64 recurrence and reduce (d², c) lexicographically — the
      // lowest index among equal distances, as the serial loop's strict '<' over ascending c
      unsigned pend = __ballot_sync(0xffffffffu, need);
      while (pend) {
        const int src = __ffs(pend) - 1;
        pend &= pend - 1;
        const float tthr = __shfl_sync(0xffffffffu, thr, src);
        float xs[MP];
#pragma unroll
        for (int f = 0; f < MP; ++f) xs[f] = __shfl_sync(0xffffffffu, lane_f32x2(xp2[f], p), src);
        double bd = 0.0;
        int bl = 0x7fffffff;
        for (int c = (int)(threadIdx.x & 31); c < k; c += 32) {
          bool cand = a.exact_only != 0;
          if (!cand) {
            float sc = s_cn[c];
#pragma unroll
            for (int f = 0; f < MP; ++f) sc = __fmaf_rn(xs[f], s_wt[(size_t)f * kp8 + c], sc);
            cand = sc <= tthr;
          }
          if (cand) {
            const double* cc = a.c64 + (size_t)c * m;
            double d2 = 0.0;
#pragma unroll
            for (int f = 0; f < MP; ++f) {
              if (f < m) {
                const double d = __dsub_rn((double)xs[f], cc[f]);
                d2 = __dadd_rn(d2, __dmul_rn(d, d));
              }
            }
            if (bl == 0x7fffffff || d2 < bd) { bd = d2; bl = c; }
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double obd = __shfl_xor_sync(0xffffffffu, bd, o);
          const int obl = __shfl_xor_sync(0xffffffffu, bl, o);
          if (obl != 0x7fffffff && (bl == 0x7fffffff || obd < bd || (obd == bd && obl < bl))) { bd = obd; bl = obl; }
        }
        if ((int)(threadIdx.x & 31) == src) {
          lab = bl;
          ++my_rechecks;
        }
      }
      if (!live[p]) continue;
      a.labels[row[p]] = lab;
      if (SMEM_ACC) {
        atomicAdd(reinterpret_cast<unsigned int*>(cnt + lab), 1u);  // counts < 2^32 per CTA
        if (DO_SUMS) {
          unsigned long long* dst = acc + (size_t)lab * m;
#pragma unroll
          for (int f = 0; f < MP; ++f)
            if (f < m) smem_add64(dst + f, (unsigned long long)to_fixed<float>(lane_f32x2(xp2[f], p), a.scale_f, a.scale_d, a.use_dscale));
        }
      } else {
        atomicAdd(cnt + lab, 1ull);
        if (DO_SUMS) {
          unsigned long long* dst = acc + (size_t)lab * m;
#pragma unroll
          for (int f = 0; f < MP; ++f)
            if (f < m) atomicAdd(dst + f, (unsigned long long)to_fixed<float>(lane_f32x2(xp2[f], p), a.scale_f, a.scale_d, a.use_dscale));
        }
      }
    }
  }
  unsigned int wsum = my_rechecks;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
  if ((tid & 31) == 0 && wsum) atomicAdd(&a.st->rechecked, (unsigned long long)wsum);
  if (SMEM_ACC) {
    __syncthreads();
    for (int i = tid; i < k * m; i += kBlkThreads)
      if (s_acc[i]) atomicAdd(g_acc + i, s_acc[i]);
    for (int i = tid; i < k; i += kBlkThreads)
      if (s_cnt[i]) atomicAdd(g_cnt + i, s_cnt[i]);
  }
}

// Per-block coordinate / cluster sums of a sample range (the COORD_SUM / CLUSTER_SUM device
// jobs, device.py:117-134, 218-239 → _kernels.coord_sums_block / cluster_sums_block,
// _kernels.py:84-113).  CTA = one chunk of ≤ kChunk samples inside one accumulation block;
// exact int64 fixed-point sums in shared memory (labels == nullptr: every sample in cluster 0),
// flushed into acc[(block · k + c) · m + f] and counts into acc[nb·k·m + block · k + c].  A label
// outside [0, k) lowers *bad to its sample index (the reference reports the first one).
constexpr int kBlockSumChunk = 8192;
template <typename T>
__global__ void __launch_bounds__(256) block_sums_kernel(const T* __restrict__ x, int m, int64_t start, int64_t stop,
                                                         int64_t block, int64_t chunks_per_block,
                                                         const int32_t* __restrict__ labels, int k, float sf,
                                                         double sd, int use_d, int64_t nb,
                                                         unsigned long long* __restrict__ acc,
                                                         unsigned long long* __restrict__ bad) {
  extern __shared__ unsigned long long s_blk[];  // k·m sums, then k counts
  const int km = k * m;
  for (int i = threadIdx.x; i < km + k; i += blockDim.x) s_blk[i] = 0ull;
  __syncthreads();
  const int64_t b = blockIdx.x / chunks_per_block, c = blockIdx.x % chunks_per_block;
  const int64_t bs = start + b * block;
  const int64_t be = min(stop, bs + block);
  const int64_t c0 = bs + c * kBlockSumChunk;
  const int64_t c1 = min(be, c0 + kBlockSumChunk);
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
    const int lab = labels ? labels[i - start] : 0;
    if (lab < 0 || lab >= k) {
      atomicMin(bad, (unsigned long long)i);
      continue;
    }
    const T* xr = x + i * m;
    for (int f = 0; f < m; ++f)
      smem_add64(s_blk + (size_t)lab * m + f, (unsigned long long)to_fixed<T>(xr[f], sf, sd, use_d));
    smem_add64(s_blk + km + lab, 1ull);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < km; i += blockDim.x)
    if (s_blk[i]) atomicAdd(acc + (size_t)b * km + i, s_blk[i]);
  for (int i = threadIdx.x; i < k; i += blockDim.x)
    if (s_blk[km + i]) atomicAdd(acc + (size_t)nb * km + (size_t)b * k + i, s_blk[km + i]);
}

__global__ void __launch_bounds__(512) lloyd_finish_kernel(FinishArgs a, int stage_cap) {
  extern __shared__ double s_stage[];
  finish_block(a, stage_cap > 0 ? s_stage : nullptr, stage_cap);
}


// The loop finish (finish_block mode 0, same decisions) for m ≤ 32 with warp per centre and lane
// per feature: fold Δ, C_t = S/N, empties, the congruence test and the filter operands in one
// parallel pass — the single-CTA serial chains of finish_block cost ~10 µs per iteration.
__global__ void __launch_bounds__(512) lloyd_finish_warp_kernel(FinishArgs a) {
  DevState* st = a.st;
  const int k = a.k, m = a.m, km = k * m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (st->done || st->need_host) return;
  __shared__ int s_flags[32];
  __shared__ float s_max[32];
  if (tid == 0 && a.recheck_count) {
    st->rechecked += *a.recheck_count;
    *a.recheck_count = 0u;
  }
  // running totals of the current labels (exact integer arithmetic)
  for (int i = tid; i < km + k; i += blockDim.x) {
    a.tot[i] = a.accumulate ? a.tot[i] + a.part[i] : a.part[i];
    a.part[i] = 0ull;
  }
  __syncthreads();
  const unsigned long long* cnts = a.tot + km;
  if (st->exhausted) {  // the final assign pass of an exhausted run: counts = bincount(L_T)
    for (int c = tid; c < k; c += blockDim.x) a.model_counts[c] = (long long)cnts[c];
    if (tid == 0) st->done = 1;
    return;
  }
  const double tol = st->tol;
  const int hw = 8 * ((m + 1 + 7) / 8);
  int flags = 0;   // bit 0: some cluster empty, bit 1: some centre moved
  float wmax = 0.f;
  for (int c = warp; c < k; c += nw) {
    const long long nc = (long long)cnts[c];
    const bool fv = lane < m;
    const long long sv = fv ? (long long)a.tot[(size_t)c * m + lane] : 0ll;
    const double v = (fv && nc > 0) ? __ddiv_rn(__dmul_rn((double)sv, a.inv_scale), (double)nc) : 0.0;
    const double vo = fv ? a.cur[(size_t)c * m + lane] : 0.0;
    if (fv) {
      a.prev[(size_t)c * m + lane] = vo;
      a.cur[(size_t)c * m + lane] = v;
    }
    if (lane == 0) a.model_counts[c] = nc;
    const double dd = fv ? __dmul_rn(__dsub_rn(vo, v), __dsub_rn(vo, v)) : 0.0;
    bool moved;
    if (tol == 0.0) {
      moved = __any_sync(0xffffffffu, dd != 0.0);
    } else {
      double acc = 0.0;  // the reference order: features ascending
      for (int f = 0; f < m; ++f) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, dd, f));
      moved = !(sqrt(acc) <= tol);
    }
    flags |= (nc == 0 ? 1 : 0) | (moved ? 2 : 0);
    // filter operands: ‖fl32(c)‖² (fp64, exact squares), max ‖c‖, SIMT w / cn, tensor-core rows
    const float v32 = __double2float_rn(v);
    const double q = fv ? (double)v32 : 0.0;
    double cn2 = q * q;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cn2 += __shfl_xor_sync(0xffffffffu, cn2, o);
    wmax = fmaxf(wmax, __double2float_ru(sqrt(cn2) * (1.0 + 1e-12)));
    if (lane == 0) a.cn[c] = __double2float_rn(cn2);
    for (int f = lane; f < a.mpad; f += 32) a.w[(size_t)c * a.mpad + f] = (f < m) ? -2.0f * v32 : 0.0f;
    if (a.wop != nullptr) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = lane + 32 * h;
        const int f = col < hw ? col : col - hw;
        const double vf = __shfl_sync(0xffffffffu, v, f < 32 ? f : 0);
        float w = 0.f;
        if (col < 2 * hw) {
          if (f < m) w = -2.0f * __double2float_rn(vf) * a.pre;
          else if (f == m) w = __double2float_rn(cn2 * (double)a.pre * (double)a.pre);
        }
        const __half wh = __float2half_rn(w);
        const __half wl = __float2half_rn(w - __half2float(wh));
        a.wop[(size_t)c * 64 + col] = (col < 2 * hw) ? __half_as_ushort(wh) : (unsigned short)0;
        a.wop[(size_t)(a.kp + c) * 64 + col] = (col < hw) ? __half_as_ushort(wl) : (unsigned short)0;
      }
    }
  }
  if (lane == 0) {
    s_flags[warp] = flags;
    s_max[warp] = wmax;
  }
  __syncthreads();
  if (tid == 0) {
    int fl = 0;
    float mx = 0.f;
    for (int w = 0; w < nw; ++w) {
      fl |= s_flags[w];
      mx = fmaxf(mx, s_max[w]);
    }
    st->t += 1;
    int ne = 0;
    for (int c = 0; c < k; ++c) ne += (cnts[c] == 0ull);
    st->n_empty = ne;
    if (fl & 1) {
      st->need_host = 1;  // empty clusters: the host repairs, then the check kernel runs the test
    } else {
      a.cmax[0] = mx;
      st->need_host = 0;
      if (!(fl & 2)) {
        st->converged = 1;
        st->done = 1;
      } else if (st->t >= st->max_iters) {
        st->exhausted = 1;  // reference: assignment = assign_fn(model) once more, then return
      }
    }
  }
}

// After a host-driven repair: congruence test + prep (no division).
__global__ void __launch_bounds__(512) lloyd_check_kernel(FinishArgs a) {
  __shared__ float s_red[32];
  __shared__ double s_redd[32];
  loop_check(a, s_redd, s_red);
}

// Filter prep only (initial centres, standalone assign).
__global__ void __launch_bounds__(512) prep_filter_kernel(const double* c, float* w, float* cn, float* cmax,
                                                          int k, int m, int mpad, unsigned short* wop, int kp,
                                                          float pre) {
  __shared__ float s_red[32];
  block_prep_filter(c, w, cn, cmax, k, m, mpad, s_red, wop, kp, pre);
}

// Start of a resident Lloyd run (km_lloyd, tensor-core path), one launch instead of a state
// upload + five memsets + the prep kernel: loop state {max_iters, tol}, zeroed Δ / totals /
// rotating delta buffers / grid-barrier counter / recheck counter, and the filter operands of C0.
// C0 of a km_lloyd call passed by value in the begin kernel's launch parameters when it fits
// (k·m ≤ 480: no host→device copy in front of the run)
constexpr int kC0Inline = 480;
struct C0Inline {
  double v[kC0Inline];
};

__global__ void __launch_bounds__(512) lloyd_begin_kernel(DevState* st, int max_iters, double tol,
                                                          unsigned long long* part, unsigned long long* tot,
                                                          unsigned long long* dlt, size_t nacc,
                                                          unsigned int* grid_sync, unsigned int* recheck_count,
                                                          double* c, float* w, float* cn, float* cmax, int k,
                                                          int m, int mpad, unsigned short* wop, int kp, float pre,
                                                          const __grid_constant__ C0Inline c0, int c0_n) {
  __shared__ float s_red[32];
  if (c0_n > 0) {  // C0 from the launch parameters (else the caller copied it to c)
    for (int i = threadIdx.x; i < c0_n; i += blockDim.x) c[i] = c0.v[i];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    DevState s{};
    s.max_iters = max_iters;
    s.tol = tol;
    *st = s;
    grid_sync[0] = grid_sync[1] = grid_sync[2] = grid_sync[3] = 0u;
    *recheck_count = 0u;
  }
  for (size_t i = threadIdx.x; i < nacc; i += blockDim.x) {
    part[i] = 0ull;
    tot[i] = 0ull;
  }
  for (size_t i = threadIdx.x; i < 3 * nacc; i += blockDim.x) dlt[i] = 0ull;
  block_prep_filter(c, w, cn, cmax, k, m, mpad, s_red, wop, kp, pre);
}

// End of a km_lloyd call: state, centres and counts straight into the caller's pinned (mapped)
// staging — one launch instead of three device→host copies.
__global__ void __launch_bounds__(256) lloyd_publish_kernel(const DevState* st, const double* cur,
                                                            const long long* counts, int km, int k, DevState* h_st,
                                                            double* h_c, long long* h_n) {
  if (threadIdx.x == 0) *h_st = *st;
  for (int i = threadIdx.x; i < km; i += blockDim.x) h_c[i] = cur[i];
  for (int i = threadIdx.x; i < k; i += blockDim.x) h_n[i] = counts[i];
}

// Standalone congruence test (km_converged).
__global__ void __launch_bounds__(512) converged_kernel(const double* prev, const double* next, int k, int m,
                                                        double tol, int* out) {
  __shared__ double s_redd[32];
  const int c = block_converged(prev, next, k, m, tol, s_redd);
  if (threadIdx.x == 0) *out = c;
}

// ---------------------------------------------------------------------------
// Empty-cluster repair (engine.py:265-276): d2_i = ‖x_i − C[label_i]‖² (fp64,
// _kernels.self_distances_block :116-126); per empty cluster (ascending):
// s = argmax d2 (first index), relabel s, move one count, C[c] = x_s, d2_s = 0.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void self_d2_kernel(const T* __restrict__ x, int64_t n, int m, const double* __restrict__ c,
                               const int32_t* __restrict__ labels, double* __restrict__ d2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d2[i] = exact_d2<T>(x + i * m, c + (size_t)labels[i] * m, m);
}

struct ArgMax { double v; long long i; };

__device__ __forceinline__ ArgMax argmax_better(ArgMax a, ArgMax b) {
  // larger value wins; equal values → lower index (np.argmax returns the first)
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

// Block-wide reduction of the per-block partials (any blockDim ≤ 1024, multiple of 32):
// argmax_better is a total order (value desc, index asc), so the result is order-independent.
// The serial one-thread loop over thousands of partials cost ~100 µs per repair.
__device__ __forceinline__ ArgMax argmax_reduce_block(const ArgMax* partial, int nparts) {
  __shared__ ArgMax s_red[32];
  ArgMax best{-1.0, 0x7fffffffffffffffLL};
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) best = argmax_better(best, partial[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax other;
    other.v = __shfl_xor_sync(0xffffffffu, best.v, o);
    other.i = __shfl_xor_sync(0xffffffffu, best.i, o);
    best = argmax_better(best, other);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) s_red[warp] = best;
  __syncthreads();
  if (warp == 0) {
    best = lane < nw ? s_red[lane] : ArgMax{-1.0, 0x7fffffffffffffffLL};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ArgMax other;
      other.v = __shfl_xor_sync(0xffffffffu, best.v, o);
      other.i = __shfl_xor_sync(0xffffffffu, best.i, o);
      best = argmax_better(best, other);
    }
  }
  return best;  // valid in thread 0
}

__global__ void argmax_partial_kernel(const double* __restrict__ d2, int64_t n, ArgMax* partial) {
  ArgMax best{-1.0, (long long)n};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    best = argmax_better(best, ArgMax{d2[i], (long long)i});
  __shared__ ArgMax s[32];
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax other{__shfl_xor_sync(0xffffffffu, best.v, o), __shfl_xor_sync(0xffffffffu, best.i, o)};
    best = argmax_better(best, other);
  }
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = argmax_better(best, s[w]);
    partial[blockIdx.x] = best;
  }
}

// One thread: reduce the partials, apply the relabel for empty cluster `c`.
// Move sample s (fixed-point coordinates) from cluster `donor` to `c` in the running totals.
__device__ __forceinline__ void move_in_totals(unsigned long long* tot, int k, int m, int donor, int c,
                                               const double* coords, double scale_d) {
  for (int f = 0; f < m; ++f) {
    const unsigned long long v = (unsigned long long)__double2ll_rn(__dmul_rn(coords[f], scale_d));
    tot[(size_t)donor * m + f] -= v;
    tot[(size_t)c * m + f] += v;
  }
  tot[(size_t)k * m + donor] -= 1ull;
  tot[(size_t)k * m + c] += 1ull;
}

template <typename T>
__global__ void repair_apply_kernel(const ArgMax* partial, int nparts, int c, const T* __restrict__ x, int k, int m,
                                    int32_t* labels, double* d2, long long* model_counts, double* cur,
                                    unsigned long long* tot, double scale_d, ArgMax* winner_out) {
  const ArgMax best = argmax_reduce_block(partial, nparts);
  if (threadIdx.x != 0) return;
  const long long s = best.i;
  const int donor = labels[s];
  labels[s] = c;
  model_counts[donor] -= 1;
  model_counts[c] += 1;
  for (int f = 0; f < m; ++f) cur[(size_t)c * m + f] = to_f64(x[s * m + f]);
  move_in_totals(tot, k, m, donor, c, cur + (size_t)c * m, scale_d);
  d2[s] = 0.0;
  if (winner_out) *winner_out = best;
}

// Local candidate only (multi-GPU repair: the caller picks the global winner).
__global__ void argmax_final_kernel(const ArgMax* partial, int nparts, ArgMax* out) {
  const ArgMax best = argmax_reduce_block(partial, nparts);
  if (threadIdx.x == 0) *out = best;
}

// Apply a repair decided across shards.
__global__ void repair_apply_global_kernel(int c, int owner, long long local_row, const double* coords, int donor,
                                           int k, int m, int32_t* labels, double* d2, long long* model_counts,
                                           double* cur, unsigned long long* tot, double scale_d) {
  if (threadIdx.x != 0) return;
  if (owner) {
    labels[local_row] = c;
    d2[local_row] = 0.0;
  }
  model_counts[donor] -= 1;
  model_counts[c] += 1;
  for (int f = 0; f < m; ++f) cur[(size_t)c * m + f] = coords[f];
  move_in_totals(tot, k, m, donor, c, coords, scale_d);
}

// ---------------------------------------------------------------------------
// Reporting neighbours of the hot path.
// ---------------------------------------------------------------------------
// wcss: Σ_i ‖x_i − C[label_i]‖² — each term exactly as _kernels.wcss_block,
// the total accumulated in 2^-(F2) fixed point (exact integer adds, so the
// total does not depend on the reduction order).
template <typename T>
__global__ void wcss_kernel(const T* __restrict__ x, int64_t n, int m, const double* __restrict__ c,
                            const int32_t* __restrict__ labels, double scale, unsigned long long* out_hi_lo) {
  long long acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = exact_d2<T>(x + i * m, c + (size_t)labels[i] * m, m);
    acc += __double2ll_rn(__dmul_rn(d, scale));
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out_hi_lo, (unsigned long long)acc);
}

// transform: out[i,c] = sqrt(exact_d2(x_i, C_c))  (_kernels.center_distances :158-170)
template <typename T>
__global__ void center_distances_kernel(const T* __restrict__ x, int64_t n, int m, const double* __restrict__ c,
                                        int k, double* __restrict__ out) {
  const int64_t total = n * (int64_t)k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / k;
    const int cc = (int)(idx - i * k);
    out[idx] = sqrt(exact_d2<T>(x + i * m, c + (size_t)cc * m, m));
  }
}

// max |x| (exact) for the fixed-point scale; flags[0] |= non-finite seen,
// flags[1] |= value not exactly representable in fp32 (fp64 input only).
template <typename T>
__global__ void absmax_kernel(const T* __restrict__ x, int64_t count, unsigned long long* out_bits,
                              int* flags) {
  double mx = 0.0;
  int bad = 0, inexact = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = to_f64(x[i]);
    if (!isfinite(v)) { bad = 1; continue; }
    mx = fmax(mx, fabs(v));
    if (sizeof(T) == 8 && (double)__double2float_rn(v) != v) inexact = 1;
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  bad = __any_sync(0xffffffffu, bad);
  inexact = __any_sync(0xffffffffu, inexact);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out_bits, (unsigned long long)__double_as_longlong(mx));
    if (bad) atomicOr(flags, 1);
    if (inexact) atomicOr(flags + 1, 1);
  }
}

// max over rows of ‖x_i‖ (fp64 sums, rounded up to fp32) for the per-launch filter bound
template <typename T>
__global__ void rownorm_max_kernel(const T* __restrict__ x, int64_t n, int m, unsigned int* out_bits) {
  float mx = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int f = 0; f < m; ++f) {
      const double v = to_f64(x[i * m + f]);
      s = __fma_rn(v, v, s);
    }
    mx = fmaxf(mx, __double2float_ru(sqrt(s) * (1.0 + 1e-12)));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out_bits, __float_as_uint(mx));  // non-negative floats order as uints
}

__global__ void narrow_f64_kernel(const double* __restrict__ in, int64_t count, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __double2float_rn(in[i]);
}

// int32 labels → int64 (download path)
__global__ void widen_labels_kernel(const int32_t* __restrict__ in, int64_t n, long long* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

}  // namespace km
