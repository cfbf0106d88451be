// kmeans_seed.cuh — seeding phase on the device: the dataset diameter
// (engine.diameter / _kernels.max_pair_rows, engine.py:141-154, _kernels.py:49-81) and the
// maximin centre choice (engine.init_centers, engine.py:171-215, _kernels.update_min_d2
// _kernels.py:144-155).
//
// Diameter: a tiled pair scan over rows i ∈ {0, s, 2s, …} (engine.scan_rows) × columns j > i.
//   Phase 1 computes every pair's squared distance in fp32 (points are fp32-exact, so the
//   only errors are the roundings of x_i − x_j, the squares and the m-term sum: relative
//   error ≤ γ = (m+4)·2^-24) and keeps the maximum M32.  Phase 2 rescans and re-evaluates
//   every pair whose fp32 value could still reach the maximum (d²₃₂ ≥ M32·(1−γ)/(1+γ)) with the
//   reference's exact fp64 recurrence, keeping the lexicographic best (largest d², then the
//   smallest i, then the smallest j — the strict '>' scan order of max_pair_rows).  Data whose
//   fp32 squares could under/overflow, or fp64-resident points, run phase 2 over every pair.
// Maximin: min_d2 (fp64, exact recurrence) is lowered by each chosen centre in one pass that
//   also produces per-block argmax partials (largest, then the lowest index = np.argmax).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace km {

struct PairBest {
  double d2;
  long long i, j;
};

__device__ __forceinline__ bool pair_better(const PairBest& b, const PairBest& a) {  // b better than a?
  if (b.d2 != a.d2) return b.d2 > a.d2;
  if (b.i != a.i) return b.i < a.i;
  return b.j < a.j;
}

constexpr int kPairRows = 32;   // rows per tile
constexpr int kPairCols = 256;  // columns per tile (= threads per block)
constexpr int kPairFeat = 16;   // features staged per step

// PHASE 1: fp32 maximum into *max_bits (non-negative float bits, atomicMax).
// PHASE 2: pairs with d²₃₂ ≥ thr get the exact fp64 value; per-block best into out[blockIdx].
template <typename T, bool PHASE2>
__global__ void __launch_bounds__(kPairCols) pair_scan_kernel(const T* __restrict__ x, int64_t n, int m,
                                                              int64_t stride, int64_t R, float thr,
                                                              unsigned int* max_bits, PairBest* out,
                                                              const long long* __restrict__ rows = nullptr) {
  // scan row r is r·stride (engine.scan_rows), or rows[r] for an explicit ascending row list
  // (a MAX_PAIR device job, device.py:117-122)
  auto row_of = [&](int64_t r) -> int64_t { return rows ? (int64_t)rows[r] : r * stride; };
  __shared__ float s_row[kPairFeat][kPairRows];
  __shared__ float s_col[kPairFeat][kPairCols];
  __shared__ PairBest s_best[kPairCols / 32];
  __shared__ float s_max[kPairCols / 32];
  const int tid = threadIdx.x;
  const int64_t RT = (R + kPairRows - 1) / kPairRows;
  const int64_t CT = (n + kPairCols - 1) / kPairCols;
  float tmax = 0.f;
  PairBest best{-1.0, -1, -1};
  for (int64_t t = blockIdx.x; t < RT * CT; t += gridDim.x) {
    const int64_t rt = t / CT, ct = t - rt * CT;
    const int64_t r0 = rt * kPairRows;
    const int64_t i_min = row_of(r0);  // rows ascending: the tile's smallest row
    const int64_t j0 = ct * kPairCols;
    if (j0 + kPairCols - 1 <= i_min) continue;  // tile entirely on or below the diagonal (block-uniform)
    const int nr = (int)((R - r0) < kPairRows ? (R - r0) : kPairRows);
    const int64_t j = j0 + tid;
    float acc[kPairRows];
#pragma unroll
    for (int r = 0; r < kPairRows; ++r) acc[r] = 0.f;
    for (int f0 = 0; f0 < m; f0 += kPairFeat) {
      const int fc = min(kPairFeat, m - f0);
      __syncthreads();
      for (int e = tid; e < kPairRows * kPairFeat; e += kPairCols) {
        const int r = e / kPairFeat, f = e - r * kPairFeat;
        s_row[f][r] = (r < nr && f < fc) ? (float)x[row_of(r0 + r) * m + f0 + f] : 0.f;
      }
      for (int f = 0; f < fc; ++f) s_col[f][tid] = (j < n) ? (float)x[j * m + f0 + f] : 0.f;
      __syncthreads();
      for (int f = 0; f < fc; ++f) {
        const float xj = s_col[f][tid];
#pragma unroll
        for (int r = 0; r < kPairRows; ++r) {
          const float d = s_row[f][r] - xj;
          acc[r] = __fmaf_rn(d, d, acc[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kPairRows; ++r) {
      const int64_t i = r < nr ? row_of(r0 + r) : n;
      const bool valid = r < nr && j < n && j > i;
      if (!PHASE2) {
        if (valid) tmax = fmaxf(tmax, acc[r]);
      } else if (valid && acc[r] >= thr) {
        double d2 = 0.0;  // the reference recurrence: features ascending, fp64, no FMA
        for (int f = 0; f < m; ++f) {
          const double d = __dsub_rn((double)x[i * m + f], (double)x[j * m + f]);
          d2 = __dadd_rn(d2, __dmul_rn(d, d));
        }
        const PairBest cand{d2, (long long)i, (long long)j};
        if (pair_better(cand, best)) best = cand;
      }
    }
  }
  const int lane = tid & 31, w = tid >> 5;
  if (!PHASE2) {
    for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    if (lane == 0) s_max[w] = tmax;
    __syncthreads();
    if (tid == 0) {
      float mx = 0.f;
      for (int k = 0; k < kPairCols / 32; ++k) mx = fmaxf(mx, s_max[k]);
      atomicMax(max_bits, __float_as_uint(mx));
    }
  } else {
    for (int o = 16; o > 0; o >>= 1) {
      const PairBest other{__shfl_xor_sync(0xffffffffu, best.d2, o), __shfl_xor_sync(0xffffffffu, best.i, o),
                           __shfl_xor_sync(0xffffffffu, best.j, o)};
      if (pair_better(other, best)) best = other;
    }
    if (lane == 0) s_best[w] = best;
    __syncthreads();
    if (tid == 0) {
      for (int k = 1; k < kPairCols / 32; ++k)
        if (pair_better(s_best[k], best)) best = s_best[k];
      out[blockIdx.x] = best;
    }
  }
}

// min_d2[i] = min(min_d2[i], d²(x_i, x_c)) with the reference recurrence (update_min_d2), then
// per-block argmax partials of the lowered array (largest, lowest index).
template <typename T>
__global__ void __launch_bounds__(256) min_d2_update_kernel(const T* __restrict__ x, int64_t n, int m, int64_t c,
                                                            double* __restrict__ min_d2, double* __restrict__ part_v,
                                                            long long* __restrict__ part_i) {
  extern __shared__ double s_c[];  // the chosen centre (m doubles)
  for (int f = threadIdx.x; f < m; f += blockDim.x) s_c[f] = (double)x[c * m + f];
  __syncthreads();
  double bv = -1.0;
  long long bi = (long long)n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double d2 = 0.0;
    for (int f = 0; f < m; ++f) {
      const double d = __dsub_rn((double)x[i * m + f], s_c[f]);
      d2 = __dadd_rn(d2, __dmul_rn(d, d));
    }
    double v = min_d2[i];
    if (d2 < v) {
      v = d2;
      min_d2[i] = v;
    }
    if (v > bv) {  // ascending i per thread: strict '>' keeps the first
      bv = v;
      bi = (long long)i;
    }
  }
  __shared__ double s_v[8];
  __shared__ long long s_i[8];
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { s_v[threadIdx.x >> 5] = bv; s_i[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (s_v[w] > bv || (s_v[w] == bv && s_i[w] < bi)) { bv = s_v[w]; bi = s_i[w]; }
    part_v[blockIdx.x] = bv;
    part_i[blockIdx.x] = bi;
  }
}

__global__ void fill_f64_kernel(double* p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace km
