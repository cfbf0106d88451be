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
// Layout: lane f of a warp owns feature f of every row it reads (lane m counts); the row's label
// is warp-uniform, so one warp instruction adds a whole row into accumulator row `label` with
// distinct addresses per lane.  PRIV: every warp owns a private [k][m+1] int64 accumulator in
// shared memory (plain LDS/IADD/STS, no atomics); otherwise (large k·m) the CTA shares one copy
// updated with 32-bit atomic pairs.  Rows are read 8 at a time per warp (8 independent loads per
// lane in flight), each warp a contiguous row range (sequential DRAM pages).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kmeans_kernels.cuh"

namespace km {

constexpr int kSumsThreads = 256;
constexpr int kSumsRows = 8;  // rows per warp batch

template <bool PRIV>
__global__ void __launch_bounds__(kSumsThreads) cluster_sums_f32_kernel(
    const float* __restrict__ x, const int32_t* __restrict__ labels, int64_t n, int m, int k, float scale_f,
    double scale_d, int use_dscale, unsigned long long* __restrict__ out /* [k·m sums][k counts] */) {
  extern __shared__ unsigned long long s_acc[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int W = kSumsThreads / 32;
  const int row_len = m + 1;
  const int per = k * row_len;
  const int copies = PRIV ? W : 1;
  for (int i = threadIdx.x; i < per * copies; i += kSumsThreads) s_acc[i] = 0ull;
  __syncthreads();
  unsigned long long* acc = s_acc + (PRIV ? (size_t)warp * per : 0);

  const int64_t gw = (int64_t)blockIdx.x * W + warp, nw = (int64_t)gridDim.x * W;
  const int64_t r_lo = n * gw / nw, r_hi = n * (gw + 1) / nw;
  const bool feat = lane < m, cnt_lane = lane == m;
  for (int64_t r = r_lo; r < r_hi; r += kSumsRows) {
    const int rows = (int)(r_hi - r < (int64_t)kSumsRows ? r_hi - r : (int64_t)kSumsRows);
    const int lab = lane < rows ? __ldg(labels + r + lane) : 0;
    float v[kSumsRows];
#pragma unroll
    for (int j = 0; j < kSumsRows; ++j) v[j] = (feat && j < rows) ? __ldg(x + (r + j) * m + lane) : 0.f;
#pragma unroll
    for (int j = 0; j < kSumsRows; ++j) {
      const int L = __shfl_sync(0xffffffffu, lab, j);
      if (j < rows && (unsigned)L < (unsigned)k) {
        unsigned long long* dst = acc + (size_t)L * row_len + lane;
        if (feat) {
          const unsigned long long q = (unsigned long long)to_fixed<float>(v[j], scale_f, scale_d, use_dscale);
          if (PRIV) *dst += q; else smem_add64(dst, q);
        } else if (cnt_lane) {
          if (PRIV) *dst += 1ull; else smem_add64(dst, 1ull);
        }
      }
    }
  }
  __syncthreads();
  // one global atomic per non-zero accumulator and CTA
  for (int i = threadIdx.x; i < per; i += kSumsThreads) {
    unsigned long long s = 0;
    for (int w = 0; w < copies; ++w) s += s_acc[(size_t)w * per + i];
    if (s) {
      const int c = i / row_len, f = i - c * row_len;
      atomicAdd(out + (f < m ? (size_t)c * m + f : (size_t)k * m + c), s);
    }
  }
}

}  // namespace km
