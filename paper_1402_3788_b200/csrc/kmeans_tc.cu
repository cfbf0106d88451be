// kmeans_tc.cu — instantiations + launcher of the tcgen05 fused pass.
#include <algorithm>
#include <cstdio>

#include "kmeans_tc.cuh"
#include "kmeans_tc_dispatch.h"

namespace km {
namespace tc {

// Exact re-decision of the queued points: the reference's fp64 recurrence over
// ALL centres (_kernels.py:22-45: features ascending, no FMA; argmin with the
// lowest index on ties), then the same Δ update of the fixed-point sums
// (global atomics).  One warp per queued point, lane = centre (each lane keeps
// the reference's sequential feature order); centres staged in shared memory.
__global__ void __launch_bounds__(256) recheck_kernel(const float* __restrict__ x, const double* __restrict__ x64,
                                                      int m, int k,
                                                      const double* __restrict__ c64, int32_t* labels,
                                                      const long long* rows, const unsigned int* count,
                                                      unsigned long long* part, float scale_f, double scale_d,
                                                      int use_dscale, int full, int no_sums, DevState* st,
                                                      int gate) {
  if (gate && (st->done || st->need_host)) return;
  const unsigned int cnt = *count;
  if (cnt == 0) return;
  extern __shared__ double s_c[];  // k × m when it fits (host decides), else global
  const bool staged = k * m <= 6144;
  if (staged) {
    for (int i = threadIdx.x; i < k * m; i += blockDim.x) s_c[i] = c64[i];
    __syncthreads();
  }
  const double* C = staged ? s_c : c64;
  const int lane = threadIdx.x & 31;
  const unsigned int warps = (gridDim.x * blockDim.x) >> 5;
  for (unsigned int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < cnt; q += warps) {
    const long long row = rows[q];
    // m ≤ 31 on the tensor-core path; fp64 points: the exact row (not the fp32 shadow)
    const double xl = lane >= m ? 0.0 : x64 ? __ldg(x64 + row * m + lane) : (double)__ldg(x + row * m + lane);
    double bd = 0.0;
    int bl = -1;
    for (int c0 = 0; c0 < k; c0 += 32) {
      const int c = c0 + lane;
      double acc = 0.0;
      for (int f = 0; f < m; ++f) {
        const double xv = __shfl_sync(0xffffffffu, xl, f);
        if (c < k) {
          const double d = __dsub_rn(xv, C[(size_t)c * m + f]);
          acc = __dadd_rn(acc, __dmul_rn(d, d));
        }
      }
      if (c < k && (bl < 0 || acc < bd)) { bd = acc; bl = c; }
    }
    // warp argmin: smaller distance, then the lower index (the reference's strict '<' scan)
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (ol >= 0 && (bl < 0 || od < bd || (od == bd && ol < bl))) { bd = od; bl = ol; }
    }
    const int old = full ? -1 : labels[row];
    if (bl != old) {
      if (no_sums) {  // first pass of a run: labels only (the cluster-sums kernel adds the points)
        if (lane == 0) labels[row] = bl;
        continue;
      }
      if (lane == 0) {
        labels[row] = bl;
        atomicAdd(part + (size_t)k * m + bl, 1ull);
        if (old >= 0) atomicAdd(part + (size_t)k * m + old, ~0ull);
        if (!full) atomicAdd(&st->changed, 1ull);
      }
      if (lane < m) {
        const long long v = use_dscale || x64 ? __double2ll_rn(__dmul_rn(xl, scale_d))
                                              : __float2ll_rn(__fmul_rn((float)xl, scale_f));
        atomicAdd(part + (size_t)bl * m + lane, (unsigned long long)v);
        if (old >= 0) atomicAdd(part + (size_t)old * m + lane, (unsigned long long)(-v));
      }
    }
  }
}


cudaError_t launch_recheck(const TcArgs& a, int num_sms, cudaStream_t stream) {
  const size_t smem = (size_t)a.k * a.m <= 6144 ? (size_t)a.k * a.m * 8 : 0;
  // one resident warp per queued point (≈ 64 warps/SM): the per-point latency is a few L2 loads
  recheck_kernel<<<num_sms * 8, 256, smem, stream>>>(a.x, a.x64, a.m, a.k, a.c64, a.labels, a.recheck_rows, a.recheck_count,
                                                     a.part, a.scale_f, a.scale_d, a.use_dscale, a.full, a.no_sums, a.st,
                                                     a.gate);
  return cudaGetLastError();
}

int launch(const TcArgs& a, int mp, int kp, int num_sms, size_t smem_optin, cudaStream_t stream,
           cudaError_t* ce, char* msg, size_t len) {
  if (a.x64) return launch_f64(a, a.m, mp, kp, num_sms, smem_optin, stream, ce, msg, len);
  if (a.exact_m) {
    const int r = launch_exact(a, a.m, kp, a.prescale != 0, num_sms, smem_optin, stream, ce, msg, len);
    if (r >= 0) return r;
  }
  return launch_bucket(a, mp, kp, num_sms, smem_optin, stream, ce, msg, len);
}

}  // namespace tc
}  // namespace km
