// kmeans_finish.cuh — block-level finish of a Lloyd iteration (device functions only; shared by
// the standalone finish kernel and the last CTA of the fused tensor-core pass).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kmeans_state.h"

namespace km {

// Exact re-decision of one point by a warp: the reference recurrence (_kernels.py:31-44:
// features ascending, d = x − c, acc += d·d, no FMA) per centre, lane = centre, argmin with the
// lowest index on ties.  x_lane holds feature `lane` (m ≤ 32).  Returns the label (all lanes).
template <int MMAX = 32, typename T = float>
__device__ __forceinline__ int exact_label_warp(T x_lane, int m, int k, const double* __restrict__ c64) {
  const int lane = threadIdx.x & 31;
  double bd = 0.0;
  int bl = -1;
  for (int c0 = 0; c0 < k; c0 += 32) {
    const int c = c0 + lane;
    const int cl = c < k ? c : 0;
    double acc = 0.0;
#pragma unroll
    for (int f = 0; f < MMAX; ++f) {  // unrolled: centre loads issue up front; fp64 chain in feature order
      if (f < m) {
        const double xv = (double)__shfl_sync(0xffffffffu, x_lane, f);
        const double d = __dsub_rn(xv, c64[(size_t)cl * m + f]);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
      }
    }
    if (c < k && (bl < 0 || acc < bd)) { bd = acc; bl = c; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
    const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
    if (ol >= 0 && (bl < 0 || od < bd || (od == bd && ol < bl))) { bd = od; bl = ol; }
  }
  return bl;
}

// NB points per warp at once (lane = centre): the centre coordinate is loaded once
// per feature and NB independent fp64 chains hide the DADD latency; each chain is
// still the reference's exact sequential recurrence.
template <int MMAX, int NB>
__device__ __forceinline__ void exact_label_warp_batch(const float (&x_lane)[NB], int m, int k,
                                                       const double* __restrict__ c64, int (&label)[NB]) {
  const int lane = threadIdx.x & 31;
  double bd[NB];
  int bl[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) { bd[j] = 0.0; bl[j] = -1; }
  for (int c0 = 0; c0 < k; c0 += 32) {
    const int c = c0 + lane;
    const int cl = c < k ? c : 0;
    double acc[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[j] = 0.0;
#pragma unroll
    for (int f = 0; f < MMAX; ++f) {
      if (f < m) {
        const double cv = c64[(size_t)cl * m + f];
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          const double d = __dsub_rn((double)__shfl_sync(0xffffffffu, x_lane[j], f), cv);
          acc[j] = __dadd_rn(acc[j], __dmul_rn(d, d));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (c < k && (bl[j] < 0 || acc[j] < bd[j])) { bd[j] = acc[j]; bl[j] = c; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const double od = __shfl_xor_sync(0xffffffffu, bd[j], o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl[j], o);
      if (ol >= 0 && (bl[j] < 0 || od < bd[j] || (od == bd[j] && ol < bl[j]))) { bd[j] = od; bl[j] = ol; }
    }
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) label[j] = bl[j];
}

// ---------------------------------------------------------------------------
// Finish (one CTA): C_t = S/N (engine._finish_update, engine.py:249-263),
// empty-cluster count, then — if no cluster is empty — the congruence test
// (engine.converged, engine.py:297-310) and the fp32 filter prep.
// ---------------------------------------------------------------------------
struct FinishArgs {
  unsigned long long* part;  // k·m sums + k counts of the last pass (Δ or full; zeroed once consumed)
  unsigned long long* tot;   // k·m sums + k counts of the current labels (running totals)
  int32_t accumulate;        // 1: tot += part (incremental pass), 0: tot = part (full pass)
  unsigned int* recheck_count;  // global recheck queue length of the last pass (reset here)
  const long long* recheck_rows;  // global recheck queue (uncertified points not yet re-decided)
  const float* x;            // fp32 points (overflow recheck)
  const double* x64;         // fp64 points: the exact rows (x is then their fp32 shadow); else null
  int32_t* labels;
  int32_t full;              // the pass had no valid previous labels
  float scale_f;
  double scale_d;
  int32_t use_dscale;
  double* cur;               // k × m current centres (in: C_{t-1}; out: C_t)
  double* prev;              // k × m (out: C_{t-1})
  long long* model_counts;   // k (out)
  float* w;                  // k × mpad (out: −2·fl32(C_t))
  float* cn;                 // k
  float* cmax;               // [0]
  unsigned short* wop;       // [2kp][64] fp16 tensor-core B operand (nullable): [wh|wh], [wl|0]
  int32_t kp;
  float pre;                 // power-of-two prescale of the tensor-core operands
  int32_t k, m, mpad;
  double inv_scale;          // 2^-F
  DevState* st;
  int32_t mode;              // 0 = loop iteration, 1 = standalone update (no state machine)
};

__device__ __forceinline__ void block_prep_filter(const double* __restrict__ c, float* w, float* cn, float* cmax,
                                                  int k, int m, int mpad, float* s_red,
                                                  unsigned short* wop = nullptr, int kp = 0, float pre = 1.f) {
  // per centre: ‖fl32(c)‖² (fp64 sum of the fp32-rounded coordinates, rounded to fp32), its root
  // rounded up for the filter bound; then the SIMT operand w = −2·fl32(c) (zero padded) and the
  // tensor-core operand (fp16 hi/lo split of W~' = 2^s·(−2·fl32(c)), 2^2s·‖fl32(c)‖² at f = m):
  // row c < kp: [wh_c | wh_c], row kp + c: [wl_c | 0]  (hw halfs per part, 64-half rows)
  __shared__ double s_cn2[512];  // tensor-core operand rows (kp ≤ 512)
  float local_max = 0.f;
  for (int cc = threadIdx.x; cc < k; cc += blockDim.x) {
    double s = 0.0;
    for (int f = 0; f < m; ++f) {
      const double v = (double)__double2float_rn(c[(size_t)cc * m + f]);
      s = __fma_rn(v, v, s);
    }
    if (cc < 512) s_cn2[cc] = s;
    cn[cc] = __double2float_rn(s);
    local_max = fmaxf(local_max, __double2float_ru(sqrt(s) * (1.0 + 1e-12)));
  }
  for (int i = threadIdx.x; i < k * mpad; i += blockDim.x) {
    const int cc = i / mpad, f = i - cc * mpad;
    w[i] = (f < m) ? -2.0f * __double2float_rn(c[(size_t)cc * m + f]) : 0.0f;
  }
  for (int o = 16; o > 0; o >>= 1) local_max = fmaxf(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = local_max;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) mx = fmaxf(mx, s_red[i]);
    cmax[0] = mx;
  }
  if (wop != nullptr) {
    const int hw = 8 * ((m + 1 + 7) / 8);
    for (int i = threadIdx.x; i < kp * 64; i += blockDim.x) {
      const int cc = i >> 6, col = i & 63;
      const int f = col < hw ? col : col - hw;  // feature of this column (part 0 or 1)
      float v = 0.f;
      if (cc < k && col < 2 * hw) {
        if (f < m) v = -2.0f * __double2float_rn(c[(size_t)cc * m + f]) * pre;
        else if (f == m) v = __double2float_rn(s_cn2[cc] * (double)pre * (double)pre);
      } else if (cc >= k && col < 2 * hw && f == m) {
        v = 65504.f;  // padded centre: score +65504 (fp16 max) > every real score, never selected
      }
      const __half h = __float2half_rn(v);
      const __half l = __float2half_rn(v - __half2float(h));
      wop[i] = (col < 2 * hw) ? __half_as_ushort(h) : (unsigned short)0;                  // [wh | wh]
      wop[kp * 64 + i] = (col < hw) ? __half_as_ushort(l) : (unsigned short)0;             // [wl | 0 ]
    }
  }
  __syncthreads();
}

// worst = max_c sqrt(Σ_f (prev−next)²) ≤ tol, fp64, no FMA (engine.py:306-310, _kernels.py:173-180)
__device__ __forceinline__ int block_converged(const double* __restrict__ prev, const double* __restrict__ next,
                                               int k, int m, double tol, double* s_redd) {
  double worst = 0.0;
  for (int cc = threadIdx.x; cc < k; cc += blockDim.x) {
    double acc = 0.0;
    for (int f = 0; f < m; ++f) {
      const double d = __dsub_rn(prev[(size_t)cc * m + f], next[(size_t)cc * m + f]);
      acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    worst = fmax(worst, sqrt(acc));
  }
  for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
  if ((threadIdx.x & 31) == 0) s_redd[threadIdx.x >> 5] = worst;
  __syncthreads();
  double w = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) w = fmax(w, s_redd[i]);
  __syncthreads();
  return w <= tol ? 1 : 0;
}

__device__ __forceinline__ void loop_check(FinishArgs& a, double* s_redd, float* s_red, const double* prev_s = nullptr,
                                           const double* cur_s = nullptr) {
  DevState* st = a.st;
  const double* P = prev_s ? prev_s : a.prev;
  const double* C = cur_s ? cur_s : a.cur;
  const int conv = block_converged(P, C, a.k, a.m, st->tol, s_redd);
  block_prep_filter(C, a.w, a.cn, a.cmax, a.k, a.m, a.mpad, s_red, a.wop, a.kp, a.pre);
  if (threadIdx.x == 0) {
    st->need_host = 0;
    if (conv) {
      st->converged = 1;
      st->done = 1;
    } else if (st->t >= st->max_iters) {
      st->exhausted = 1;  // reference: assignment = assign_fn(model) once more, then return
    }
  }
}

// Re-decide the globally queued points (overflow of the per-CTA queues) with the whole block
// (warp per point) and apply their Δ to the partial buffer.  Centres: a.cur = C_t of the pass.
__device__ __forceinline__ void recheck_global_queue(FinishArgs& a) {
  const unsigned int cnt = *a.recheck_count;
  const int lane = threadIdx.x & 31, m = a.m, k = a.k;
  for (unsigned int q = threadIdx.x >> 5; q < cnt; q += blockDim.x >> 5) {
    const long long row = a.recheck_rows[q];
    // (fp64 points: the exact fp64 row, not the fp32 shadow the pass streamed)
    const double xl = lane >= m ? 0.0 : a.x64 ? a.x64[row * m + lane] : (double)a.x[row * m + lane];
    const int bl = exact_label_warp(xl, m, k, a.cur);
    const int old = a.full ? -1 : a.labels[row];
    if (bl != old) {
      if (lane == 0) {
        a.labels[row] = bl;
        atomicAdd(a.part + (size_t)k * m + bl, 1ull);
        if (old >= 0) atomicAdd(a.part + (size_t)k * m + old, ~0ull);
        if (!a.full) atomicAdd(&a.st->changed, 1ull);
      }
      if (lane < m) {
        const long long v = a.use_dscale || a.x64 ? __double2ll_rn(__dmul_rn(xl, a.scale_d))
                                                  : __float2ll_rn(__fmul_rn((float)xl, a.scale_f));
        atomicAdd(a.part + (size_t)bl * m + lane, (unsigned long long)v);
        if (old >= 0) atomicAdd(a.part + (size_t)old * m + lane, (unsigned long long)(-v));
      }
    }
  }
  __threadfence_block();
}

// Block-level finish (any block size that is a multiple of 32, ≤ 1024).  Runs as its own
// one-CTA kernel after a pass, or in the last CTA of the fused tensor-core pass.
// `stage` (shared memory, `stage_cap` doubles) holds C_{t-1} and C_t while the congruence test and
// the filter prep read them (global memory otherwise).
static __device__ __noinline__ void finish_block(FinishArgs a, double* stage, int stage_cap,
                                                long long* fts = nullptr) {
#define FTS(i) do { if (fts != nullptr && threadIdx.x == 0) fts[i] = clock64(); } while (0)
  FTS(0);
  __shared__ float s_red[32];
  __shared__ double s_redd[32];
  __shared__ int s_empty[32];
  DevState* st = a.st;
  const int k = a.k, m = a.m;
  if (a.mode == 0) {
    if (st->done || st->need_host) return;
    if (a.recheck_rows && a.recheck_count && *a.recheck_count) {  // overflow queue not yet re-decided
      recheck_global_queue(a);
      __syncthreads();
    }
    if (threadIdx.x == 0 && a.recheck_count) st->rechecked += *a.recheck_count;
    __syncthreads();
    if (threadIdx.x == 0 && a.recheck_count) *a.recheck_count = 0u;
    if (st->exhausted) {  // the final assign pass has run: fold its Δ so tot counts = bincount(L_T)
      for (int i = threadIdx.x; i < k * m + k; i += blockDim.x) {
        a.tot[i] = a.accumulate ? a.tot[i] + a.part[i] : a.part[i];
        a.part[i] = 0ull;
      }
      __syncthreads();
      for (int cc = threadIdx.x; cc < k; cc += blockDim.x) a.model_counts[cc] = (long long)a.tot[(size_t)k * m + cc];
      if (threadIdx.x == 0) st->done = 1;
      return;
    }
  }
  FTS(1);
  // running totals of the current labels (exact integer arithmetic: Δ-updates == recomputation)
  for (int i = threadIdx.x; i < k * m + k; i += blockDim.x) {
    a.tot[i] = a.accumulate ? a.tot[i] + a.part[i] : a.part[i];
    a.part[i] = 0ull;
  }
  __syncthreads();
  FTS(2);
  unsigned long long* sums = a.tot;
  unsigned long long* cnts = a.tot + (size_t)k * m;
  // prev ← cur ; cur ← S/N  (engine._finish_update, engine.py:249-263)
  const bool staged = stage != nullptr && 2 * k * m <= stage_cap;
  for (int i = threadIdx.x; i < k * m; i += blockDim.x) {
    const int cc = i / m;
    const long long nc = (long long)cnts[cc];
    const double old = a.cur[i];
    double v = 0.0;  // placeholder for empty clusters; every one is re-seeded by the repair
    if (nc > 0) v = __ddiv_rn(__dmul_rn((double)(long long)sums[i], a.inv_scale), (double)nc);
    a.prev[i] = old;
    a.cur[i] = v;
    if (staged) {
      stage[i] = old;
      stage[k * m + i] = v;
    }
  }
  FTS(3);
  int empties = 0;
  for (int cc = threadIdx.x; cc < k; cc += blockDim.x) {
    const long long nc = (long long)cnts[cc];
    a.model_counts[cc] = nc;
    empties += (nc == 0);
  }
  for (int o = 16; o > 0; o >>= 1) empties += __shfl_xor_sync(0xffffffffu, empties, o);
  if ((threadIdx.x & 31) == 0) s_empty[threadIdx.x >> 5] = empties;
  __syncthreads();
  int total_empty = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) total_empty += s_empty[i];
  if (a.mode == 1) {
    if (threadIdx.x == 0) st->n_empty = total_empty;
    return;
  }
  if (threadIdx.x == 0) {
    st->t += 1;
    st->n_empty = total_empty;
  }
  __syncthreads();
  if (total_empty > 0) {
    if (threadIdx.x == 0) st->need_host = 1;
    return;
  }
  FTS(4);
  loop_check(a, s_redd, s_red, staged ? stage : nullptr, staged ? stage + k * m : nullptr);
  FTS(5);
#undef FTS
}


}  // namespace km
