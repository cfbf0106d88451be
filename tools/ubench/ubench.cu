// ubench.cu — design microbenchmarks for the fused Lloyd pass on B200.
// Not part of the product; results are summarised in profiles/ubench_r01.txt.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o ubench ubench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int K = 16, M = 25, MP = 28, TR = 256;
__constant__ float c_w[K * M];
__constant__ float c_cn[K];

__device__ __forceinline__ void stage(float* s, const float* g, int64_t row0, int rows) {
  const int64_t bytes = (int64_t)rows * M * 4;
  const float4* s4 = reinterpret_cast<const float4*>(g + row0 * M);
  float4* d4 = reinterpret_cast<float4*>(s);
  const int nv = (int)(bytes >> 4);
  for (int i = threadIdx.x; i < nv; i += blockDim.x) d4[i] = __ldg(s4 + i);
}

__device__ __forceinline__ void track(float s, int c, float& best, float& min2, int& bi) {
  const bool lt = s < best;
  min2 = lt ? best : fminf(min2, s);
  bi = lt ? c : bi;
  best = lt ? s : best;
}

// B) memory only: stage + label write
__global__ void __launch_bounds__(256) k_mem(const float* x, int64_t n, int* labels) {
  __shared__ __align__(16) float tile[TR * M];
  const int64_t ntiles = (n + TR - 1) / TR;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    __syncthreads();
    stage(tile, x, t * TR, TR);
    __syncthreads();
    labels[t * TR + threadIdx.x] = (int)tile[threadIdx.x * M] ;
  }
}

// A) assign variants.  P points per thread (block handles TR*P rows per tile).
template <int P, bool CONST_W>
__global__ void __launch_bounds__(256) k_assign(const float* x, int64_t n, const float* gw, const float* gcn,
                                                int* labels, float E) {
  extern __shared__ __align__(16) float sm[];
  float* s_w = sm;                 // K*MP
  float* s_cn = sm + K * MP;       // K (pad 16)
  float* tile = sm + K * MP + 16;  // TR*P*M
  for (int i = threadIdx.x; i < K * MP; i += 256) s_w[i] = gw[i];
  if (threadIdx.x < K) s_cn[threadIdx.x] = gcn[threadIdx.x];
  const int64_t rows_per_tile = (int64_t)TR * P;
  const int64_t ntiles = (n + rows_per_tile - 1) / rows_per_tile;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    __syncthreads();
    stage(tile, x, t * rows_per_tile, (int)rows_per_tile);
    __syncthreads();
    float xr[P][MP];
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int f = 0; f < MP; ++f) xr[p][f] = f < M ? tile[(threadIdx.x + p * TR) * M + f] : 0.f;
    float best[P], min2[P];
    int bi[P];
#pragma unroll
    for (int p = 0; p < P; ++p) { best[p] = 3.0e38f; min2[p] = 3.0e38f; bi[p] = 0; }
#pragma unroll 4
    for (int c = 0; c < K; ++c) {
      float a[P];
      if (CONST_W) {
#pragma unroll
        for (int p = 0; p < P; ++p) a[p] = c_cn[c];
#pragma unroll
        for (int f = 0; f < M; ++f) {
          const float w = c_w[c * M + f];
#pragma unroll
          for (int p = 0; p < P; ++p) a[p] = __fmaf_rn(xr[p][f], w, a[p]);
        }
      } else {
        const float cn = s_cn[c];
#pragma unroll
        for (int p = 0; p < P; ++p) a[p] = cn;
#pragma unroll
        for (int f = 0; f < MP; f += 4) {
          const float4 w4 = *reinterpret_cast<const float4*>(s_w + c * MP + f);
#pragma unroll
          for (int p = 0; p < P; ++p) {
            a[p] = __fmaf_rn(xr[p][f], w4.x, a[p]);
            a[p] = __fmaf_rn(xr[p][f + 1], w4.y, a[p]);
            a[p] = __fmaf_rn(xr[p][f + 2], w4.z, a[p]);
            a[p] = __fmaf_rn(xr[p][f + 3], w4.w, a[p]);
          }
        }
      }
#pragma unroll
      for (int p = 0; p < P; ++p) track(a[p], c, best[p], min2[p], bi[p]);
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int lab = (min2[p] > best[p] + E) ? bi[p] : -1 - bi[p];
      labels[t * rows_per_tile + threadIdx.x + p * TR] = lab;
    }
  }
}

// A6) packed fp32x2 FMA: 2 points per lane-op, P2 pairs per thread
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
template <int PAIRS>
__global__ void __launch_bounds__(256) k_assign_f2(const float* x, int64_t n, const float* gw, const float* gcn,
                                                   int* labels, float E) {
  extern __shared__ __align__(16) float sm[];
  float* s_w2 = sm;                      // K*MP*2 (w duplicated)
  float* s_cn = sm + K * MP * 2;
  float* tile = s_cn + 16;
  for (int i = threadIdx.x; i < K * MP; i += 256) { s_w2[2 * i] = gw[i]; s_w2[2 * i + 1] = gw[i]; }
  if (threadIdx.x < K) s_cn[threadIdx.x] = gcn[threadIdx.x];
  constexpr int P = 2 * PAIRS;
  const int64_t rows_per_tile = (int64_t)TR * P;
  const int64_t ntiles = (n + rows_per_tile - 1) / rows_per_tile;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    __syncthreads();
    stage(tile, x, t * rows_per_tile, (int)rows_per_tile);
    __syncthreads();
    unsigned long long xr[PAIRS][MP];
#pragma unroll
    for (int q = 0; q < PAIRS; ++q)
#pragma unroll
      for (int f = 0; f < MP; ++f) {
        const float lo = f < M ? tile[(threadIdx.x + (2 * q) * TR) * M + f] : 0.f;
        const float hi = f < M ? tile[(threadIdx.x + (2 * q + 1) * TR) * M + f] : 0.f;
        xr[q][f] = pack2(lo, hi);
      }
    float best[P], min2[P];
    int bi[P];
#pragma unroll
    for (int p = 0; p < P; ++p) { best[p] = 3.0e38f; min2[p] = 3.0e38f; bi[p] = 0; }
#pragma unroll 2
    for (int c = 0; c < K; ++c) {
      unsigned long long a[PAIRS];
      const float cn = s_cn[c];
#pragma unroll
      for (int q = 0; q < PAIRS; ++q) a[q] = pack2(cn, cn);
#pragma unroll
      for (int f = 0; f < MP; f += 2) {
        const float4 w4 = *reinterpret_cast<const float4*>(s_w2 + (c * MP + f) * 2);
        const unsigned long long wa = pack2(w4.x, w4.y), wb = pack2(w4.z, w4.w);
#pragma unroll
        for (int q = 0; q < PAIRS; ++q) {
          a[q] = ffma2(xr[q][f], wa, a[q]);
          a[q] = ffma2(xr[q][f + 1], wb, a[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < PAIRS; ++q) {
        track(__uint_as_float((unsigned)(a[q] & 0xffffffffu)), c, best[2 * q], min2[2 * q], bi[2 * q]);
        track(__uint_as_float((unsigned)(a[q] >> 32)), c, best[2 * q + 1], min2[2 * q + 1], bi[2 * q + 1]);
      }
    }
#pragma unroll
    for (int q = 0; q < PAIRS; ++q)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = 2 * q + h;
        const int lab = (min2[p] > best[p] + E) ? bi[p] : -1 - bi[p];
        labels[t * rows_per_tile + threadIdx.x + p * TR] = lab;
      }
  }
}

// C) update variants (labels given).  U1: smem atomics per element.
__global__ void __launch_bounds__(256) k_upd_atomics(const float* x, int64_t n, const int* labels,
                                                     unsigned long long* out, float scale) {
  __shared__ __align__(16) float tile[TR * M];
  __shared__ unsigned long long acc[K * M + K];
  for (int i = threadIdx.x; i < K * M + K; i += 256) acc[i] = 0;
  const int64_t ntiles = (n + TR - 1) / TR;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    __syncthreads();
    stage(tile, x, t * TR, TR);
    __syncthreads();
    const int lab = labels[t * TR + threadIdx.x] & 15;
    atomicAdd(&acc[K * M + lab], 1ull);
    for (int f = 0; f < M; ++f)
      atomicAdd(&acc[lab * M + f], (unsigned long long)__float2ll_rn(tile[threadIdx.x * M + f] * scale));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < K * M + K; i += 256) atomicAdd(&out[i], acc[i]);
}

// U2: lane = feature; warp walks its 32 points; register accumulators per cluster via uniform switch.
__global__ void __launch_bounds__(256) k_upd_lanefeat(const float* x, int64_t n, const int* labels,
                                                      unsigned long long* out, float scale) {
  __shared__ __align__(16) float tile[TR * M];
  __shared__ int s_lab[TR];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long acc[K];
#pragma unroll
  for (int c = 0; c < K; ++c) acc[c] = 0;
  int cnt = 0;
  const int64_t ntiles = (n + TR - 1) / TR;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    __syncthreads();
    stage(tile, x, t * TR, TR);
    s_lab[threadIdx.x] = labels[t * TR + threadIdx.x] & 15;
    __syncthreads();
    const int f = lane < M ? lane : 0;
    for (int j = warp * 32; j < warp * 32 + 32; ++j) {
      const int lab = s_lab[j];
      const long long v = lane < M ? __float2ll_rn(tile[j * M + f] * scale) : 0;
      switch (lab) {
#define CASE(c) case c: acc[c] += v; break;
        CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
        CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
      }
      cnt += (lane == lab);
    }
  }
  if (lane < M) {
#pragma unroll
    for (int c = 0; c < K; ++c) if (acc[c]) atomicAdd(&out[c * M + lane], (unsigned long long)acc[c]);
  }
  if (lane < K && cnt) atomicAdd(&out[K * M + lane], (unsigned long long)cnt);
}

// U3: thread-per-point, predicated register accumulation for K clusters (K selects per element)
// -- too many instructions for K=16; kept as a reference point only for K<=4.

template <typename F>
float time_it(F launch, int reps = 20) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) launch();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  CK(cudaGetLastError());
  return ms / reps;
}

int main(int argc, char** argv) {
  const int64_t n = 2000000 - 2000000 % (TR * 4 * 2);
  std::vector<float> hx((size_t)n * M), hw(K * MP, 0.f), hcn(K), hwc(K * M);
  std::mt19937 rng(1);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::uniform_real_distribution<float> ud(-10.f, 10.f);
  std::vector<float> cent(K * M);
  for (auto& v : cent) v = ud(rng);
  for (int64_t i = 0; i < n; ++i) {
    int c = (int)(rng() % K);
    for (int f = 0; f < M; ++f) hx[i * M + f] = cent[c * M + f] + nd(rng);
  }
  for (int c = 0; c < K; ++c) {
    double s = 0;
    for (int f = 0; f < M; ++f) {
      float cc = hx[(size_t)c * M + f];
      hw[c * MP + f] = -2.f * cc;
      hwc[c * M + f] = -2.f * cc;
      s += (double)cc * cc;
    }
    hcn[c] = (float)s;
  }
  float *dx, *dw, *dcn;
  int* dl;
  unsigned long long* dout;
  CK(cudaMalloc(&dx, hx.size() * 4));
  CK(cudaMalloc(&dw, hw.size() * 4));
  CK(cudaMalloc(&dcn, 64));
  CK(cudaMalloc(&dl, n * 4));
  CK(cudaMalloc(&dout, 8 * (K * M + K)));
  CK(cudaMemcpy(dx, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dcn, hcn.data(), K * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpyToSymbol(c_w, hwc.data(), K * M * 4));
  CK(cudaMemcpyToSymbol(c_cn, hcn.data(), K * 4));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const double bytes = (double)n * (4 * M + 4);
  auto report = [&](const char* name, float ms) {
    printf("%-34s %8.2f us  %7.0f GB/s (alg bytes)  %.3f of 6534\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9,
           bytes / (ms * 1e-3) / 1e9 / 6534.1);
  };
  auto occ_grid = [&](const void* kern, size_t smem) {
    int per = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, smem));
    return per * sms;
  };
  {
    int g = occ_grid((const void*)k_mem, 0);
    report("mem only (stage+label)", time_it([&] { k_mem<<<g, 256>>>(dx, n, dl); }));
  }
  const float E = 1e-3f;
#define RUN_A(P, CW)                                                                                 \
  {                                                                                                  \
    size_t sm = (K * MP + 16 + (size_t)TR * P * M) * 4;                                              \
    auto kern = k_assign<P, CW>;                                                                     \
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));           \
    int g = occ_grid((const void*)kern, sm);                                                         \
    char nm[64];                                                                                     \
    snprintf(nm, 64, "assign P=%d const_w=%d (grid %d)", P, (int)CW, g);                             \
    report(nm, time_it([&] { kern<<<g, 256, sm>>>(dx, n, dw, dcn, dl, E); }));                      \
  }
  RUN_A(1, false) RUN_A(2, false) RUN_A(4, false) RUN_A(1, true) RUN_A(2, true) RUN_A(4, true)
#define RUN_F2(PAIRS)                                                                                \
  {                                                                                                  \
    size_t sm = (K * MP * 2 + 16 + (size_t)TR * 2 * PAIRS * M) * 4;                                  \
    auto kern = k_assign_f2<PAIRS>;                                                                  \
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));           \
    int g = occ_grid((const void*)kern, sm);                                                         \
    char nm[64];                                                                                     \
    snprintf(nm, 64, "assign ffma2 pairs=%d (grid %d)", PAIRS, g);                                   \
    report(nm, time_it([&] { kern<<<g, 256, sm>>>(dx, n, dw, dcn, dl, E); }));                      \
  }
  RUN_F2(1) RUN_F2(2)
  // correctness cross-check of label outputs between variants
  {
    std::vector<int> l1(n), l2(n);
    size_t sm = (K * MP + 16 + (size_t)TR * 1 * M) * 4;
    k_assign<1, false><<<occ_grid((const void*)k_assign<1, false>, sm), 256, sm>>>(dx, n, dw, dcn, dl, E);
    CK(cudaMemcpy(l1.data(), dl, n * 4, cudaMemcpyDeviceToHost));
    size_t sm2 = (K * MP * 2 + 16 + (size_t)TR * 2 * 2 * M) * 4;
    k_assign_f2<2><<<occ_grid((const void*)k_assign_f2<2>, sm2), 256, sm2>>>(dx, n, dw, dcn, dl, E);
    CK(cudaMemcpy(l2.data(), dl, n * 4, cudaMemcpyDeviceToHost));
    int64_t diff = 0, amb = 0;
    for (int64_t i = 0; i < n; ++i) { diff += l1[i] != l2[i]; amb += l1[i] < 0; }
    printf("labels p1 vs ffma2: %lld differ, %lld uncertified (E=%g)\n", (long long)diff, (long long)amb, E);
  }
  {
    int g = occ_grid((const void*)k_upd_atomics, 0);
    report("update smem atomics", time_it([&] { k_upd_atomics<<<g, 256>>>(dx, n, dl, dout, 65536.f); }));
  }
  {
    int g = occ_grid((const void*)k_upd_lanefeat, 0);
    report("update lane=feature switch", time_it([&] { k_upd_lanefeat<<<g, 256>>>(dx, n, dl, dout, 65536.f); }));
  }
  return 0;
}
