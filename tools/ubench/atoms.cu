// atoms.cu — shared-memory 64-bit accumulation throughput on B200 (design microbenchmark for the
// Δ / cluster-sum updates).  Each warp adds a row (lanes 0..24 = features, warp-uniform label) into
// a [16][26] int64 accumulator, ITERS times; variants: two 32-bit atomics with carry (smem_add64),
// native 64-bit atomicAdd, red.shared.add.u64, warp-private plain LDS/STS.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms atoms.cu && ./atoms
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
constexpr int ITERS = 4096, K = 16, M = 25, WARPS = 6;

__device__ __forceinline__ void add64_pair(unsigned long long* addr, unsigned long long v) {
  unsigned int* p = reinterpret_cast<unsigned int*>(addr);
  const unsigned int lo = (unsigned int)v, hi = (unsigned int)(v >> 32);
  const unsigned int old = atomicAdd(p, lo);
  atomicAdd(p + 1, hi + ((old + lo) < old ? 1u : 0u));
}

template <int MODE>
__global__ void __launch_bounds__(WARPS * 32, 1) k_acc(unsigned long long* out, unsigned seed) {
  __shared__ unsigned long long acc[WARPS][K * (M + 1) * 2];
  for (int i = threadIdx.x; i < WARPS * K * (M + 1) * 2; i += blockDim.x) (&acc[0][0])[i] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned s = seed ^ (blockIdx.x * 7919u + warp * 104729u);
  unsigned long long* mine = MODE == 3 ? acc[warp] : acc[0];
  if (lane <= M) {
    for (int it = 0; it < ITERS; ++it) {
      s = s * 1664525u + 1013904223u;
      const int L = (s >> 20) & (K - 1);  // warp-uniform
      unsigned long long* dst = mine + L * (M + 1) + lane;
      const unsigned long long v = (unsigned long long)(s ^ lane) << 7;
      if (MODE == 0) add64_pair(dst, v);
      else if (MODE == 1) atomicAdd(dst, v);
      else if (MODE == 2) asm volatile("red.shared.add.u64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(v) : "memory");
      else if (MODE == 4) {  // four 16-bit limbs, 32-bit reductions without return
        unsigned* d32 = reinterpret_cast<unsigned*>(mine) + 4 * (L * (M + 1) + lane);
        const unsigned sa = (unsigned)__cvta_generic_to_shared(d32);
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(sa), "r"((unsigned)(v & 0xffff)) : "memory");
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(sa + 4), "r"((unsigned)((v >> 16) & 0xffff)) : "memory");
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(sa + 8), "r"((unsigned)((v >> 32) & 0xffff)) : "memory");
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(sa + 12), "r"((unsigned)((long long)v >> 48)) : "memory");
      }
      else *dst += v;
    }
  }
  __syncthreads();
  unsigned long long t = 0;
  for (int i = threadIdx.x; i < WARPS * K * (M + 1) * 2; i += blockDim.x) t += (&acc[0][0])[i];
  atomicAdd(out, t);
}

template <int MODE>
int run(const char* name, int sms) {
  unsigned long long* d;
  CK(cudaMalloc(&d, 8));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_acc<MODE><<<sms, WARPS * 32>>>(d, 1);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  k_acc<MODE><<<sms, WARPS * 32>>>(d, 2);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double lane_ops = (double)sms * WARPS * (M + 1) * ITERS;
  printf("%-28s %8.3f ms  %6.2f lane-ops/clk/SM (at 1.965 GHz)  %6.2f warp-rows/clk/SM\n", name, ms,
         lane_ops / sms / (ms * 1e-3 * 1.965e9), lane_ops / (M + 1) / sms / (ms * 1e-3 * 1.965e9));
  cudaFree(d);
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("2x32-bit atomics (carry)", sms);
  run<1>("atomicAdd u64 (shared)", sms);
  run<2>("red.shared.add.u64", sms);
  run<3>("warp-private LDS/STS", sms);
  run<4>("4x red.shared.add.u32 (limbs)", sms);
  return 0;
}
