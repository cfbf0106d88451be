// TMA 1-D bulk streaming probe (tuning only): 1 CTA/SM, producer lane + consumer warps, ring of RS slots.
#include <cstdio>
#ifndef HINTS
#define HINTS 0, 1
#endif
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, uint64_t* b, uint64_t pol, int hint) {
  if (hint)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)), "l"(pol) : "memory");
  else
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}
__global__ void stream(const char* x, long long bytes, int tile, int RS, int hint, int consumers, float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t full[16], empty[16];
  const long long ntiles = bytes / tile;
  const long long lo = ntiles * blockIdx.x / gridDim.x, hi = ntiles * (blockIdx.x + 1) / gridDim.x;
  const int my = (int)(hi - lo);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < RS; ++s) { init(full + s, 1); init(empty + s, consumers / 2 * 0 + 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  uint64_t pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int nw = blockDim.x / 32;
  if (warp == nw - 1) {
    if (lane == 0)
      for (int i = 0; i < my; ++i) {
        const int s = i % RS;
        if (i >= RS) wait(empty + s, ((i / RS) - 1) & 1);
        expect(full + s, tile);
        g2s(sm + s * tile, x + (lo + i) * (long long)tile, tile, full + s, pol, hint);
      }
  } else {
    // consumer warps: warp w takes tiles i ≡ w (mod nw-1); touches one float per lane
    float acc = 0.f;
    for (int i = warp; i < my; i += nw - 1) {
      const int s = i % RS;
      wait(full + s, (i / RS) & 1);
      acc += reinterpret_cast<const float*>(sm + s * tile)[lane];
      __syncwarp();
      if (lane == 0) arrive(empty + s);
    }
    if (acc == 12345.f) sink[0] = acc;
  }
}
int main() {
  const long long bytes = 200ll * 1000 * 1000;
  char* x; float* sink; cudaMalloc(&x, bytes + (1 << 20)); cudaMalloc(&sink, 64); cudaMemset(x, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int hint : {HINTS})
    for (int tile : {12800, 16384, 25600})
      for (int RS : {4, 6, 8, 12}) {
        if ((long long)tile * RS > 200 * 1024) continue;
        for (int consumers : {2}) {
          for (int rep = 0; rep < 2; ++rep) stream<<<sms, (consumers + 1) * 32, tile * RS>>>(x, bytes, tile, RS, hint, consumers, sink);
          cudaEventRecord(a);
          const int reps = 10;
          for (int rep = 0; rep < reps; ++rep) stream<<<sms, (consumers + 1) * 32, tile * RS>>>(x, bytes, tile, RS, hint, consumers, sink);
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b);
          printf("hint %d tile %6d RS %2d: %7.1f us/pass  %6.0f GB/s  %s\n", hint, tile, RS, ms * 1e3 / reps, bytes / (ms * 1e-3 / reps) / 1e9,
                 cudaGetErrorString(cudaGetLastError()));
        }
      }
  return 0;
}
