// conv.cu — throughput of the per-element ops of the transform stage on B200.
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)
constexpr int ITERS = 4096;

__global__ void k_f2fp(const float* in, uint32_t* out) {
  float a = in[threadIdx.x], b = in[threadIdx.x + 1];
  uint32_t acc = 0;
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    __half2 h = __floats2half2_rn(a, b);
    acc ^= *reinterpret_cast<uint32_t*>(&h);
    a += 1.0f; b += 1.0f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_split(const float* in, uint32_t* out) {  // full hi/lo split of a pair
  float a = in[threadIdx.x], b = in[threadIdx.x + 1];
  uint32_t acc = 0;
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    const __half2 h2 = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h2);
    const __half2 l2 = __floats2half2_rn(a - hf.x, b - hf.y);
    acc ^= *reinterpret_cast<const uint32_t*>(&h2) ^ *reinterpret_cast<const uint32_t*>(&l2);
    a += 1.0f; b += 1.0f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_tf32(const float* in, uint32_t* out) {  // tf32 hi/lo split of a pair (mask + sub)
  float a = in[threadIdx.x], b = in[threadIdx.x + 1];
  uint32_t acc = 0;
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    const float ha = __uint_as_float(__float_as_uint(a) & 0xffffe000u), hb = __uint_as_float(__float_as_uint(b) & 0xffffe000u);
    acc ^= __float_as_uint(ha) ^ __float_as_uint(a - ha) ^ __float_as_uint(hb) ^ __float_as_uint(b - hb);
    a += 1.0f; b += 1.0f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_bits(const float* in, uint32_t* out) {  // fp16 hi via integer rounding of the fp32 bits
  float a = in[threadIdx.x], b = in[threadIdx.x + 1];
  uint32_t acc = 0;
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    // round-to-nearest-even to 11 significant bits, kept as fp32 (exactly representable in fp16 when normal)
    const uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
    const uint32_t ra = (ua + 0x0fffu + ((ua >> 13) & 1u)) & 0xffffe000u;
    const uint32_t rb = (ub + 0x0fffu + ((ub >> 13) & 1u)) & 0xffffe000u;
    acc ^= ra ^ rb ^ __float_as_uint(a - __uint_as_float(ra)) ^ __float_as_uint(b - __uint_as_float(rb));
    a += 1.0f; b += 1.0f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_f2i64(const float* in, uint32_t* out) {
  float a = in[threadIdx.x];
  uint32_t acc = 0;
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) { acc ^= (uint32_t)__float2ll_rn(a * 1024.f); a += 1.0f; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <typename K>
float run(K k, const float* in, uint32_t* out, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<sms * 4, 256>>>(in, out);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<sms * 4, 256>>>(in, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* in; uint32_t* out;
  CK(cudaMalloc(&in, 4096)); CK(cudaMalloc(&out, (size_t)sms * 4 * 256 * 4)); CK(cudaMemset(in, 0, 4096));
  const double thr = (double)sms * 4 * 256 * ITERS;  // loop iterations (thread-level)
  struct { const char* n; float ms; double per; } r[] = {
    {"F2FP pack (2 values)", run(k_f2fp, in, out, sms), 2},
    {"fp16 hi/lo split (2 values)", run(k_split, in, out, sms), 2},
    {"tf32 hi/lo split (2 values)", run(k_tf32, in, out, sms), 2},
    {"int-rounded hi/lo (2 values)", run(k_bits, in, out, sms), 2},
    {"F2I.S64 (1 value)", run(k_f2i64, in, out, sms), 1},
  };
  for (auto& x : r) {
    const double cyc = x.ms * 1e-3 * clk * 1e3;
    printf("%-30s %8.3f ms  %7.2f values/clk/SM\n", x.n, x.ms, thr * x.per / cyc / sms);
  }
  CK(cudaGetLastError());
  return 0;
}
