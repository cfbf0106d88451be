// fp64 latency/throughput probes on sm_100a (tuning only)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat_dadd(double* out, double a, double b, int n, long long* t) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void lat_dmul(double* out, double a, double b, int n, long long* t) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, b);
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void lat_step(double* out, const double* c, double a, int n, int m, long long* t) {
  __shared__ double sc[64];
  if (threadIdx.x < 64) sc[threadIdx.x] = c[threadIdx.x];
  __syncthreads();
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int f = 0; f < 25; ++f) {
      const double d = __dsub_rn(a + f, sc[f]);
      acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void lat_div(double* out, double a, double b, int n, long long* t) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __ddiv_rn(x, b) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void lat_sqrt(double* out, double a, int n, long long* t) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 2.0;
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void lat_f2f(double* out, float a, int n, long long* t) {
  float x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = (float)((double)x * 1.0000001);
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void thr_dadd(double* out, double a, double b, int n, long long* t) {
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = __dadd_rn(x0, b); x1 = __dadd_rn(x1, b); x2 = __dadd_rn(x2, b); x3 = __dadd_rn(x3, b);
    x4 = __dadd_rn(x4, b); x5 = __dadd_rn(x5, b); x6 = __dadd_rn(x6, b); x7 = __dadd_rn(x7, b);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0 && blockIdx.x == 0) t[0] = t1 - t0;
}
int main() {
  double* out; long long* t; double* c;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&t, 64); cudaMalloc(&c, 64 * 8); cudaMemset(c, 0, 512);
  long long h;
  const int n = 4096;
  auto rd = [&](const char* name, double per) { cudaDeviceSynchronize(); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("%-28s %8.2f cyc\n", name, h / per); };
  lat_dadd<<<1, 32>>>(out, 1.0, 1e-9, n, t); lat_dadd<<<1, 32>>>(out, 1.0, 1e-9, n, t); rd("DADD dep latency", n);
  lat_dmul<<<1, 32>>>(out, 1.0, 1.0000001, n, t); lat_dmul<<<1, 32>>>(out, 1.0, 1.0000001, n, t); rd("DMUL dep latency", n);
  lat_step<<<1, 32>>>(out, c, 1.0, n / 16, 25, t); lat_step<<<1, 32>>>(out, c, 1.0, n / 16, 25, t); rd("sub/mul/add step (smem c)", (n / 16) * 25.0);
  lat_div<<<1, 32>>>(out, 1.0, 3.0, n / 8, t); lat_div<<<1, 32>>>(out, 1.0, 3.0, n / 8, t); rd("DDIV(+DADD) dep latency", n / 8);
  lat_sqrt<<<1, 32>>>(out, 5.0, n / 8, t); lat_sqrt<<<1, 32>>>(out, 5.0, n / 8, t); rd("DSQRT(+DADD) dep latency", n / 8);
  lat_f2f<<<1, 32>>>(out, 1.0f, n, t); lat_f2f<<<1, 32>>>(out, 1.0f, n, t); rd("F2F64+DMUL+F2F32 dep", n);
  for (int w : {1, 4, 16, 32}) {
    thr_dadd<<<148, 32 * w>>>(out, 1.0, 1e-9, n, t); thr_dadd<<<148, 32 * w>>>(out, 1.0, 1e-9, n, t);
    cudaDeviceSynchronize(); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    printf("DADD throughput %2d warps/SM: %.2f lane-ops/cyc/SM\n", w, 32.0 * w * 8 * n / h);
  }
  return 0;
}
