// kmeans_tc.cu — instantiations + launcher of the tcgen05 fused pass.
#include <algorithm>
#include <cstdio>

#include "kmeans_tc.cuh"

namespace km {
namespace tc {

template <int MP, int KP>
static int launch_t(const TcArgs& a, int num_sms, size_t smem_optin, cudaStream_t stream, cudaError_t* ce,
                    char* msg, size_t len) {
  auto kern = lloyd_pass_tc_kernel<MP, KP>;
  const size_t smem = TcSmem<MP, KP>(a.m).total;
  if (smem > smem_optin) {
    snprintf(msg, len, "tensor-core pass needs %zu B of shared memory (max %zu)", smem, smem_optin);
    return 2;
  }
  cudaError_t c = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (c != cudaSuccess) { *ce = c; snprintf(msg, len, "cudaFuncSetAttribute(tc smem)"); return 1; }
  c = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (c != cudaSuccess) { *ce = c; snprintf(msg, len, "cudaFuncSetAttribute(tc carveout)"); return 1; }
  int per_sm = 0;
  c = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreadsTC, smem);
  if (c != cudaSuccess) { *ce = c; snprintf(msg, len, "occupancy(tc)"); return 1; }
  if (per_sm < 1) { snprintf(msg, len, "tensor-core pass does not fit on an SM"); return 2; }
  per_sm = std::min(per_sm, 1);  // one persistent CTA per SM (two ping-pong warpgroups inside)
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)per_sm * num_sms));
  kern<<<(unsigned)grid, kThreadsTC, smem, stream>>>(a);
  c = cudaGetLastError();
  if (c != cudaSuccess) { *ce = c; snprintf(msg, len, "lloyd_pass_tc_kernel launch"); return 1; }
  return 0;
}

template <int MP>
static int launch_kp(const TcArgs& a, int kp, int num_sms, size_t smem_optin, cudaStream_t stream, cudaError_t* ce,
                     char* msg, size_t len) {
  switch (kp) {
    case 16: return launch_t<MP, 16>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 32: return launch_t<MP, 32>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 48: return launch_t<MP, 48>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 64: return launch_t<MP, 64>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 96: return launch_t<MP, 96>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 128: return launch_t<MP, 128>(a, num_sms, smem_optin, stream, ce, msg, len);
    default: snprintf(msg, len, "tensor-core pass: unsupported k padding %d", kp); return 2;
  }
}

int launch(const TcArgs& a, int mp, int kp, int num_sms, size_t smem_optin, cudaStream_t stream,
           cudaError_t* ce, char* msg, size_t len) {
  switch (mp) {
    case 7: return launch_kp<7>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    case 15: return launch_kp<15>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    case 23: return launch_kp<23>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    case 31: return launch_kp<31>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    default: snprintf(msg, len, "tensor-core pass: unsupported feature padding %d", mp); return 2;
  }
}

}  // namespace tc
}  // namespace km
