// kmeans_tc_bucket.cu — tcgen05 pass instantiations for a runtime feature count (buckets of 8).
#include <cstdio>

#include "kmeans_tc.cuh"
#include "kmeans_tc_dispatch.h"

namespace km {
namespace tc {

template <int MT>
static int by_kp(const TcArgs& a, int kp, int num_sms, size_t smem_optin, cudaStream_t stream, cudaError_t* ce,
                 char* msg, size_t len) {
  switch (kp) {
    case 16: return launch_t<MT, 16, true, false>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 32: return launch_t<MT, 32, true, false>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 48: return launch_t<MT, 48, true, false>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 64: return launch_t<MT, 64, true, false>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 96: return launch_t<MT, 96, true, false>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 128: return launch_t<MT, 128, true, false>(a, num_sms, smem_optin, stream, ce, msg, len);
    default: snprintf(msg, len, "tensor-core pass: unsupported k padding %d", kp); return 2;
  }
}

int launch_bucket(const TcArgs& a, int mp, int kp, int num_sms, size_t smem_optin, cudaStream_t stream,
                  cudaError_t* ce, char* msg, size_t len) {
  switch (mp) {
    case 7: return by_kp<-7>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    case 15: return by_kp<-15>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    case 23: return by_kp<-23>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    case 31: return by_kp<-31>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    default: snprintf(msg, len, "tensor-core pass: unsupported feature padding %d", mp); return 2;
  }
}

}  // namespace tc
}  // namespace km
