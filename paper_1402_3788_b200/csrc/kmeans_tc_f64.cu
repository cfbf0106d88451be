// kmeans_tc_f64.cu — tcgen05 pass instantiations for fp64 points (X64: the pass streams the fp32
// shadow, the exact fp64 rows feed the recheck and the Δ of changed points).
#include <cstdio>

#include "kmeans_tc.cuh"
#include "kmeans_tc_dispatch.h"

namespace km {
namespace tc {

template <int MT>
static int by_kp64(const TcArgs& a, int kp, int num_sms, size_t smem_optin, cudaStream_t stream, cudaError_t* ce,
                   char* msg, size_t len) {
  switch (kp) {
    case 16: return launch_t<MT, 16, true, true>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 32: return launch_t<MT, 32, true, true>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 48: return launch_t<MT, 48, true, true>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 64: return launch_t<MT, 64, true, true>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 96: return launch_t<MT, 96, true, true>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 128: return launch_t<MT, 128, true, true>(a, num_sms, smem_optin, stream, ce, msg, len);
    default: snprintf(msg, len, "tensor-core pass: unsupported k padding %d", kp); return 2;
  }
}

int launch_f64(const TcArgs& a, int m, int mp, int kp, int num_sms, size_t smem_optin, cudaStream_t stream,
               cudaError_t* ce, char* msg, size_t len) {
  if (m == 25 && (kp == 16 || kp == 64)) {  // the BASELINE feature count
    return kp == 16 ? launch_t<25, 16, true, true>(a, num_sms, smem_optin, stream, ce, msg, len)
                    : launch_t<25, 64, true, true>(a, num_sms, smem_optin, stream, ce, msg, len);
  }
  switch (mp) {
    case 7: return by_kp64<-7>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    case 15: return by_kp64<-15>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    case 23: return by_kp64<-23>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    case 31: return by_kp64<-31>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    default: snprintf(msg, len, "tensor-core pass: unsupported feature padding %d", mp); return 2;
  }
}

}  // namespace tc
}  // namespace km
