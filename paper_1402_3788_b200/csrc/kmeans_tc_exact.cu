// kmeans_tc_exact.cu — tcgen05 pass instantiations with a compile-time feature count.
#include <cstdio>

#include "kmeans_tc.cuh"
#include "kmeans_tc_dispatch.h"

namespace km {
namespace tc {

template <int MT, bool PRE>
static int by_kp(const TcArgs& a, int kp, int num_sms, size_t smem_optin, cudaStream_t stream, cudaError_t* ce,
                 char* msg, size_t len) {
  switch (kp) {
    case 16: return launch_t<MT, 16, PRE, false>(a, num_sms, smem_optin, stream, ce, msg, len);
    case 64: return launch_t<MT, 64, PRE, false>(a, num_sms, smem_optin, stream, ce, msg, len);
    default: return -1;
  }
}

int launch_exact(const TcArgs& a, int m, int kp, bool pre, int num_sms, size_t smem_optin, cudaStream_t stream,
                 cudaError_t* ce, char* msg, size_t len) {
  switch (m) {
    case 5: return pre ? by_kp<5, true>(a, kp, num_sms, smem_optin, stream, ce, msg, len)
                       : by_kp<5, false>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    case 10: return pre ? by_kp<10, true>(a, kp, num_sms, smem_optin, stream, ce, msg, len)
                        : by_kp<10, false>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    case 25: return pre ? by_kp<25, true>(a, kp, num_sms, smem_optin, stream, ce, msg, len)
                        : by_kp<25, false>(a, kp, num_sms, smem_optin, stream, ce, msg, len);
    default: return -1;  // not instantiated: the caller uses the bucket kernels
  }
}

}  // namespace tc
}  // namespace km
