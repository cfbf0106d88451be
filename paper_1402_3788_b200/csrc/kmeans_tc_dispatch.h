// kmeans_tc_dispatch.h — instantiation table of the tcgen05 pass (split across TUs for build speed).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include "kmeans_tc.h"

namespace km {
namespace tc {

template <int MT, int KP, bool PRE, bool X64>
int launch_t(const TcArgs& a, int num_sms, size_t smem_optin, cudaStream_t stream, cudaError_t* ce, char* msg,
             size_t len);

// exact feature counts (compile-time m): the BASELINE shapes
int launch_exact(const TcArgs& a, int m, int kp, bool pre, int num_sms, size_t smem_optin, cudaStream_t stream,
                 cudaError_t* ce, char* msg, size_t len);
// runtime m in buckets of 8 (≤ 31), always prescaled
int launch_bucket(const TcArgs& a, int mp, int kp, int num_sms, size_t smem_optin, cudaStream_t stream,
                  cudaError_t* ce, char* msg, size_t len);
// fp64 points (a.x64): the same buckets (+ m = 25 exact), X64 instantiations
int launch_f64(const TcArgs& a, int m, int mp, int kp, int num_sms, size_t smem_optin, cudaStream_t stream,
               cudaError_t* ce, char* msg, size_t len);

}  // namespace tc
}  // namespace km
