// kmeans_tc.h — host-side launcher of the tcgen05 fused pass (kmeans_tc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "kmeans_state.h"

namespace km {
namespace tc {

constexpr int kTile = 128;

struct TcArgs {
  const float* x;          // n × m fp32 row-major
  int64_t n;
  int32_t m, k;
  const float* wsplit;     // [2][KP][32] : tf32 hi, lo of W~ rows (prepared by the finish kernel)
  const float* cmax;       // [0] max ‖fl32(c)‖ rounded up
  const double* c64;       // k × m fp64 centres (exact recheck)
  int32_t* labels;
  unsigned long long* part;  // k·m sums + k counts (int64 fixed point)
  float scale_f;           // 2^F
  double scale_d;
  int32_t use_dscale;
  float err_coef;          // certified bound coefficient for the tensor-core scores
  float err_floor;
  float nx_inflate;
  int32_t exact_only;
  DevState* st;
  int32_t gate;
  int32_t do_sums;         // 0: assign only (counts still accumulated)
  float* dbg_scores;       // optional n × k raw tensor-core scores (tests)
  int32_t dbg_flags;       // tuning experiments only: 1 = skip update MMAs, 2 = skip assign MMAs
  long long* dbg_times;    // tuning experiments only: per-tile clock64 stamps of CTA 0
};

// Launch lloyd_pass_tc_kernel<mp, kp>.  Returns 0 on success, 1 on a CUDA error
// (*cuda_err set), 2 if the shape does not fit; msg receives a description.
int launch(const TcArgs& a, int mp, int kp, int num_sms, size_t smem_optin, cudaStream_t stream,
           cudaError_t* cuda_err, char* msg, size_t msg_len);

}  // namespace tc
}  // namespace km
