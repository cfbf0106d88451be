// kmeans_tc.h — host-side launcher of the tcgen05 fused pass (kmeans_tc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "kmeans_state.h"
#include "kmeans_finish.cuh"

namespace km {
namespace tc {

constexpr int kTile = 128;

struct TcArgs {
  const float* x;          // n × m fp32 row-major (fp64 points: their fp32 shadow, streamed by the pass)
  const double* x64;       // fp64 points: the exact rows (recheck, Δ); null for fp32 points
  int64_t n;
  int32_t m, k;
  const unsigned short* wop;  // [2KP][64] fp16 B operand rows ([wh|wh], [wl|0]) from the prep/finish kernel
  const float* cmax;       // [0] max ‖fl32(c)‖ (unscaled, rounded up)
  float xnorm_max;         // max ‖x‖ over the resident points (rounded up)
  const double* c64;       // k × m fp64 centres (exact recheck)
  int32_t* labels;         // in: L_{t-1} (incremental) / out: L_t (written where changed)
  unsigned long long* part;  // Δ (incremental) or full per-cluster fixed-point sums + counts
  float pre;               // 2^s operand prescale (|x·pre| < 1)
  float scale_f;           // 2^F fixed point
  double scale_d;
  int32_t use_dscale;
  float err_coef;          // certified bound coefficient for the tensor-core scores
  float err_floor;         // absolute floor (prescaled units)
  float nx_inflate;
  int32_t exact_only;
  int32_t exact_m;         // 1: use a compile-time-m instantiation when one exists for m
  int32_t prescale;        // 1: multiply x by `pre` (else the data are fp16-safe as is; pre == 1)
  int32_t full;            // 1: old labels invalid (first pass / standalone assign): add every point
  int32_t no_sums;         // 1: labels only (no Δ / sums): the first pass of a run, whose sums the
                           //    cluster-sums kernel computes in one stream afterwards
  int32_t skip_first;      // resident: the sums of the current labels are already in fin.tot
                           //    (first pass run separately): start the loop at the finish
  long long* recheck_rows;      // global overflow queue of uncertified points
  unsigned int* recheck_count;
  int32_t fuse_finish;     // 1: the last CTA to finish runs finish_block(fin) (single-GPU loop)
  unsigned int* cta_done;  // completion counter for the fused finish (self-resetting)
  FinishArgs fin;
  int32_t resident;        // 1: run the whole loop in this (cooperative) launch, see lloyd_pass_tc_kernel
  unsigned int* grid_sync; // resident: [0] barrier arrivals (zeroed before the launch)
  unsigned long long* dlt; // resident: [3][k·m + k] per-pass deltas (zeroed before the launch)
  // Row-sharded multi-GPU resident loop: after its local grid barrier every rank pushes its Δ
  // into every rank's exchange buffer over NVLink peer memory (CUDA IPC mappings) and sums the
  // `world` rows it received — one fused compute + all-reduce per iteration, no collective launch.
  // Buffer of each rank: [2 slots][world][k·m + k] u64 data, then [2][world] u64 sequence flags.
  unsigned long long* const* xch_peers;  // device array [world]: each rank's exchange buffer (null: single GPU)
  unsigned long long* xch_local;         // this rank's exchange buffer
  int32_t world, rank;
  uint32_t epoch;                        // run id (identical on every rank, new per km_lloyd_peer call)
  DevState* st;
  int32_t gate;
  float* dbg_scores;       // optional n × k raw tensor-core scores, unscaled (tests)
  int32_t dbg_flags;       // tuning experiments only: 2 = skip assign MMAs
  long long* dbg_times;    // tuning experiments only: per-tile clock64 stamps of CTA 0
};

// Launch lloyd_pass_tc_kernel<mp, kp>.  Returns 0 on success, 1 on a CUDA error
// (*cuda_err set), 2 if the shape does not fit, 3 if only the resident variant does not
// fit (the launch-per-iteration variant may); msg receives a description.
int launch(const TcArgs& a, int mp, int kp, int num_sms, size_t smem_optin, cudaStream_t stream,
           cudaError_t* cuda_err, char* msg, size_t msg_len);

// Re-decide the queued points exactly (after launch(), before the finish kernel).
cudaError_t launch_recheck(const TcArgs& a, int num_sms, cudaStream_t stream);

}  // namespace tc
}  // namespace km
