// kmeans_state.h — device-side Lloyd loop state shared by all kernels.
#pragma once
#include <stdint.h>

namespace km {

// Device-side loop state (lives in device memory, mirrored to pinned host).
struct DevState {
  int32_t t;          // updates performed (reference `iterations`)
  int32_t done;       // loop finished
  int32_t converged;  // finished by convergence
  int32_t exhausted;  // t == max_iters without convergence: one more assign pass, then done
  int32_t need_host;  // empty clusters: host must run the repair before the check
  int32_t n_empty;
  int32_t max_iters;
  int32_t bad_label;  // first invalid label seen by a sums-only pass (+1), 0 = none
  unsigned long long rechecked;
  double tol;
};

}  // namespace km
