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
  unsigned long long changed;   // labels that changed in incremental passes
  double tol;
  int32_t passes;     // passes run by resident launches (statistics)
  int32_t pad_;
};

#ifdef __CUDACC__
// Exact 64-bit (mod 2^64) add into shared memory with two native 32-bit atomics
// (a 64-bit shared atomicAdd compiles to a CAS spin loop on sm_100a).
__device__ __forceinline__ void smem_add64(unsigned long long* addr, unsigned long long v) {
  unsigned int* p = reinterpret_cast<unsigned int*>(addr);
  const unsigned int lo = (unsigned int)v, hi = (unsigned int)(v >> 32);
  const unsigned int old = atomicAdd(p, lo);
  // unconditional (no branch on the returned value): independent adds pipeline
  atomicAdd(p + 1, hi + ((old + lo) < old ? 1u : 0u));
}

#endif

}  // namespace km
