// kmeans_engine.cu — host engine + C ABI (include/kmeans_b200.h).
//
// The engine owns one CUDA stream on one device, the resident point matrix and
// the per-k device buffers.  km_lloyd reproduces engine.iterate
// (/root/reference/pkg/src/kmeans_regimes/engine.py:320-343) with the loop
// control on the device: every kernel checks the device-side DevState and the
// host reads that state once per batch of iterations (one 48-byte D2H).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/kmeans_b200.h"
#include "kmeans_kernels.cuh"
#include "kmeans_seed.cuh"
#include "kmeans_sums.cuh"
#include "kmeans_tc.h"

using namespace km;

static thread_local std::string g_global_err;

struct km_engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  std::string err;

  // resident points
  void* x = nullptr;
  bool x_owned = false;
  // grow-only device buffers (a reload / a new k reuses them when large enough; freed at destroy)
  void* xbuf = nullptr;             // owned points (fp32, or fp64 when narrowing would lose bits)
  void* stage = nullptr;            // fp64 upload staging
  void* x32 = nullptr;              // fp64 points: fp32 shadow streamed by the tensor-core pass (else null)
  bool no_shadow = false;           // KM_NO_FP32_SHADOW=1: fp64 points take the SIMT fp64 pass (A/B)
  size_t xbuf_cap = 0, stage_cap = 0, labels_cap = 0, rr_cap = 0, d2_cap = 0, l64_cap = 0, partials_cap = 0;
  // seeding: per-block pair-scan bests, min_d2 argmax partials
  PairBest* pair_best = nullptr;
  double* seed_pv = nullptr;
  long long* seed_pi = nullptr;
  size_t pair_best_cap = 0, seed_pv_cap = 0, seed_pi_cap = 0;
  // device jobs (MAX_PAIR rows, COORD_SUM / CLUSTER_SUM per-block sums)
  void* rows_dev = nullptr;
  void* job_acc = nullptr;
  void* job_lab = nullptr;
  size_t rows_cap = 0, job_acc_cap = 0, job_lab_cap = 0;
  bool seed_ready = false;
  int64_t n = 0;
  int32_t m = 0;
  int32_t point_bytes = 4;
  double absmax = 0.0;
  double op_absmax = 0.0;  // max(|x|, |C|) the tensor-core operand scale was chosen for
  int32_t frac_bits = 0;
  bool frac_user = false;

  // per-k buffers
  int32_t k = 0;
  int32_t mpad = 0;
  int32_t* labels = nullptr;        // n
  unsigned long long* part = nullptr;  // k*m + k
  double* cur = nullptr;            // k*m
  double* prev = nullptr;           // k*m
  long long* model_counts = nullptr;  // k
  float* w = nullptr;               // k*mpad
  float* cn = nullptr;              // k
  float* cmax = nullptr;            // 1
  DevState* st = nullptr;           // device
  DevState* st_host = nullptr;      // pinned
  double* d2 = nullptr;             // n (repair, lazily)
  ArgMax* partials = nullptr;       // argmax partials
  ArgMax* winner = nullptr;         // 1
  int32_t* scratch_i = nullptr;     // small device scratch
  double* scratch_d = nullptr;      // 2*k*m device scratch
  unsigned long long* scratch_u = nullptr;  // 2
  long long* labels64 = nullptr;    // n (download staging)
  int n_partials = 0;

  unsigned short* wop = nullptr;    // [2kp][64] fp16 tensor-core B operand ([wh|wh], [wl|0])
  int32_t kp = 0;                   // k padded for the tensor-core N dimension (16..128)
  float pre = 1.f;                  // power-of-two prescale of the tensor-core operands
  float xnorm_max = 0.f;            // max ‖x_i‖ over the resident points (rounded up)
  bool prescale = true;             // multiply x by `pre` in the tensor-core pass
  unsigned long long* tot = nullptr;  // running per-cluster totals (k·m sums + k counts)
  bool next_full = true;            // next TC pass must add every point (no valid previous labels)
  long long* recheck_rows = nullptr;     // queue of uncertified points (n)
  unsigned int* recheck_count = nullptr;
  unsigned int* cta_done = nullptr;      // fused-finish completion counter
  unsigned int* grid_sync = nullptr;     // resident loop: barrier arrivals
  unsigned long long* dlt = nullptr;     // resident loop: [3][k·m + k] per-pass deltas
  bool resident_unfit = false;           // the resident TC loop does not fit this shape (use per-iteration launches)
  bool last_pass_full = true;       // the most recent pass produced full sums (finish: tot = part)
  int32_t path_pref = 0;            // 0 auto, 1 SIMT only, 2 tensor-core required, 3 SIMT without register blocking
  float* dbg_scores = nullptr;      // test hook: raw tensor-core scores
  // environment knobs, read once at km_create (tuning / A-B experiments only)
  int full_first_pass = -1;         // KM_FULL_FIRST_PASS=1 / 0: force the fused / split first pass (-1: by n)
  bool no_resident = false;         // KM_NO_RESIDENT=1: launch-per-iteration loop
  bool call_trace = false;          // KM_CALL_TRACE=1: per-step device/host times of km_lloyd (stderr)
  int dbg_flags = 0;                // KM_TC_DBG
  const char* times_path = nullptr; // KM_TC_TIMES
  size_t sums_key = 0;              // cluster-sums launch geometry cache
  bool resident_zeroed = false;     // grid barrier + delta buffers are zero (next resident launch)
  // row-sharded multi-GPU resident loop (km_peer_*): in-kernel Δ exchange over NVLink peer memory
  int32_t world = 1, rank = 0;
  unsigned long long* xch = nullptr;         // this rank's exchange buffer (IPC-exported)
  size_t xch_nacc = 0;                       // k·m + k it was sized for
  unsigned long long** xch_peers_dev = nullptr;  // device array [world] of every rank's buffer
  std::vector<void*> xch_opened;             // IPC mappings of the peers' buffers
  uint32_t epoch = 0;                        // run id of the exchange's sequence flags
  bool peer_active = false;                  // the current km_lloyd_peer call uses the exchange
  void* pin = nullptr;              // pinned staging of the resident loop's C0 / model
  size_t pin_cap = 0;
  int sums_per_sm = 1;

  km_stats stats{};
  bool profiling = false;
  std::vector<cudaEvent_t> ev;  // profiling event pool (pairs)
};

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
static int set_err(km_engine* e, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (e) e->err = buf; else g_global_err = buf;
  return code;
}

static int cuda_fail(km_engine* e, cudaError_t c, const char* what) {
  const int code = (c == cudaErrorMemoryAllocation) ? KM_ERR_CAPACITY
                   : (c == cudaErrorNoDevice || c == cudaErrorInsufficientDriver || c == cudaErrorInvalidDevice)
                       ? KM_ERR_DEVICE_UNAVAILABLE
                       : KM_ERR_DEVICE_LOST;
  cudaGetLastError();  // clear sticky-free errors
  return set_err(e, code, "%s: %s (%s)", what, cudaGetErrorString(c), cudaGetErrorName(c));
}

#define CK(call)                                          \
  do {                                                    \
    cudaError_t _c = (call);                              \
    if (_c != cudaSuccess) return cuda_fail(e, _c, #call); \
  } while (0)

#define CK_LAUNCH(what)                                   \
  do {                                                    \
    cudaError_t _c = cudaGetLastError();                  \
    if (_c != cudaSuccess) return cuda_fail(e, _c, what); \
  } while (0)

template <typename P>
static int dalloc(km_engine* e, P** p, size_t bytes) {
  if (*p) { cudaFree(*p); *p = nullptr; }
  if (bytes == 0) bytes = 16;
  cudaError_t c = cudaMalloc((void**)p, bytes);
  if (c != cudaSuccess) { *p = nullptr; return cuda_fail(e, c, "cudaMalloc"); }
  return KM_OK;
}

static void dfree(void* p) { if (p) cudaFree(p); }

static int grow(km_engine* e, void** p, size_t* cap, size_t bytes) {
  if (*p && *cap >= bytes) return KM_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t c = cudaMalloc(p, bytes ? bytes : 16);
  if (c != cudaSuccess) { *p = nullptr; return cuda_fail(e, c, "cudaMalloc"); }
  *cap = bytes;
  return KM_OK;
}
template <typename P>
static int grow(km_engine* e, P** p, size_t* cap, size_t bytes) {
  return grow(e, reinterpret_cast<void**>(p), cap, bytes);
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
static int mp_for(int m) {
  static const int mps[] = {4, 8, 12, 16, 20, 24, 28, 32, 40, 48, 64};
  for (int v : mps) if (m <= v) return v;
  return 0;  // generic
}

static size_t pass_smem_bytes(const km_engine* e, bool assign, bool smem_acc, int elem_bytes) {
  auto a16 = [](size_t v) { return (v + 15) & ~size_t(15); };
  size_t b = 0;
  if (assign) b = a16(b + (size_t)e->k * e->mpad * 4) + 0, b = a16(b + (size_t)e->k * 4);
  if (smem_acc) b = a16(b + ((size_t)e->k * e->m + e->k) * 8);
  b += (size_t)kTileRows * e->m * elem_bytes;
  return b;
}

template <typename T, int MP, bool A, bool S, bool SA>
static int launch_pass_t(km_engine* e, const PassArgs& a, size_t smem) {
  auto kern = lloyd_pass_kernel<T, MP, A, S, SA>;
  if (smem > 48 * 1024) {
    cudaError_t c = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (c != cudaSuccess) return cuda_fail(e, c, "cudaFuncSetAttribute(pass smem)");
  }
  int per_sm = 0;
  cudaError_t c = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (c != cudaSuccess) return cuda_fail(e, c, "occupancy");
  if (per_sm < 1) return set_err(e, KM_ERR_CAPACITY, "pass kernel does not fit on an SM (smem %zu B)", smem);
  const int64_t ntiles = (a.n + kTileRows - 1) / kTileRows;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)per_sm * e->num_sms));
  kern<<<(unsigned)grid, kThreads, smem, e->stream>>>(a);
  CK_LAUNCH("lloyd_pass_kernel launch");
  e->stats.kernel_launches += 1;
  return KM_OK;
}

template <typename T, bool A, bool S, bool SA>
static int launch_pass_mp(km_engine* e, const PassArgs& a, size_t smem) {
  if (!A) return launch_pass_t<T, 0, A, S, SA>(e, a, smem);
  switch (mp_for(e->m)) {
    case 4: return launch_pass_t<T, 4, A, S, SA>(e, a, smem);
    case 8: return launch_pass_t<T, 8, A, S, SA>(e, a, smem);
    case 12: return launch_pass_t<T, 12, A, S, SA>(e, a, smem);
    case 16: return launch_pass_t<T, 16, A, S, SA>(e, a, smem);
    case 20: return launch_pass_t<T, 20, A, S, SA>(e, a, smem);
    case 24: return launch_pass_t<T, 24, A, S, SA>(e, a, smem);
    case 28: return launch_pass_t<T, 28, A, S, SA>(e, a, smem);
    case 32: return launch_pass_t<T, 32, A, S, SA>(e, a, smem);
    case 40: return launch_pass_t<T, 40, A, S, SA>(e, a, smem);
    case 48: return launch_pass_t<T, 48, A, S, SA>(e, a, smem);
    case 64: return launch_pass_t<T, 64, A, S, SA>(e, a, smem);
    default: return launch_pass_t<T, 0, A, S, SA>(e, a, smem);
  }
}

enum PassMode { PASS_ASSIGN_SUMS = 0, PASS_ASSIGN_ONLY = 1, PASS_SUMS_ONLY = 2 };
// register-blocked large-K pass (fp32 points, m ≤ 32, k ≥ kBlockedMinK): MP = the register row
static int blk_mp_for(int m) { return m <= 8 ? 8 : m <= 16 ? 16 : m <= 24 ? 24 : m == 25 ? 25 : m <= 28 ? 28 : m <= 32 ? 32 : 0; }
constexpr int kBlockedMinK = 32;
static size_t blocked_smem_bytes(const km_engine* e, int mp, bool smem_acc) {
  const size_t kp8 = ((size_t)e->k + 7) & ~size_t(7);
  return (size_t)mp * kp8 * 4 + kp8 * 4 + (smem_acc ? ((size_t)e->k * e->m + e->k) * 8 : 0);
}

template <int MP, bool S, bool SA>
static int launch_blocked_t(km_engine* e, const PassArgs& a, size_t smem) {
  auto kern = lloyd_pass_blocked_kernel<MP, S, SA>;
  if (smem > 48 * 1024) {
    cudaError_t c = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (c != cudaSuccess) return cuda_fail(e, c, "cudaFuncSetAttribute(blocked pass smem)");
  }
  int per_sm = 0;
  cudaError_t c = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlkThreads, smem);
  if (c != cudaSuccess) return cuda_fail(e, c, "occupancy");
  if (per_sm < 1) return set_err(e, KM_ERR_CAPACITY, "blocked pass kernel does not fit on an SM (smem %zu B)", smem);
  const int64_t ntiles = (a.n + kBlkTileRows - 1) / kBlkTileRows;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)per_sm * e->num_sms));
  kern<<<(unsigned)grid, kBlkThreads, smem, e->stream>>>(a, (e->k + 7) & ~7);
  CK_LAUNCH("lloyd_pass_blocked_kernel launch");
  e->stats.kernel_launches += 1;
  return KM_OK;
}

template <bool S, bool SA>
static int launch_blocked_mp(km_engine* e, const PassArgs& a, size_t smem, int mp) {
  switch (mp) {
    case 8: return launch_blocked_t<8, S, SA>(e, a, smem);
    case 16: return launch_blocked_t<16, S, SA>(e, a, smem);
    case 24: return launch_blocked_t<24, S, SA>(e, a, smem);
    case 25: return launch_blocked_t<25, S, SA>(e, a, smem);
    case 28: return launch_blocked_t<28, S, SA>(e, a, smem);
    default: return launch_blocked_t<32, S, SA>(e, a, smem);
  }
}


// tensor-core path: fp32 resident points, m ≤ 31 ([xh|xl] + the ones column fit one 128-byte
// fp16 row), k ≤ 128 (N = 2·KP ≤ 256 per MMA; 2 warpgroups × 2·KP TMEM columns ≤ 512)
static bool tc_eligible(const km_engine* e) {
  return (e->point_bytes == 4 || e->x32 != nullptr) && e->m <= 31 && e->kp >= 16 && e->kp <= 128;
}
static bool use_tc(const km_engine* e) { return e->path_pref != 1 && e->path_pref != 3 && tc_eligible(e); }

static int tc_mp_for(int m) { return m <= 7 ? 7 : m <= 15 ? 15 : m <= 23 ? 23 : 31; }

static float host_err_coef_tc(int m, int mp) {
  // |S_tc − S| ≤ coef·(‖x‖ + max‖c‖)² for the kind::f16 scores (fp16 hi/lo split of both
  // operands, fp32 accumulation): the split residue (|x − xh − xl| ≤ 2⁻²²|x|, same for w) and the
  // dropped xl·wl term (≤ 3·2⁻²¹ of Σ|x_f w_f| ≤ 2‖x‖‖c‖), the accumulation of the k-steps (the
  // products are exact; each k-step's sum and the fp32 accumulator are charged 2⁻²³ of the
  // largest product per step), the fp32 rounding of c and ‖c‖², and the reference's own fp64
  // rounding.  The hardware adder's alignment width is not documented, so the coefficient is
  // checked adversarially: tests/test_gpu_tensorcore.py sweeps product ratios 2⁻⁸ … 2⁻³⁰ with one
  // large and 24 small same-sign (or alternating) products per k-step and requires the worst
  // observed error ≤ coef/4 (profiles/r02_tensorcore_margins.txt has the margins).
  const int ks = (mp + 1 + 7) / 8;
  return (float)std::max((m + 8 + 12 * ks) * std::ldexp(1.0, -23), std::ldexp(1.0, -18));
}

static FinishArgs finish_args(km_engine* e, int mode, bool accumulate);
static int finish_threads(int k, int m);

// resident: the whole Lloyd loop in one cooperative launch (returns KM_RESIDENT_UNFIT when the
// shape only fits the launch-per-iteration kernel)
constexpr int KM_RESIDENT_UNFIT = -3;
static int launch_tc(km_engine* e, bool full, bool gated, bool fuse = false, bool resident = false,
                     bool no_sums = false, bool skip_first = false) {
  tc::TcArgs a{};
  // fp64 points: the pass streams the fp32 shadow; the exact rows come from x64
  a.x = (const float*)(e->point_bytes == 8 ? e->x32 : e->x);
  a.x64 = e->point_bytes == 8 ? (const double*)e->x : nullptr;
  a.n = e->n;
  a.m = e->m;
  a.k = e->k;
  a.wop = e->wop;
  a.cmax = e->cmax;
  a.xnorm_max = e->xnorm_max;
  a.c64 = e->cur;
  a.labels = e->labels;
  a.part = e->part;
  a.pre = e->pre;
  const int F = e->frac_bits;
  a.scale_d = std::ldexp(1.0, F);
  a.use_dscale = (F > 120 || F < -120) ? 1 : 0;
  a.scale_f = a.use_dscale ? 1.0f : (float)std::ldexp(1.0, F);
  const int mp = tc_mp_for(e->m);
  // (+ the fp32 rounding of the shadow coordinates, |fl32(x) − x| ≤ 2⁻²⁴|x|, for fp64 points)
  a.err_coef = host_err_coef_tc(e->m, mp) + (e->point_bytes == 8 ? (float)std::ldexp(1.0, -22) : 0.f);
  // absolute floor (operand units): fp16 subnormal spacing 2^-24 per element times |w| ≤ 2·max‖x‖·pre
  a.err_floor = (float)((e->m + 2) * std::ldexp(1.0, -23) * (1.0 + 2.0 * e->xnorm_max * e->pre));
  a.nx_inflate = (float)(1.0 + (e->m + 2) * std::ldexp(1.0, -24));
  a.exact_only = (e->op_absmax > std::ldexp(1.0, 50)) ? 1 : 0;
  a.full = full ? 1 : 0;
  a.no_sums = no_sums ? 1 : 0;
  a.skip_first = skip_first ? 1 : 0;
  a.exact_m = 1;
  a.prescale = e->prescale ? 1 : 0;
  a.recheck_rows = e->recheck_rows;
  a.recheck_count = e->recheck_count;
  a.fuse_finish = fuse ? 1 : 0;
  a.cta_done = e->cta_done;
  a.fin = finish_args(e, 0, !full);
  a.fin.recheck_rows = e->recheck_rows;  // the fused finish re-decides the overflow queue itself
  a.fin.full = full ? 1 : 0;
  a.resident = resident ? 1 : 0;
  a.grid_sync = e->grid_sync;
  a.dlt = e->dlt;

  if (resident && e->peer_active) {
    a.xch_peers = e->xch_peers_dev;
    a.xch_local = e->xch;
    a.world = e->world;
    a.rank = e->rank;
    a.epoch = e->epoch;
  } else {
    a.xch_peers = nullptr;
    a.xch_local = nullptr;
    a.world = 1;
    a.rank = 0;
    a.epoch = 0;
  }
  if (resident && !e->resident_zeroed) {  // (the begin kernel zeroed them for the first launch of a run)
    CK(cudaMemsetAsync(e->grid_sync, 0, 16, e->stream));
    CK(cudaMemsetAsync(e->dlt, 0, 3 * 8 * ((size_t)e->k * e->m + e->k), e->stream));
  }
  if (resident) e->resident_zeroed = false;
  a.st = e->st;
  a.gate = gated ? 1 : 0;
  a.dbg_scores = e->dbg_scores;
  a.dbg_flags = e->dbg_flags;
  a.dbg_times = nullptr;
  if (e->times_path) {  // tuning only: dump per-tile stamps of CTA 0 to a file after the pass
    static long long* dt = nullptr;
    if (!dt) cudaMalloc((void**)&dt, 1024 * 8 * 8);
    cudaMemsetAsync(dt, 0, 1024 * 8 * 8, e->stream);
    a.dbg_times = dt;
  }
  char msg[256] = {0};
  cudaError_t c = cudaSuccess;
  const int rc = tc::launch(a, mp, e->kp, e->num_sms, e->smem_optin, e->stream, &c, msg, sizeof msg);
  if (rc == 1) return cuda_fail(e, c, msg);
  if (rc == 2) return set_err(e, KM_ERR_CAPACITY, "%s", msg);
  if (rc == 3) return KM_RESIDENT_UNFIT;
  e->stats.kernel_launches += 1;
  // (no recheck launch: the tensor-core pass re-decides every uncertified point itself — its
  // per-CTA queue overflows are decided inline — and never writes the global recheck queue)
  if (a.dbg_times) {
    static long long h[1024 * 8];
    cudaMemcpyAsync(h, a.dbg_times, sizeof h, cudaMemcpyDeviceToHost, e->stream);
    cudaStreamSynchronize(e->stream);
    FILE* f = fopen(e->times_path, "a");
    if (f) {
      for (int i = 0; i < 64; ++i) {
        if (!h[i * 8]) continue;
        const long long* t = h + i * 8;  // transform: 0 start, 1 raw ok, 7 raw released, 2 A ok, 3 a_full; epilogue: 4 start, 5 got, 6 done
        const long long* u = h + 3072 + i * 4;  // MMA: 0 start, 1 a_full ok, 2 s_empty ok, 3 issued
        const long long z = h[0];
        fprintf(f, "tile %2d T[%6lld raw+%4lld comp+%4lld A+%4lld sts+%4lld] M[%6lld af+%4lld se+%4lld is+%4lld] E[%6lld got+%4lld body+%4lld]\n", i,
                t[0] - z, t[1] - t[0], t[7] - t[1], t[2] - t[7], t[3] - t[2], u[0] - z, u[1] - u[0], u[2] - u[1], u[3] - u[2],
                t[4] - z, t[5] - t[4], t[6] - t[5]);
      }
      if (resident && h[6144]) {  // per-CTA main loop of pass 100 (ns)
        long long s0 = h[6144], s1 = h[6144], dmin = 1ll << 60, dmax = 0, dsum = 0, e1 = 0;
        int nb = 0, bmax = 0;
        for (int b = 0; b < 148 && h[6144 + 2 * b]; ++b, ++nb) {
          const long long st0 = h[6144 + 2 * b], en = h[6144 + 2 * b + 1], d = en - st0;
          s0 = std::min(s0, st0); s1 = std::max(s1, st0); e1 = std::max(e1, en);
          dmin = std::min(dmin, d); dsum += d;
          if (d > dmax) { dmax = d; bmax = b; }
        }
        fprintf(f, "pass 100 main loop per CTA (ns): min %lld avg %lld max %lld (cta %d)  start skew %lld  span %lld\n",
                dmin, dsum / std::max(1, nb), dmax, bmax, s1 - s0, e1 - s0);
        for (int b = 0; b < nb; b += 8) {
          fprintf(f, "  cta %3d..:", b);
          for (int j = b; j < std::min(nb, b + 8); ++j) fprintf(f, " %6lld", h[6144 + 2 * j + 1] - h[6144 + 2 * j]);
          fprintf(f, "\n");
        }
      }
      if (resident && h[6144] && h[6444] && h[6744]) {  // is the per-CTA pass time systematic? (passes 100/101/150)
        double a[3][148];
        int nb = 0;
        for (int b = 0; b < 148 && h[6144 + 2 * b]; ++b, ++nb)
          for (int q = 0; q < 3; ++q) a[q][b] = (double)(h[6144 + 300 * q + 2 * b + 1] - h[6144 + 300 * q + 2 * b]);
        auto corr = [&](int p, int q) {
          double mp = 0, mq = 0, spq = 0, spp = 0, sqq = 0;
          for (int b = 0; b < nb; ++b) { mp += a[p][b]; mq += a[q][b]; }
          mp /= nb; mq /= nb;
          for (int b = 0; b < nb; ++b) {
            spq += (a[p][b] - mp) * (a[q][b] - mq); spp += (a[p][b] - mp) * (a[p][b] - mp); sqq += (a[q][b] - mq) * (a[q][b] - mq);
          }
          return spq / std::sqrt(spp * sqq + 1e-30);
        };
        fprintf(f, "per-CTA main-loop time correlation: pass100~101 %.3f  pass100~150 %.3f  pass101~150 %.3f\n",
                corr(0, 1), corr(0, 2), corr(1, 2));
      }
      if (resident) {  // per-pass phase ends of the resident loop (ns, max over CTAs, from CTA 0's start)
        const unsigned long long* q = reinterpret_cast<const unsigned long long*>(h + 4096);
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int cnt = 0;
        for (int it = 20; it < 256; ++it) {
          const unsigned long long* u = q + it * 8;
          if (!u[7] || !u[6]) break;
          for (int j = 1; j < 8; ++j) acc[j] += (double)(long long)(u[j] - u[0]);
          ++cnt;
        }
        if (cnt)
          fprintf(f, "resident passes 20..%d (ns after CTA0 start): main %.0f recheck %.0f flush %.0f barrier-passed %.0f "
                  "finish %.0f conv %.0f prep %.0f\n", 20 + cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt,
                  acc[4] / cnt, acc[5] / cnt, acc[6] / cnt, acc[7] / cnt);
      }
      fprintf(f, "----\n");
      fclose(f);
    }
  }
  return KM_OK;
}

static float host_err_coef(int m) { return (float)((m + 8) * std::ldexp(1.0, -24) * 1.25); }

static int launch_pass(km_engine* e, PassMode mode, bool gated, bool fuse_finish = false) {
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if (mode != PASS_SUMS_ONLY && use_tc(e)) {
    // the TC pass updates the sums by exact deltas against the previous labels; the first
    // pass of a run (and any standalone assign) adds every point
    const bool full = e->next_full || mode == PASS_ASSIGN_ONLY;
    const int r = launch_tc(e, full, gated, fuse_finish && mode == PASS_ASSIGN_SUMS);
    if (!r && mode == PASS_ASSIGN_SUMS) e->next_full = false;  // tot will track the labels from here on
    e->last_pass_full = full;
    return r;
  }
  e->last_pass_full = true;  // SIMT passes recompute the sums
  if (e->path_pref == 2) return set_err(e, KM_ERR_CAPACITY, "tensor-core path not available for m=%d k=%d (%d-byte points)",
                                        e->m, e->k, e->point_bytes);
  const bool A = mode != PASS_SUMS_ONLY;
  PassArgs a{};
  a.x = e->x;
  a.n = e->n;
  a.m = e->m;
  a.k = e->k;
  a.w = e->w;
  a.cn = e->cn;
  a.cmax = e->cmax;
  a.c64 = e->cur;
  a.labels = e->labels;
  a.part = e->part;
  const int F = e->frac_bits;
  a.scale_d = std::ldexp(1.0, F);
  a.use_dscale = (F > 120 || F < -120) ? 1 : 0;
  a.scale_f = a.use_dscale ? 1.0f : (float)std::ldexp(1.0, F);
  a.mpad = e->mpad;
  a.err_coef = host_err_coef(e->m);
  a.err_floor = (float)((e->m + 2) * std::ldexp(1.0, -140));
  a.nx_inflate = (float)(1.0 + (e->m + 2) * std::ldexp(1.0, -24));
  const bool huge = e->absmax > std::ldexp(1.0, 50);
  const bool tiny64 = e->point_bytes == 8 && e->absmax > 0 && e->absmax < std::ldexp(1.0, -100);
  a.exact_only = (huge || tiny64) ? 1 : 0;
  a.st = e->st;
  a.gate = gated ? 1 : 0;
  const PassArgs& a2 = a;
  const int eb = e->point_bytes;
  size_t smem_sa = pass_smem_bytes(e, A, true, eb);
  const bool sa = smem_sa <= e->smem_optin;
  size_t smem = sa ? smem_sa : pass_smem_bytes(e, A, false, eb);
  if (smem > e->smem_optin)
    return set_err(e, KM_ERR_CAPACITY, "k=%d, m=%d needs %zu B of shared memory per CTA (max %zu)", e->k, e->m, smem,
                   e->smem_optin);
  if (eb == 4 && A && e->k >= kBlockedMinK && blk_mp_for(e->m) > 0 && e->path_pref != 3) {
    const int mp = blk_mp_for(e->m);
    const size_t bs_sa = blocked_smem_bytes(e, mp, true), bs_g = blocked_smem_bytes(e, mp, false);
    if (bs_g <= e->smem_optin) {
      const bool bsa = bs_sa <= e->smem_optin;
      const size_t bsm = bsa ? bs_sa : bs_g;
      if (mode == PASS_ASSIGN_SUMS) return bsa ? launch_blocked_mp<true, true>(e, a2, bsm, mp) : launch_blocked_mp<true, false>(e, a2, bsm, mp);
      return bsa ? launch_blocked_mp<false, true>(e, a2, bsm, mp) : launch_blocked_mp<false, false>(e, a2, bsm, mp);
    }
  }
  if (eb == 4) {
    if (mode == PASS_ASSIGN_SUMS) return sa ? launch_pass_mp<float, true, true, true>(e, a2, smem) : launch_pass_mp<float, true, true, false>(e, a2, smem);
    if (mode == PASS_ASSIGN_ONLY) return sa ? launch_pass_mp<float, true, false, true>(e, a2, smem) : launch_pass_mp<float, true, false, false>(e, a2, smem);
    return sa ? launch_pass_mp<float, false, true, true>(e, a2, smem) : launch_pass_mp<float, false, true, false>(e, a2, smem);
  } else {
    if (mode == PASS_ASSIGN_SUMS) return sa ? launch_pass_mp<double, true, true, true>(e, a2, smem) : launch_pass_mp<double, true, true, false>(e, a2, smem);
    if (mode == PASS_ASSIGN_ONLY) return sa ? launch_pass_mp<double, true, false, true>(e, a2, smem) : launch_pass_mp<double, true, false, false>(e, a2, smem);
    return sa ? launch_pass_mp<double, false, true, true>(e, a2, smem) : launch_pass_mp<double, false, true, false>(e, a2, smem);
  }
}

static FinishArgs finish_args(km_engine* e, int mode, bool accumulate) {
  FinishArgs f{};
  f.part = e->part;
  f.tot = e->tot;
  f.accumulate = accumulate ? 1 : 0;
  f.recheck_count = e->recheck_count;
  f.recheck_rows = nullptr;  // standalone finish: the recheck kernel already re-decided the overflow
  f.x = (const float*)(e->point_bytes == 8 ? e->x32 : e->x);
  f.x64 = e->point_bytes == 8 ? (const double*)e->x : nullptr;
  f.labels = e->labels;
  f.full = 0;
  f.scale_d = std::ldexp(1.0, e->frac_bits);
  f.use_dscale = (e->frac_bits > 120 || e->frac_bits < -120) ? 1 : 0;
  f.scale_f = f.use_dscale ? 1.0f : (float)f.scale_d;
  f.cur = e->cur;
  f.prev = e->prev;
  f.model_counts = e->model_counts;
  f.w = e->w;
  f.cn = e->cn;
  f.cmax = e->cmax;
  f.wop = tc_eligible(e) ? e->wop : nullptr;
  f.kp = e->kp;
  f.pre = e->pre;
  f.k = e->k;
  f.m = e->m;
  f.mpad = e->mpad;
  f.inv_scale = std::ldexp(1.0, -e->frac_bits);
  f.st = e->st;
  f.mode = mode;
  return f;
}

static int finish_threads(int k, int m) {
  const int work = std::max(k, k * m);
  int t = 128;
  while (t < 512 && t < work) t *= 2;
  return t;
}

static int launch_finish(km_engine* e, int mode, bool accumulate) {
  FinishArgs f = finish_args(e, mode, accumulate);
  const int cap = 2 * e->k * e->m <= 6144 ? 2 * e->k * e->m : 0;  // stage C_{t-1}, C_t in ≤ 48 KB
  lloyd_finish_kernel<<<1, finish_threads(e->k, e->m), (size_t)cap * 8, e->stream>>>(f, cap);
  CK_LAUNCH("lloyd_finish_kernel launch");
  e->stats.kernel_launches += 1;
  return KM_OK;
}

static int launch_check(km_engine* e) {
  FinishArgs f = finish_args(e, 0, false);
  lloyd_check_kernel<<<1, finish_threads(e->k, e->m), 0, e->stream>>>(f);
  CK_LAUNCH("lloyd_check_kernel launch");
  e->stats.kernel_launches += 1;
  return KM_OK;
}

static int launch_prep(km_engine* e) {
  prep_filter_kernel<<<1, finish_threads(e->k, e->m), 0, e->stream>>>(
      e->cur, e->w, e->cn, e->cmax, e->k, e->m, e->mpad, tc_eligible(e) ? e->wop : nullptr, e->kp, e->pre);
  CK_LAUNCH("prep_filter_kernel launch");
  e->stats.kernel_launches += 1;
  return KM_OK;
}

static int read_state(km_engine* e) {
  CK(cudaMemcpyAsync(e->st_host, e->st, sizeof(DevState), cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  e->stats.host_syncs += 1;
  return KM_OK;
}

static int reset_state(km_engine* e, int max_iters, double tol) {
  DevState s{};
  s.max_iters = max_iters;
  s.tol = tol;
  *e->st_host = s;
  CK(cudaMemcpyAsync(e->st, e->st_host, sizeof(DevState), cudaMemcpyHostToDevice, e->stream));
  return KM_OK;
}

static int grid_for(km_engine* e, int64_t n, int per_sm = 8) {
  int64_t g = (n + 255) / 256;
  g = std::min<int64_t>(g, (int64_t)e->num_sms * per_sm);
  return (int)std::max<int64_t>(1, g);
}

// ---------------------------------------------------------------------------
// buffers
// ---------------------------------------------------------------------------
// k-sized buffers only; the n-sized ones (labels, recheck queue, d2, label staging, partials) are
// grow-only and live until destroy
static void free_k(km_engine* e) {
  dfree(e->part); dfree(e->cur); dfree(e->prev); dfree(e->model_counts);
  dfree(e->w); dfree(e->cn); dfree(e->cmax); dfree(e->winner);
  dfree(e->scratch_d); dfree(e->wop); dfree(e->tot);
  dfree(e->recheck_count); dfree(e->cta_done); dfree(e->grid_sync); dfree(e->dlt);
  e->dlt = nullptr;
  e->part = nullptr; e->cur = nullptr; e->prev = nullptr; e->model_counts = nullptr;
  e->w = nullptr; e->cn = nullptr; e->cmax = nullptr; e->winner = nullptr;
  e->scratch_d = nullptr; e->wop = nullptr; e->tot = nullptr;
  e->recheck_count = nullptr; e->cta_done = nullptr; e->grid_sync = nullptr;
  e->resident_unfit = false;
  e->k = 0;
  e->kp = 0;
}

static int ensure_k(km_engine* e, int32_t k) {
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if (k < 1) return set_err(e, KM_ERR_CONTRACT, "k must be >= 1, got %d", k);
  if (k == e->k && e->labels) return KM_OK;
  free_k(e);
  const int m = e->m;
  e->mpad = mp_for(m) ? mp_for(m) : ((m + 3) & ~3);
  int r;
  if ((r = grow(e, &e->labels, &e->labels_cap, sizeof(int32_t) * (size_t)e->n))) return r;
  if ((r = dalloc(e, &e->part, 8 * ((size_t)k * m + k)))) return r;
  if ((r = dalloc(e, &e->cur, 8 * (size_t)k * m))) return r;
  if ((r = dalloc(e, &e->prev, 8 * (size_t)k * m))) return r;
  if ((r = dalloc(e, &e->model_counts, 8 * (size_t)k))) return r;
  if ((r = dalloc(e, &e->w, 4 * (size_t)k * e->mpad))) return r;
  if ((r = dalloc(e, &e->cn, 4 * (size_t)k))) return r;
  if ((r = dalloc(e, &e->cmax, 16))) return r;
  if ((r = dalloc(e, &e->scratch_d, 8 * 2 * (size_t)k * m))) return r;
  e->n_partials = grid_for(e, e->n);
  if ((r = grow(e, &e->partials, &e->partials_cap, sizeof(ArgMax) * (size_t)e->n_partials))) return r;
  if ((r = dalloc(e, &e->winner, sizeof(ArgMax)))) return r;
  // tensor-core N padding: 16s to 64, 32s to 128 (K > 128 takes the SIMT blocked pass)
  e->kp = k <= 64 ? ((k + 15) & ~15) : k <= 128 ? ((k + 31) & ~31) : 1024;
  if ((r = dalloc(e, &e->wop, sizeof(unsigned short) * 2 * 64 * (size_t)e->kp))) return r;
  CK(cudaMemsetAsync(e->wop, 0, sizeof(unsigned short) * 2 * 64 * (size_t)e->kp, e->stream));
  if ((r = dalloc(e, &e->tot, 8 * ((size_t)k * m + k)))) return r;
  if ((r = grow(e, &e->recheck_rows, &e->rr_cap, 8 * (size_t)e->n))) return r;
  if ((r = dalloc(e, &e->recheck_count, 16))) return r;
  CK(cudaMemsetAsync(e->recheck_count, 0, 16, e->stream));
  if ((r = dalloc(e, &e->cta_done, 16))) return r;
  if ((r = dalloc(e, &e->grid_sync, 16))) return r;
  if ((r = dalloc(e, &e->dlt, 3 * 8 * ((size_t)k * m + k)))) return r;
  CK(cudaMemsetAsync(e->cta_done, 0, 16, e->stream));
  CK(cudaMemsetAsync(e->tot, 0, 8 * ((size_t)k * m + k), e->stream));
  e->next_full = true;
  CK(cudaMemsetAsync(e->part, 0, 8 * ((size_t)k * m + k), e->stream));
  CK(cudaMemsetAsync(e->labels, 0, sizeof(int32_t) * (size_t)e->n, e->stream));
  e->k = k;
  return KM_OK;
}

static int compute_frac_bits(double absmax, int64_t n_total) {
  if (n_total < 1) n_total = 1;
  double bound = std::max(absmax, 1e-300) * (double)n_total;
  int ex = 0;
  std::frexp(bound, &ex);  // bound < 2^ex
  int F = 62 - ex;
  if (absmax == 0.0) F = 62 - 1 - (int)std::ceil(std::log2((double)n_total));
  F = std::max(-60, std::min(1000, F));
  return F;
}

// exact max |x| (+ finiteness) on the device; sets the fixed-point scale.
static int scan_points(km_engine* e, const void* x, int bytes_per, int64_t count, int* flags_out) {
  unsigned long long zero = 0;
  int zf[2] = {0, 0};
  CK(cudaMemcpyAsync(e->scratch_u, &zero, 8, cudaMemcpyHostToDevice, e->stream));
  CK(cudaMemcpyAsync(e->scratch_i, zf, 8, cudaMemcpyHostToDevice, e->stream));
  const int g = grid_for(e, count, 4);
  if (bytes_per == 4)
    absmax_kernel<float><<<g, 256, 0, e->stream>>>((const float*)x, count, e->scratch_u, e->scratch_i);
  else
    absmax_kernel<double><<<g, 256, 0, e->stream>>>((const double*)x, count, e->scratch_u, e->scratch_i);
  CK_LAUNCH("absmax_kernel");
  e->stats.kernel_launches += 1;
  unsigned long long bits = 0;
  CK(cudaMemcpyAsync(&bits, e->scratch_u, 8, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaMemcpyAsync(flags_out, e->scratch_i, 8, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  double v;
  std::memcpy(&v, &bits, 8);
  e->absmax = v;
  return KM_OK;
}

// Tensor-core operand range (fp16 hi/lo): `amax` bounds every |x_f| AND every |c_f| the pass
// will see.  Data already in a safe range (amax ≥ 2^-4, every score |S| ≤ ‖c‖² + 2|x·c| ≤
// 3·m·amax² ≤ 2^15 < the +65504 padding score) go as is; otherwise both operands are prescaled
// by an exact power of two 2^s with |v·2^s| < 1.  Lloyd iterates are means of points (|c_f| ≤
// max|x_f|), but caller-supplied centres (km_assign, C0 of km_lloyd / km_step_begin) may be far
// larger than the data, so those entry points widen amax to max(max|x|, max|C|).
static void choose_operand_scale(km_engine* e, double amax) {
  e->op_absmax = amax;
  e->pre = 1.f;
  e->prescale = true;
  if (amax >= std::ldexp(1.0, -4) && 4.0 * e->m * amax * amax <= 32768.0) {
    e->prescale = false;
  } else if (amax > 0.0 && amax < std::ldexp(1.0, 100)) {
    const int s = -(std::ilogb(amax) + 1);
    e->pre = (float)std::ldexp(1.0, std::max(-120, std::min(120, s)));
  }
}

// widen the operand range to the centres a run starts from (see choose_operand_scale)
static void scale_for_centers(km_engine* e, const double* c, int32_t k) {
  double cm = 0.0;
  for (int64_t i = 0; i < (int64_t)k * e->m; ++i) cm = std::max(cm, std::fabs(c[i]));
  choose_operand_scale(e, std::max(e->absmax, cm));
}

static int after_points_loaded(km_engine* e) {
  {  // max ‖x_i‖ for the tensor-core filter bound
    unsigned int zero = 0, bits = 0;
    CK(cudaMemcpyAsync(e->scratch_u, &zero, 4, cudaMemcpyHostToDevice, e->stream));
    const int g = grid_for(e, e->n, 4);
    if (e->point_bytes == 4)
      rownorm_max_kernel<float><<<g, 256, 0, e->stream>>>((const float*)e->x, e->n, e->m, (unsigned int*)e->scratch_u);
    else
      rownorm_max_kernel<double><<<g, 256, 0, e->stream>>>((const double*)e->x, e->n, e->m, (unsigned int*)e->scratch_u);
    CK_LAUNCH("rownorm_max_kernel");
    e->stats.kernel_launches += 1;
    CK(cudaMemcpyAsync(&bits, e->scratch_u, 4, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    std::memcpy(&e->xnorm_max, &bits, 4);
  }
  if (!e->frac_user) e->frac_bits = compute_frac_bits(e->absmax, e->n);
  choose_operand_scale(e, e->absmax);
  e->next_full = true;
  e->stats.frac_bits = e->frac_bits;
  e->stats.point_bytes = e->point_bytes;
  return KM_OK;
}

static int drop_points(km_engine* e) {
  free_k(e);
  e->seed_ready = false;
  e->x = nullptr;  // an owned copy lives on in xbuf / stage for the next load
  e->x32 = nullptr;
  e->x_owned = false;
  e->n = 0;
  e->m = 0;
  // a fixed-point scale set for the previous points (km_set_frac_bits) is not valid for new
  // ones: a larger n·max|x| would overflow the int64 sums
  e->frac_user = false;
  return KM_OK;
}

static int validate_points_shape(km_engine* e, const void* x, int64_t n, int32_t m) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!x) return set_err(e, KM_ERR_CONTRACT, "null point buffer");
  if (n < 1 || m < 1) return set_err(e, KM_ERR_CONTRACT, "points must be non-empty, got shape (%lld, %d)", (long long)n, m);
  if (n > (int64_t)INT32_MAX * 64) return set_err(e, KM_ERR_CONTRACT, "n too large");
  return KM_OK;
}

// ---------------------------------------------------------------------------
// repair (engine.py:265-276), single shard
// ---------------------------------------------------------------------------
static int self_d2(km_engine* e) {
  { int r = grow(e, &e->d2, &e->d2_cap, 8 * (size_t)e->n); if (r) return r; }
  const int g = grid_for(e, e->n);
  if (e->point_bytes == 4)
    self_d2_kernel<float><<<g, 256, 0, e->stream>>>((const float*)e->x, e->n, e->m, e->cur, e->labels, e->d2);
  else
    self_d2_kernel<double><<<g, 256, 0, e->stream>>>((const double*)e->x, e->n, e->m, e->cur, e->labels, e->d2);
  CK_LAUNCH("self_d2_kernel");
  e->stats.kernel_launches += 1;
  return KM_OK;
}

static int empty_list(km_engine* e, std::vector<int32_t>& out) {
  std::vector<long long> cnt(e->k);
  CK(cudaMemcpyAsync(cnt.data(), e->model_counts, 8 * (size_t)e->k, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  out.clear();
  for (int c = 0; c < e->k; ++c) if (cnt[c] == 0) out.push_back(c);
  return KM_OK;
}

static int repair_local(km_engine* e) {
  std::vector<int32_t> empties;
  int r;
  if ((r = empty_list(e, empties))) return r;
  if (empties.empty()) return KM_OK;
  if ((r = self_d2(e))) return r;
  for (int32_t c : empties) {
    argmax_partial_kernel<<<e->n_partials, 256, 0, e->stream>>>(e->d2, e->n, e->partials);
    CK_LAUNCH("argmax_partial_kernel");
    if (e->point_bytes == 4)
      repair_apply_kernel<float><<<1, 512, 0, e->stream>>>(e->partials, e->n_partials, c, (const float*)e->x, e->k,
                                                          e->m, e->labels, e->d2, e->model_counts, e->cur, e->tot,
                                                          std::ldexp(1.0, e->frac_bits), e->winner);
    else
      repair_apply_kernel<double><<<1, 512, 0, e->stream>>>(e->partials, e->n_partials, c, (const double*)e->x,
                                                           e->k, e->m, e->labels, e->d2, e->model_counts, e->cur,
                                                           e->tot, std::ldexp(1.0, e->frac_bits), e->winner);
    CK_LAUNCH("repair_apply_kernel");
    e->stats.repairs += 1;
    e->stats.kernel_launches += 2;
  }
  return KM_OK;
}

static int download_labels(km_engine* e, int64_t* out) {
  { int r = grow(e, &e->labels64, &e->l64_cap, 8 * (size_t)e->n); if (r) return r; }
  widen_labels_kernel<<<grid_for(e, e->n), 256, 0, e->stream>>>(e->labels, e->n, e->labels64);
  CK_LAUNCH("widen_labels_kernel");
  e->stats.kernel_launches += 1;
  CK(cudaMemcpyAsync(out, e->labels64, 8 * (size_t)e->n, cudaMemcpyDeviceToHost, e->stream));
  return KM_OK;
}

// Exact fixed-point sums + counts of every resident point by its current label, added into `out`
// ([k·m sums][k counts], zeroed by the caller): one HBM stream, warp-private accumulators where
// they fit (kmeans_sums.cuh).  Also clears the recheck overflow counter of the pass before it.
static int launch_sums(km_engine* e, unsigned long long* out) {
  if (e->m > 31) return set_err(e, KM_ERR_INTERNAL, "cluster-sums kernel: m <= 31 only");
  const bool f64 = e->point_bytes == 8;  // fp64 points: sums of the exact fp64 coordinates
  const size_t per = (size_t)e->k * (e->m + 1) * 8;
  const bool use_d = e->frac_bits > 120 || e->frac_bits < -120;
  // shared-memory accumulators, warp-private where they fit.  (Measured and dropped: cluster-owner
  // warps with register accumulators, 120 µs vs 70 µs at cfg3; label-grouped 32-row batches,
  // 133 µs — both latency-bound ballot loops.)
  const bool priv = per * kSumsWarps <= 100 * 1024;
  const size_t smem = sums_smem_bytes(e->m, e->k, priv, f64 ? 8 : 4);
  if (smem > e->smem_optin) return set_err(e, KM_ERR_CAPACITY, "cluster-sums kernel: k·m too large for shared memory");
  using Kern = void (*)(const float*, const int32_t*, int64_t, int, int, float, double, unsigned long long*);
  // compile-time feature counts for the BASELINE shapes
  auto accum = [&](auto mt) -> Kern {
    constexpr int MT = decltype(mt)::value;
    return priv ? (use_d ? cluster_sums_f32_kernel<float, MT, true, true> : cluster_sums_f32_kernel<float, MT, true, false>)
                : (use_d ? cluster_sums_f32_kernel<float, MT, false, true> : cluster_sums_f32_kernel<float, MT, false, false>);
  };
  auto pick = [&](auto mt) -> Kern { return accum(mt); };
  using Kern64 = void (*)(const double*, const int32_t*, int64_t, int, int, float, double, unsigned long long*);
  Kern kern = nullptr;
  Kern64 kern64 = nullptr;
  if (f64) {  // (to_fixed<double> always uses the fp64 scale)
    kern64 = e->m == 25 ? (priv ? cluster_sums_f32_kernel<double, 25, true, true> : cluster_sums_f32_kernel<double, 25, false, true>)
                        : (priv ? cluster_sums_f32_kernel<double, 0, true, true> : cluster_sums_f32_kernel<double, 0, false, true>);
  } else {
    kern = e->m == 25 ? pick(std::integral_constant<int, 25>{})
           : e->m == 10 ? pick(std::integral_constant<int, 10>{})
           : e->m == 5 ? pick(std::integral_constant<int, 5>{})
                       : pick(std::integral_constant<int, 0>{});
  }
  const void* kfn = f64 ? (const void*)kern64 : (const void*)kern;
  // launch geometry per (k, m) shape, computed once (no attribute / occupancy queries per call)
  const size_t key = ((smem * 4 + (priv ? 1 : 0) + (use_d ? 2 : 0)) * 64 + (size_t)e->m) * 2 + (f64 ? 1 : 0);
  if (e->sums_key != key) {
    CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kSumsThreads, smem));
    e->sums_per_sm = std::max(1, per_sm);
    e->sums_key = key;
  }
  const int64_t ntiles = (e->n + kSumsTile - 1) / kSumsTile;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)e->sums_per_sm * e->num_sms, ntiles));
  if (f64)
    kern64<<<(unsigned)grid, kSumsThreads, smem, e->stream>>>((const double*)e->x, e->labels, e->n, e->m, e->k,
                                                              (float)std::ldexp(1.0, e->frac_bits),
                                                              std::ldexp(1.0, e->frac_bits), out);
  else
    kern<<<(unsigned)grid, kSumsThreads, smem, e->stream>>>((const float*)e->x, e->labels, e->n, e->m, e->k,
                                                            (float)std::ldexp(1.0, e->frac_bits),
                                                            std::ldexp(1.0, e->frac_bits), out);
  CK_LAUNCH("cluster_sums_f32_kernel");
  e->stats.kernel_launches += 1;
  return KM_OK;
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* km_version(void) { return "kmeans_b200 0.1.0 (sm_100a)"; }

int km_device_count(int32_t* out) {
  int c = 0;
  cudaError_t r = cudaGetDeviceCount(&c);
  if (r != cudaSuccess) {
    if (out) *out = 0;
    cudaGetLastError();
    return set_err(nullptr, KM_ERR_DEVICE_UNAVAILABLE, "cudaGetDeviceCount: %s", cudaGetErrorString(r));
  }
  if (out) *out = c;
  return KM_OK;
}

const char* km_last_error(const km_engine* e) { return e ? e->err.c_str() : g_global_err.c_str(); }

int km_create(int32_t device, km_engine** out) {
  if (!out) return set_err(nullptr, KM_ERR_CONTRACT, "null out pointer");
  *out = nullptr;
  int count = 0;
  cudaError_t r = cudaGetDeviceCount(&count);
  if (r != cudaSuccess || count == 0) {
    cudaGetLastError();
    return set_err(nullptr, KM_ERR_DEVICE_UNAVAILABLE, "no CUDA device: %s",
                   r == cudaSuccess ? "device count is 0" : cudaGetErrorString(r));
  }
  if (device < 0 || device >= count)
    return set_err(nullptr, KM_ERR_DEVICE_UNAVAILABLE, "device %d out of range [0, %d)", device, count);
  r = cudaSetDevice(device);
  if (r != cudaSuccess) return set_err(nullptr, KM_ERR_DEVICE_UNAVAILABLE, "cudaSetDevice: %s", cudaGetErrorString(r));
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10)
    return set_err(nullptr, KM_ERR_DEVICE_UNAVAILABLE, "device %d is sm_%d%d; this build targets sm_100a", device,
                   prop.major, prop.minor);
  km_engine* e = new km_engine();
  e->device = device;
  e->full_first_pass = getenv("KM_FULL_FIRST_PASS") ? (atoi(getenv("KM_FULL_FIRST_PASS")) != 0 ? 1 : 0) : -1;
  e->no_resident = getenv("KM_NO_RESIDENT") != nullptr;
  e->call_trace = getenv("KM_CALL_TRACE") != nullptr;
  e->no_shadow = getenv("KM_NO_FP32_SHADOW") != nullptr;
  e->dbg_flags = getenv("KM_TC_DBG") ? atoi(getenv("KM_TC_DBG")) : 0;
  e->times_path = getenv("KM_TC_TIMES");
  e->num_sms = prop.multiProcessorCount;
  e->smem_optin = prop.sharedMemPerBlockOptin;
  if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete e;
    return set_err(nullptr, KM_ERR_DEVICE_LOST, "cudaStreamCreate failed");
  }
  e->own_stream = true;
  if (cudaMalloc((void**)&e->st, sizeof(DevState)) != cudaSuccess ||
      cudaMallocHost((void**)&e->st_host, sizeof(DevState)) != cudaSuccess ||
      cudaMalloc((void**)&e->scratch_u, 16) != cudaSuccess || cudaMalloc((void**)&e->scratch_i, 16) != cudaSuccess) {
    km_destroy(e);
    return set_err(nullptr, KM_ERR_CAPACITY, "allocation of engine state failed");
  }
  std::memset(e->st_host, 0, sizeof(DevState));
  cudaMemset(e->st, 0, sizeof(DevState));
  *out = e;
  return KM_OK;
}

static void peer_release(km_engine* e);

int km_destroy(km_engine* e) {
  if (!e) return KM_OK;
  cudaSetDevice(e->device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  drop_points(e);
  peer_release(e);
  dfree(e->xbuf); dfree(e->stage); dfree(e->labels); dfree(e->recheck_rows); dfree(e->d2);
  dfree(e->labels64); dfree(e->partials);
  dfree(e->pair_best); dfree(e->seed_pv); dfree(e->seed_pi);
  dfree(e->rows_dev); dfree(e->job_acc); dfree(e->job_lab);
  for (cudaEvent_t ev : e->ev) cudaEventDestroy(ev);
  dfree(e->st);
  dfree(e->scratch_u);
  dfree(e->scratch_i);
  if (e->st_host) cudaFreeHost(e->st_host);
  if (e->pin) cudaFreeHost(e->pin);
  if (e->own_stream && e->stream) cudaStreamDestroy(e->stream);
  delete e;
  return KM_OK;
}

int km_set_stream(km_engine* e, void* stream) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  if (stream == nullptr) {
    if (!e->own_stream) {
      if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess)
        return set_err(e, KM_ERR_DEVICE_LOST, "cudaStreamCreate failed");
      e->own_stream = true;
    }
    return KM_OK;
  }
  if (e->own_stream && e->stream) {
    cudaStreamSynchronize(e->stream);
    cudaStreamDestroy(e->stream);
  }
  e->stream = (cudaStream_t)stream;
  e->own_stream = false;
  return KM_OK;
}

int km_load_points_f32(km_engine* e, const float* x, int64_t n, int32_t m) {
  int r = validate_points_shape(e, x, n, m);
  if (r) return r;
  cudaSetDevice(e->device);
  drop_points(e);
  if ((r = grow(e, &e->xbuf, &e->xbuf_cap, sizeof(float) * (size_t)n * m))) return r;
  void* d = e->xbuf;
  e->x = d;
  e->x_owned = true;
  e->n = n;
  e->m = m;
  e->point_bytes = 4;
  CK(cudaMemcpyAsync(d, x, sizeof(float) * (size_t)n * m, cudaMemcpyHostToDevice, e->stream));
  int flags[2] = {0, 0};
  if ((r = scan_points(e, d, 4, n * (int64_t)m, flags))) return r;
  if (flags[0]) { drop_points(e); return set_err(e, KM_ERR_CONTRACT, "coords contains NaN or infinite values"); }
  return after_points_loaded(e);
}

int km_load_points_f64(km_engine* e, const double* x, int64_t n, int32_t m) {
  int r = validate_points_shape(e, x, n, m);
  if (r) return r;
  cudaSetDevice(e->device);
  const int64_t count = n * (int64_t)m;
  drop_points(e);
  if ((r = grow(e, &e->stage, &e->stage_cap, sizeof(double) * (size_t)count))) return r;
  void* d64 = e->stage;
  CK(cudaMemcpyAsync(d64, x, sizeof(double) * (size_t)count, cudaMemcpyHostToDevice, e->stream));
  int flags[2] = {0, 0};
  if ((r = scan_points(e, d64, 8, count, flags))) return r;
  if (flags[0]) return set_err(e, KM_ERR_CONTRACT, "coords contains NaN or infinite values");
  if (!flags[1]) {  // lossless: keep the fp32 copy only (half the bytes per pass)
    if ((r = grow(e, &e->xbuf, &e->xbuf_cap, sizeof(float) * (size_t)count))) return r;
    narrow_f64_kernel<<<grid_for(e, count, 4), 256, 0, e->stream>>>((const double*)d64, count, (float*)e->xbuf);
    CK_LAUNCH("narrow_f64_kernel");
    e->stats.kernel_launches += 1;
    e->x = e->xbuf;
    e->point_bytes = 4;
  } else {
    e->x = d64;
    e->point_bytes = 8;
    // fp32 shadow (round to nearest) for the tensor-core filter: the pass streams 4 bytes per
    // coordinate; the exact fp64 rows are read only by the recheck and the Δ of changed points.
    // Magnitudes outside the fp32 normal range keep the SIMT fp64 pass (no shadow).
    const double amax = e->absmax;
    if (!e->no_shadow && amax < std::ldexp(1.0, 60) && (amax == 0.0 || amax > std::ldexp(1.0, -60))) {
      if ((r = grow(e, &e->xbuf, &e->xbuf_cap, sizeof(float) * (size_t)count))) return r;
      narrow_f64_kernel<<<grid_for(e, count, 4), 256, 0, e->stream>>>((const double*)d64, count, (float*)e->xbuf);
      CK_LAUNCH("narrow_f64_kernel");
      e->stats.kernel_launches += 1;
      e->x32 = e->xbuf;
    }
  }
  e->x_owned = true;
  e->n = n;
  e->m = m;
  return after_points_loaded(e);
}

int km_attach_points_device_f32(km_engine* e, const float* dev_x, int64_t n, int32_t m) {
  int r = validate_points_shape(e, dev_x, n, m);
  if (r) return r;
  if (((uintptr_t)dev_x & 15) != 0) return set_err(e, KM_ERR_CONTRACT, "device point buffer must be 16-byte aligned");
  cudaSetDevice(e->device);
  drop_points(e);
  e->x = (void*)dev_x;
  e->x_owned = false;
  e->n = n;
  e->m = m;
  e->point_bytes = 4;
  int flags[2] = {0, 0};
  if ((r = scan_points(e, dev_x, 4, n * (int64_t)m, flags))) return r;
  if (flags[0]) { drop_points(e); return set_err(e, KM_ERR_CONTRACT, "coords contains NaN or infinite values"); }
  return after_points_loaded(e);
}

int km_points_info(km_engine* e, int64_t* n, int32_t* m, int32_t* point_bytes, double* absmax) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (n) *n = e->n;
  if (m) *m = e->m;
  if (point_bytes) *point_bytes = e->point_bytes;
  if (absmax) *absmax = e->absmax;
  return KM_OK;
}

static int check_centers(km_engine* e, const double* c, int32_t k) {
  if (!c) return set_err(e, KM_ERR_CONTRACT, "null centers");
  if (k < 1) return set_err(e, KM_ERR_CONTRACT, "k must be >= 1, got %d", k);
  for (int64_t i = 0; i < (int64_t)k * e->m; ++i)
    if (!std::isfinite(c[i])) return set_err(e, KM_ERR_CONTRACT, "centers contains NaN or infinite values");
  return KM_OK;
}

int km_assign(km_engine* e, const double* centers, int32_t k, int64_t* labels_out, int64_t* counts_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  int r;
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if ((r = check_centers(e, centers, k))) return r;
  if ((r = ensure_k(e, k))) return r;
  CK(cudaMemcpyAsync(e->cur, centers, 8 * (size_t)k * e->m, cudaMemcpyHostToDevice, e->stream));
  if ((r = reset_state(e, 1, 0.0))) return r;
  scale_for_centers(e, centers, k);
  if ((r = launch_prep(e))) return r;
  CK(cudaMemsetAsync(e->part, 0, 8 * ((size_t)k * e->m + k), e->stream));
  if ((r = launch_pass(e, PASS_ASSIGN_ONLY, false))) return r;
  e->stats.passes += 1;
  CK(cudaMemsetAsync(e->recheck_count, 0, 4, e->stream));
  if (labels_out && (r = download_labels(e, labels_out))) return r;
  if (counts_out)
    CK(cudaMemcpyAsync(counts_out, e->part + (size_t)k * e->m, 8 * (size_t)k, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaMemsetAsync(e->part, 0, 8 * ((size_t)k * e->m + k), e->stream));
  if ((r = read_state(e))) return r;
  e->stats.rechecked = (int64_t)e->st_host->rechecked + 0;
  return KM_OK;
}

int km_update(km_engine* e, int64_t* labels_inout, int32_t k, double* centers_out, int64_t* counts_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  int r;
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if (!labels_inout) return set_err(e, KM_ERR_CONTRACT, "null labels");
  if (k < 1) return set_err(e, KM_ERR_CONTRACT, "k must be >= 1, got %d", k);
  std::vector<int32_t> lab((size_t)e->n);
  for (int64_t i = 0; i < e->n; ++i) {
    const int64_t v = labels_inout[i];
    if (v < 0 || v >= k) return set_err(e, KM_ERR_CONTRACT, "labels must lie in [0, %d)", k);
    lab[i] = (int32_t)v;
  }
  if ((r = ensure_k(e, k))) return r;
  CK(cudaMemcpyAsync(e->labels, lab.data(), 4 * (size_t)e->n, cudaMemcpyHostToDevice, e->stream));
  if ((r = reset_state(e, 1, 0.0))) return r;
  CK(cudaMemsetAsync(e->part, 0, 8 * ((size_t)k * e->m + k), e->stream));
  // labels were validated on the host: fp32 points with m ≤ 31 take the streaming cluster-sums
  // kernel (kmeans_sums.cuh), other shapes the SIMT pass in sums-only mode
  if (e->m <= 31) {
    if ((r = launch_sums(e, e->part))) return r;
  } else if ((r = launch_pass(e, PASS_SUMS_ONLY, false))) {
    return r;
  }
  if ((r = launch_finish(e, 1, false))) return r;
  e->next_full = true;
  if ((r = read_state(e))) return r;
  if (e->st_host->bad_label) return set_err(e, KM_ERR_VALIDATION, "label out of range [0, %d) on device", k);
  const bool repaired = e->st_host->n_empty > 0;
  if (repaired && (r = repair_local(e))) return r;
  if (centers_out) CK(cudaMemcpyAsync(centers_out, e->cur, 8 * (size_t)k * e->m, cudaMemcpyDeviceToHost, e->stream));
  if (counts_out) CK(cudaMemcpyAsync(counts_out, e->model_counts, 8 * (size_t)k, cudaMemcpyDeviceToHost, e->stream));
  if (repaired) {
    CK(cudaMemcpyAsync(lab.data(), e->labels, 4 * (size_t)e->n, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    for (int64_t i = 0; i < e->n; ++i) labels_inout[i] = lab[i];
  }
  CK(cudaStreamSynchronize(e->stream));
  return KM_OK;
}

int km_converged(km_engine* e, const double* prev, const double* next, int32_t k, int32_t m, double tol,
                 int32_t* out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!prev || !next || !out) return set_err(e, KM_ERR_CONTRACT, "null argument");
  if (k < 1 || m < 1) return set_err(e, KM_ERR_CONTRACT, "bad shape (%d, %d)", k, m);
  if (!(tol >= 0.0)) return set_err(e, KM_ERR_CONTRACT, "tol must be >= 0, got %g", tol);
  cudaSetDevice(e->device);
  double* buf = nullptr;
  int r;
  if ((r = dalloc(e, &buf, 8 * 2 * (size_t)k * m))) return r;
  int32_t* flag = e->scratch_i;
  cudaMemcpyAsync(buf, prev, 8 * (size_t)k * m, cudaMemcpyHostToDevice, e->stream);
  cudaMemcpyAsync(buf + (size_t)k * m, next, 8 * (size_t)k * m, cudaMemcpyHostToDevice, e->stream);
  converged_kernel<<<1, finish_threads(k, 1), 0, e->stream>>>(buf, buf + (size_t)k * m, k, m, tol, flag);
  cudaError_t c = cudaGetLastError();
  int32_t h = 0;
  if (c == cudaSuccess) c = cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, e->stream);
  if (c == cudaSuccess) c = cudaStreamSynchronize(e->stream);
  cudaFree(buf);
  if (c != cudaSuccess) return cuda_fail(e, c, "km_converged");
  *out = h;
  return KM_OK;
}

// Tensor-core resident loop: the whole Lloyd iteration runs inside one cooperative launch
// (lloyd_pass_tc_kernel with a.resident); the host only steps in for empty-cluster repairs.
// Host cost per call (the bench times whole calls): one pinned H2D of C0, one begin kernel
// (state, zeroed accumulators, filter operands), the first pass + cluster sums + the resident
// launch, and ONE synchronisation that also brings back the state, the centres and the counts
// (pinned).  Returns KM_RESIDENT_UNFIT when the shape only fits the launch-per-iteration kernel.
static int lloyd_resident(km_engine* e, const double* c0, int max_iters, double tol, bool resume = false) {
  int r;
  const int k = e->k, m = e->m;
  const size_t km = (size_t)k * m, nacc = km + k;
  // pinned staging: [C0 | C out | counts out]
  const size_t pin_bytes = 8 * (2 * km + k);
  if (e->pin_cap < pin_bytes) {
    if (e->pin) cudaFreeHost(e->pin);
    e->pin = nullptr;
    e->pin_cap = 0;
    CK(cudaMallocHost(&e->pin, pin_bytes));
    e->pin_cap = pin_bytes;
  }
  double* pin_c0 = reinterpret_cast<double*>(e->pin);
  double* pin_c = pin_c0 + km;
  long long* pin_n = reinterpret_cast<long long*>(pin_c + km);
  // KM_CALL_TRACE: device (events) and host (clock) time of each step of the call, on stderr
  cudaEvent_t tev[6] = {};
  double th[6] = {};
  int nt = 0;
  auto trace = [&]() {
    if (!e->call_trace || nt >= 6) return;
    if (!tev[nt]) cudaEventCreate(&tev[nt]);
    cudaEventRecord(tev[nt], e->stream);
    th[nt++] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  trace();
  if (!resume) {
    // C0: in the begin kernel's parameters when it fits, else one pinned H2D copy
    C0Inline c0p{};  // (by-value launch parameter; only the first k·m entries are read)
    const bool inl = km <= (size_t)kC0Inline;
    if (inl) {
      std::memcpy(c0p.v, c0, 8 * km);
    } else {
      std::memcpy(pin_c0, c0, 8 * km);
      CK(cudaMemcpyAsync(e->cur, pin_c0, 8 * km, cudaMemcpyHostToDevice, e->stream));
    }
    lloyd_begin_kernel<<<1, 512, 0, e->stream>>>(e->st, max_iters, tol, e->part, e->tot, e->dlt, nacc, e->grid_sync,
                                                 e->recheck_count, e->cur, e->w, e->cn, e->cmax, k, m, e->mpad,
                                                 tc_eligible(e) ? e->wop : nullptr, e->kp, e->pre, c0p,
                                                 inl ? (int)km : 0);
    CK_LAUNCH("lloyd_begin_kernel launch");
    e->stats.kernel_launches += 1;
    e->resident_zeroed = true;
    e->next_full = true;
  }
  // First pass split in two: L0 = A(C0) writes labels only (tensor cores), then one cluster-sums
  // stream adds every point to its cluster (S(L0) into tot); the resident loop starts at the
  // finish of iteration 1.  Small point sets take the fused full first pass inside the resident
  // launch instead (two launches fewer: cfg1 9.2 → 8.7, cfg2 11.8 → 11.4 µs per step; at cfg3 the
  // split is 85 µs per call faster).  KM_FULL_FIRST_PASS=1 / 0 forces either (A/B timing).
  constexpr int64_t kSplitFirstMinRows = 500000;
  const bool split = e->peer_active ||  // (the peer loop exchanges the split's local sums)
                     (e->full_first_pass < 0 ? e->n >= kSplitFirstMinRows : e->full_first_pass == 0);
  bool full = !split && !resume, first = !resume;
  DevState* hs = e->st_host;
  for (;;) {
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (e->profiling) {
      while (e->ev.size() < 2) {
        cudaEvent_t ev;
        CK(cudaEventCreate(&ev));
        e->ev.push_back(ev);
      }
      ev0 = e->ev[0];
      ev1 = e->ev[1];
      CK(cudaEventRecord(ev0, e->stream));
    }
    const int passes_before = first ? 0 : hs->passes;  // (the begin kernel zeroed the device state)
    const bool skip = split && first;
    if (skip) {
      trace();
      if ((r = launch_tc(e, true, false, false, false, true))) return r;  // labels of C0 only
      trace();
      if ((r = launch_sums(e, e->tot))) return r;
      trace();
    }
    if ((r = launch_tc(e, full, true, false, true, false, skip))) return r;
    trace();
    if (e->profiling) CK(cudaEventRecord(ev1, e->stream));
    // one round trip: state + (if the loop is done) the model, written into the pinned staging by
    // one small kernel (mapped host memory)
    lloyd_publish_kernel<<<1, 256, 0, e->stream>>>(e->st, e->cur, e->model_counts, (int)km, k, hs, pin_c, pin_n);
    CK_LAUNCH("lloyd_publish_kernel launch");
    e->stats.kernel_launches += 1;
    CK(cudaStreamSynchronize(e->stream));
    e->stats.host_syncs += 1;
    if (e->call_trace && nt > 1) {
      const double t_end = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
      fprintf(stderr, "km_lloyd trace (device us | host us): ");
      for (int i = 1; i < nt; ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tev[i - 1], tev[i]);
        fprintf(stderr, "[%d] %.1f | %.1f  ", i, ms * 1e3, th[i] - th[i - 1]);
      }
      fprintf(stderr, "sync wait %.1f\n", t_end - th[nt - 1]);
      for (int i = 0; i < nt; ++i) cudaEventDestroy(tev[i]);
      nt = 6;
    }
    const DevState s = *hs;
    const int ran = s.passes - passes_before + (skip ? 1 : 0);
    if (e->profiling && ran > 0) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ev0, ev1));
      e->stats.pass_ms_total += ms;
      e->stats.pass_timed += ran;
    }
    full = false;
    first = false;
    e->next_full = false;
    if (s.done) return KM_OK;
    if (!s.need_host) return set_err(e, KM_ERR_INTERNAL, "resident Lloyd loop stopped without a decision");
    if (e->peer_active) return KM_OK;  // row shards: the caller runs the global repair (all ranks)
    if ((r = repair_local(e))) return r;
    if ((r = launch_check(e))) return r;
    if ((r = read_state(e))) return r;
    if (hs->done) {  // the repaired model converged: bring it back
      CK(cudaMemcpyAsync(pin_c, e->cur, 8 * km, cudaMemcpyDeviceToHost, e->stream));
      CK(cudaMemcpyAsync(pin_n, e->model_counts, 8 * (size_t)k, cudaMemcpyDeviceToHost, e->stream));
      CK(cudaStreamSynchronize(e->stream));
      return KM_OK;
    }
  }
}

int km_lloyd(km_engine* e, const double* c0, int32_t k, int32_t max_iters, double tol, double* centers_out,
             int64_t* counts_out, int64_t* labels_out, int32_t* iterations_out, int32_t* converged_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  int r;
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if (max_iters < 1) return set_err(e, KM_ERR_CONTRACT, "max_iters must be >= 1, got %d", max_iters);
  if (!(tol >= 0.0)) return set_err(e, KM_ERR_CONTRACT, "tol must be >= 0, got %g", tol);
  if (k > e->n) return set_err(e, KM_ERR_CONTRACT, "k=%d exceeds sample count n=%lld", k, (long long)e->n);
  if ((r = check_centers(e, c0, k))) return r;
  if ((r = ensure_k(e, k))) return r;
  scale_for_centers(e, c0, k);
  if (use_tc(e) && !e->resident_unfit && !e->no_resident) {
    r = lloyd_resident(e, c0, max_iters, tol);
    if (r == KM_OK) {
      const DevState s = *e->st_host;
      const size_t km = (size_t)k * e->m;
      const double* pin_c = reinterpret_cast<const double*>(e->pin) + km;
      e->stats.passes += 1 + s.t - (s.converged ? 1 : 0);
      e->stats.rechecked += (int64_t)s.rechecked;
      e->stats.changed += (int64_t)s.changed;
      if (centers_out) std::memcpy(centers_out, pin_c, 8 * km);
      if (counts_out) std::memcpy(counts_out, pin_c + km, 8 * (size_t)k);
      if (labels_out) {
        if ((r = download_labels(e, labels_out))) return r;
        CK(cudaStreamSynchronize(e->stream));
      }
      if (iterations_out) *iterations_out = s.t;
      if (converged_out) *converged_out = s.converged;
      return KM_OK;
    }
    if (r != KM_RESIDENT_UNFIT) return r;
    e->resident_unfit = true;
  }
  CK(cudaMemcpyAsync(e->cur, c0, 8 * (size_t)k * e->m, cudaMemcpyHostToDevice, e->stream));
  if ((r = reset_state(e, max_iters, tol))) return r;
  if ((r = launch_prep(e))) return r;
  CK(cudaMemsetAsync(e->part, 0, 8 * ((size_t)k * e->m + k), e->stream));
  e->next_full = true;  // the labels buffer does not hold L of this run yet
  // Tensor-core path: ONE launch per iteration — pass t + (last CTA) finish t+1.
  // SIMT path: finish and pass are separate launches.
  const bool fused = use_tc(e);
  bool prev_full = true;
  int batch = 1;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed;
  auto timed_pass = [&](void) -> int {
    cudaEvent_t a = nullptr, b = nullptr;
    if (e->profiling) {
      const size_t need = 2 * (timed.size() + 1);
      while (e->ev.size() < need) {
        cudaEvent_t ev;
        CK(cudaEventCreate(&ev));
        e->ev.push_back(ev);
      }
      a = e->ev[need - 2];
      b = e->ev[need - 1];
      CK(cudaEventRecord(a, e->stream));
    }
    const int rr = launch_pass(e, PASS_ASSIGN_SUMS, true, fused);
    if (rr) return rr;
    prev_full = e->last_pass_full;
    if (e->profiling) {
      CK(cudaEventRecord(b, e->stream));
      timed.push_back({a, b});
    }
    return KM_OK;
  };
  // account the passes of a batch that actually ran (gated launches after done / need_host
  // exit immediately and are not counted)
  auto account = [&](int n_ran) -> int {
    for (int i = 0; i < (int)timed.size() && i < n_ran; ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, timed[i].first, timed[i].second));
      e->stats.pass_ms_total += ms;
      e->stats.pass_timed += 1;
    }
    timed.clear();
    return KM_OK;
  };
  // L0 = A(C0) (engine.py:328), fused with the sums U(L0) needs (and, fused, the first update).
  if ((r = timed_pass())) return r;
  int first = 1;
  int t_before = 0;
  for (;;) {
    for (int b = 0; b < batch; ++b) {
      if (!fused && (r = launch_finish(e, 0, !prev_full))) return r;
      if ((r = timed_pass())) return r;
    }
    if ((r = read_state(e))) return r;
    const DevState s = *e->st_host;
    const int ran_updates = s.t - t_before;
    int ran;
    if (fused) {  // launch j = pass j + finish j+1; the exhausted final launch folds without t += 1
      ran = ran_updates + ((s.done && !s.converged) ? 1 : 0);
    } else {
      const int stopped = (s.done && s.converged) || s.need_host ? 1 : 0;
      ran = first + std::max(0, ran_updates - stopped);
    }
    if ((r = account(ran))) return r;
    first = 0;
    t_before = s.t;
    if (s.done) break;
    if (s.need_host) {
      if ((r = repair_local(e))) return r;
      if ((r = launch_check(e))) return r;
      if (!fused) {
        if ((r = timed_pass())) return r;
        // the check may have finished the loop (converged): then the pass was gated
        if ((r = read_state(e))) return r;
        if ((r = account(e->st_host->done ? 0 : 1))) return r;
        if (e->st_host->done) break;
      } else {
        if ((r = read_state(e))) return r;
        if (e->st_host->done) break;
        t_before = e->st_host->t;
      }
      batch = 1;
      continue;
    }
    batch = std::min(batch * 2, 16);
  }
  const DevState s = *e->st_host;
  e->stats.passes += 1 + s.t - (s.converged ? 1 : 0);
  e->stats.rechecked += (int64_t)s.rechecked;
  e->stats.changed += (int64_t)s.changed;
  if (centers_out) CK(cudaMemcpyAsync(centers_out, e->cur, 8 * (size_t)k * e->m, cudaMemcpyDeviceToHost, e->stream));
  if (counts_out)  // converged: counts of the update; exhausted: the final finish folded bincount(L_T)
    CK(cudaMemcpyAsync(counts_out, e->model_counts, 8 * (size_t)k, cudaMemcpyDeviceToHost, e->stream));
  if (labels_out && (r = download_labels(e, labels_out))) return r;
  CK(cudaMemsetAsync(e->part, 0, 8 * ((size_t)k * e->m + k), e->stream));
  CK(cudaStreamSynchronize(e->stream));
  if (iterations_out) *iterations_out = s.t;
  if (converged_out) *converged_out = s.converged;
  return KM_OK;
}

int km_wcss(km_engine* e, const double* centers, int32_t k, const int64_t* labels, double* out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  int r;
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if (!out || !labels) return set_err(e, KM_ERR_CONTRACT, "null argument");
  if ((r = check_centers(e, centers, k))) return r;
  std::vector<int32_t> lab((size_t)e->n);
  for (int64_t i = 0; i < e->n; ++i) {
    if (labels[i] < 0 || labels[i] >= k) return set_err(e, KM_ERR_CONTRACT, "labels must lie in [0, %d)", k);
    lab[i] = (int32_t)labels[i];
  }
  if ((r = ensure_k(e, k))) return r;
  CK(cudaMemcpyAsync(e->scratch_d, centers, 8 * (size_t)k * e->m, cudaMemcpyHostToDevice, e->stream));
  CK(cudaMemcpyAsync(e->labels, lab.data(), 4 * (size_t)e->n, cudaMemcpyHostToDevice, e->stream));
  // bound every term: d2 ≤ m·(2·max(|x|,|c|))²
  double cm = e->absmax;
  for (int64_t i = 0; i < (int64_t)k * e->m; ++i) cm = std::max(cm, std::fabs(centers[i]));
  const double term = (double)e->m * 4.0 * cm * cm;
  const int F2 = compute_frac_bits(std::max(term, 1e-300), e->n);
  unsigned long long zero = 0;
  CK(cudaMemcpyAsync(e->scratch_u, &zero, 8, cudaMemcpyHostToDevice, e->stream));
  const int g = grid_for(e, e->n);
  if (e->point_bytes == 4)
    wcss_kernel<float><<<g, 256, 0, e->stream>>>((const float*)e->x, e->n, e->m, e->scratch_d, e->labels,
                                                 std::ldexp(1.0, F2), e->scratch_u);
  else
    wcss_kernel<double><<<g, 256, 0, e->stream>>>((const double*)e->x, e->n, e->m, e->scratch_d, e->labels,
                                                  std::ldexp(1.0, F2), e->scratch_u);
  CK_LAUNCH("wcss_kernel");
  unsigned long long v = 0;
  CK(cudaMemcpyAsync(&v, e->scratch_u, 8, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  *out = std::ldexp((double)(long long)v, -F2);
  return KM_OK;
}

// ---------------------------------------------------------------------------
// Seeding: diameter pair scan + maximin / random-far primitives
// ---------------------------------------------------------------------------
// Best pair (largest exact d², then smallest i, then smallest j) over scan rows × columns j > i:
// rows r·stride for r < R, or rows[r] (device, ascending) when given.  best.i < 0: no pair.
static int pair_scan_best(km_engine* e, int64_t stride, int64_t R, const long long* rows, PairBest* best_out) {
  const int64_t n = e->n;
  const int m = e->m;
  const int grid = e->num_sms * 4;
  int r;
  if ((r = grow(e, &e->pair_best, &e->pair_best_cap, sizeof(PairBest) * (size_t)grid))) return r;
  // fp32 estimates are certified only for fp32-exact points whose squares stay normal
  bool exact = e->point_bytes != 4 || !(e->absmax < std::ldexp(1.0, 60));
  float thr = -1.0f;
  if (!exact) {
    unsigned int zero = 0, bits = 0;
    CK(cudaMemcpyAsync(e->scratch_u, &zero, 4, cudaMemcpyHostToDevice, e->stream));
    pair_scan_kernel<float, false><<<grid, kPairCols, 0, e->stream>>>((const float*)e->x, n, m, stride, R, 0.f,
                                                                      (unsigned int*)e->scratch_u, e->pair_best, rows);
    CK_LAUNCH("pair_scan_kernel (phase 1)");
    e->stats.kernel_launches += 1;
    CK(cudaMemcpyAsync(&bits, e->scratch_u, 4, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    float max32;
    std::memcpy(&max32, &bits, 4);
    if (!(max32 >= std::ldexp(1.0f, -100))) {
      exact = true;
    } else {
      // relative error of a fp32 squared distance of fp32 points (+ the reference's fp64 rounding)
      const double g = (m + 4) * std::ldexp(1.0, -24) * 1.01 + (m + 2) * std::ldexp(1.0, -52);
      const double t = (double)max32 * (1.0 - g) / (1.0 + g) - m * std::ldexp(1.0, -120);
      thr = std::nextafter((float)t, -INFINITY);
    }
  }
  if (e->point_bytes == 4)
    pair_scan_kernel<float, true><<<grid, kPairCols, 0, e->stream>>>((const float*)e->x, n, m, stride, R,
                                                                     exact ? -1.0f : thr, nullptr, e->pair_best, rows);
  else
    pair_scan_kernel<double, true><<<grid, kPairCols, 0, e->stream>>>((const double*)e->x, n, m, stride, R, -1.0f,
                                                                      nullptr, e->pair_best, rows);
  CK_LAUNCH("pair_scan_kernel (phase 2)");
  e->stats.kernel_launches += 1;
  std::vector<PairBest> h(grid);
  CK(cudaMemcpyAsync(h.data(), e->pair_best, sizeof(PairBest) * grid, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  PairBest best{-1.0, -1, -1};
  for (const PairBest& b : h) {
    if (b.i < 0) continue;
    if (best.i < 0 || b.d2 > best.d2 || (b.d2 == best.d2 && (b.i < best.i || (b.i == best.i && b.j < best.j))))
      best = b;
  }
  *best_out = best;
  return KM_OK;
}

int km_diameter(km_engine* e, int64_t pair_cap, double* d_out, int64_t* i_out, int64_t* j_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  cudaSetDevice(e->device);
  const int64_t n = e->n;
  const int m = e->m;
  if (n < 2) return set_err(e, KM_ERR_CONTRACT, "diameter needs at least 2 samples, got %lld", (long long)n);
  // engine.scan_rows (engine.py:124-138): every row, or every stride-th row under a pair cap
  const unsigned __int128 total = (unsigned __int128)n * (unsigned __int128)(n - 1) / 2;
  int64_t stride = 1;
  if (pair_cap > 0 && total > (unsigned __int128)pair_cap) {
    const unsigned __int128 q = (total + (unsigned __int128)pair_cap - 1) / (unsigned __int128)pair_cap;
    stride = std::max<int64_t>(2, (int64_t)q);
  }
  const int64_t R = (n - 1 + stride - 1) / stride;
  int r;
  PairBest best;
  if ((r = pair_scan_best(e, stride, R, nullptr, &best))) return r;
  if (d_out) *d_out = std::sqrt(best.d2);
  if (i_out) *i_out = best.i;
  if (j_out) *j_out = best.j;
  return KM_OK;
}

// MAX_PAIR device job (device.max_pair_job / HostReferenceDevice._execute, device.py:117-122,
// 213-216 → _kernels.max_pair_rows, _kernels.py:48-81): best pair over the given ascending rows ×
// columns j > i; (-1, -1, -1) when the rows produce no pair.
int km_max_pair_rows(km_engine* e, const int64_t* rows, int64_t nrows, double* d2_out, int64_t* i_out,
                     int64_t* j_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if (nrows < 0 || (nrows > 0 && !rows)) return set_err(e, KM_ERR_CONTRACT, "bad row list");
  for (int64_t r = 0; r < nrows; ++r) {
    if (rows[r] < 0 || rows[r] >= e->n) return set_err(e, KM_ERR_CONTRACT, "scan rows must lie in [0, %lld)", (long long)e->n);
    if (r && rows[r] <= rows[r - 1]) return set_err(e, KM_ERR_CONTRACT, "scan rows must be strictly ascending");
  }
  cudaSetDevice(e->device);
  PairBest best{-1.0, -1, -1};
  if (nrows > 0 && e->n >= 2) {
    int r;
    if ((r = grow(e, &e->rows_dev, &e->rows_cap, sizeof(long long) * (size_t)nrows))) return r;
    CK(cudaMemcpyAsync(e->rows_dev, rows, sizeof(long long) * (size_t)nrows, cudaMemcpyHostToDevice, e->stream));
    if ((r = pair_scan_best(e, 1, nrows, (const long long*)e->rows_dev, &best))) return r;
  }
  if (d2_out) *d2_out = best.i < 0 ? -1.0 : best.d2;
  if (i_out) *i_out = best.i;
  if (j_out) *j_out = best.j;
  return KM_OK;
}

static int seed_argmax(km_engine* e, int grid, double* v_out, int64_t* i_out) {
  std::vector<double> pv(grid);
  std::vector<long long> pi(grid);
  CK(cudaMemcpyAsync(pv.data(), e->seed_pv, 8 * (size_t)grid, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaMemcpyAsync(pi.data(), e->seed_pi, 8 * (size_t)grid, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  double bv = -1.0;
  long long bi = -1;
  for (int b = 0; b < grid; ++b)
    if (pi[b] < e->n && (bi < 0 || pv[b] > bv || (pv[b] == bv && pi[b] < bi))) { bv = pv[b]; bi = pi[b]; }
  if (v_out) *v_out = bv;
  if (i_out) *i_out = bi;
  return KM_OK;
}

int km_seed_reset(km_engine* e) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  cudaSetDevice(e->device);
  int r;
  if ((r = grow(e, &e->d2, &e->d2_cap, 8 * (size_t)e->n))) return r;
  fill_f64_kernel<<<grid_for(e, e->n, 4), 256, 0, e->stream>>>(e->d2, e->n, INFINITY);
  CK_LAUNCH("fill_f64_kernel");
  e->stats.kernel_launches += 1;
  e->seed_ready = true;
  return KM_OK;
}

int km_seed_add(km_engine* e, int64_t c, double* max_v, int64_t* max_i) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->x || !e->seed_ready) return set_err(e, KM_ERR_CONTRACT, "call km_seed_reset first");
  if (c < 0 || c >= e->n) return set_err(e, KM_ERR_CONTRACT, "centre index %lld out of range", (long long)c);
  cudaSetDevice(e->device);
  const int grid = grid_for(e, e->n, 4);
  int r;
  if ((r = grow(e, &e->seed_pv, &e->seed_pv_cap, 8 * (size_t)grid))) return r;
  if ((r = grow(e, &e->seed_pi, &e->seed_pi_cap, 8 * (size_t)grid))) return r;
  const size_t smem = 8 * (size_t)e->m;
  if (e->point_bytes == 4)
    min_d2_update_kernel<float><<<grid, 256, smem, e->stream>>>((const float*)e->x, e->n, e->m, c, e->d2, e->seed_pv,
                                                                 e->seed_pi);
  else
    min_d2_update_kernel<double><<<grid, 256, smem, e->stream>>>((const double*)e->x, e->n, e->m, c, e->d2,
                                                                  e->seed_pv, e->seed_pi);
  CK_LAUNCH("min_d2_update_kernel");
  e->stats.kernel_launches += 1;
  return seed_argmax(e, grid, max_v, max_i);
}

int km_seed_min_d2(km_engine* e, int64_t i, double* out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->x || !e->seed_ready) return set_err(e, KM_ERR_CONTRACT, "call km_seed_reset first");
  if (i < 0 || i >= e->n) return set_err(e, KM_ERR_CONTRACT, "sample index %lld out of range", (long long)i);
  CK(cudaMemcpyAsync(out, e->d2 + i, 8, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  return KM_OK;
}

int km_center_distances(km_engine* e, const double* centers, int32_t k, double* out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  int r;
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if (!out) return set_err(e, KM_ERR_CONTRACT, "null argument");
  if ((r = check_centers(e, centers, k))) return r;
  double* cbuf = nullptr;
  double* obuf = nullptr;
  if ((r = dalloc(e, &cbuf, 8 * (size_t)k * e->m))) return r;
  if ((r = dalloc(e, &obuf, 8 * (size_t)e->n * k))) { cudaFree(cbuf); return r; }
  cudaMemcpyAsync(cbuf, centers, 8 * (size_t)k * e->m, cudaMemcpyHostToDevice, e->stream);
  const int g = grid_for(e, e->n * (int64_t)k);
  if (e->point_bytes == 4)
    center_distances_kernel<float><<<g, 256, 0, e->stream>>>((const float*)e->x, e->n, e->m, cbuf, k, obuf);
  else
    center_distances_kernel<double><<<g, 256, 0, e->stream>>>((const double*)e->x, e->n, e->m, cbuf, k, obuf);
  cudaError_t c = cudaGetLastError();
  if (c == cudaSuccess) c = cudaMemcpyAsync(out, obuf, 8 * (size_t)e->n * k, cudaMemcpyDeviceToHost, e->stream);
  if (c == cudaSuccess) c = cudaStreamSynchronize(e->stream);
  cudaFree(cbuf);
  cudaFree(obuf);
  if (c != cudaSuccess) return cuda_fail(e, c, "km_center_distances");
  return KM_OK;
}

// ---- step API (row-sharded multi-GPU) --------------------------------------
int km_frac_bits_for(double absmax, int64_t n_total, int32_t* out) {
  if (!out) return set_err(nullptr, KM_ERR_CONTRACT, "null out");
  *out = compute_frac_bits(absmax, n_total);
  return KM_OK;
}

int km_set_frac_bits(km_engine* e, int32_t frac_bits) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  e->frac_bits = frac_bits;
  e->frac_user = true;
  e->stats.frac_bits = frac_bits;
  return KM_OK;
}

int km_step_begin(km_engine* e, const double* c0, int32_t k) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  int r;
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if ((r = check_centers(e, c0, k))) return r;
  if ((r = ensure_k(e, k))) return r;
  CK(cudaMemcpyAsync(e->cur, c0, 8 * (size_t)k * e->m, cudaMemcpyHostToDevice, e->stream));
  if ((r = reset_state(e, INT32_MAX, 0.0))) return r;
  scale_for_centers(e, c0, k);
  if ((r = launch_prep(e))) return r;
  CK(cudaMemsetAsync(e->part, 0, 8 * ((size_t)k * e->m + k), e->stream));
  e->next_full = true;
  CK(cudaStreamSynchronize(e->stream));
  return KM_OK;
}

int km_step_partials(km_engine* e, void** dev_ptr, int64_t* n_int64) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->part) return set_err(e, KM_ERR_CONTRACT, "call km_step_begin first");
  if (dev_ptr) *dev_ptr = e->part;
  if (n_int64) *n_int64 = (int64_t)e->k * e->m + e->k;
  return KM_OK;
}

int km_step_pass(km_engine* e) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->part) return set_err(e, KM_ERR_CONTRACT, "call km_step_begin first");
  cudaSetDevice(e->device);
  int r = launch_pass(e, PASS_ASSIGN_SUMS, false);
  if (r) return r;
  e->stats.passes += 1;
  CK(cudaStreamSynchronize(e->stream));
  return KM_OK;
}

int km_step_finish(km_engine* e, double tol, int32_t* status_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->part) return set_err(e, KM_ERR_CONTRACT, "call km_step_begin first");
  cudaSetDevice(e->device);
  int r;
  // keep the loop ungated: clear done/need_host, set tol
  CK(cudaMemcpyAsync(e->st_host, e->st, sizeof(DevState), cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  e->st_host->done = 0;
  e->st_host->need_host = 0;
  e->st_host->exhausted = 0;
  e->st_host->converged = 0;
  e->st_host->tol = tol;
  e->st_host->max_iters = INT32_MAX;
  CK(cudaMemcpyAsync(e->st, e->st_host, sizeof(DevState), cudaMemcpyHostToDevice, e->stream));
  if ((r = launch_finish(e, 0, !e->last_pass_full))) return r;
  if ((r = read_state(e))) return r;
  if (status_out) {
    status_out[0] = e->st_host->n_empty;
    status_out[1] = e->st_host->converged;
  }
  return KM_OK;
}

int km_step_fold(km_engine* e) {
  // exhausted run: fold the (allreduced) final pass into the totals so counts = bincount(L_T)
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  int r;
  CK(cudaMemcpyAsync(e->st_host, e->st, sizeof(DevState), cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  e->st_host->done = 0;
  e->st_host->need_host = 0;
  e->st_host->exhausted = 1;
  CK(cudaMemcpyAsync(e->st, e->st_host, sizeof(DevState), cudaMemcpyHostToDevice, e->stream));
  if ((r = launch_finish(e, 0, !e->last_pass_full))) return r;
  CK(cudaStreamSynchronize(e->stream));
  return KM_OK;
}

int km_step_repair_prepare(km_engine* e) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  return self_d2(e);
}

int km_step_repair_candidate(km_engine* e, double* d2_out, int64_t* row_out, double* coords_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->d2) return set_err(e, KM_ERR_CONTRACT, "call km_step_repair_prepare first");
  cudaSetDevice(e->device);
  argmax_partial_kernel<<<e->n_partials, 256, 0, e->stream>>>(e->d2, e->n, e->partials);
  CK_LAUNCH("argmax_partial_kernel");
  argmax_final_kernel<<<1, 512, 0, e->stream>>>(e->partials, e->n_partials, e->winner);
  CK_LAUNCH("argmax_final_kernel");
  ArgMax h{};
  CK(cudaMemcpyAsync(&h, e->winner, sizeof h, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  if (d2_out) *d2_out = h.v;
  if (row_out) *row_out = h.i;
  if (coords_out && h.i >= 0 && h.i < e->n) {
    if (e->point_bytes == 4) {
      std::vector<float> row(e->m);
      CK(cudaMemcpy(row.data(), (const float*)e->x + h.i * e->m, 4 * (size_t)e->m, cudaMemcpyDeviceToHost));
      for (int f = 0; f < e->m; ++f) coords_out[f] = row[f];
    } else {
      CK(cudaMemcpy(coords_out, (const double*)e->x + h.i * e->m, 8 * (size_t)e->m, cudaMemcpyDeviceToHost));
    }
  }
  return KM_OK;
}

int km_step_label_of(km_engine* e, int64_t local_row, int32_t* label_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (local_row < 0 || local_row >= e->n) return set_err(e, KM_ERR_CONTRACT, "row out of range");
  cudaSetDevice(e->device);
  CK(cudaMemcpyAsync(label_out, e->labels + local_row, 4, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  return KM_OK;
}

int km_step_repair_apply(km_engine* e, int32_t empty_cluster, int32_t owner_is_me, int64_t local_row,
                         const double* coords, int32_t donor) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!coords) return set_err(e, KM_ERR_CONTRACT, "null coords");
  if (empty_cluster < 0 || empty_cluster >= e->k || donor < 0 || donor >= e->k)
    return set_err(e, KM_ERR_CONTRACT, "cluster index out of range");
  cudaSetDevice(e->device);
  double* dc = e->scratch_d;
  CK(cudaMemcpyAsync(dc, coords, 8 * (size_t)e->m, cudaMemcpyHostToDevice, e->stream));
  repair_apply_global_kernel<<<1, 32, 0, e->stream>>>(empty_cluster, owner_is_me, local_row, dc, donor, e->k,
                                                      e->m, e->labels, e->d2, e->model_counts, e->cur, e->tot,
                                                      std::ldexp(1.0, e->frac_bits));
  CK_LAUNCH("repair_apply_global_kernel");
  CK(cudaStreamSynchronize(e->stream));
  e->stats.repairs += 1;
  return KM_OK;
}

int km_step_empty_list(km_engine* e, int32_t* empties_out, int32_t* n_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  std::vector<int32_t> v;
  int r = empty_list(e, v);
  if (r) return r;
  if (n_out) *n_out = (int32_t)v.size();
  if (empties_out) std::copy(v.begin(), v.end(), empties_out);
  return KM_OK;
}

// Batched step loop: the device keeps the loop state (DevState) exactly as km_lloyd does, so a
// driver can enqueue [allreduce, finish, pass] for several iterations and read the state once.
int km_step_loop_begin(km_engine* e, int32_t max_iters, double tol) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->part) return set_err(e, KM_ERR_CONTRACT, "call km_step_begin first");
  if (max_iters < 1) return set_err(e, KM_ERR_CONTRACT, "max_iters must be >= 1, got %d", max_iters);
  if (!(tol >= 0.0)) return set_err(e, KM_ERR_CONTRACT, "tol must be >= 0, got %g", tol);
  cudaSetDevice(e->device);
  return reset_state(e, max_iters, tol);
}

int km_step_loop_pass(km_engine* e) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->part) return set_err(e, KM_ERR_CONTRACT, "call km_step_begin first");
  cudaSetDevice(e->device);
  return launch_pass(e, PASS_ASSIGN_SUMS, true);  // gated: no work once done / waiting for the host
}

int km_step_loop_finish(km_engine* e) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->part) return set_err(e, KM_ERR_CONTRACT, "call km_step_begin first");
  cudaSetDevice(e->device);
  if (e->m > 32) return launch_finish(e, 0, !e->last_pass_full);  // engine.iterate's update/test/exhaustion rules
  FinishArgs f = finish_args(e, 0, !e->last_pass_full);
  lloyd_finish_warp_kernel<<<1, 512, 0, e->stream>>>(f);
  CK_LAUNCH("lloyd_finish_warp_kernel launch");
  e->stats.kernel_launches += 1;
  return KM_OK;
}

int km_step_loop_check(km_engine* e) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  return launch_check(e);  // after a host repair: congruence test, filter prep, exhaustion
}

int km_step_loop_state(km_engine* e, int32_t* out4) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  int r;
  if ((r = read_state(e))) return r;
  if (out4) {
    out4[0] = e->st_host->t;
    out4[1] = e->st_host->done;
    out4[2] = e->st_host->converged;
    out4[3] = e->st_host->need_host;
  }
  return KM_OK;
}

int km_step_check(km_engine* e, double tol, int32_t* converged_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  int r;
  CK(cudaMemcpyAsync(e->st_host, e->st, sizeof(DevState), cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  e->st_host->tol = tol;
  e->st_host->max_iters = INT32_MAX;
  CK(cudaMemcpyAsync(e->st, e->st_host, sizeof(DevState), cudaMemcpyHostToDevice, e->stream));
  if ((r = launch_check(e))) return r;
  if ((r = read_state(e))) return r;
  if (converged_out) *converged_out = e->st_host->converged;
  return KM_OK;
}

int km_step_read(km_engine* e, double* centers_out, int64_t* counts_out, int64_t* labels_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  int r;
  if (centers_out) CK(cudaMemcpyAsync(centers_out, e->cur, 8 * (size_t)e->k * e->m, cudaMemcpyDeviceToHost, e->stream));
  if (counts_out) CK(cudaMemcpyAsync(counts_out, e->model_counts, 8 * (size_t)e->k, cudaMemcpyDeviceToHost, e->stream));
  if (labels_out && (r = download_labels(e, labels_out))) return r;
  CK(cudaStreamSynchronize(e->stream));
  return KM_OK;
}

// ---- row-sharded resident loop with the in-kernel NVLink exchange -------------------------
static void peer_release(km_engine* e) {
  for (void* p : e->xch_opened) cudaIpcCloseMemHandle(p);
  e->xch_opened.clear();
  dfree(e->xch_peers_dev);
  e->xch_peers_dev = nullptr;
  dfree(e->xch);
  e->xch = nullptr;
  e->xch_nacc = 0;
  e->world = 1;
  e->rank = 0;
}

int km_peer_init(km_engine* e, int32_t world, int32_t rank, int32_t k, void* handle_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if (world < 1 || rank < 0 || rank >= world) return set_err(e, KM_ERR_CONTRACT, "bad world/rank %d/%d", world, rank);
  if (k < 1) return set_err(e, KM_ERR_CONTRACT, "k must be >= 1, got %d", k);
  if (!handle_out) return set_err(e, KM_ERR_CONTRACT, "null handle_out");
  cudaSetDevice(e->device);
  peer_release(e);
  const size_t nacc = (size_t)k * e->m + k;
  const size_t words = 2 * (size_t)world * nacc + 2 * (size_t)world;
  int r;
  if ((r = dalloc(e, &e->xch, 8 * words))) return r;
  CK(cudaMemset(e->xch, 0, 8 * words));  // sequence flags start below every run's values
  cudaIpcMemHandle_t h{};
  CK(cudaIpcGetMemHandle(&h, e->xch));
  std::memcpy(handle_out, &h, sizeof h);
  e->world = world;
  e->rank = rank;
  e->xch_nacc = nacc;
  return KM_OK;
}

int km_peer_connect(km_engine* e, const void* handles) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->xch) return set_err(e, KM_ERR_CONTRACT, "call km_peer_init first");
  if (!handles) return set_err(e, KM_ERR_CONTRACT, "null handles");
  cudaSetDevice(e->device);
  std::vector<unsigned long long*> ptrs((size_t)e->world, nullptr);
  for (int p = 0; p < e->world; ++p) {
    if (p == e->rank) {
      ptrs[p] = e->xch;
      continue;
    }
    cudaIpcMemHandle_t h{};
    std::memcpy(&h, static_cast<const unsigned char*>(handles) + (size_t)p * sizeof h, sizeof h);
    void* d = nullptr;
    CK(cudaIpcOpenMemHandle(&d, h, cudaIpcMemLazyEnablePeerAccess));
    e->xch_opened.push_back(d);
    ptrs[p] = static_cast<unsigned long long*>(d);
  }
  int r;
  if ((r = dalloc(e, &e->xch_peers_dev, sizeof(void*) * (size_t)e->world))) return r;
  CK(cudaMemcpy(e->xch_peers_dev, ptrs.data(), sizeof(void*) * (size_t)e->world, cudaMemcpyHostToDevice));
  return KM_OK;
}

static void peer_state(km_engine* e, int32_t* out4) {
  if (!out4) return;
  out4[0] = e->st_host->t;
  out4[1] = e->st_host->done;
  out4[2] = e->st_host->converged;
  out4[3] = e->st_host->need_host;
}

int km_lloyd_peer(km_engine* e, const double* c0, int32_t k, int32_t max_iters, double tol, int32_t* state_out4) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  int r;
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if (!e->xch_peers_dev) return set_err(e, KM_ERR_CONTRACT, "call km_peer_init and km_peer_connect first");
  if (max_iters < 1) return set_err(e, KM_ERR_CONTRACT, "max_iters must be >= 1, got %d", max_iters);
  if (!(tol >= 0.0)) return set_err(e, KM_ERR_CONTRACT, "tol must be >= 0, got %g", tol);
  if ((r = check_centers(e, c0, k))) return r;
  if ((size_t)k * e->m + k != e->xch_nacc) return set_err(e, KM_ERR_CONTRACT, "k differs from km_peer_init's");
  if ((r = ensure_k(e, k))) return r;
  scale_for_centers(e, c0, k);
  if (!use_tc(e) || e->resident_unfit)
    return set_err(e, KM_ERR_CAPACITY, "the resident peer loop needs the tensor-core pass (fp32, m <= 31, k <= 128)");
  e->epoch += 1;
  e->peer_active = true;
  r = lloyd_resident(e, c0, max_iters, tol);
  e->peer_active = false;
  if (r == KM_RESIDENT_UNFIT) {
    e->resident_unfit = true;
    return set_err(e, KM_ERR_CAPACITY, "shape does not fit the resident loop");
  }
  if (r) return r;
  peer_state(e, state_out4);
  return KM_OK;
}

int km_lloyd_peer_resume(km_engine* e, int32_t* state_out4) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  if (!e->xch_peers_dev || !e->part) return set_err(e, KM_ERR_CONTRACT, "call km_lloyd_peer first");
  e->peer_active = true;
  const int r = lloyd_resident(e, nullptr, 0, 0.0, true);
  e->peer_active = false;
  if (r) return r;
  peer_state(e, state_out4);
  return KM_OK;
}

int km_set_kernel_path(km_engine* e, int32_t path) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (path < 0 || path > 3)
    return set_err(e, KM_ERR_CONTRACT, "path must be 0 (auto), 1 (SIMT), 2 (tensor core) or 3 (SIMT, one point per thread)");
  e->path_pref = path;
  return KM_OK;
}

int km_kernel_path(km_engine* e, int32_t* out) {
  if (!e || !out) return set_err(e, KM_ERR_CONTRACT, "null argument");
  *out = use_tc(e) ? 2 : 1;
  return KM_OK;
}

int km_debug_filter_scores(km_engine* e, const double* centers, int32_t k, float* out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  cudaSetDevice(e->device);
  int r;
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if (!out) return set_err(e, KM_ERR_CONTRACT, "null out");
  if ((r = check_centers(e, centers, k))) return r;
  if ((r = ensure_k(e, k))) return r;
  if (!use_tc(e)) return set_err(e, KM_ERR_CAPACITY, "tensor-core filter not available for this shape");
  scale_for_centers(e, centers, k);
  float* dbg = nullptr;
  if ((r = dalloc(e, &dbg, sizeof(float) * (size_t)e->n * k))) return r;
  CK(cudaMemcpyAsync(e->cur, centers, 8 * (size_t)k * e->m, cudaMemcpyHostToDevice, e->stream));
  if ((r = reset_state(e, 1, 0.0))) { cudaFree(dbg); return r; }
  if ((r = launch_prep(e))) { cudaFree(dbg); return r; }
  CK(cudaMemsetAsync(e->part, 0, 8 * ((size_t)k * e->m + k), e->stream));
  e->dbg_scores = dbg;
  r = launch_pass(e, PASS_ASSIGN_ONLY, false);
  e->dbg_scores = nullptr;
  cudaMemsetAsync(e->recheck_count, 0, 4, e->stream);
  cudaError_t c = cudaSuccess;
  if (!r) c = cudaMemcpyAsync(out, dbg, sizeof(float) * (size_t)e->n * k, cudaMemcpyDeviceToHost, e->stream);
  if (!r && c == cudaSuccess) c = cudaMemsetAsync(e->part, 0, 8 * ((size_t)k * e->m + k), e->stream);
  if (!r && c == cudaSuccess) c = cudaStreamSynchronize(e->stream);
  cudaFree(dbg);
  if (r) return r;
  if (c != cudaSuccess) return cuda_fail(e, c, "km_debug_filter_scores");
  return KM_OK;
}

int km_reset_stats(km_engine* e) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  const int32_t fb = e->stats.frac_bits, pb = e->stats.point_bytes;
  e->stats = km_stats{};
  e->stats.frac_bits = fb;
  e->stats.point_bytes = pb;
  return KM_OK;
}

int km_set_profiling(km_engine* e, int32_t enable) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  e->profiling = enable != 0;
  return KM_OK;
}

int km_get_stats(km_engine* e, km_stats* out) {
  if (!e || !out) return set_err(e, KM_ERR_CONTRACT, "null argument");
  *out = e->stats;
  return KM_OK;
}

}  // extern "C"

// COORD_SUM / CLUSTER_SUM device jobs (device.py:117-134; HostReferenceDevice._execute :218-239):
// per-block sums of samples [start, stop) (start on a block boundary), blocks of `block`
// samples.  labels == NULL: coordinate sums, sums_out (nb, m).  Otherwise cluster sums,
// sums_out (nb, k, m) and counts_out (nb, k); *bad_out = the first sample whose label lies
// outside [0, k) (then KM_ERR_VALIDATION), else -1.  The sums are exact int64 fixed point
// rounded once to fp64 (the reference's sequential fp64 block sums agree to ~1e-15 relative).
int km_block_sums(km_engine* e, const int64_t* labels, int32_t k, int64_t start, int64_t stop, int64_t block,
                  double* sums_out, int64_t* counts_out, int64_t* bad_out) {
  if (!e) return set_err(nullptr, KM_ERR_CONTRACT, "null engine");
  if (!e->x) return set_err(e, KM_ERR_CONTRACT, "no points loaded");
  if (bad_out) *bad_out = -1;
  if (!(0 <= start && start <= stop && stop <= e->n))
    return set_err(e, KM_ERR_CONTRACT, "job range [%lld, %lld) must lie within [0, %lld]", (long long)start,
                   (long long)stop, (long long)e->n);
  if (block < 1) return set_err(e, KM_ERR_CONTRACT, "block size must be >= 1, got %lld", (long long)block);
  if (start % block)
    return set_err(e, KM_ERR_CONTRACT, "job range must start on an accumulation-block boundary (start=%lld, block=%lld)",
                   (long long)start, (long long)block);
  const bool cluster = labels != nullptr;
  if (cluster && k < 1) return set_err(e, KM_ERR_CONTRACT, "k must be >= 1, got %d", k);
  const int kk = cluster ? k : 1;
  const int m = e->m;
  const int64_t len = stop - start;
  const int64_t nb = (len + block - 1) / block;
  if (nb == 0) return KM_OK;
  if (!sums_out || (cluster && !counts_out)) return set_err(e, KM_ERR_CONTRACT, "null output");
  const size_t smem = 8 * ((size_t)kk * m + kk);
  if (smem > e->smem_optin) return set_err(e, KM_ERR_CAPACITY, "k*m too large for a device sum job");
  cudaSetDevice(e->device);
  int r;
  const size_t nacc = (size_t)nb * kk * m + (size_t)nb * kk + 1;  // + the bad-label slot
  if ((r = grow(e, &e->job_acc, &e->job_acc_cap, 8 * nacc))) return r;
  unsigned long long* acc = (unsigned long long*)e->job_acc;
  CK(cudaMemsetAsync(acc, 0, 8 * (nacc - 1), e->stream));
  const unsigned long long nobad = ~0ull;
  CK(cudaMemcpyAsync(acc + nacc - 1, &nobad, 8, cudaMemcpyHostToDevice, e->stream));
  const int32_t* dlab = nullptr;
  std::vector<int32_t> lab32;
  if (cluster) {
    lab32.resize((size_t)len);
    for (int64_t i = 0; i < len; ++i) {
      const int64_t v = labels[start + i];
      lab32[i] = (v < 0 || v >= k) ? -1 : (int32_t)v;
    }
    if ((r = grow(e, &e->job_lab, &e->job_lab_cap, 4 * (size_t)len))) return r;
    CK(cudaMemcpyAsync(e->job_lab, lab32.data(), 4 * (size_t)len, cudaMemcpyHostToDevice, e->stream));
    dlab = (const int32_t*)e->job_lab;
  }
  const int64_t cpb = (std::min<int64_t>(block, len) + kBlockSumChunk - 1) / kBlockSumChunk;
  const int F = e->frac_bits;
  const double sd = std::ldexp(1.0, F);
  const int use_d = (F > 120 || F < -120) ? 1 : 0;
  const float sf = use_d ? 1.0f : (float)sd;
  if (nb * cpb > INT32_MAX) return set_err(e, KM_ERR_CAPACITY, "too many blocks");
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(block_sums_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(block_sums_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  if (e->point_bytes == 4)
    block_sums_kernel<float><<<(unsigned)(nb * cpb), 256, smem, e->stream>>>(
        (const float*)e->x, m, start, stop, block, cpb, dlab, kk, sf, sd, use_d, nb, acc, acc + nacc - 1);
  else
    block_sums_kernel<double><<<(unsigned)(nb * cpb), 256, smem, e->stream>>>(
        (const double*)e->x, m, start, stop, block, cpb, dlab, kk, sf, sd, use_d, nb, acc, acc + nacc - 1);
  CK_LAUNCH("block_sums_kernel");
  e->stats.kernel_launches += 1;
  std::vector<unsigned long long> h(nacc);
  CK(cudaMemcpyAsync(h.data(), acc, 8 * nacc, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  if (h[nacc - 1] != nobad) {
    if (bad_out) *bad_out = (int64_t)h[nacc - 1];
    return set_err(e, KM_ERR_VALIDATION, "label out of range [0, %d) at sample %lld", k, (long long)h[nacc - 1]);
  }
  const double inv = std::ldexp(1.0, -F);
  const size_t ns = (size_t)nb * kk * m;
  for (size_t i = 0; i < ns; ++i) sums_out[i] = (double)(long long)h[i] * inv;
  if (cluster)
    for (size_t i = 0; i < (size_t)nb * kk; ++i) counts_out[i] = (int64_t)h[ns + i];
  return KM_OK;
}
