/*
 * kmeans_b200.h — C ABI of the B200-native Lloyd engine (assign → update →
 * congruence test), the drop-in for the reference's hot path.
 *
 * The reference (`kmeans-regimes`, /root/reference/pkg) has no C ABI: its hot
 * path is Python calling numba kernels.  Each entry point below names the
 * reference function whose contract it replaces (file:line relative to
 * /root/reference/pkg/src/kmeans_regimes/).  Plain pointers and sizes only; no
 * torch or CUDA types cross this boundary (streams are passed as void*).
 *
 * Ownership: the caller owns every host buffer; the library owns device
 * buffers.  Points uploaded with km_load_points_* stay resident on the device
 * until the next load or km_destroy (the reference keeps one immutable
 * Dataset per run, model.py:34-47; the bridge ships coordinates once by
 * digest, bridge.py:103-119).
 *
 * Errors: every call returns a km_status; the message of the most recent
 * failure on a handle is km_last_error(handle) (km_last_error(NULL) for
 * failures before a handle exists).  Codes map 1:1 onto the reference's
 * exception classes (exceptions.py:4-74).  There is no CPU fallback: a CUDA
 * error surfaces as KM_ERR_DEVICE_LOST / KM_ERR_DEVICE_UNAVAILABLE.
 *
 * Threading: calls on one handle must be serialised by the caller (the
 * reference's Device serialises with a lock, device.py:167,181-193).  A handle
 * owns one CUDA stream on one device.
 */
#ifndef KMEANS_B200_H
#define KMEANS_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define KM_API __attribute__((visibility("default")))
#else
#define KM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum km_status {
  KM_OK = 0,
  KM_ERR_CONTRACT = 1,           /* ContractViolationError   (validation.py:8-52, engine.py:223-226) */
  KM_ERR_VALIDATION = 2,         /* ValidationFailureError   (device.py:234-238: label out of range on device) */
  KM_ERR_DEVICE_UNAVAILABLE = 3, /* DeviceUnavailableError   (device.py:253-261) */
  KM_ERR_DEVICE_LOST = 4,        /* DeviceLostError          (device.py:377-382) */
  KM_ERR_CAPACITY = 5,           /* CapacityExceededError    (device.py:175-179: device memory exhausted) */
  KM_ERR_INTERNAL = 6            /* ClusteringError (root)   */
} km_status;

typedef struct km_engine km_engine;

/* Per-iteration loop state, readable after km_lloyd / km_step_* calls. */
typedef struct km_stats {
  int64_t passes;          /* fused assign+update passes launched            */
  int64_t rechecked;       /* points whose fp32 label was not certified and were
                              re-decided in exact fp64 (cumulative)            */
  int64_t repairs;         /* empty clusters repaired (cumulative)             */
  int64_t host_syncs;      /* host<->device synchronisations in km_lloyd       */
  int32_t frac_bits;       /* fixed-point fraction bits F of the cluster sums  */
  int32_t point_bytes;     /* 4 (fp32 resident points) or 8 (fp64)            */
  int64_t kernel_launches; /* kernels this handle launched (cumulative)       */
  int64_t changed;         /* labels changed by incremental passes (last run) */
  int64_t pass_timed;      /* fused passes timed with CUDA events (profiling) */
  double pass_ms_total;    /* their summed device time, ms                    */
} km_stats;

/* ---- lifetime ---------------------------------------------------------- */
KM_API const char* km_version(void);
KM_API int km_device_count(int32_t* out);
KM_API int km_create(int32_t device, km_engine** out);
KM_API int km_destroy(km_engine* e);
KM_API const char* km_last_error(const km_engine* e);
/* Use an external CUDA stream (cudaStream_t as void*; NULL = the handle's own). */
KM_API int km_set_stream(km_engine* e, void* stream);

/* ---- dataset (reference: model.Dataset, model.py:34-75) ---------------- */
/* Upload n×m row-major points once; they stay resident.  fp32 input is kept
 * as fp32.  fp64 input is stored as fp32 when every value is exactly
 * representable (lossless), else as fp64 — results are the same either way. */
KM_API int km_load_points_f32(km_engine* e, const float* x, int64_t n, int32_t m);
KM_API int km_load_points_f64(km_engine* e, const double* x, int64_t n, int32_t m);
/* Borrow an existing device buffer of n×m fp32 points (no copy; caller keeps
 * it alive).  Used by the bench's device-resident leg. */
KM_API int km_attach_points_device_f32(km_engine* e, const float* dev_x, int64_t n, int32_t m);
KM_API int km_points_info(km_engine* e, int64_t* n, int32_t* m, int32_t* point_bytes, double* absmax);

/* ---- hot-path steps ---------------------------------------------------- */
/* engine.assign_step (engine.py:218-230) / _kernels.assign_block
 * (_kernels.py:22-45): nearest centre by squared distance, ties → lowest
 * index; counts_out = bincount(labels).  centers: k×m fp64 row-major. */
KM_API int km_assign(km_engine* e, const double* centers, int32_t k,
              int64_t* labels_out, int64_t* counts_out);

/* engine.update_step (engine.py:281-294) + _finish_update (engine.py:249-278):
 * centres = per-cluster means of `labels`; empty clusters repaired in
 * ascending order at the sample farthest from its own new centre, which is
 * relabelled IN PLACE in labels_inout (engine.py:258,272).  Labels outside
 * [0,k) → KM_ERR_CONTRACT. */
KM_API int km_update(km_engine* e, int64_t* labels_inout, int32_t k,
              double* centers_out, int64_t* counts_out);

/* engine.converged (engine.py:297-310): max_c sqrt(Σ_f (prev−next)²) ≤ tol,
 * fp64 left-to-right without FMA (tol = 0 ⇒ exact fixed point). */
KM_API int km_converged(km_engine* e, const double* prev, const double* next,
                 int32_t k, int32_t m, double tol, int32_t* out);

/* engine.iterate (engine.py:320-343) with the single-regime closures, from
 * explicit initial centres c0 (k×m fp64).  Same counting/return rules:
 * converged at update t ⇒ (C_t, L_{t-1} repaired, t, 1); exhaustion ⇒
 * (C_T, L_T = A(C_T), T, 0) with counts = bincount(L_T).
 * labels_out may be NULL (skip the n×8 B download). */
KM_API int km_lloyd(km_engine* e, const double* c0, int32_t k, int32_t max_iters, double tol,
             double* centers_out, int64_t* counts_out, int64_t* labels_out,
             int32_t* iterations_out, int32_t* converged_out);

/* wcss / inertia_ (model.py:206-217, _kernels.wcss_block :129-141) of the
 * given centres and labels (fp64 self-distances, exact fixed-point total). */
KM_API int km_wcss(km_engine* e, const double* centers, int32_t k, const int64_t* labels, double* out);

/* transform (estimator.py:183-189, _kernels.center_distances :158-170):
 * out (n×k fp64) = Euclidean distance of every resident point to every centre. */
KM_API int km_center_distances(km_engine* e, const double* centers, int32_t k, double* out);

/* ---- seeding ----
 * km_diameter: largest pairwise distance over rows scan_rows(n, pair_cap) × all j > i
 *   (engine.diameter / _kernels.max_pair_rows, engine.py:124-154, _kernels.py:49-81): exact
 *   fp64 value of the reference recurrence, ties → smallest (i, j).  pair_cap <= 0: every pair.
 * km_seed_reset / km_seed_add / km_seed_min_d2: the per-sample minimum squared distance to the
 *   chosen centres (engine._append_center / _kernels.update_min_d2, engine.py:157-160,
 *   _kernels.py:144-155, fp64, same recurrence); km_seed_add lowers it with sample c and returns
 *   np.argmax of the result (largest, lowest index) — the maximin step (engine.py:162-168). */
KM_API int km_diameter(km_engine* e, int64_t pair_cap, double* d_out, int64_t* i_out, int64_t* j_out);
KM_API int km_seed_reset(km_engine* e);
KM_API int km_seed_add(km_engine* e, int64_t c, double* max_v, int64_t* max_i);
KM_API int km_seed_min_d2(km_engine* e, int64_t i, double* out);

/* ---- device jobs (the reference's offload-device protocol) ----
 * The B200 side of a `Device._execute(job)` (device.py:153-239) for the three job kinds:
 * km_max_pair_rows: MAX_PAIR (device.max_pair_job :117-122 → _kernels.max_pair_rows,
 *   _kernels.py:48-81): best pair over the given strictly ascending rows × columns j > i, exact
 *   fp64 d² (not its root), ties → smallest (i, j); (-1, -1, -1) when the rows give no pair.
 * km_block_sums: COORD_SUM (labels == NULL; sums_out (nb, m)) and CLUSTER_SUM (sums_out
 *   (nb, k, m), counts_out (nb, k)) over samples [start, stop), start on a `block` boundary
 *   (device._check_range :139-150, HostReferenceDevice._execute :218-239 →
 *   _kernels.coord_sums_block / cluster_sums_block, _kernels.py:84-113); nb = ceil((stop −
 *   start)/block).  A label outside [0, k) → KM_ERR_VALIDATION with *bad_out = its sample index
 *   (device.py:233-238).  Sums are exact fixed point rounded once to fp64. */
KM_API int km_max_pair_rows(km_engine* e, const int64_t* rows, int64_t nrows, double* d2_out, int64_t* i_out,
                            int64_t* j_out);
KM_API int km_block_sums(km_engine* e, const int64_t* labels, int32_t k, int64_t start, int64_t stop, int64_t block,
                         double* sums_out, int64_t* counts_out, int64_t* bad_out);

/* ---- row-sharded multi-GPU step API (partition.py:84-100,237-261) ------
 * One process per GPU holds a contiguous row shard.  Per iteration:
 *   km_step_pass      fused assign + per-cluster fixed-point sums of the shard
 *   (caller)          allreduce-sum the int64 partial buffer across ranks
 *   km_step_finish    divide, empty-cluster count, convergence flag
 * The partial buffer is (k·m sums + k counts) int64 on the device; its device
 * address is returned by km_step_partials so an NCCL allreduce (e.g.
 * torch.distributed) can run on it in place. */
KM_API int km_set_frac_bits(km_engine* e, int32_t frac_bits);   /* agree on a global F */
KM_API int km_frac_bits_for(double absmax, int64_t n_total, int32_t* out);
KM_API int km_step_begin(km_engine* e, const double* c0, int32_t k);
KM_API int km_step_partials(km_engine* e, void** dev_ptr, int64_t* n_int64);
KM_API int km_step_pass(km_engine* e);
/* status_out[0] = #empty clusters, [1] = converged (only valid when no empties) */
KM_API int km_step_finish(km_engine* e, double tol, int32_t* status_out);
/* empty-cluster repair across shards: local candidate = (max self-distance,
 * first local row); the caller picks the global winner (largest d², lowest
 * global row) and calls km_step_repair_apply on every rank. */
KM_API int km_step_repair_prepare(km_engine* e);                 /* self-distances of the shard */
KM_API int km_step_repair_candidate(km_engine* e, double* d2_out, int64_t* row_out, double* coords_out);
KM_API int km_step_repair_apply(km_engine* e, int32_t empty_cluster, int32_t owner_is_me,
                         int64_t local_row, const double* coords, int32_t donor_cluster_or_neg);
/* exhausted run: after the final pass and its allreduce, fold it into the
 * totals so km_step_read returns counts = bincount(L_T) */
KM_API int km_step_fold(km_engine* e);
KM_API int km_step_empty_list(km_engine* e, int32_t* empties_out, int32_t* n_out);
KM_API int km_step_label_of(km_engine* e, int64_t local_row, int32_t* label_out);
KM_API int km_step_check(km_engine* e, double tol, int32_t* converged_out);

/* Batched form of the same loop (no host round trip per iteration): after km_step_begin and
 * km_step_loop_begin, enqueue km_step_loop_pass (L0), then per iteration [allreduce of the
 * partial buffer, km_step_loop_finish, km_step_loop_pass]; read {t, done, converged, need_host}
 * with km_step_loop_state every few iterations.  Kernels are gated on the device state, so
 * iterations enqueued past the end do no work.  need_host: run the global repair with the
 * km_step_repair_* calls, then km_step_loop_check. */
KM_API int km_step_loop_begin(km_engine* e, int32_t max_iters, double tol);
KM_API int km_step_loop_pass(km_engine* e);
KM_API int km_step_loop_finish(km_engine* e);
KM_API int km_step_loop_check(km_engine* e);
KM_API int km_step_loop_state(km_engine* e, int32_t* out4);
KM_API int km_step_read(km_engine* e, double* centers_out, int64_t* counts_out, int64_t* labels_out);

/* Resident form of the row-sharded loop (the fast path): one cooperative launch per GPU runs
 * the whole Lloyd loop, and every iteration's (k·m + k) int64 Δ is exchanged INSIDE the kernel
 * over NVLink peer memory — each rank pushes its Δ into every rank's exchange buffer (CUDA IPC
 * mapping) and sums the `world` rows it receives — instead of an allreduce launch per iteration.
 *   km_peer_init      allocate this rank's exchange buffer for k; export its IPC handle (64 bytes)
 *   km_peer_connect   map every rank's buffer (handles[world][64], gathered by the caller)
 *   km_lloyd_peer     run from C0 until the loop is done or needs the host (empty clusters)
 *   km_lloyd_peer_resume   after the global repair (km_step_repair_*) and km_step_loop_check
 * state_out4 = {t, done, converged, need_host}; results through km_step_read.  Every rank must
 * call these in lockstep with the same C0 / max_iters / tol and a global km_set_frac_bits. */
KM_API int km_peer_init(km_engine* e, int32_t world, int32_t rank, int32_t k, void* handle_out);
KM_API int km_peer_connect(km_engine* e, const void* handles);
KM_API int km_lloyd_peer(km_engine* e, const double* c0, int32_t k, int32_t max_iters, double tol,
                         int32_t* state_out4);
KM_API int km_lloyd_peer_resume(km_engine* e, int32_t* state_out4);

KM_API int km_get_stats(km_engine* e, km_stats* out);
KM_API int km_reset_stats(km_engine* e);
/* Kernel path for the fused pass: 0 = auto (tcgen05 tensor-core pass when the
 * shape allows: fp32 points, m ≤ 31, k ≤ 128; SIMT otherwise — register-blocked
 * for fp32 points with m ≤ 32, k ≥ 32), 1 = SIMT only, 2 = tensor core required
 * (error if not available), 3 = SIMT one point per thread (no register blocking;
 * a test hook for the blocked kernel). */
KM_API int km_set_kernel_path(km_engine* e, int32_t path);
KM_API int km_kernel_path(km_engine* e, int32_t* out);   /* path the next pass uses: 1 SIMT, 2 tensor core */
/* Test hook: raw tensor-core filter scores S~[n×k] = ‖c~‖² − 2x·c~ (fp32) for the given centres. */
KM_API int km_debug_filter_scores(km_engine* e, const double* centers, int32_t k, float* out);
/* Record a CUDA event pair around every fused pass km_lloyd launches (on the
 * handle's stream) and accumulate the device time of the passes that ran. */
KM_API int km_set_profiling(km_engine* e, int32_t enable);

#ifdef __cplusplus
}
#endif
#endif /* KMEANS_B200_H */
