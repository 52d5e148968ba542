/*
 * parsmc_b200.h -- C ABI of the B200-native particle filtering / particle
 * learning engine (libparsmc_b200.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types cross this boundary.
 * Every entry point returns a status code (PF_OK on success); the message and
 * failing time step of the last error on the calling thread are available
 * from pf_last_error_message() / pf_last_error_step().  Codes map 1:1 onto
 * the reference's exception classes (parsmc errors.py:4-35):
 *
 *   PF_ERR_ALL_WEIGHTS_ZERO   AllWeightsZeroError(step=t)  filtering.py:294-296,
 *                                                          prefix_sum.py:97-100
 *   PF_ERR_NON_FINITE_WEIGHT  NonFiniteWeightError         core.py:26-27
 *   PF_ERR_NOT_POWER_OF_TWO   NotPowerOfTwoError           core.py:16-18
 *   PF_ERR_VALUE              ValueError                   filtering.py:205-208
 *
 * Reference paths below are relative to the reference's pkg/src/parsmc/.
 * Indices crossing the boundary are 1-based int64, as in the reference
 * (resampling.py:15-16).
 */
#ifndef PARSMC_B200_H
#define PARSMC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PF_OK = 0,
  PF_ERR_ALL_WEIGHTS_ZERO = 1,
  PF_ERR_NON_FINITE_WEIGHT = 2,
  PF_ERR_NOT_POWER_OF_TWO = 3,
  PF_ERR_VALUE = 4,
  PF_ERR_CUDA = 5,
  PF_ERR_OUT_OF_MEMORY = 6,
  PF_ERR_NOT_IMPLEMENTED = 7
};

enum { PF_DTYPE_F64 = 0, PF_DTYPE_F32 = 1 };

/* ------------------------------------------------------------ library --- */
const char* pf_version(void);
const char* pf_last_error_message(void);
/* sizeof(pf_config), sizeof(pf_outputs), sizeof(pf_feed) as compiled into
 * the library: lets a binding check its struct mirrors (no device needed). */
int pf_abi_sizes(int64_t* sizes3);
int64_t pf_last_error_step(void);
/* Number of visible CUDA devices (0 on a host without a GPU; never fails). */
int pf_device_count(void);
/* Kernels launched by this process so far (the bench's gpu_launches). */
int64_t pf_launch_count(void);

/* ------------------------------------------------------ engine (L3) --- */
/* Replaces filtering._run_loop (filtering.py:200-374) behind
 * run_particle_learning (filtering.py:178-197) and run_particle_filter
 * (filtering.py:165-175).  One engine = one device-resident particle system
 * of n slots; runs are repeatable and bit-identical for a fixed seed. */
typedef struct pf_config {
  int64_t n;               /* particle count, a power of two (cut-point) */
  uint64_t seed;           /* Philox key word 0; slot j uses stream j */
  int32_t learn;           /* 1: run_particle_learning, 0: run_particle_filter */
  int32_t learn_sigma2;    /* sigma2 ~ IG(shape, scale) learned (models.py:82-88) */
  int32_t learn_tau2;
  int32_t precision;       /* PF_DTYPE_F64 ("double") / PF_DTYPE_F32 ("single") */
  double x0_mean, x0_var;
  double sqrt_x0_var;      /* math.sqrt(x0_var), host-computed (filtering.py:235) */
  double sigma2_shape, sigma2_scale;
  double tau2_shape, tau2_scale;
  double sigma2_fixed;     /* used when the parameter is not learned */
  double tau2_fixed;
  double sqrt_tau2_fixed;  /* np.sqrt(tau2) (filtering.py:274) */
  double log_term_fixed;   /* -0.5*(LOG_TWO_PI + np.log(sigma2)) (filtering.py:293) */
  int32_t track_quantiles; /* weighted 5/50/95% state quantiles per step */
  int32_t keep_indices;    /* resampled_indices [T, n] (1-based) */
  int32_t keep_final;      /* final_particles */
  int32_t store_particles; /* particle_history, one snapshot per step */
  int32_t phase_timing;    /* per-phase CUDA-event timings (PhaseTimings) */
  int32_t gamma_method;    /* 0: per-step table (default), 1: accurate per draw */
  int32_t device;          /* CUDA device ordinal */
  int32_t resampler;       /* PF_RESAMPLE_*: cutpoint (the exact parallel path) or one
                              of the reference's sequential baselines */
} pf_config;

/* Resampling schemes (filtering.py:305-317, resampling.py:29-177).  The
 * baselines run on the reference's sequential CDF (a left-to-right cumsum,
 * prefix_sum.py:130-134) and accept any n >= 1; cutpoint needs a power of 2.
 * PF_RESAMPLE_SPACINGS (perf mode, not in the reference) is exact multinomial
 * resampling like the reference's `sorted` (resampling.py:57-67), but its
 * sorted uniforms are generated in order -- U_(k) = S_k / S_(N+1), S the
 * prefix sums of standard exponentials drawn from each slot's Philox word 3
 * -- and looked up in the cut-point tables, so ancestors are nondecreasing in
 * the slot: record gathers stream, and a shard's ancestors stay in the shard
 * except at its boundaries.  Power of 2 like cutpoint. */
enum { PF_RESAMPLE_CUTPOINT = 0, PF_RESAMPLE_NAIVE = 1, PF_RESAMPLE_SORTED = 2,
       PF_RESAMPLE_STRATIFIED = 3, PF_RESAMPLE_SYSTEMATIC = 4, PF_RESAMPLE_SPACINGS = 5 };

/* Oracle mode: host arrays [T+1][n] (row 0 = initialisation) that replace the
 * ndtri / gammaincinv outputs (and optionally the normalised weights) with
 * the reference's own draws.  NULL members are computed on the device. */
typedef struct pf_feed {
  const double* z;        /* ndtri(u)        rng.py:223-224 */
  const double* g_sigma;  /* gammaincinv     rng.py:226-229, filtering.py:280 */
  const double* g_tau;    /*                 filtering.py:286 */
  const double* w;        /* exp(lw - max)   filtering.py:297 (rows 1..T) */
} pf_feed;

/* Caller-allocated host outputs; NULL members are not produced. */
typedef struct pf_outputs {
  double* filtered_mean;        /* [T] */
  double* filtered_quantiles;   /* [T][3]  probs (0.05, 0.5, 0.95) */
  double* sigma2_mean;          /* [T] */
  double* sigma2_sd;            /* [T] */
  double* sigma2_quantiles;     /* [T][5]  probs (0.005, 0.05, 0.5, 0.95, 0.995) */
  double* tau2_mean;
  double* tau2_sd;
  double* tau2_quantiles;
  int64_t* indices;             /* [T][n] 1-based ancestors */
  /* final particles (post-resample system at step T; init system if T == 0) */
  double* final_states;         /* [n] (float32 values when precision single) */
  double* final_sigma2;         /* [n] */
  double* final_tau2;
  double* final_a_sigma;
  double* final_b_sigma;
  double* final_a_tau;
  double* final_b_tau;
  /* store_particles: [T][n] snapshots of the same seven arrays */
  double* hist_states;
  double* hist_sigma2;
  double* hist_tau2;
  double* hist_a_sigma;
  double* hist_b_sigma;
  double* hist_a_tau;
  double* hist_b_tau;
  /* PhaseTimings (filtering.py:44-74): initialize, cdf, resample,
   * resample_sort_only, propagate, store, other (nanoseconds) */
  int64_t phase_ns[7];
  int64_t failed_step;          /* step of AllWeightsZeroError, else 0 */
  /* [T] effective sample size (sum w)^2 / sum w^2 of the pre-resample weights
   * (an extension: the reference reports no ESS); reduced with the other
   * per-shard sums in sharded runs */
  double* ess;
} pf_outputs;

typedef struct pf_engine pf_engine;

int pf_engine_create(const pf_config* cfg, pf_engine** out);
/* Replace the model / seed / output flags of an engine; n, precision and
 * device must not change (the device buffers are sized by them). */
int pf_engine_reconfigure(pf_engine* e, const pf_config* cfg);
int pf_engine_run(pf_engine* e, const double* y, int64_t t_len,
                  const pf_feed* feed, pf_outputs* out);
/* Device-resident repeat of the last run's workload: y is already on the
 * device; no host outputs are copied.  Used by bench.py for the kernel-only
 * throughput (value); pf_engine_run is the end-to-end path (e2e). */
/* Batched replications (BASELINE configs[4]; the paper's timing experiment,
 * replication r = an independent run with seed seeds[r]): `reps` filters of
 * the engine's n particles on the same series, every kernel launch covering
 * all of them.  Outputs are the per-step summaries only, each [reps][t_len]
 * row-major (quantiles [reps][t_len][k]); indices, store and final states
 * must be NULL.  Each replication follows pf_engine_run with that seed:
 * the same particles and ancestors; means / sds to rounding and quantiles
 * except at exact near-ties (the weight sums are split over fewer CTAs per
 * replication).  reps > 1 needs
 * cut-point resampling, gamma_method 0 and 2^11 <= n < 2^21. */
int pf_engine_run_batch(pf_engine* e, const uint64_t* seeds, int32_t reps, const double* y,
                        int64_t t_len, pf_outputs* out);
int pf_engine_run_resident(pf_engine* e, int64_t t_len);
/* Device time (ms, CUDA events) of the last run / resident run, and the
 * average duration and launch count of the step kernel inside it. */
int pf_engine_last_timing(pf_engine* e, double* total_ms, double* step_kernel_ms,
                          int64_t* step_kernel_launches, int64_t* kernels_launched);
/* Weighted-quantile diagnostics of the last run: [0] quantiles resolved on
 * a truncated candidate set (should be 0), [1] window misses that needed
 * the fallback pass, [2] largest candidate list, [3] resolves performed. */
int pf_engine_quantile_stats(pf_engine* e, int64_t* stats4);
/* Kernel path the last run took (bit mask): PF_PATH_FUSED_DRAWS -- draws
 * computed inside the step kernel; PF_PATH_RANK_TABLES -- strata rank-table
 * lookups (N >= 2^21); PF_PATH_FUSED_TOP -- top tree in K2's last CTA.
 * Lets parity tests assert they covered the benchmarked path. */
enum { PF_PATH_FUSED_DRAWS = 1, PF_PATH_RANK_TABLES = 2, PF_PATH_FUSED_TOP = 4 };
int pf_engine_last_path(pf_engine* e, int32_t* flags);
int pf_engine_destroy(pf_engine* e);

/* ----------------------------------------- sharded run (multi-GPU) --- */
/* One filter of cfg->n particles split into nshards (1, 2, 4, 8) shards of
 * n/nshards consecutive slots, shard s on devices[s] (NULL: all on device 0;
 * distinct devices need P2P access, e.g. NVLink / NVSwitch).  Same drop-in
 * boundary as pf_engine_run (filtering.py:200-374) and bit-identical to it
 * in ancestors and particles; the per-step exchange is one partial record
 * and one subtree total per shard, plus the cross-shard resampling reads.
 * Oracle feeds and store_particles are not supported. */
typedef struct pf_group pf_group;
int pf_group_create(const pf_config* cfg, int32_t nshards, const int32_t* devices, pf_group** out);
int pf_group_reconfigure(pf_group* g, const pf_config* cfg);
int pf_group_run(pf_group* g, const double* y, int64_t t_len, pf_outputs* out);
int pf_group_last_timing(pf_group* g, double* total_ms);
int pf_group_destroy(pf_group* g);

/* ------------------------- sharded run, one process per GPU (torchrun) --- */
/* The same sharded filter with one OS process per GPU: rank r of world
 * (1, 2, 4, 8) owns slots [r N/world, (r+1) N/world) on cfg->device.  The
 * caller owns the process group and drives, per step t = 1..T:
 *   pf_shard_phase(s, 1, t)   ancestors + step kernel -> partial record
 *   all-gather PF_XCHG_PARTIAL (in place, one slot per rank)
 *   pf_shard_phase(s, 2, t)   combine + local tree reduce -> subtree total
 *   all-gather PF_XCHG_TOTAL
 *   pf_shard_phase(s, 3, t)   top tree, cut table / q, quantile classification
 *   barrier (any collective)
 *   pf_shard_phase(s, 4, t)   rank 0: exact weighted-quantile resolve
 * then pf_shard_finish.  The collectives may run on pf_shard_stream (NCCL:
 * no host sync) or through host memory (pf_shard_exchange_host, gloo).
 * Data-dependent peer reads go through CUDA IPC: every rank exports
 * pf_shard_ipc_handle_bytes() of handles and opens all ranks' handles
 * (rank-major) once, after create.  Results are bit-identical to
 * pf_engine_run; rank 0's pf_outputs receive the summaries, every rank its
 * own slots of indices (T x N/world) and final particles.  Replaces the same
 * _run_loop (filtering.py:200-374) as pf_group_run. */
typedef struct pf_shard pf_shard;
enum { PF_XCHG_PARTIAL = 0, PF_XCHG_TOTAL = 1 };
int pf_shard_create(const pf_config* cfg, int32_t rank, int32_t world, pf_shard** out);
/* Same n, precision, device and tracked outputs (seed, priors may change). */
int pf_shard_reconfigure(pf_shard* s, const pf_config* cfg);
int32_t pf_shard_ipc_handle_bytes(void);
int pf_shard_ipc_handles(pf_shard* s, void* handles);
int pf_shard_open_peers(pf_shard* s, const void* all_handles);
/* Device pointer of an exchange array (world slots) and its slot size. */
int pf_shard_exchange(pf_shard* s, int32_t which, void** dptr, int64_t* slot_bytes);
/* to_host != 0: synchronise and copy this rank's slot to host; else copy
 * all world slots from host to the device array. */
int pf_shard_exchange_host(pf_shard* s, int32_t which, int32_t to_host, void* host);
int pf_shard_stream(pf_shard* s, void** stream);
int pf_shard_synchronize(pf_shard* s);
int pf_shard_begin(pf_shard* s, const double* y, int64_t t_len, pf_outputs* out);
int pf_shard_phase(pf_shard* s, int32_t phase, int64_t t);
int pf_shard_finish(pf_shard* s);
int pf_shard_last_timing(pf_shard* s, double* total_ms);
/* Unmap the peers' buffers.  Every rank should call it, then meet at a
 * barrier, before any rank destroys (frees what its peers mapped). */
int pf_shard_close_peers(pf_shard* s);
int pf_shard_destroy(pf_shard* s);

/* ------------------------------------------------- kernel level (L2) --- */
/* These kernel-level entries take HOST pointers and run synchronously on
 * the current device; they exist for parity tests and for the reference's
 * kernel-level API surface.  The *_d forms below take device pointers and
 * a stream. */

/* philox_block_lanes (rng.py:103-110): words_out is [4][n]. */
int pf_philox_block(uint64_t seed, const uint64_t* stream_ids, int64_t n,
                    uint64_t block, uint64_t* words_out);
/* philox4x64_block (rng.py:49-63) with arbitrary counters: counters is
 * [4][n] (c0..c3), keys [2][n] (k0, k1), words_out [4][n]. */
int pf_philox4x64(const uint64_t* counters, const uint64_t* keys, int64_t n, uint64_t* words_out);
/* uniforms_at (rng.py:122-140). */
int pf_uniforms_at(uint64_t seed, const uint64_t* stream_ids,
                   const uint64_t* counters, int64_t n, double* u_out);
/* scipy.special.ndtri as used at rng.py:223-224. */
int pf_ndtri(const double* u, int64_t n, double* out);
/* The hot-path normal draw: the piecewise u-space table of ndtri that the
 * draws kernel evaluates (replaces the same ndtri call, rng.py:223-224). */
int pf_ndtri_table(const double* u, int64_t n, double* out);
/* scipy.special.gammaincinv(a, u) as used at rng.py:226-229.  method 0 uses
 * the per-step table (hot path), 1 the accurate Halley solver. */
int pf_gammaincinv(double a, const double* u, int64_t n, int32_t method, double* out);
/* parallel_cdf (prefix_sum.py:109-127): w -> q, dtype PF_DTYPE_F64/F32.
 * total_out (optional) receives the adder-tree root. */
int pf_tree_cdf(const void* w, int64_t n, int32_t dtype, void* q_out, double* total_out);
/* forward_adder + backward_adder (prefix_sum.py:46-91): levels_out holds the
 * 2n-1 tree nodes level by level (level 0 first), prefix_out the inclusive
 * prefix sums. */
int pf_adder_tree(const void* w, int64_t n, int32_t dtype, void* levels_out, void* prefix_out);
/* cut_points_parallel (resampling.py:110-134): 1-based cut table. */
int pf_cut_table(const void* q, int64_t n, int32_t dtype, int64_t* cuts_out);
/* cutpoint_indices (resampling.py:146-158) over m uniforms. */
int pf_cutpoint_lookup(const void* q, const int64_t* cuts, int64_t n, int32_t dtype,
                       const double* u, int64_t m, int64_t* idx_out);
/* merge_indices (resampling.py:29-36): searchsorted(q, u, 'right') + 1 for m
 * uniforms (u >= 0), the search of the reference's naive / sorted /
 * stratified / systematic resamplers; sort_first sorts u ascending first
 * (resample_sorted, resampling.py:57-67). */
int pf_merge_indices(const void* q, int64_t n, int32_t dtype, const double* u, int64_t m,
                     int32_t sort_first, int64_t* idx_out);
/* resample_cutpoint (resampling.py:161-177): uniforms of streams 0..n-1 at
 * `counter`, cut table, lookup. */
int pf_resample_cutpoint(const void* q, int64_t n, int32_t dtype, uint64_t seed,
                         uint64_t counter, int64_t* idx_out);
/* weighted_quantiles (filtering.py:135-140); weights dtype PF_DTYPE_F64/F32. */
int pf_weighted_quantiles(const double* values, const void* weights, int32_t wdtype,
                          int64_t n, const double* probs, int32_t nprobs, double* out);

/* ------------------- kernel level, device pointers + stream (L2d) --- */
/* The same operations on DEVICE-resident buffers (every pointer argument is
 * device memory on the current device), enqueued on `stream` (a
 * cudaStream_t; NULL = the legacy default stream) and returning without a
 * host synchronisation.  Scratch comes from the stream's memory pool
 * (cudaMallocAsync) and is returned stream-ordered.  Size and dtype checks
 * return an error code as above; data-dependent conditions cannot (nothing
 * is read back), so each entry documents where they show up instead.
 * Results are bit-identical to the host-pointer forms on the same inputs. */

/* uniforms_at (rng.py:122-140). */
int pf_uniforms_at_d(uint64_t seed, const uint64_t* stream_ids, const uint64_t* counters,
                     int64_t n, double* u_out, void* stream);
/* parallel_cdf (prefix_sum.py:109-127).  total_out (device f64, optional)
 * receives the adder-tree root: the caller's all-zero / non-finite check
 * (prefix_sum.py:94-106 raises there) is `!(total > 0) || !isfinite(total)`. */
int pf_tree_cdf_d(const void* w, int64_t n, int32_t dtype, void* q_out, double* total_out,
                  void* stream);
/* cut_points_parallel (resampling.py:110-134): 1-based cut table. */
int pf_cut_table_d(const void* q, int64_t n, int32_t dtype, int64_t* cuts_out, void* stream);
/* cutpoint_indices (resampling.py:146-158) over m device uniforms. */
int pf_cutpoint_lookup_d(const void* q, const int64_t* cuts, int64_t n, int32_t dtype,
                         const double* u, int64_t m, int64_t* idx_out, void* stream);
/* resample_cutpoint (resampling.py:161-177), as pf_resample_cutpoint. */
int pf_resample_cutpoint_d(const void* q, int64_t n, int32_t dtype, uint64_t seed,
                           uint64_t counter, int64_t* idx_out, void* stream);
/* weighted_quantiles (filtering.py:135-140); probs and out are device
 * arrays of nprobs doubles. */
int pf_weighted_quantiles_d(const double* values, const void* weights, int32_t wdtype,
                            int64_t n, const double* probs, int32_t nprobs, double* out,
                            void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PARSMC_B200_H */
