/* turnstile_b200.h - C ABI of the B200-native iterative NUTS engine.
 *
 * The reference (turnstile, pure Python + numba) has no native boundary: its
 * hot path is the Python call chain
 *   chains.run -> run_chain -> nuts_transition_from -> build_tree_iterative
 *   -> integrator.leapfrog -> model.potential / model.gradient -> kernels.*
 * Each entry point below replaces one link of that chain; the Python package
 * paper_1912_11554_b200 binds them with ctypes (INTEGRATION.md shows the
 * binding) and keeps the reference's Python API on top.
 *
 * Conventions:
 *  - every pointer argument named *_dev is device memory owned by the caller
 *    (torch tensors); the library owns only ts_model handles and transient
 *    workspaces;
 *  - return 0 on success; TS_EINVAL for contract violations (the Python layer
 *    raises ValueError, as the reference does), TS_ECUDA / TS_EUNSUPPORTED
 *    otherwise (RuntimeError); ts_last_error() describes the last failure of
 *    the calling thread;
 *  - numerical events are data, never errors: +inf energies, divergence
 *    flags and -inf log weights are returned in the outputs;
 *  - calls are ordered on the given CUDA stream (NULL = legacy stream).
 */
#ifndef TURNSTILE_B200_H
#define TURNSTILE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_ABI_VERSION 1

enum { TS_OK = 0, TS_EINVAL = 1, TS_ECUDA = 2, TS_EUNSUPPORTED = 3 };

/* Model kinds.  Reference constructors: models.py:67-144 (std_normal,
 * gaussian, logistic_regression, funnel); eight_schools is the SURVEY 8(d)
 * config-3 model (no reference built-in; oracle twin in oracle/). */
enum { TS_STD_NORMAL = 0, TS_GAUSSIAN = 1, TS_LOGISTIC = 2, TS_FUNNEL = 3, TS_EIGHT_SCHOOLS = 4, TS_DENSE_GAUSS = 5 };

/* Arithmetic policy of the logistic data pass (ts_logistic.cuh) and of the
 * dense-Gaussian GEMM (FP64: SIMT fp64; FP32/TF32: tcgen05 TF32 tensor cores).
 * Logistic: FP64 / FP32 stream X stored as fp32 (x_dev float); FP64X streams X
 * stored as fp64 (x_dev double: data that are not fp32-exact, as the
 * reference's LogisticRegressionData keeps them, models.py:43-64); TF32 =
 * many chains sharing X on the tensor cores (ts_k_logistic_many.cu). */
enum { TS_PREC_FP64 = 0, TS_PREC_FP32 = 1, TS_PREC_TF32 = 2, TS_PREC_FP64X = 3 };

/* U-turn criterion (tree.py:36-37). */
enum { TS_GENERALIZED = 0, TS_CLASSIC = 1 };

/* Team layout for small models: one chain per thread (default; the
 * reference's summation order, bit for bit), per CTA, or per warp (vectors in
 * shared memory, shuffle-tree reductions: fastest for many small chains). */
typedef enum { TS_EXEC_THREAD = 0, TS_EXEC_BLOCK = 1, TS_EXEC_WARP = 2 } ts_exec_mode;

/* SamplerConfig (sampler.py:38-59). */
typedef struct {
  double step_size;
  int32_t max_tree_depth;
  int32_t criterion;
  double divergence_threshold;
} ts_sampler_cfg;

/* RunConfig (chains.py:36-57) minus model/mode/seed, which the host resolves. */
typedef struct {
  int32_t num_warmup;
  int32_t num_samples;
  double target_accept;
  int32_t has_sampler; /* RunConfig.sampler is not None (chains.py:137-143) */
  int32_t keep_warmup; /* 1: samples holds [C][W+S][dim], the warmup draws first (adaptation audits) */
  ts_sampler_cfg sampler;
} ts_run_cfg;

typedef struct ts_model ts_model;

const char* ts_last_error(void);
int ts_abi_version(void);

/* Replaces models.py:67-144 + LogisticRegressionData (models.py:43-64): builds
 * a device model.  params (host): gaussian inv_var[dim]; eight_schools
 * y[J], sigma[J] (dim = J + 2); dense_gauss A[dim][dim] (U = x'Ax/2, the
 * SURVEY 8(d) config-4 target after the dense-mass reparametrisation x =
 * L^-1 q; dim % 4 == 0 for TF32).  Logistic: x_dev row-major (n_rows x
 * n_feat), fp32 or - precision TS_PREC_FP64X - fp64, y_dev uint8 in {0,1};
 * the library re-tiles X into its own HBM layout. */
int ts_model_create(int kind, int dim, const double* params, int n_params, const void* x_dev, const uint8_t* y_dev,
                    int64_t n_rows, int n_feat, int precision, ts_model** out);
int ts_model_destroy(ts_model* m);
int ts_model_dim(const ts_model* m);
/* Sticky device error word of a model (synchronises the device): 0, or
 * TS_STATUS_SYNC_TIMEOUT once any wait of a persistent kernel on this model
 * (grid barrier, peer mailbox, served flag) exceeded TS_SPIN_TIMEOUT_S
 * seconds (default 30) - e.g. a row-shard peer that never launched.  The
 * kernel then gives up instead of hanging the GPU; the model is poisoned
 * (recreate it).  No reference counterpart (the reference is single-process). */
enum { TS_STATUS_SYNC_TIMEOUT = 2 };
int ts_model_error(const ts_model* m, int* code);
/* Cap the number of CTAs of the persistent logistic grid (0 = one per SM). */
int ts_model_set_grid(ts_model* m, int grid);

/* Replaces model.potential + model.gradient (models.py:110-118 ->
 * kernels.py:90-123): one fused pass per point.  q_dev [n][dim];
 * out_dev [n][1 + dim] = (U, gradient).  U is returned raw (may be inf/nan). */
int ts_potential_grad(const ts_model* m, const double* q_dev, int n_points, double* out_dev, void* stream);

/* Benchmark helper: `repeats` evaluations of the same point inside one
 * persistent launch (the per-leapfrog model cost of the device loop).
 * out_dev[6]: U, kernel-internal ns (globaltimer, CTA 0), then 4 uint64
 * CTA-0 cycle counters (prior, data pass, barrier, cross-CTA reduce). */
int ts_eval_bench(const ts_model* m, const double* q_dev, int repeats, double* out_dev, void* stream);

/* Replaces integrator.leapfrog (integrator.py:90-103).
 * z = [q dim | r dim | grad dim | U]; z_out same layout. */
int ts_leapfrog(const ts_model* m, const double* inv_dev, const double* z_in, double eps, double* z_out, int exec_mode,
                void* stream);

/* Replaces tree.build_tree_iterative (tree.py:344-453).  z_in as above; the
 * tree's uniforms come from the device Philox stream of key (== numpy's
 * RngKey(key).generator()).  tree_out [8*dim + 10]:
 *   left.q, left.r, right.q, right.r, right.grad, proposal.q, proposal.grad,
 *   momentum_sum, then lw, sum_metropolis, leapfrog_count, turning,
 *   diverging, proposal.U, proposal.H, proposal leaf index, left.U, right.U.
 * Optional trace (TreeTrace, tree.py:165-187): events int32[cap][5], leaf
 * log weights, counts int32[3] = (events, leaf weights, max occupied). */
int ts_build_tree(const ts_model* m, const ts_sampler_cfg* cfg, const double* inv_dev, const double* z_in, int depth,
                  double eps, double h_ref, uint64_t key_hi, uint64_t key_lo, double* tree_out, int32_t* trace_ev,
                  int trace_cap, double* leaf_lw, int lw_cap, int32_t* trace_counts, int exec_mode, void* stream);

/* Replaces sampler.nuts_transition_from (sampler.py:83-148).  z_in as above
 * (momentum ignored).  normals_or_null: injected standard normals for the
 * momentum refresh, else drawn on device from fold(key, 0) exactly as numpy
 * does.  out [2*dim + 8]: q, grad, U, depth, leapfrogs, diverged,
 * accept_stat, energy, proposal tree, proposal leaf. */
int ts_transition(const ts_model* m, const ts_sampler_cfg* cfg, const double* inv_dev, const double* z_in,
                  const double* normals_or_null, uint64_t key_hi, uint64_t key_lo, double* out, int32_t* trace_ev,
                  int trace_cap, int32_t* trace_counts, int exec_mode, void* stream);

/* Replaces sampler.hmc_transition (sampler.py:163-203): num_steps leapfrogs of
 * cfg->step_size, then Metropolis accept with fold(key, 1).random().  z_in as
 * for ts_transition.  out [2*dim + 7]: q, grad, U (the kept state), depth (0),
 * leapfrogs, diverged, accept_stat, energy, accepted. */
int ts_hmc_transition(const ts_model* m, const ts_sampler_cfg* cfg, const double* inv_dev, const double* z_in,
                      const double* normals_or_null, uint64_t key_hi, uint64_t key_lo, int num_steps, double* out,
                      int exec_mode, void* stream);

/* Replaces adapt.find_reasonable_step_size (adapt.py:172-204). out[1]. */
int ts_find_step_size(const ts_model* m, const double* inv_dev, const double* z_in, const double* normals_or_null,
                      uint64_t key_hi, uint64_t key_lo, double init, double* out, int exec_mode, void* stream);

/* Replaces chains.run_chain for every chain (chains.py:98-163, adapt.py:207-236):
 * warmup adaptation and sampling entirely on device, one launch.
 * chain_keys_dev [C][2] (hi, lo); inv0_dev [dim]; schedule_dev [W] (bit0 in a
 * covariance window, bit1 window end: WarmupSchedule.window_steps,
 * adapt.py:119-127); da_weight_dev [W] = t^-kappa.  Outputs: samples
 * [C][S][dim], stats [C][W+S][5] (depth, leapfrogs, diverged, accept_stat,
 * energy), adapt [C][2+W+dim] (initial step, final step, step trace,
 * inverse mass), status [C] (0 ok, 1 invalid mass install, TS_STATUS_SYNC_TIMEOUT:
 * an inter-CTA / inter-GPU wait exceeded TS_SPIN_TIMEOUT_S, see ts_model_error), evals [C] or NULL
 * (model evaluations = passes over the data, incl. step-size search). */
int ts_run_chains(const ts_model* m, const ts_run_cfg* rc, const uint64_t* chain_keys_dev, int n_chains,
                  const double* inv0_dev, const uint8_t* schedule_dev, const double* da_weight_dev, double* samples,
                  double* stats, double* adapt, int32_t* status, int64_t* evals, int exec_mode, void* stream);

/* Row sharding of one logistic model across GPUs (SURVEY.md 8(e), config 5:
 * the reference evaluates kernels.py:90-123 over all N rows in one process;
 * here rank g of `world` holds rows [g*N/world, (g+1)*N/world)).  Every rank
 * builds its model from its own row shard with ts_model_create, then
 *   ts_peer_mailbox_create(m, rank, world, handle_out)  writes the 64-byte
 *       CUDA IPC handle of this rank's exchange mailbox;
 *   the host all-gathers the handles (rank order), e.g. torch.distributed;
 *   ts_peer_mailbox_connect(m, handles)                  maps the peers.
 * From then on every launch on m (potential/gradient, trees, transitions,
 * runs) combines the per-pass partial sums of all ranks inside the
 * persistent kernel: after its grid barrier each GPU pushes its exact
 * fixed-point totals (p+2 values as int64 pairs) to every peer's mailbox
 * over NVLink and sums the `world` copies it receives.  Integer sums are
 * order-free, so every rank sees the same U and gradient -- bit-identical to
 * one GPU holding all rows -- and runs the identical (replicated) chain.  All
 * ranks must issue the same sequence of calls with the same arguments.
 * world == 1 connects the mailbox to itself (the same device code path). */
#define TS_MAX_PEERS 8
int ts_peer_mailbox_create(ts_model* m, int rank, int world, void* ipc_handle_out);
int ts_peer_mailbox_connect(ts_model* m, const void* ipc_handles);

/* Test helper for row sharding on one GPU: emulate `vranks` row-sharded ranks
 * inside one cooperative launch (equal groups of CTAs, each with its own rows,
 * grid barrier and accumulators, exchanging through in-memory mailboxes with
 * the same device code as ts_peer_mailbox_*).  1 = off. */
int ts_model_set_virtual_ranks(ts_model* m, int vranks);

/* Test helper for row sharding: the raw cross-CTA fixed-point totals of ONE
 * potential/gradient evaluation at q_dev over this model's rows (before any
 * peer exchange): words_dev[2*(p+2)+1] uint64 = (hi, lo) pairs for the p
 * feature sums, the residual sum and the log-likelihood sum, then the
 * out-of-range flag.  value = hi * 2^-10 + lo * 2^-63 (two's complement). */
int ts_logistic_partial_sums(const ts_model* m, const double* q_dev, uint64_t* words_dev, void* stream);

/* Test probe of the tcgen05 TF32 GEMM (csrc/ts_umma.cuh) behind the
 * dense-Gaussian model: gt[n][m] = sum_k a[m][k] * xt[n][k] with a (M x K)
 * and xt (N x K) row-major fp32 (K % 4 == 0), gt (N x M).  grid <= 0: one
 * CTA per 128 x 64 tile.  Replaces nothing in the reference. */
int ts_gemm_tf32_probe(const float* a_dev, const float* xt_dev, float* gt_dev, int M, int N, int K, int grid, void* stream);

/* Parity probe of the device randomness (csrc/ts_rng.cuh): kind 0 writes n
 * Generator.random() doubles of RngKey(key).generator(), kind 1 n
 * standard_normal() values, kind 2 the keys fold(0..n-1) as raw 64-bit
 * words [n][2].  Replaces nothing in the reference; used by tests. */
int ts_rng_probe(uint64_t key_hi, uint64_t key_lo, int kind, int n, double* out_dev, void* stream);

/* Test probe: y = exp(x) (kind 0), log1p(x) (1) or log(x) (2) as the device
 * engine evaluates them (csrc/ts_libm.cuh: glibc's exp and log1p bit for bit,
 * log correctly rounded), the functions the reference calls through math at
 * tree.py:131-156, 276, 410-416, sampler.py:127, adapt.py:44-57, 192. */
int ts_libm_probe(int kind, const double* x_dev, double* y_dev, int64_t n, void* stream);

/* Pooled sample covariance of n_rows draws (row-major n_rows x D fp64 in
 * device memory, e.g. the (C, S, D) samples of a many-chain warmup pooled
 * over chains): mean_dev[D] and cov_dev[D*D] with ddof = 1; regularize != 0
 * applies the shrinkage of welford_regularized_variance (adapt.py:91-94) to
 * the full matrix: n/(n+5) cov + 5/(n+5) 1e-3 I.  work_dev holds
 * ts_pooled_covariance_workspace(n_rows, D) doubles.  Deterministic (no atomics).
 * Extends adapt.py:73-108 (diagonal, per chain) to a dense mass pooled
 * across chains - no reference entry point is replaced. */
int ts_pooled_covariance(const double* x_dev, int64_t n_rows, int D, int regularize, double* mean_dev,
                         double* cov_dev, double* work_dev, void* stream);
int64_t ts_pooled_covariance_workspace(int64_t n_rows, int D);

/* Dense-mass reparametrisation: the run
 * samples x = L^-1 q (M^-1 = L L^T); this maps every draw back,
 * q_dev[r] = L x_dev[r] for r < rows (row-major [rows][dim], L lower
 * triangular [dim][dim], fp64, not in place).  Replaces the reference's
 * nothing (its mass is diagonal, integrator.py:21-31). */
int ts_dense_transform(const double* l_dev, const double* x_dev, double* q_dev, int64_t rows, int dim, void* stream);

/* Replaces diagnostics.ess (diagnostics.py:49-86) and diagnostics.split_rhat
 * (diagnostics.py:89-105) for samples already in device memory: samples_dev
 * (n_chains, n_draws, dim) fp64 C-contiguous -> ess_dev[dim], rhat_dev[dim]
 * (NaN for a constant dimension, as the reference).  Split-chain estimator,
 * autocovariance by direct lag sums in blocks of 64 lags until Geyer's
 * truncation (csrc/ts_k_diagnostics.cu); deterministic; agrees with the host
 * estimator to rounding.  work_dev holds ts_chain_diagnostics_workspace()
 * doubles.  Synchronises `stream` once per lag block (reads one flag). */
int ts_chain_diagnostics(const double* samples_dev, int n_chains, int n_draws, int dim, double* ess_dev,
                         double* rhat_dev, double* work_dev, void* stream);
int64_t ts_chain_diagnostics_workspace(int n_chains, int n_draws, int dim);

#ifdef __cplusplus
}
#endif
#endif
