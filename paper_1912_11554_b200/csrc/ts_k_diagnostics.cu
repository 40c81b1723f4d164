// Split-chain ESS and split R-hat of draws already in HBM (SURVEY.md 8(f)
// item 1): the reference estimators diagnostics.py:49-86 (ess) and
// diagnostics.py:89-105 (split_rhat), for (C, S, D) fp64 samples of a
// many-chain run, without copying the samples to the host.
//
// Split sequences: chain c's first half (draws [0, n)) is sequence c, its
// second half (draws [n, 2n)) is sequence C + c, n = S / 2, m = 2C
// (_split_halves).  The reference's FFT autocovariance acov_s[k] =
// sum_t y_t y_{t+k} / n of the centred sequence y is evaluated directly,
// lag block by lag block; Geyer's monotone pairs only ever need the lags up
// to the first non-positive pair, so blocks of kLagBlock lags are computed
// until every dimension has truncated (typically one block).
//
//   k_diag_lags     grid (chain groups, dimension chunks): a CTA stages one
//                   chain's 2 x DB sequences in shared memory (coalesced
//                   row reads), centres them (fixed-order warp sums; the
//                   means go to HBM for the between-chain variance), then
//                   each thread forms 8 consecutive lags of one sequence
//                   with a register shift window (2 shared loads per 8
//                   FMAs); the two halves and the CTA's chains accumulate
//                   in a fixed order into part[group][d][k].
//   k_diag_finalize one thread per dimension: fixed-order sums over the
//                   groups; lag block 0 also gives W = mean chain variance
//                   and B/n = variance of the 2C sequence means (two-pass);
//                   rho_k = 1 - (W - A_k) / var_plus, Geyer pairs with the
//                   running minimum, then ESS = m n / tau (capped at m n,
//                   m n if tau <= 0) and R-hat = sqrt(var_plus / W).
// Deterministic (no atomics); summation order differs from numpy's FFT, so
// results agree with the host estimator to rounding (tests: <= 1e-10).
#include "ts_internal.cuh"

namespace {

constexpr int kLagBlock = 64;   // lags per block (even: Geyer pairs never straddle blocks)
constexpr int kLagsPerThread = 8;
constexpr int kDiagThreads = 256;
constexpr int kDiagSmemMax = 96 * 1024;

struct DiagState {  // per dimension, carried across lag blocks
  double w, var_plus, tau, prev;
  int done, nan;
};

// smem: seq[2][DB][n + kLagBlock + 8] (zero tail) | sums[2 * DB * kLagBlock]
__global__ void __launch_bounds__(kDiagThreads) k_diag_lags(const double* __restrict__ x, int C, int S, int D, int DB,
                                                          int k0, double* __restrict__ part,
                                                          double* __restrict__ means) {
  extern __shared__ double sm[];
  const int n = S / 2;
  const int ld = n + kLagBlock + 8;
  const int d0 = blockIdx.y * DB;
  const int db = D - d0 < DB ? D - d0 : DB;
  const int nseq = 2 * db;
  double* seq = sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = kDiagThreads / 32;
  // this thread's items: (sequence, 8-lag group); kLagBlock / 8 groups per sequence
  constexpr int kGroups = kLagBlock / kLagsPerThread;
  const int nitems = nseq * kGroups;
  constexpr int kMaxItems = 2;  // items per thread (nseq * kGroups <= 2 * 256)
  double acc[kMaxItems][kLagsPerThread];
#pragma unroll
  for (int i = 0; i < kMaxItems; ++i)
#pragma unroll
    for (int j = 0; j < kLagsPerThread; ++j) acc[i][j] = 0.0;

  for (int c = blockIdx.x; c < C; c += gridDim.x) {
    __syncthreads();
    // stage: row t of chain c holds D doubles; sequence (h, dd) = column d0 + dd of rows [h n, (h+1) n)
    const double* xc = x + (int64_t)c * S * D;
    for (int i = threadIdx.x; i < 2 * n * db; i += kDiagThreads) {
      const int t = i / db, dd = i - t * db;  // consecutive threads: consecutive columns of one row
      const int h = t >= n ? 1 : 0;
      seq[(h * db + dd) * ld + (t - h * n)] = xc[(int64_t)t * D + d0 + dd];
    }
    for (int i = threadIdx.x; i < nseq * (ld - n); i += kDiagThreads) {
      const int s = i / (ld - n);
      seq[s * ld + n + (i - s * (ld - n))] = 0.0;
    }
    __syncthreads();
    // centre each sequence (warp per sequence, fixed order)
    for (int s = warp; s < nseq; s += nwarps) {
      double* y = seq + s * ld;
      double a = 0.0;
      for (int t = lane; t < n; t += 32) a += y[t];
#pragma unroll
      for (int off = 16; off; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
      const double mu = a / (double)n;
      for (int t = lane; t < n; t += 32) y[t] = y[t] - mu;
      if (k0 == 0 && lane == 0) {
        const int h = s / db, dd = s - h * db;
        means[((int64_t)h * C + c) * D + d0 + dd] = mu;
      }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kMaxItems; ++it) {
      const int item = threadIdx.x + it * kDiagThreads;
      if (item >= nitems) continue;
      const int s = item / kGroups, kb = k0 + (item - s * kGroups) * kLagsPerThread;
      if (kb >= n) continue;
      const double* y = seq + s * ld;
      double w[kLagsPerThread];
#pragma unroll
      for (int j = 0; j < kLagsPerThread; ++j) w[j] = (kb + j < ld) ? y[kb + j] : 0.0;
      // y_t y_{t+k} for k = kb..kb+7; y is zero past n (lags past the end contribute nothing)
      double lacc[kLagsPerThread];
#pragma unroll
      for (int j = 0; j < kLagsPerThread; ++j) lacc[j] = 0.0;
      const int tmax = n - kb;  // t + kb < n
      for (int t = 0; t < tmax; ++t) {
        const double yt = y[t];
#pragma unroll
        for (int j = 0; j < kLagsPerThread; ++j) lacc[j] = __fma_rn(yt, w[j], lacc[j]);
#pragma unroll
        for (int j = 0; j < kLagsPerThread - 1; ++j) w[j] = w[j + 1];
        w[kLagsPerThread - 1] = y[t + kb + kLagsPerThread];
      }
#pragma unroll
      for (int j = 0; j < kLagsPerThread; ++j) acc[it][j] += lacc[j];
    }
  }
  // combine the two halves (sequence s and s + db) and write this group's partial sums
  __syncthreads();
  double* sums = sm + (size_t)nseq * ld;
#pragma unroll
  for (int it = 0; it < kMaxItems; ++it) {
    const int item = threadIdx.x + it * kDiagThreads;
    if (item >= nitems) continue;
    const int s = item / kGroups, g = item - s * kGroups;
#pragma unroll
    for (int j = 0; j < kLagsPerThread; ++j) sums[s * kLagBlock + g * kLagsPerThread + j] = acc[it][j];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < db * kLagBlock; i += kDiagThreads) {
    const int dd = i / kLagBlock, k = i - dd * kLagBlock;
    part[((int64_t)blockIdx.x * D + d0 + dd) * kLagBlock + k] = sums[dd * kLagBlock + k] + sums[(db + dd) * kLagBlock + k];
  }
}

// One thread per dimension.  flag[0] += dimensions still open after this block.
__global__ void k_diag_finalize(const double* __restrict__ part, int G, const double* __restrict__ means, int C, int S,
                                int D, int k0, DiagState* __restrict__ st, double* __restrict__ ess,
                                double* __restrict__ rhat, int* __restrict__ open) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= D) return;
  const int n = S / 2;
  const double m = 2.0 * C, nn = (double)n;
  DiagState s = st[d];
  if (k0 == 0) {
    // lag 0: W = mean over sequences of acov[0] * n / (n - 1)
    double a0 = 0.0;
    for (int g = 0; g < G; ++g) a0 += part[((int64_t)g * D + d) * kLagBlock];
    const double w = (a0 / nn) / m * nn / (nn - 1.0);
    // between-sequence variance of the 2C means (ddof = 1), two-pass
    double mu = 0.0;
    for (int i = 0; i < 2 * C; ++i) mu += means[(int64_t)i * D + d];
    mu /= m;
    double ss = 0.0;
    for (int i = 0; i < 2 * C; ++i) {
      const double e = means[(int64_t)i * D + d] - mu;
      ss = __fma_rn(e, e, ss);
    }
    const double b_over_n = ss / (m - 1.0);
    s.w = w;
    s.var_plus = w * (nn - 1.0) / nn + b_over_n;
    s.tau = 0.0;
    s.prev = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    s.done = 0;
    s.nan = !(s.var_plus > 0.0 && isfinite(s.var_plus));
    rhat[d] = (s.w > 0.0 && isfinite(s.w)) ? sqrt(s.var_plus / s.w) : __longlong_as_double(0x7ff8000000000000LL);
    if (s.nan) s.done = 1;
  }
  if (!s.done) {
    for (int k = k0; k < k0 + kLagBlock && k + 1 < n; k += 2) {
      // pair (k, k + 1): rho_k = 1 - (W - A_k) / var_plus, rho_0 = 1
      double ak = 0.0, ak1 = 0.0;
      for (int g = 0; g < G; ++g) {
        ak += part[((int64_t)g * D + d) * kLagBlock + (k - k0)];
        ak1 += part[((int64_t)g * D + d) * kLagBlock + (k + 1 - k0)];
      }
      ak = ak / nn / m;
      ak1 = ak1 / nn / m;
      const double r0 = (k == 0) ? 1.0 : 1.0 - (s.w - ak) / s.var_plus;
      const double r1 = 1.0 - (s.w - ak1) / s.var_plus;
      double pair = r0 + r1;
      if (pair <= 0.0) { s.done = 1; break; }
      pair = fmin(pair, s.prev);
      s.tau += 2.0 * pair;
      s.prev = pair;
    }
    if (!s.done && k0 + kLagBlock + 1 >= n) s.done = 1;  // no pair (2k, 2k+1) with 2k + 1 < n left
  }
  st[d] = s;
  if (s.done) {
    const double mnv = m * nn;
    if (s.nan) {
      ess[d] = __longlong_as_double(0x7ff8000000000000LL);
    } else {
      const double tau = s.tau - 1.0;
      ess[d] = tau <= 0.0 ? mnv : fmin(mnv / tau, mnv);
    }
  } else {
    atomicAdd(open, 1);
  }
}

struct DiagPlan {
  int DB, gy, gx;
  size_t smem;
};

DiagPlan plan(int C, int S, int D) {
  DiagPlan p;
  const int n = S / 2;
  const size_t per_seq = (size_t)(n + kLagBlock + 8) * sizeof(double);
  // sequences of one CTA: 2 * DB, items 2 * DB * kLagBlock / 8 <= 2 * 256
  int DB = (int)(kDiagSmemMax / (2 * per_seq + 2 * kLagBlock * sizeof(double)));
  if (DB > 32) DB = 32;
  if (DB > D) DB = D;
  if (DB > 0) {  // balance the dimension chunks (D = 10, DB <= 9: 5 + 5, not 9 + 1)
    const int chunks = (D + DB - 1) / DB;
    DB = (D + chunks - 1) / chunks;
  }
  p.DB = DB;
  p.gy = DB > 0 ? (D + DB - 1) / DB : 0;
  int gx = p.gy > 0 ? (2 * 148 + p.gy - 1) / p.gy : 0;
  if (gx > C) gx = C;
  if (gx < 1) gx = 1;
  p.gx = gx;
  p.smem = (size_t)2 * DB * per_seq + (size_t)2 * DB * kLagBlock * sizeof(double);
  return p;
}

}  // namespace

using namespace ts_internal;

extern "C" int64_t ts_chain_diagnostics_workspace(int n_chains, int n_draws, int dim) {
  if (n_chains < 1 || n_draws < 4 || dim < 1) return 0;
  const DiagPlan p = plan(n_chains, n_draws, dim);
  const int64_t part = (int64_t)p.gx * dim * kLagBlock;
  const int64_t means = 2 * (int64_t)n_chains * dim;
  const int64_t state = ((int64_t)dim * sizeof(DiagState) + 7) / 8;
  return part + means + state + 2;
}

extern "C" int ts_chain_diagnostics(const double* samples_dev, int n_chains, int n_draws, int dim, double* ess_dev,
                                    double* rhat_dev, double* work_dev, void* stream) {
  if (!samples_dev || !ess_dev || !rhat_dev || !work_dev) return set_err(TS_EINVAL, "null argument");
  if (n_chains < 1 || dim < 1) return set_err(TS_EINVAL, "need at least one chain and one dimension");
  if (n_draws / 2 < 2) return set_err(TS_EINVAL, "need at least 4 draws per chain to split");
  const DiagPlan p = plan(n_chains, n_draws, dim);
  if (p.DB < 1) return set_err(TS_EUNSUPPORTED, "draws per chain too many for the shared-memory staging (> ~5900)");
  cudaStream_t st = (cudaStream_t)stream;
  double* part = work_dev;
  double* means = part + (int64_t)p.gx * dim * kLagBlock;
  DiagState* state = reinterpret_cast<DiagState*>(means + 2 * (int64_t)n_chains * dim);
  int* open = reinterpret_cast<int*>(work_dev + ts_chain_diagnostics_workspace(n_chains, n_draws, dim) - 2);
  TS_CUDA(cudaFuncSetAttribute(k_diag_lags, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  const int n = n_draws / 2;
  for (int k0 = 0; k0 < n; k0 += kLagBlock) {
    k_diag_lags<<<dim3(p.gx, p.gy), kDiagThreads, p.smem, st>>>(samples_dev, n_chains, n_draws, dim, p.DB, k0, part,
                                                                 means);
    TS_CUDA(cudaGetLastError());
    TS_CUDA(cudaMemsetAsync(open, 0, sizeof(int), st));
    k_diag_finalize<<<(dim + 127) / 128, 128, 0, st>>>(part, p.gx, means, n_chains, n_draws, dim, k0, state, ess_dev,
                                                       rhat_dev, open);
    TS_CUDA(cudaGetLastError());
    int h_open = 0;
    TS_CUDA(cudaMemcpyAsync(&h_open, open, sizeof(int), cudaMemcpyDeviceToHost, st));
    TS_CUDA(cudaStreamSynchronize(st));
    if (h_open == 0) break;
  }
  return TS_OK;
}
