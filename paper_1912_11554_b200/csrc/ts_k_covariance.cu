// Pooled sample covariance of draws already in HBM: the dense-mass
// extension of the reference's Welford variance (adapt.py:73-108, diagonal
// and per-chain only), SURVEY.md 8(f) item 3.
//
// Input: rows x (n_rows x D, row-major fp64) -- e.g. the samples tensor
// (C, S, D) of a many-chain warmup run, pooled over chains.  Output: the
// column means and the D x D covariance with ddof = 1, optionally shrunk
// toward 1e-3 * I like welford_regularized_variance (adapt.py:91-94):
//   cov_reg = n/(n+5) * cov + 5/(n+5) * 1e-3 * I.
//
// Deterministic (fixed summation order, no atomics):
//   k_colsum_partial : grid (D/128, kChunks), each thread one column of one
//                      row chunk -> partial[chunk][D] (coalesced row reads)
//   k_colmean        : fixed-order sum over chunks -> mean[D]
//   k_cov_tile       : one CTA per 64x64 lower-triangular output tile; rows
//                      streamed in 16-row slabs through shared memory, centred
//                      on load; 4x4 fp64 register micro-tile per thread with
//                      explicit __fma_rn; the tile and its mirror are stored.
// Bound: the FP64 pipe (2 N D^2 / 2 flops for the triangle); the samples are
// L2-resident re-reads across tiles (N x D x 8 B in HBM once per tile row).

#include "ts_internal.cuh"

namespace {

constexpr int kColThreads = 128;
constexpr int kChunks = 64;
constexpr int kTile = 64;
constexpr int kSlab = 16;

__global__ void k_colsum_partial(const double* __restrict__ x, int64_t n, int D, double* __restrict__ partial) {
  const int d = blockIdx.x * kColThreads + threadIdx.x;
  if (d >= D) return;
  const int64_t per = (n + kChunks - 1) / kChunks;
  const int64_t r0 = (int64_t)blockIdx.y * per;
  const int64_t r1 = r0 + per < n ? r0 + per : n;
  double s = 0.0;
  for (int64_t r = r0; r < r1; ++r) s += x[r * D + d];
  partial[(int64_t)blockIdx.y * D + d] = s;
}

__global__ void k_colmean(const double* __restrict__ partial, int64_t n, int D, double* __restrict__ mean) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= D) return;
  double s = 0.0;
  for (int c = 0; c < kChunks; ++c) s += partial[(int64_t)c * D + d];
  mean[d] = s / (double)n;
}

__global__ void __launch_bounds__(256) k_cov_tile(const double* __restrict__ x, const double* __restrict__ mean,
                                                  int64_t n, int D, int regularize, double* __restrict__ cov) {
  // linear triangle index -> (ti, tj) with tj <= ti
  const int t = blockIdx.x;
  int ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  while (ti * (ti + 1) / 2 > t) --ti;
  const int tj = t - ti * (ti + 1) / 2;
  const int i0 = ti * kTile, j0 = tj * kTile;

  __shared__ double As[kSlab][kTile];
  __shared__ double Bs[kSlab][kTile];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 outputs each
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

  // loader: 256 threads x 4 elements = one 16 x 64 slab per operand
  const int lc = threadIdx.x & 63, lr = threadIdx.x >> 6;  // column, row 0..3 (+4 k)
  const double mi = (i0 + lc < D) ? mean[i0 + lc] : 0.0;
  const double mj = (j0 + lc < D) ? mean[j0 + lc] : 0.0;
  for (int64_t r0 = 0; r0 < n; r0 += kSlab) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int rr = lr + 4 * k;
      const int64_t r = r0 + rr;
      const bool rin = r < n;
      As[rr][lc] = (rin && i0 + lc < D) ? x[r * D + i0 + lc] - mi : 0.0;
      Bs[rr][lc] = (rin && j0 + lc < D) ? x[r * D + j0 + lc] - mj : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kSlab; ++k) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[k][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[k][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = __fma_rn(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
  const double inv = 1.0 / (double)(n - 1);
  const double shrink = regularize ? (double)n / ((double)n + 5.0) : 1.0;
  const double ridge = regularize ? 1e-3 * (5.0 / ((double)n + 5.0)) : 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = i0 + ty + 16 * a;
    if (i >= D) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = j0 + tx + 16 * b;
      if (j >= D || j > i) continue;
      double v = acc[a][b] * inv * shrink;
      if (i == j) v += ridge;
      cov[(int64_t)i * D + j] = v;
      cov[(int64_t)j * D + i] = v;
    }
  }
}

}  // namespace

extern "C" int ts_pooled_covariance(const double* x_dev, int64_t n_rows, int D, int regularize, double* mean_dev,
                                    double* cov_dev, double* work_dev, void* stream) {
  if (!x_dev || !mean_dev || !cov_dev || !work_dev || D < 1)
    return ts_internal::set_err(TS_EINVAL, "bad covariance arguments");
  if (n_rows < 2) return ts_internal::set_err(TS_EINVAL, "covariance needs at least two draws");
  cudaStream_t st = (cudaStream_t)stream;
  k_colsum_partial<<<dim3((D + kColThreads - 1) / kColThreads, kChunks), kColThreads, 0, st>>>(x_dev, n_rows, D,
                                                                                               work_dev);
  TS_CUDA(cudaGetLastError());
  k_colmean<<<(D + 127) / 128, 128, 0, st>>>(work_dev, n_rows, D, mean_dev);
  TS_CUDA(cudaGetLastError());
  const int nt = (D + kTile - 1) / kTile;
  k_cov_tile<<<nt * (nt + 1) / 2, 256, 0, st>>>(x_dev, mean_dev, n_rows, D, regularize, cov_dev);
  TS_CUDA(cudaGetLastError());
  return TS_OK;
}

extern "C" int64_t ts_pooled_covariance_workspace(int D) { return (int64_t)kChunks * (D > 0 ? D : 0); }
