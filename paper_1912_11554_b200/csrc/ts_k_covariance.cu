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
//   k_cov_tile       : one CTA per (64x64 lower-triangular output tile, row
//                      split); rows streamed in 16-row slabs through shared
//                      memory (next slab prefetched into registers), centred
//                      on load; 4x4 fp64 register micro-tile per thread with
//                      explicit __fma_rn -> one partial tile per split
//   k_cov_finish     : fixed-order sum over splits, scaling, mirror store.
// Splits give ~6 resident CTAs per SM whatever D is.
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

__device__ __forceinline__ void tri_index(int t, int& ti, int& tj) {
  ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  while (ti * (ti + 1) / 2 > t) --ti;
  tj = t - ti * (ti + 1) / 2;
}

// blockIdx.x: lower-triangular tile, blockIdx.y: row split.  Writes the
// split's raw centred cross-product tile to part[split][tile][64*64].
__global__ void __launch_bounds__(256, 3) k_cov_tile(const double* __restrict__ x, const double* __restrict__ mean,
                                                  int64_t n, int D, int64_t rows_per_split,
                                                  double* __restrict__ part) {
  int ti, tj;
  tri_index(blockIdx.x, ti, tj);
  const int i0 = ti * kTile, j0 = tj * kTile;
  const int64_t rbeg = (int64_t)blockIdx.y * rows_per_split;
  const int64_t rend = rbeg + rows_per_split < n ? rbeg + rows_per_split : n;

  __shared__ double As[kSlab][kTile];
  __shared__ double Bs[kSlab][kTile];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 outputs each
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

  // loader: 256 threads x 4 elements = one 16 x 64 slab per operand; the
  // next slab is fetched into registers while the current one is consumed
  const int lc = threadIdx.x & 63, lr = threadIdx.x >> 6;
  const bool ci = i0 + lc < D, cj = j0 + lc < D;
  const double mi = ci ? mean[i0 + lc] : 0.0;
  const double mj = cj ? mean[j0 + lc] : 0.0;
  double ra[4], rb[4];
  auto fetch = [&](int64_t r0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t r = r0 + lr + 4 * k;
      const bool rin = r < rend;
      ra[k] = (rin && ci) ? x[r * D + i0 + lc] - mi : 0.0;
      rb[k] = (rin && cj) ? x[r * D + j0 + lc] - mj : 0.0;
    }
  };
  if (rbeg < rend) fetch(rbeg);
  for (int64_t r0 = rbeg; r0 < rend; r0 += kSlab) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      As[lr + 4 * k][lc] = ra[k];
      Bs[lr + 4 * k][lc] = rb[k];
    }
    __syncthreads();
    if (r0 + kSlab < rend) fetch(r0 + kSlab);
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
  double* out = part + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (kTile * kTile);
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) out[(ty + 16 * a) * kTile + tx + 16 * b] = acc[a][b];
}

// Fixed-order sum over splits, ddof-1 scaling, optional shrinkage, mirror.
__global__ void k_cov_finish(const double* __restrict__ part, int tiles, int splits, int64_t n, int D,
                             int regularize, double* __restrict__ cov) {
  int ti, tj;
  tri_index(blockIdx.x, ti, tj);
  const double inv = 1.0 / (double)(n - 1);
  const double shrink = regularize ? (double)n / ((double)n + 5.0) : 1.0;
  const double ridge = regularize ? 1e-3 * (5.0 / ((double)n + 5.0)) : 0.0;
  for (int e = threadIdx.x; e < kTile * kTile; e += blockDim.x) {
    const int i = ti * kTile + e / kTile, j = tj * kTile + e % kTile;
    if (i >= D || j >= D || j > i) continue;
    double s = 0.0;
    for (int sp = 0; sp < splits; ++sp) s += part[((int64_t)sp * tiles + blockIdx.x) * (kTile * kTile) + e];
    double v = s * inv * shrink;
    if (i == j) v += ridge;
    cov[(int64_t)i * D + j] = v;
    cov[(int64_t)j * D + i] = v;
  }
}

int cov_splits(int64_t n, int D) {
  const int nt = (D + kTile - 1) / kTile;
  const int tiles = nt * (nt + 1) / 2;
  int64_t s = (6 * 148 + tiles - 1) / tiles;           // ~6 resident CTAs per SM
  const int64_t max_s = (n + 8 * kSlab - 1) / (8 * kSlab);  // >= 8 slabs per split
  if (s > max_s) s = max_s;
  return s < 1 ? 1 : (int)s;
}

}  // namespace

extern "C" int ts_pooled_covariance(const double* x_dev, int64_t n_rows, int D, int regularize, double* mean_dev,
                                    double* cov_dev, double* work_dev, void* stream) {
  if (!x_dev || !mean_dev || !cov_dev || !work_dev || D < 1)
    return ts_internal::set_err(TS_EINVAL, "bad covariance arguments");
  if (n_rows < 2) return ts_internal::set_err(TS_EINVAL, "covariance needs at least two draws");
  cudaStream_t st = (cudaStream_t)stream;
  // workspace: [kChunks * D] column partial sums, then the split tiles
  double* part = work_dev + (int64_t)kChunks * D;
  k_colsum_partial<<<dim3((D + kColThreads - 1) / kColThreads, kChunks), kColThreads, 0, st>>>(x_dev, n_rows, D,
                                                                                               work_dev);
  TS_CUDA(cudaGetLastError());
  k_colmean<<<(D + 127) / 128, 128, 0, st>>>(work_dev, n_rows, D, mean_dev);
  TS_CUDA(cudaGetLastError());
  const int nt = (D + kTile - 1) / kTile;
  const int tiles = nt * (nt + 1) / 2;
  const int splits = cov_splits(n_rows, D);
  int64_t rps = (n_rows + splits - 1) / splits;
  rps = (rps + kSlab - 1) / kSlab * kSlab;
  k_cov_tile<<<dim3(tiles, splits), 256, 0, st>>>(x_dev, mean_dev, n_rows, D, rps, part);
  TS_CUDA(cudaGetLastError());
  k_cov_finish<<<tiles, 256, 0, st>>>(part, tiles, splits, n_rows, D, regularize, cov_dev);
  TS_CUDA(cudaGetLastError());
  return TS_OK;
}

extern "C" int64_t ts_pooled_covariance_workspace(int64_t n_rows, int D) {
  if (D < 1 || n_rows < 2) return 0;
  const int nt = (D + kTile - 1) / kTile;
  return (int64_t)kChunks * D + (int64_t)cov_splits(n_rows, D) * (nt * (nt + 1) / 2) * kTile * kTile;
}

// ---------------------------------------------------------------- dense mass: q = L x
// Samples of the reparametrised dense-mass run come back as q = L x
// (chains.run_device; L lower triangular, M^-1 = L L^T).  Q (rows x D) =
// X (rows x D) . L^T: 64 x 64 output tiles per CTA (256 threads, 4 x 4 each),
// k in chunks of 16 through shared memory, fp64 FMAs in k order; the upper
// triangle of L (zeros) is skipped by the k range of each column block.
namespace {
constexpr int kTB = 64, kTK = 16;
__global__ void __launch_bounds__(256) k_lower_transform(const double* __restrict__ L, const double* __restrict__ X,
                                                         double* __restrict__ Q, int64_t rows, int D) {
  __shared__ double xs[kTK][kTB + 1];  // [k][row]
  __shared__ double ls[kTK][kTB + 1];  // [k][col]
  const int64_t r0 = (int64_t)blockIdx.x * kTB;
  const int c0 = blockIdx.y * kTB;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  // columns c0 .. c0+63 of Q need L[c][k] for k <= c < c0 + 64
  const int kend = (c0 + kTB < D) ? c0 + kTB : D;
  for (int k0 = 0; k0 < kend; k0 += kTK) {
    for (int i = threadIdx.x; i < kTK * kTB; i += 256) {
      const int kk = i % kTK, rr = i / kTK;
      const int64_t row = r0 + rr;
      const int k = k0 + kk;
      xs[kk][rr] = (row < rows && k < D) ? X[row * D + k] : 0.0;
      const int col = c0 + rr;
      ls[kk][rr] = (col < D && k < D && k <= col) ? L[(int64_t)col * D + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = xs[kk][ty * 4 + i]; b[i] = ls[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = r0 + ty * 4 + i;
    if (row >= rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = c0 + tx * 4 + j;
      if (col < D) Q[row * D + col] = acc[i][j];
    }
  }
}
}  // namespace

extern "C" int ts_dense_transform(const double* l_dev, const double* x_dev, double* q_dev, int64_t rows, int dim,
                                  void* stream) {
  using ts_internal::set_err;
  if (!l_dev || !x_dev || !q_dev || rows < 0 || dim < 1) return set_err(TS_EINVAL, "bad dense transform arguments");
  if (x_dev == q_dev) return set_err(TS_EINVAL, "dense transform cannot run in place");
  if (rows == 0) return TS_OK;
  const dim3 grid((unsigned)((rows + kTB - 1) / kTB), (unsigned)((dim + kTB - 1) / kTB));
  k_lower_transform<<<grid, 256, 0, (cudaStream_t)stream>>>(l_dev, x_dev, q_dev, rows, dim);
  TS_CUDA(cudaGetLastError());
  return TS_OK;
}
