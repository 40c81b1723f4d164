// Fused logistic-regression potential + gradient: ONE pass over X.
//
// Reference: turnstile/kernels.py:90-123 (numba) / :194-211 (numpy) computes
//   U(theta) = 0.5|theta|^2 - sum_i [ y_i eta_i - log1pexp(eta_i) ]
//   g_j      = theta_j - sum_i (y_i - sigma(eta_i)) x_ij ,  g_p = theta_p - sum_i (y_i - sigma(eta_i))
// with eta_i = theta_p + sum_j x_ij theta_j, streaming X twice (once per call,
// integrator.py:98-101).  Here every row's eta, residual, log-likelihood term
// and gradient contribution come from a single read of the row.
//
// HBM layout (built once by ts_model_create): X is re-tiled
// into 32-row tiles; inside a tile, feature group g (4 features; the last
// group holds p % 4) stores lane r's features contiguously, so each warp
// reads a group with one fully coalesced LDG.128 (LDG.64/32 for the tail).
// A warp owns whole tiles; lane r owns row 32*t + r.
//
// Precision policies:
//   FP64 - eta, transcendentals and accumulators in double (fp32 data is
//          exact in double).  Differs from the reference only by summation
//          order: the bit-exact parity mode.
//   FP32 - eta, log1pexp and sigma in float; per-lane float accumulation
//          over that lane's rows, then double across lanes, warps and CTAs.
//          Tolerance mode (<= 1e-5 relative, tests/test_gpu_parity.py).
//
// Cross-CTA reduction: each CTA writes its (p+2)-vector of partial sums to a
// parity-double-buffered slot, one grid barrier, then every CTA reduces all
// slots in the same fixed order, so every CTA holds the identical gradient
// and runs the (replicated) tree logic without a second barrier.
#pragma once
#include <stdint.h>
#include "ts_team.cuh"

namespace ts {

struct LogisticArgs {
  const float* xt;        // tiled X, ntiles * 32 * p floats
  const uint8_t* yt;      // labels, ntiles * 32 (padding rows 0)
  int64_t n_rows;
  int p;
  int64_t ntiles;
  double* pbuf;           // [2][grid][p+2] partial sums
  unsigned long long* bar;  // grid barrier counter (zeroed before launch)
  int fp64;               // precision policy
  int pmax;               // compile-time feature capacity of the pass (8/32/56/64)
};

__device__ __forceinline__ float4 ld_stream4(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ld_stream2(const float2* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream1(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

// Load lane's row of one tile into x[0..PMAX) (zeros past p).
template <int PMAX>
__device__ __forceinline__ void load_row(const float* __restrict__ tile, int p, int lane, float (&x)[PMAX]) {
#pragma unroll
  for (int g = 0; g < PMAX / 4; ++g) {
    if (4 * g + 4 <= p) {
      float4 v = ld_stream4(reinterpret_cast<const float4*>(tile + 128 * g) + lane);
      x[4 * g] = v.x; x[4 * g + 1] = v.y; x[4 * g + 2] = v.z; x[4 * g + 3] = v.w;
    } else if (4 * g < p) {
      const int w = p - 4 * g;
      const float* tb = tile + 128 * g + lane * w;
      if (w == 2) {
        float2 v = ld_stream2(reinterpret_cast<const float2*>(tb));
        x[4 * g] = v.x; x[4 * g + 1] = v.y;
      } else {
        x[4 * g] = ld_stream1(tb);
        x[4 * g + 1] = (w > 1) ? ld_stream1(tb + 1) : 0.f;
      }
      x[4 * g + 2] = (w > 2) ? ld_stream1(tb + 2) : 0.f;
      x[4 * g + 3] = 0.f;
    } else {
      x[4 * g] = 0.f; x[4 * g + 1] = 0.f; x[4 * g + 2] = 0.f; x[4 * g + 3] = 0.f;
    }
  }
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Grid barrier #epoch (0-based) over gridDim.x co-resident CTAs.
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned long long epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long target = (epoch + 1) * (unsigned long long)gridDim.x;
    red_release_add_u64(bar, 1ULL);
    while (ld_acquire_u64(bar) < target) {
    }
  }
  __syncthreads();
}

// Per-CTA streaming pass.  Writes this CTA's partial sums
// red_out[0..p) = sum resid*x_j, red_out[p] = sum resid, red_out[p+1] = sum (y eta - log1pexp)
// into smem `wred` (>= nwarps*(PMAX+2) doubles) and reduces them to red_out.
template <int PMAX, bool FP64>
__device__ __noinline__ void logistic_cta_pass(const LogisticArgs& a, const double* __restrict__ theta_s, double* wred, double* red_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int p = a.p;
  const int64_t G = gridDim.x;
  const int64_t t_begin = (a.ntiles * (int64_t)blockIdx.x) / G;
  const int64_t t_end = (a.ntiles * ((int64_t)blockIdx.x + 1)) / G;
  constexpr int NA = PMAX + 2;

  using acc_t = typename std::conditional<FP64, double, float>::type;
  acc_t acc[PMAX + 1];
  acc_t accl = 0;
#pragma unroll
  for (int j = 0; j <= PMAX; ++j) acc[j] = 0;

  float th32[PMAX];
  float thb32 = 0.f;
  if constexpr (!FP64) {
#pragma unroll
    for (int j = 0; j < PMAX; ++j) th32[j] = (j < p) ? (float)theta_s[j] : 0.f;
    thb32 = (float)theta_s[p];
  }

  for (int64_t t = t_begin + warp; t < t_end; t += nwarps) {
    const float* tile = a.xt + t * 32 * (int64_t)p;
    float x[PMAX];
    load_row<PMAX>(tile, p, lane, x);
    const int64_t row = t * 32 + lane;
    const bool valid = row < a.n_rows;
    const uint8_t yb = a.yt[row];
    if constexpr (FP64) {
      double e0 = theta_s[p], e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll
      for (int j = 0; j < PMAX; j += 4) {
        e0 = __fma_rn((double)x[j], (j < p) ? theta_s[j] : 0.0, e0);
        e1 = __fma_rn((double)x[j + 1], (j + 1 < p) ? theta_s[j + 1] : 0.0, e1);
        e2 = __fma_rn((double)x[j + 2], (j + 2 < p) ? theta_s[j + 2] : 0.0, e2);
        e3 = __fma_rn((double)x[j + 3], (j + 3 < p) ? theta_s[j + 3] : 0.0, e3);
      }
      const double eta = (e0 + e1) + (e2 + e3);
      const double e = exp(-fabs(eta));
      const double l = fmax(eta, 0.0) + log1p(e);
      const double sig = __ddiv_rn(eta >= 0.0 ? 1.0 : e, 1.0 + e);
      const double yv = (double)yb;
      const double resid = valid ? yv - sig : 0.0;
      accl += valid ? (yv * eta - l) : 0.0;
#pragma unroll
      for (int j = 0; j < PMAX; ++j) acc[j] = __fma_rn(resid, (double)x[j], acc[j]);
      acc[PMAX] += resid;
    } else {
      float e0 = thb32, e1 = 0.f, e2 = 0.f, e3 = 0.f;
#pragma unroll
      for (int j = 0; j < PMAX; j += 4) {
        e0 = __fmaf_rn(x[j], th32[j], e0);
        e1 = __fmaf_rn(x[j + 1], th32[j + 1], e1);
        e2 = __fmaf_rn(x[j + 2], th32[j + 2], e2);
        e3 = __fmaf_rn(x[j + 3], th32[j + 3], e3);
      }
      const float eta = (e0 + e1) + (e2 + e3);
      const float e = expf(-fabsf(eta));
      const float l = fmaxf(eta, 0.f) + log1pf(e);
      const float sig = __fdiv_rn(eta >= 0.f ? 1.f : e, 1.f + e);
      const float yv = (float)yb;
      const float resid = valid ? yv - sig : 0.f;
      accl += valid ? __fmaf_rn(yv, eta, -l) : 0.f;
#pragma unroll
      for (int j = 0; j < PMAX; ++j) acc[j] = __fmaf_rn(resid, x[j], acc[j]);
      acc[PMAX] += resid;
    }
  }

  // warp reduction in double, fixed shuffle tree
#pragma unroll
  for (int j = 0; j < NA; ++j) {
    double v = (j <= PMAX) ? (double)acc[j <= PMAX ? j : PMAX] : (double)accl;
    if (j < p || j >= PMAX) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) wred[warp * NA + j] = v;
    }
  }
  __syncthreads();
  // CTA reduction in warp order; output index: [0,p) features, p bias, p+1 loglik
  for (int d = threadIdx.x; d < p + 2; d += blockDim.x) {
    const int j = (d < p) ? d : (d == p ? PMAX : PMAX + 1);
    double s = 0.0;
    for (int w = 0; w < nwarps; ++w) s += wred[w * NA + j];
    red_out[d] = s;
  }
}

// Full logistic evaluation over the grid for the team's q (vector qid):
// returns U, writes the gradient to vector gid.  `epoch` counts grid
// barriers already passed by this kernel (identical in every CTA).
static __device__ __forceinline__ void logistic_cta_dispatch(const LogisticArgs& a, const double* theta, double* wred, double* red_s) {
  switch (a.pmax * 2 + (a.fp64 ? 1 : 0)) {
    case 16: logistic_cta_pass<8, false>(a, theta, wred, red_s); break;
    case 17: logistic_cta_pass<8, true>(a, theta, wred, red_s); break;
    case 64: logistic_cta_pass<32, false>(a, theta, wred, red_s); break;
    case 65: logistic_cta_pass<32, true>(a, theta, wred, red_s); break;
    case 112: logistic_cta_pass<56, false>(a, theta, wred, red_s); break;
    case 113: logistic_cta_pass<56, true>(a, theta, wred, red_s); break;
    case 128: logistic_cta_pass<64, false>(a, theta, wred, red_s); break;
    case 129: logistic_cta_pass<64, true>(a, theta, wred, red_s); break;
    default: break;
  }
}

static __device__ double logistic_eval_grid(const BlockTeam& T, const LogisticArgs& a, const VecStore& S, int qid, int gid,
                                     double* wred, double* red_s, unsigned long long& epoch) {
  const int p = a.p;
  const int P2 = p + 2;
  const int64_t G = gridDim.x;
  const double* theta = S.v(qid);  // smem, contiguous (dstride 1)
  // prior term 0.5 * |theta|^2 (kernels.py:92-95)
  double pr = 0.0;
  for (int d = threadIdx.x; d <= p; d += blockDim.x) pr += 0.5 * theta[d] * theta[d];
  pr = T.sum(pr);

  logistic_cta_dispatch(a, theta, wred, red_s);
  __syncthreads();
  double* slot = a.pbuf + ((epoch & 1ULL) * G + blockIdx.x) * P2;
  for (int d = threadIdx.x; d < P2; d += blockDim.x) slot[d] = red_s[d];
  if (G > 1) grid_barrier(a.bar, epoch);
  else __syncthreads();
  epoch += 1;

  // Every CTA reduces all partial slots in the same fixed order.
  const double* base = a.pbuf + (((epoch - 1) & 1ULL) * G) * P2;
  const int ngrp = ((int)blockDim.x / P2) > 1 ? (int)blockDim.x / P2 : 1;
  double* grp = wred;  // reuse: ngrp * P2 doubles
  for (int idx = threadIdx.x; idx < ngrp * P2; idx += blockDim.x) {
    const int gi = idx / P2, d0 = idx % P2;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t b = gi;
    for (; b + 3 * ngrp < G; b += 4 * ngrp) {
      s0 += __ldcg(base + b * P2 + d0);
      s1 += __ldcg(base + (b + ngrp) * P2 + d0);
      s2 += __ldcg(base + (b + 2 * ngrp) * P2 + d0);
      s3 += __ldcg(base + (b + 3 * ngrp) * P2 + d0);
    }
    for (; b < G; b += ngrp) s0 += __ldcg(base + b * P2 + d0);
    grp[gi * P2 + d0] = (s0 + s1) + (s2 + s3);
  }
  __syncthreads();
  double* g = S.v(gid);
  for (int d = threadIdx.x; d < P2; d += blockDim.x) {
    double s = 0.0;
    for (int gi = 0; gi < ngrp; ++gi) s += grp[gi * P2 + d];
    if (d <= p) g[d] = theta[d] - s;
    else red_s[0] = s;  // sum of log-likelihood terms
  }
  __syncthreads();
  const double U = pr - red_s[0];
  __syncthreads();
  return U;
}

}  // namespace ts
