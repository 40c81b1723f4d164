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
// into 32-row tiles of 128*p contiguous bytes; inside a tile, feature group g
// (4 features; the last group holds p % 4) stores lane r's features
// contiguously, so a lane reads its row with LDS.128s and a warp's reads are
// bank-conflict free.  y is a separate uint8 array, 32 bytes per tile.
//
// Memory pipeline: each warp owns a ring of NSTAGE shared-memory stages fed
// by TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx) issued by lane
// 0; the warp's tiles form a periodic sequence (the same tiles every pass,
// since X never changes), so the producer stays NSTAGE tiles ahead ACROSS
// passes: the first tiles of pass k+1 are in flight while the grid barrier,
// the cross-CTA reduction and the tree logic of pass k run.
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

struct WarpPipe {
  unsigned long long issued;    // tiles issued into the ring (periodic sequence index)
  unsigned long long consumed;  // tiles consumed
};

struct LogisticArgs {
  const float* xt;          // tiled X, ntiles * 32 * p floats
  const uint8_t* yt;        // labels, ntiles * 32 (padding rows 0)
  int64_t n_rows;
  int p;
  int64_t ntiles;
  double* pbuf;             // [2][grid][p+2] partial sums
  unsigned long long* bar;  // grid barrier counter (zeroed before launch)
  int fp64;                 // precision policy
  int pmax;                 // compile-time feature capacity of the pass (8/32/56/64)
  // shared-memory pipeline of this CTA (set by the kernel)
  unsigned char* stages;    // [nwarps][nstage][stage_bytes]
  uint64_t* mbar;           // [nwarps][nstage]
  WarpPipe* pipe;           // [nwarps]
  int nstage;
  int stage_bytes;
  int l2_keep_tiles;        // tiles [0, l2_keep_tiles) loaded with L2::evict_last, rest evict_first
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA 1-D bulk copy global -> shared, completion signalled on `bar`, with an L2 cache hint.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
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

// ------------------------------------------------------------- tile pipeline
struct WarpTiles {
  int64_t first;  // first tile of this warp
  int64_t count;  // number of tiles (stride nwarps)
  int nwarps;
};

__device__ __forceinline__ WarpTiles warp_tiles(const LogisticArgs& a) {
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int64_t G = gridDim.x;
  const int64_t t_begin = (a.ntiles * (int64_t)blockIdx.x) / G;
  const int64_t t_end = (a.ntiles * ((int64_t)blockIdx.x + 1)) / G;
  WarpTiles w;
  w.first = t_begin + warp;
  w.count = (t_end - w.first + nwarps - 1) / nwarps;
  if (w.count < 0) w.count = 0;
  w.nwarps = nwarps;
  return w;
}

// lane 0: issue periodic-sequence tile `seq` of this warp into its stage
__device__ __forceinline__ void issue_tile(const LogisticArgs& a, const WarpTiles& wt, unsigned long long seq) {
  const int warp = threadIdx.x >> 5;
  const int s = (int)(seq % (unsigned long long)a.nstage);
  const int64_t tile = wt.first + (int64_t)(seq % (unsigned long long)wt.count) * wt.nwarps;
  unsigned char* dst = a.stages + ((int64_t)warp * a.nstage + s) * a.stage_bytes;
  uint64_t* bar = a.mbar + warp * a.nstage + s;
  const uint32_t xb = 128u * (uint32_t)a.p;
  const uint64_t pol = tile < a.l2_keep_tiles ? policy_evict_last() : policy_evict_first();
  mbar_expect_tx(bar, xb + 32u);
  bulk_g2s(dst, a.xt + tile * 32 * (int64_t)a.p, xb, bar, pol);
  bulk_g2s(dst + xb, a.yt + tile * 32, 32u, bar, pol);
}

// Kernel prologue (all threads of the CTA): mbarriers and pipe counters.
static __device__ void logistic_pipeline_init(const LogisticArgs& a) {
  const int nwarps = blockDim.x >> 5;
  for (int i = threadIdx.x; i < nwarps * a.nstage; i += blockDim.x) mbar_init(a.mbar + i, 1);
  for (int i = threadIdx.x; i < nwarps; i += blockDim.x) { a.pipe[i].issued = 0; a.pipe[i].consumed = 0; }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
}

// Kernel epilogue: wait for the tiles the producer prefetched for a pass that
// never came, so no bulk copy targets the shared memory of an exited CTA.
static __device__ void logistic_pipeline_drain(const LogisticArgs& a) {
  const int warp = threadIdx.x >> 5;
  const WarpTiles wt = warp_tiles(a);
  if (wt.count > 0) {
    const unsigned long long c = a.pipe[warp].consumed, iss = a.pipe[warp].issued;
    for (unsigned long long seq = c; seq < iss; ++seq)
      mbar_wait(a.mbar + warp * a.nstage + (int)(seq % a.nstage), (uint32_t)((seq / a.nstage) & 1ULL));
  }
  __syncthreads();
}

// Lane's row of a tile in shared memory -> x[0..PMAX) (zeros past p), y.
template <int PMAX>
__device__ __forceinline__ void row_from_stage(const unsigned char* sb, int p, int lane, float (&x)[PMAX], uint8_t& y) {
  const float* f = reinterpret_cast<const float*>(sb);
#pragma unroll
  for (int g = 0; g < PMAX / 4; ++g) {
    if (4 * g + 4 <= p) {
      const float4 v = reinterpret_cast<const float4*>(f + 128 * g)[lane];
      x[4 * g] = v.x; x[4 * g + 1] = v.y; x[4 * g + 2] = v.z; x[4 * g + 3] = v.w;
    } else if (4 * g < p) {
      const int w = p - 4 * g;
      const float* tb = f + 128 * g + lane * w;
      if (w == 2) {
        const float2 v = *reinterpret_cast<const float2*>(tb);
        x[4 * g] = v.x; x[4 * g + 1] = v.y;
      } else {
        x[4 * g] = tb[0];
        x[4 * g + 1] = (w > 1) ? tb[1] : 0.f;
      }
      x[4 * g + 2] = (w > 2) ? tb[2] : 0.f;
      x[4 * g + 3] = 0.f;
    } else {
      x[4 * g] = 0.f; x[4 * g + 1] = 0.f; x[4 * g + 2] = 0.f; x[4 * g + 3] = 0.f;
    }
  }
  y = sb[128 * p + lane];
}

// Per-CTA streaming pass.  Writes this CTA's partial sums
// red_out[0..p) = sum resid*x_j, red_out[p] = sum resid, red_out[p+1] = sum (y eta - log1pexp)
// (wred: >= nwarps*(PMAX+2) doubles of scratch).
template <int PMAX, bool FP64>
__device__ __noinline__ void logistic_cta_pass(const LogisticArgs& a, const double* __restrict__ theta_s, double* wred,
                                               double* red_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int p = a.p;
  constexpr int NA = PMAX + 2;
  const WarpTiles wt = warp_tiles(a);

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

  if (wt.count > 0) {
    WarpPipe& pipe = a.pipe[warp];
    const unsigned long long c0 = pipe.consumed;
    unsigned long long issued = pipe.issued;
    if (lane == 0) {
      while (issued < c0 + (unsigned long long)a.nstage) issue_tile(a, wt, issued++);
    }
    for (int64_t j = 0; j < wt.count; ++j) {
      const unsigned long long seq = c0 + (unsigned long long)j;
      const int s = (int)(seq % (unsigned long long)a.nstage);
      mbar_wait(a.mbar + warp * a.nstage + s, (uint32_t)((seq / a.nstage) & 1ULL));
      const unsigned char* sb = a.stages + ((int64_t)warp * a.nstage + s) * a.stage_bytes;
      float x[PMAX];
      uint8_t yb;
      row_from_stage<PMAX>(sb, p, lane, x, yb);
      __syncwarp();
      // stage s is free again: keep the producer NSTAGE tiles ahead (wrapping
      // into the next pass; X is read-only for the whole kernel)
      if (lane == 0) issue_tile(a, wt, issued++);
      const int64_t row = (wt.first + (int64_t)(seq % (unsigned long long)wt.count) * wt.nwarps) * 32 + lane;
      const bool valid = row < a.n_rows;
      if constexpr (FP64) {
        double e0 = theta_s[p], e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll
        for (int k = 0; k < PMAX; k += 4) {
          e0 = __fma_rn((double)x[k], (k < p) ? theta_s[k] : 0.0, e0);
          e1 = __fma_rn((double)x[k + 1], (k + 1 < p) ? theta_s[k + 1] : 0.0, e1);
          e2 = __fma_rn((double)x[k + 2], (k + 2 < p) ? theta_s[k + 2] : 0.0, e2);
          e3 = __fma_rn((double)x[k + 3], (k + 3 < p) ? theta_s[k + 3] : 0.0, e3);
        }
        const double eta = (e0 + e1) + (e2 + e3);
        const double e = exp(-fabs(eta));
        const double l = fmax(eta, 0.0) + log1p(e);
        const double sig = __ddiv_rn(eta >= 0.0 ? 1.0 : e, 1.0 + e);
        const double yv = (double)yb;
        const double resid = valid ? yv - sig : 0.0;
        accl += valid ? (yv * eta - l) : 0.0;
#pragma unroll
        for (int k = 0; k < PMAX; ++k) acc[k] = __fma_rn(resid, (double)x[k], acc[k]);
        acc[PMAX] += resid;
      } else {
        float e0 = thb32, e1 = 0.f, e2 = 0.f, e3 = 0.f;
#pragma unroll
        for (int k = 0; k < PMAX; k += 4) {
          e0 = __fmaf_rn(x[k], th32[k], e0);
          e1 = __fmaf_rn(x[k + 1], th32[k + 1], e1);
          e2 = __fmaf_rn(x[k + 2], th32[k + 2], e2);
          e3 = __fmaf_rn(x[k + 3], th32[k + 3], e3);
        }
        const float eta = (e0 + e1) + (e2 + e3);
        const float e = expf(-fabsf(eta));
        const float l = fmaxf(eta, 0.f) + log1pf(e);
        const float sig = __fdiv_rn(eta >= 0.f ? 1.f : e, 1.f + e);
        const float yv = (float)yb;
        const float resid = valid ? yv - sig : 0.f;
        accl += valid ? __fmaf_rn(yv, eta, -l) : 0.f;
#pragma unroll
        for (int k = 0; k < PMAX; ++k) acc[k] = __fmaf_rn(resid, x[k], acc[k]);
        acc[PMAX] += resid;
      }
    }
    __syncwarp();
    if (lane == 0) { pipe.consumed = c0 + (unsigned long long)wt.count; pipe.issued = issued; }
    __syncwarp();
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

static __device__ __forceinline__ void logistic_cta_dispatch(const LogisticArgs& a, const double* theta, double* wred,
                                                             double* red_s) {
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

// Full logistic evaluation over the grid for the team's q (vector qid):
// returns U, writes the gradient to vector gid.  `epoch` counts grid
// barriers already passed by this kernel (identical in every CTA).
static __device__ double logistic_eval_grid(const BlockTeam& T, const LogisticArgs& a, const VecStore& S, int qid,
                                            int gid, double* wred, double* red_s, unsigned long long& epoch) {
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
