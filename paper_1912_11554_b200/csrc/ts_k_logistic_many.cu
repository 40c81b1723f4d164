// Many chains of one logistic-regression model sharing X on the tcgen05
// tensor cores (BASELINE north star "many-chain batching": >= 64 chains
// sharing X form a dense contraction).  Reference: chains.run over
// num_chains independent run_chain calls (chains.py:98-191), each leapfrog
// evaluating kernels.logistic_potential/gradient (kernels.py:90-123) over
// all N rows.  Here one X stream per batched step serves every chain with an
// outstanding request:
//
//   eta[i][c]  = sum_k Xa[i][k] Th[c][k]          GEMM 1 (M = 128 rows, N = 64 chains)
//   r[i][c]    = y_i - sigma(eta),  ll[i][c] = y_i eta - log1pexp(eta)   (CUDA cores)
//   G[c][k]    = sum_i r[i][c] Xa[i][k]           GEMM 2 (M = 128, N = 64 features)
//
// Xa = [X | 1 | y] (N x KA fp32, KA = p + 2 rounded up to 8, row pitch 4 KA
// bytes): the ones column gives the bias in eta and the residual sum (bias
// gradient) in G; the label column is where the epilogue reads y_i.  Th[c] =
// (theta_c, 0).  One 2-D TMA box pair (128 rows x 32 columns, 128-byte
// swizzle) per row tile is read as the K-major A operand of GEMM 1 AND as the
// MN-major B operand of GEMM 2 (same bytes, two shared-memory descriptors).
//
// Precision ("tf32" policy): GEMM 1 in 3xTF32 - tcgen05 kind::tf32 reads
// the top 19 bits of each fp32, so every operand is split v = hi + lo (hi =
// tf32(v) rounded to nearest, lo = tf32(v - hi): both unbiased) and the MMAs
// issue Xhi.Thhi + Xhi.Thlo + Xlo.Thhi (dropped lo.lo ~2^-22 relative).  GEMM 2
// needs Xa with K = rows, i.e. MN-major; tcgen05 takes 32-bit MN-major
// operands only in the 32-byte-atom swizzle (a second X layout), so GEMM 2
// runs in 3xBF16 (kind::f16): the SIMT pass that forms Xlo also writes X as
// bf16 hi | lo (MN-major, 128-byte swizzle), the epilogue writes [Rhi; Rlo]
// bf16 stacked as M = 128 (64 chains x 2) -> Rhi.Xhi + Rhi.Xlo + Rlo.Xhi at
// ~2^-16 relative per product.  Stated tolerance in
// tests/test_gpu_logistic_many.py.  Accumulation is fp32 in TMEM within a
// CTA's row slice, then exact fixed-point int64 pairs across CTAs
// (deterministic, as the single-chain pass).
//
// Execution: one persistent cooperative CTA per SM = 4 server warps + 8
// chain warps.  A chain warp runs one chain's NUTS engine (Engine<WarpTeam>,
// vectors in HBM) and requests gradients through posted/served flags exactly
// like the dense-Gaussian model (ts_k_dense.cu).  The server warps of all
// CTAs run batched steps: snapshot the outstanding requests, grid barrier,
// every CTA streams its row slice of Xa once per 64-chain tile with at least
// one request (TMA ring -> split -> GEMM 1 -> epilogue -> GEMM 2),
// fixed-point atomics of the CTA partials, grid barrier, release.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>
#include "ts_internal.cuh"
#include "ts_umma.cuh"
#include <cuda_bf16.h>

namespace ts_internal {

int make_tmap_f32(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int box_rows);

namespace {

constexpr int kLmRows = 128;     // rows per tile (GEMM 1 M)
constexpr int kLmChains = 64;    // chains per tile (GEMM 1 N)
constexpr int kLmSW = 8;         // server warps per CTA (2 per SM sub-partition: the epilogue is latency-bound)
constexpr int kLmSrv = 32 * kLmSW;
constexpr int kLmCW = 4;         // chain warps per CTA (runs with more chains than 148 x 4 are chunked)
constexpr int kLmThreads = kLmSrv + 32 * kLmCW;
constexpr int kLmBox = 16384;    // one 128-row x 128-B box
constexpr int kLmXBytes = 2 * kLmBox;                  // a row tile: columns 0..31 | 32..63
constexpr int kLmThBytes = 2 * (kLmChains * 128);      // theta tile: 64 chains x 64 columns
constexpr int kLmRBytes = 2 * kLmBox;                  // bf16 [Rhi; Rlo]: 128 x 128 rows (2 K-blocks of 64 rows)
constexpr int kLmXbBytes = 2 * kLmBox;                 // bf16 X tile hi | lo: 128 rows x 64 columns each
constexpr int kLmStages = 2;
// smem: X ring | Xlo | Th hi | Th lo | R | Xb (R + Xb reused by epilogue 2) | mbarriers + TMEM slot | chain-warp slot scalars
constexpr int kLmOffXlo = kLmStages * kLmXBytes;
constexpr int kLmOffThHi = kLmOffXlo + kLmXBytes;
constexpr int kLmOffThLo = kLmOffThHi + kLmThBytes;
constexpr int kLmOffR = kLmOffThLo + kLmThBytes;
constexpr int kLmOffXb = kLmOffR + kLmRBytes;
constexpr int kLmOffBar = kLmOffXb + kLmXbBytes;
constexpr int kLmOffSlots = kLmOffBar + 256;
static_assert(128 * 65 * 4 + 4 * kLmChains * 8 <= kLmRBytes + kLmXbBytes, "epilogue-2 scratch reuses R + Xb");
constexpr int kLmSmem = kLmOffSlots + kLmCW * kMaxSlots * (int)sizeof(SlotScalars) + 1024;
constexpr unsigned long long kLmGatherNs = 20000;
constexpr int kLmAcc = 2 * 64 + 2;  // per chain: 64 (hi, lo) pairs (gradient sums, ll at KA..), flag, pad

struct LManyArgs {
  int p, KA, C, Cpad, nv, chain0;
  int64_t n_rows, ntiles;
  float* thhi;  // [Cpad][64] posted theta, tf32 hi part (bias at column p)
  float* thlo;  // [Cpad][64] lo part
  unsigned long long* acc;  // [Cpad][kLmAcc] fixed-point sums (zeroed by the chain after reading)
  double* ws;               // chain workspaces [C][nv][D]
  unsigned long long* bar;  // grid barrier counter (zeroed before launch)
  int* done;
  unsigned long long* posted;   // [Cpad]
  unsigned long long* served;   // [Cpad]
  unsigned long long* pending;  // [Cpad]
  unsigned long long* npend;    // [4]
  unsigned int* fin;            // [Cpad] chain warp finished
  unsigned int* err;
  unsigned long long spin_ns;
  unsigned long long* prof;  // TS_PROF counters (CTA 0)
};

// tf32 (round to nearest, ties away): the split v = hi + lo with both parts
// rounded keeps the error of lo unbiased (the tensor core itself truncates).
// (Integer-op variants of these conversions measured slower: the epilogue is
// latency-bound, not conversion-pipe-bound.)
__device__ __forceinline__ float tf32_rna(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}
__device__ __forceinline__ uint32_t bf16_rne_bits(float v) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v));
}
// bf16 bits of v (round to nearest even) and of the remainder
__device__ __forceinline__ void bf16_split(float v, uint32_t& hi, uint32_t& lo) {
  hi = bf16_rne_bits(v);
  lo = bf16_rne_bits(v - __uint_as_float(hi << 16));
}
__device__ __forceinline__ void u_mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D f32, A/B bf16, A K-major, B MN-major
__host__ __device__ constexpr uint32_t idesc_bf16_bmn(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---------------------------------------------------------------- chain side
struct LogisticManyW : NoTraj {
  static constexpr bool kAsync = true;
  static constexpr bool kVecOps = false;
  int p;
  int64_t n_rows;
  float* thhi;
  float* thlo;
  unsigned long long* acc;
  unsigned long long* posted;
  unsigned long long* served;
  unsigned long long seq;
  int chain;
  unsigned int* err;
  unsigned long long spin_ns;
  VecStore S;
  int pq, pg;

  __device__ void post(int q, int g) {
    pq = q;
    pg = g;
    const int lane = threadIdx.x & 31;
    const double* qv = S.v(q);
    float* hrow = thhi + (int64_t)chain * 64;
    float* lrow = thlo + (int64_t)chain * 64;
    for (int k = lane; k < 64; k += 32) {
      const double v = k <= p ? qv[k] : 0.0;  // theta_0..p-1, bias theta_p; the label column gets 0
      const float h = tf32_rna((float)v);
      hrow[k] = h;
      lrow[k] = tf32_rna((float)(v - (double)h));
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");  // read by TMA in other CTAs
    __threadfence();
    __syncwarp();
    seq += 1;
    if (lane == 0) st_release_u64(posted + chain, seq);
  }
  __device__ double wait() {
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
      // a request waits at least one batched step (tens of us): back off so
      // the spinning chain warps leave the issue slots to the server warps
      SpinGuard sg(err, spin_ns);
      while (ld_relaxed_u64(served + chain) < seq) {
        __nanosleep(500);
        if (sg.expired()) break;
      }
      (void)ld_acquire_u64(served + chain);
    }
    __syncwarp();
    unsigned long long* a = acc + (int64_t)chain * kLmAcc;
    const bool bad = __ldcg(a + 2 * 64) != 0ULL;
    const double* th = S.v(pq);
    double* gv = S.v(pg);
    double ll = 0.0;
    for (int k = lane; k <= p + 1; k += 32) {  // p features, bias, log-likelihood at k = p + 1
      unsigned long long hi = __ldcg(a + 2 * k), lo = __ldcg(a + 2 * k + 1);
      fx_canon(hi, lo);
      const double s = bad ? __longlong_as_double(0x7ff8000000000000LL) : fx_join((long long)hi, lo);
      if (k <= p) gv[k] = th[k] - s;
      else ll = s;
    }
    __syncwarp();
    for (int k = lane; k < kLmAcc; k += 32) a[k] = 0ULL;  // this chain's slot is free for its next request
    // U = prior - loglik (kernels.py:90-104); prior left to right, bias first
    ll = __shfl_sync(0xffffffffu, ll, (p + 1) & 31);
    double pr = 0.0;
    if (lane == 0) {
      pr = 0.5 * th[p] * th[p];
      for (int d = 0; d < p; ++d) pr += 0.5 * th[d] * th[d];
    }
    pr = __shfl_sync(0xffffffffu, pr, 0);
    __syncwarp();
    return pr - ll;
  }
  template <class Team>
  __device__ double eval(const Team&, const VecStore&, int q, int g) {
    post(q, g);
    return wait();
  }
};

__device__ __forceinline__ void lm_grid_barrier(const LManyArgs& a, unsigned long long& epoch) {
  asm volatile("bar.sync 4, %0;" ::"r"(kLmSrv) : "memory");
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long target = (epoch + 1) * (unsigned long long)gridDim.x;
    red_release_add_u64(a.bar, 1ULL);
    SpinGuard sg(a.err, a.spin_ns);
    while (ld_relaxed_u64(a.bar) < target) {
      if (sg.expired()) break;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  epoch += 1;
  asm volatile("bar.sync 4, %0;" ::"r"(kLmSrv) : "memory");
}

// mbarrier wait with a bound: a transaction that never completes (it should
// not happen) raises the model's error word and traps instead of hanging.
__device__ __forceinline__ void lm_wait(uint32_t bar, uint32_t parity, unsigned int* err) {
  uint32_t done = 0;
  asm volatile(
      "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  if (done) return;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (unsigned n = 1;; ++n) {
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    if (done) return;
    if ((n & 1023u) == 0) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ULL) {
        if (err) atomicOr(err, 2u);
        __trap();
      }
    }
  }
}

// OR-reduction barrier over the server threads (named barrier 4)
__device__ __forceinline__ int lm_sync_or(int v) {
  int r;
  asm volatile(
      "{\n"
      ".reg .pred p, q;\n"
      "setp.ne.s32 p, %1, 0;\n"
      "bar.red.or.pred q, 4, %2, p;\n"
      "selp.s32 %0, 1, 0, q;\n"
      "}\n"
      : "=r"(r)
      : "r"(v), "r"(kLmSrv)
      : "memory");
  return r;
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// MN-major bf16 (B operand of GEMM 2), 128-byte swizzle: the 64 columns are
// one 128-B atom (LBO unused), SBO = 8 rows x 128 B.
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Server state of one CTA (the kLmSrv threads of warps 0..kLmSW-1).
struct LmServer {
  unsigned char* sm;  // 1024-aligned base
  uint32_t s_base;    // its shared address
  uint32_t full0, thb, d1b, d2b;  // mbarriers: full[2], theta, GEMM1 done, GEMM2 done
  uint32_t tmem;      // D1 at columns [0, 64), D2 at [64, 128)
  uint32_t x_issued, x_used, th_used, d1_used, d2_used;
  uint64_t x_pol;

  __device__ void init(unsigned char* base) {
    sm = base;
    s_base = u_smem(base);
    full0 = s_base + kLmOffBar;
    thb = full0 + 16;
    d1b = thb + 8;
    d2b = d1b + 8;
    const uint32_t tslot = d2b + 8;
    if (threadIdx.x == 0) {
      u_mbar_init(full0, 1);
      u_mbar_init(full0 + 8, 1);
      u_mbar_init(thb, 1);
      u_mbar_init(d1b, 1);
      u_mbar_init(d2b, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) u_tmem_alloc(tslot, 128);
    u_fence_before();
    asm volatile("bar.sync 4, %0;" ::"r"(kLmSrv) : "memory");
    u_fence_after();
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(tslot));
    x_issued = x_used = th_used = d1_used = d2_used = 0;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(x_pol));
  }
  __device__ void release() {
    asm volatile("bar.sync 4, %0;" ::"r"(kLmSrv) : "memory");
    if (threadIdx.x < 32) u_tmem_dealloc(tmem, 128);
  }
  // thread 0: TMA of row tile `tile` into ring stage x_issued % 2
  __device__ void issue_x(const CUtensorMap* tmx, int64_t tile) {
    const int s = (int)(x_issued & 1u);
    const uint32_t dst = s_base + s * kLmXBytes;
    const uint32_t bar = full0 + 8 * s;
    u_mbar_expect_tx(bar, kLmXBytes);
    const int r0 = (int)(tile * kLmRows);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
        ::"r"(dst), "l"(tmx), "r"(0), "r"(r0), "r"(bar), "l"(x_pol) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
        ::"r"(dst + kLmBox), "l"(tmx), "r"(32), "r"(r0), "r"(bar), "l"(x_pol) : "memory");
    ++x_issued;
  }
};

// One chain tile over this CTA's row slice: G partials and log-likelihood
// partials of the tile's 64 chains, added into the global fixed-point sums
// of the pending ones.
__device__ void lm_chain_tile(LmServer& S, const LManyArgs& a, const CUtensorMap* tmx, const CUtensorMap* tmh,
                              const CUtensorMap* tml, int n0, int64_t t_lo, int64_t t_hi) {
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  const int KA = a.KA;
  const int nk1 = KA / 8;  // GEMM 1 k-steps (K = 8 tf32 each)
  const uint32_t idesc1 = u_idesc_tf32(128, 64);
  const uint32_t idesc2 = idesc_bf16_bmn(128, 64);            // GEMM 2: bf16, B (Xa rows) MN-major
  const uint32_t xlo = S.s_base + kLmOffXlo, thh = S.s_base + kLmOffThHi, thl = S.s_base + kLmOffThLo;
  const uint32_t rA = S.s_base + kLmOffR, xbh = S.s_base + kLmOffXb, xbl = xbh + kLmBox;
  const int64_t nt = t_hi - t_lo;
  // TS_PROF: CTA 0 / thread 0 cycle counters [0] X wait, [1] GEMM 2 wait,
  // [2] SIMT X pass, [3] GEMM 1, [4] epilogue 1, [5] ll reduce, [6] epilogue 2, [7] tiles, [8] chain tiles
  const bool pf = a.prof != nullptr && blockIdx.x == 0 && t == 0;
  long long pc = pf ? clock64() : 0;
#define LM_PROF(k)                              \
  if (pf) {                                     \
    const long long c_ = clock64();             \
    a.prof[24 + (k)] += (unsigned long long)(c_ - pc); \
    pc = c_;                                    \
  }
  // theta tile (hi, lo) once per chain tile
  if (t == 0) {
    u_mbar_expect_tx(S.thb, 2 * kLmThBytes);
    u_tma_load_2d(thh, tmh, 0, n0, S.thb);
    u_tma_load_2d(thh + kLmChains * 128, tmh, 32, n0, S.thb);
    u_tma_load_2d(thl, tml, 0, n0, S.thb);
    u_tma_load_2d(thl + kLmChains * 128, tml, 32, n0, S.thb);
    if (nt > 0) S.issue_x(tmx, t_lo);
    if (nt > 1) S.issue_x(tmx, t_lo + 1);
  }
  double llacc0 = 0.0;  // chain t & 63, rows 32 (t >> 6) .. + 31 of every tile
  lm_wait(S.thb, S.th_used & 1u, a.err);
  ++S.th_used;
  for (int64_t tile = t_lo; tile < t_hi; ++tile) {
    const int s = (int)(S.x_used & 1u);
    LM_PROF(6)
    lm_wait(S.full0 + 8 * s, (S.x_used >> 1) & 1u, a.err);
    LM_PROF(0)
    const uint32_t xs = S.s_base + s * kLmXBytes;
    if (tile > t_lo) {  // GEMM 2 of the previous tile has read R, Xlo and the other stage
      lm_wait(S.d2b, S.d2_used & 1u, a.err);
      ++S.d2_used;
      u_fence_after();
      if (t == 0 && tile + 1 < t_hi) S.issue_x(tmx, tile + 1);
    }
    LM_PROF(1)
    // Xhi (in place) and Xlo = X - Xhi at the same (swizzled) positions for GEMM 1, and X as
    // bf16 hi | lo rows (64 columns = one 128-B swizzled line per row) for
    // GEMM 2: 2048 float4 groups, 16 per thread
    {
      float4* src = reinterpret_cast<float4*>(S.sm + s * kLmXBytes);
      float4* dst = reinterpret_cast<float4*>(S.sm + kLmOffXlo);
      unsigned char* xb = S.sm + kLmOffXb;
#pragma unroll
      for (int i = t; i < kLmXBytes / 16; i += kLmSrv) {
        const float4 v = src[i];
        const float4 h = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
        src[i] = h;  // the stage becomes Xhi (rounded; y and the ones column are exact)
        dst[i] = make_float4(tf32_rna(v.x - h.x), tf32_rna(v.y - h.y), tf32_rna(v.z - h.z), tf32_rna(v.w - h.w));
        const int box = i >> 10, r = (i >> 3) & 127, c = (i & 7) ^ (r & 7);  // logical 16-B chunk of the fp32 row
        const int cb = 4 * box + (c >> 1);                                  // bf16 16-B chunk
        const int off = r * 128 + ((cb ^ (r & 7)) << 4) + (c & 1) * 8;
        uint32_t h0, l0, h1, l1, h2, l2, h3, l3;
        bf16_split(v.x, h0, l0);
        bf16_split(v.y, h1, l1);
        bf16_split(v.z, h2, l2);
        bf16_split(v.w, h3, l3);
        *reinterpret_cast<uint2*>(xb + off) = make_uint2(h0 | (h1 << 16), h2 | (h3 << 16));
        *reinterpret_cast<uint2*>(xb + kLmBox + off) = make_uint2(l0 | (l1 << 16), l2 | (l3 << 16));
      }
    }
    fence_async_smem();
    u_fence_before();
    asm volatile("bar.sync 4, %0;" ::"r"(kLmSrv) : "memory");
    u_fence_after();
    LM_PROF(2)
    if (t == 0) {
      // GEMM 1: D1 = Xhi.Thhi + Xhi.Thlo + Xlo.Thhi   (128 rows x 64 chains)
      for (int kk = 0; kk < nk1; ++kk) {
        const uint32_t ko = (uint32_t)((kk >> 2) * kLmBox + (kk & 3) * 32);
        const uint32_t kt = (uint32_t)((kk >> 2) * (kLmChains * 128) + (kk & 3) * 32);
        const uint64_t ah = u_desc_sw128(xs + ko), al = u_desc_sw128(xlo + ko);
        const uint64_t bh = u_desc_sw128(thh + kt), bl = u_desc_sw128(thl + kt);
        u_mma_tf32(S.tmem, ah, bh, idesc1, kk != 0);
        u_mma_tf32(S.tmem, ah, bl, idesc1, 1);
        u_mma_tf32(S.tmem, al, bh, idesc1, 1);
      }
      u_mma_commit(S.d1b);
    }
    __syncwarp();
    lm_wait(S.d1b, S.d1_used & 1u, a.err);
    ++S.d1_used;
    u_fence_after();
    LM_PROF(3)
    // epilogue 1: thread = row (TMEM lane 32 q + lane, q = w & 3); warp w
    // handles the tile's chains 32 (w >> 2) .. + 31
    const int q4 = w & 3, ch0 = 32 * (w >> 2);
    const int row = q4 * 32 + lane;
    const int64_t grow = tile * kLmRows + row;
    const bool valid = grow < a.n_rows;
    // y from the label column KA - 1 of the row's swizzled smem line
    float yv;
    {
      const int col = a.p + 1, box = col >> 5, cb = col & 31;
      const int chunk = (cb >> 2) ^ (row & 7);
      yv = *reinterpret_cast<const float*>(S.sm + s * kLmXBytes + box * kLmBox + row * 128 + chunk * 16 + (cb & 3) * 4);
    }
    // bf16 A of GEMM 2: K-block (q >> 1) holds rows 64 (q >> 1) ..; this
    // warp's rows are k = 32 (q & 1) + lane within it (16-bit stores)
    unsigned char* R = S.sm + kLmOffR + (q4 >> 1) * kLmBox;
    const int kk64 = 32 * (q4 & 1) + lane;
    const int rsub = (kk64 & 7) * 2;
    // log-likelihood terms per (row, chain) -> LL[row][chain ^ (row & 31)] in
    // the Xlo buffer (GEMM 1, its only reader, is complete): conflict-free
    // writes by row and reads by chain
    float* LL = reinterpret_cast<float*>(S.sm + kLmOffXlo);
#pragma unroll
    for (int c0 = ch0; c0 < ch0 + 32; c0 += 16) {
      float e16[16];
      u_tmem_ld16(S.tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)c0, e16);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float eta = e16[j];
        // MUFU exp / log2 (the policy's stated tolerance; the fp32 single-chain
        // pass uses the unbiased polynomials instead)
        const float e = __expf(-fabsf(eta));
        const float op = 1.f + e;
        const float sig = __fdividef(eta >= 0.f ? 1.f : e, op);
        const float r = valid ? yv - sig : 0.f;
        LL[row * 64 + ((c0 + j) ^ (row & 31))] = valid ? yv * eta - (fmaxf(eta, 0.f) + __logf(op)) : 0.f;
        const __nv_bfloat16 bh = __float2bfloat16_rn(r);
        const uint32_t rh = __bfloat16_as_ushort(bh), rl = bf16_rne_bits(r - __bfloat162float(bh));
        const int mh = c0 + j, ml = 64 + c0 + j;
        *reinterpret_cast<unsigned short*>(R + mh * 128 + ((((kk64 >> 3) ^ (mh & 7))) << 4) + rsub) = (unsigned short)rh;
        *reinterpret_cast<unsigned short*>(R + ml * 128 + ((((kk64 >> 3) ^ (ml & 7))) << 4) + rsub) = (unsigned short)rl;
      }
    }
    u_fence_before();
    fence_async_smem();
    asm volatile("bar.sync 4, %0;" ::"r"(kLmSrv) : "memory");
    u_fence_after();
    if (t == 0) {
      // GEMM 2: D2 += [Rhi; Rlo] . Xhi + [Rhi; Rlo] . Xlo   (128 x 64 features, K = 128 rows)
      const bool first = tile == t_lo;
      // K = 16 bf16 rows per MMA: A (R) K-block kk >> 2, 32-B step; B (Xb) 16 rows = 2 KB
#pragma unroll 1
      for (int kk = 0; kk < kLmRows / 16; ++kk) {
        const uint64_t ad = u_desc_sw128(rA + (kk >> 2) * kLmBox + (kk & 3) * 32);
        const uint64_t bh = desc_mn_sw128(xbh + kk * 2048), bl = desc_mn_sw128(xbl + kk * 2048);
        u_mma_bf16(S.tmem + 64, ad, bh, idesc2, !(first && kk == 0));
        u_mma_bf16(S.tmem + 64, ad, bl, idesc2, 1);
      }
      u_mma_commit(S.d2b);
    }
    __syncwarp();
    ++S.x_used;
    LM_PROF(4)
    // log-likelihood: thread t sums chain (t & 63) over rows 32 (t >> 6) ..
    // + 31 of this tile (fixed order), accumulated in double over tiles
    {
      const int c = t & 63, r0 = (t >> 6) * 32;
      float acc = 0.f;
#pragma unroll 8
      for (int r = r0; r < r0 + 32; ++r) acc += LL[r * 64 + (c ^ (r & 31))];
      llacc0 += (double)acc;
      asm volatile("bar.sync 4, %0;" ::"r"(kLmSrv) : "memory");  // LL (= Xlo) is rewritten by the next tile's SIMT pass
    }
    LM_PROF(5)
    if (pf) a.prof[24 + 7] += 1;
  }
  // drain: GEMM 2 of the last tile
  if (nt > 0) {
    lm_wait(S.d2b, S.d2_used & 1u, a.err);
    ++S.d2_used;
    u_fence_after();
  }
  // epilogue 2 (R is free now): D2 lanes 0..63 = chains (hi residuals),
  // 64..127 = the same chains (lo residuals); exchanged through shared
  // memory as [128][65] floats (padded rows: conflict-free), plus the
  // per-warp log-likelihood sums [4][64] doubles after them
  float* gx = reinterpret_cast<float*>(S.sm + kLmOffR);
  double* llw = reinterpret_cast<double*>(S.sm + kLmOffR + 128 * 65 * 4);
  llw[t] = nt > 0 ? llacc0 : 0.0;  // [quarter][chain]: rows 32 k .. 32 k + 31 of every tile
  {
    const int q4 = w & 3, col0 = 32 * (w >> 2);
    const int mm = q4 * 32 + lane;  // D2 lane
#pragma unroll
    for (int c0 = col0; c0 < col0 + 32; c0 += 16) {
      float v[16];
      if (nt > 0) u_tmem_ld16(S.tmem + 64 + ((uint32_t)(q4 * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) gx[mm * 65 + c0 + j] = nt > 0 ? v[j] : 0.f;
    }
  }
  const int m = t;  // threads 0..63: one chain each
  u_fence_before();
  asm volatile("bar.sync 4, %0;" ::"r"(kLmSrv) : "memory");
  u_fence_after();
  if (m < 64) {
    const int c = n0 + m;
    if (c < a.Cpad && __ldcg(a.pending + c) != 0ULL) {
      unsigned long long* acc = a.acc + (int64_t)c * kLmAcc;
      bool bad = false;
      for (int k = 0; k <= a.p + 1; ++k) {
        double v;
        if (k <= a.p) v = (double)gx[m * 65 + k] + (double)gx[(m + 64) * 65 + k];
        else v = ((llw[m] + llw[kLmChains + m]) + llw[2 * kLmChains + m]) + llw[3 * kLmChains + m];
        long long h, l;
        bad |= !fx_split(v, h, l);
        red_add_u64(acc + 2 * k, (unsigned long long)h);
        red_add_u64(acc + 2 * k + 1, (unsigned long long)l);
      }
      if (bad) red_add_u64(acc + 2 * 64, 1ULL);
    }
  }
  LM_PROF(6)
  if (pf) a.prof[24 + 8] += 1;
#undef LM_PROF
  u_fence_before();
  asm volatile("bar.sync 4, %0;" ::"r"(kLmSrv) : "memory");  // TMEM / scratch free for the next chain tile
  u_fence_after();
}

__global__ void __launch_bounds__(kLmThreads, 1)
    k_logistic_many(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmh,
                    const __grid_constant__ CUtensorMap tml, LManyArgs a, int nslots, OpArgs A) {
  extern __shared__ __align__(1024) unsigned char lm_dsm[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(lm_dsm) + 1023) & ~(uintptr_t)1023);
  volatile int* flag = reinterpret_cast<volatile int*>(base + kLmOffBar + 64);
  SlotScalars* ss_all = reinterpret_cast<SlotScalars*>(base + kLmOffSlots);
  const int warp = threadIdx.x >> 5;
  if (warp < kLmSW) {
    LmServer S;
    S.init(base);
    if (threadIdx.x == 0) { u_prefetch_tmap(&tmx); u_prefetch_tmap(&tmh); u_prefetch_tmap(&tml); }
    const int t = threadIdx.x;
    const int total = (int)gridDim.x * kLmCW;
    const int my_chain = blockIdx.x * kLmCW + t;
    unsigned long long srv = 0, epoch = 0;
    const int64_t G = gridDim.x;
    const int64_t t_lo = a.ntiles * blockIdx.x / G, t_hi = a.ntiles * (blockIdx.x + 1) / G;
    const int ntile_c = a.Cpad / kLmChains;
    for (int step = 0;; ++step) {
      unsigned long long mine = 0;
      if (t < kLmCW) {
        unsigned long long p = ld_acquire_u64(a.posted + my_chain);
        if (p <= srv) {
          // gather: give a chain that is still running up to kLmGatherNs to
          // post its next request, so a step serves the whole batch instead
          // of splitting chains across alternate steps
          unsigned long long g0, g1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
          for (;;) {
            if (*reinterpret_cast<volatile unsigned int*>(a.fin + my_chain) != 0u) break;
            p = ld_relaxed_u64(a.posted + my_chain);
            if (p > srv) { p = ld_acquire_u64(a.posted + my_chain); break; }
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
            if (g1 - g0 > kLmGatherNs) break;
          }
        }
        mine = p > srv ? p : 0ULL;
        a.pending[my_chain] = mine;
        if (mine) atomicAdd(a.npend + (step & 1), 1ULL);
      }
      if (t == 0 && blockIdx.x == 0)
        a.npend[2 + (step & 1)] = (*reinterpret_cast<volatile int*>(a.done) >= total) ? 1ULL : 0ULL;
      lm_grid_barrier(a, epoch);
      if (t == 0) {
        const unsigned long long np = ld_relaxed_u64(a.npend + (step & 1));
        const bool all_done = ld_relaxed_u64(a.npend + 2 + (step & 1)) != 0ULL;
        *flag = (np == 0ULL && all_done) ? 0 : (np ? 1 : 2);
        if (blockIdx.x == 0) a.npend[(step + 1) & 1] = 0ULL;
      }
      asm volatile("bar.sync 4, %0;" ::"r"(kLmSrv) : "memory");
      const int f = *flag;
      if (f == 0) break;
      if (f == 1) {
        if (t == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
        for (int ct = 0; ct < ntile_c; ++ct) {
          int any = 0;
          for (int j = t; j < kLmChains; j += kLmSrv) any |= __ldcg(a.pending + ct * kLmChains + j) != 0ULL;
          any = lm_sync_or(any);
          if (!any) continue;
          lm_chain_tile(S, a, &tmx, &tmh, &tml, ct * kLmChains, t_lo, t_hi);
        }
      }
      lm_grid_barrier(a, epoch);  // every CTA's partials are in
      if (t < kLmCW && mine) {
        srv = mine;
        st_release_u64(a.served + my_chain, mine);
      }
    }
    S.release();
    return;
  }
  // ---------------- chain warps
  const int cw = warp - kLmSW;
  const int chain = blockIdx.x * kLmCW + cw;
  const int n_active = (A.op == OP_RUN) ? a.C : 1;
  if (chain < n_active) {
    LogisticManyW M;
    M.p = a.p;
    M.n_rows = a.n_rows;
    M.thhi = a.thhi;
    M.thlo = a.thlo;
    M.acc = a.acc;
    M.posted = a.posted;
    M.served = a.served;
    M.seq = 0;
    M.chain = chain;
    M.err = a.err;
    M.spin_ns = a.spin_ns;
    Engine<WarpTeam, LogisticManyW> E;
    E.D = a.p + 1;
    E.S.base = a.ws + (int64_t)chain * a.nv * (a.p + 1);
    E.S.vstride = a.p + 1;
    E.S.dstride = 1;
    M.S = E.S;
    E.M = M;
    E.prof = nullptr;
    E.prof_last = 0;
    E.tr = nullptr;
    E.ss = ss_all + cw * kMaxSlots;
    __syncwarp();
    do_op(E, A, A.op == OP_RUN ? a.chain0 + chain : 0, chain == 0 || A.op == OP_RUN);
  }
  __syncwarp();
  __threadfence();
  if ((threadIdx.x & 31) == 0) {
    *reinterpret_cast<volatile unsigned int*>(a.fin + chain) = 1u;
    atomicAdd(a.done, 1);
  }
}

// Xa = [X | 1 | y | 0 ...] (n x KA fp32)
__global__ void k_build_xaug(const float* __restrict__ x, const uint8_t* __restrict__ y, int64_t n, int p, int KA,
                             float* __restrict__ xa) {
  const int64_t total = n * KA;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / KA;
    const int k = (int)(i - r * KA);
    xa[i] = k < p ? x[r * p + k] : (k == p ? 1.f : (k == p + 1 ? (float)y[r] : 0.f));
  }
}

int launch_lm_chunk(const ts_model* m, int nslots, OpArgs& A, int C, int chain0, cudaStream_t st) {
  ts_model* mm = const_cast<ts_model*>(m);
  const int D = m->dim;
  const int nv = num_vecs(nslots);
  int dev = 0, nsm = 0;
  TS_CUDA(cudaGetDevice(&dev));
  TS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  auto kern = k_logistic_many;
  TS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kLmSmem));
  int occ = 0;
  TS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kLmThreads, kLmSmem));
  if (occ < 1) return set_err(TS_EUNSUPPORTED, "many-chain logistic kernel cannot be resident");
  const int grid = nsm;
  if ((int64_t)grid * kLmCW < C) return set_err(TS_EINVAL, "too many chains for one co-resident grid");
  const int Cpad = ((grid * kLmCW + kLmChains - 1) / kLmChains) * kLmChains;
  const size_t need = 64 + (size_t)Cpad * 64 * 4 * 2 + (size_t)Cpad * kLmAcc * 8 + (size_t)C * nv * D * 8 +
                      (size_t)Cpad * 24 + 64 + (size_t)Cpad * 4;
  if (mm->dws_size < need) {
    if (mm->dws) cudaFree(mm->dws);
    mm->dws = nullptr;
    mm->dws_size = 0;
    TS_CUDA(cudaMalloc((void**)&mm->dws, need));
    mm->dws_size = need;
    TS_CUDA(cudaMemset(mm->dws, 0, need));
  }
  LManyArgs a;
  memset(&a, 0, sizeof a);
  a.p = m->p; a.KA = m->ka; a.C = C; a.Cpad = Cpad; a.nv = nv; a.chain0 = chain0;
  a.n_rows = m->n_rows;
  a.ntiles = (m->n_rows + kLmRows - 1) / kLmRows;
  unsigned char* p = mm->dws;
  a.bar = reinterpret_cast<unsigned long long*>(p);
  a.done = reinterpret_cast<int*>(p + 8);
  p += 64;
  a.thhi = reinterpret_cast<float*>(p); p += (size_t)Cpad * 64 * 4;
  a.thlo = reinterpret_cast<float*>(p); p += (size_t)Cpad * 64 * 4;
  a.acc = reinterpret_cast<unsigned long long*>(p); p += (size_t)Cpad * kLmAcc * 8;
  a.ws = reinterpret_cast<double*>(p); p += (size_t)C * nv * D * 8;
  a.posted = reinterpret_cast<unsigned long long*>(p);
  a.served = a.posted + Cpad;
  a.pending = a.served + Cpad;
  a.npend = a.pending + Cpad;
  a.fin = reinterpret_cast<unsigned int*>(a.npend + 4);
  a.err = m->errw;
  a.spin_ns = spin_limit_ns();
  a.prof = A.prof;
  CUtensorMap tx, th, tl;
  memset(&tx, 0, sizeof tx);
  memset(&th, 0, sizeof th);
  memset(&tl, 0, sizeof tl);
  int rc = make_tmap_f32(&tx, m->xaug, m->n_rows, m->ka, kLmRows);
  if (rc) return rc;
  rc = make_tmap_f32(&th, a.thhi, Cpad, 64, kLmChains);
  if (rc) return rc;
  rc = make_tmap_f32(&tl, a.thlo, Cpad, 64, kLmChains);
  if (rc) return rc;
  TS_CUDA(cudaMemsetAsync(mm->dws, 0, 64, st));
  TS_CUDA(cudaMemsetAsync(a.acc, 0, (size_t)Cpad * kLmAcc * 8, st));
  TS_CUDA(cudaMemsetAsync(a.posted, 0, ((size_t)Cpad * 3 + 4) * sizeof(unsigned long long) + (size_t)Cpad * 4, st));
  int ns = nslots;
  void* args[] = {&tx, &th, &tl, &a, &ns, &A};
  TS_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3((unsigned)grid), dim3(kLmThreads), args, kLmSmem, st));
  return TS_OK;
}

}  // namespace

int build_logistic_xaug(ts_model* m, const float* x_dev, const uint8_t* y_dev) {
  m->ka = ((m->p + 2) + 7) / 8 * 8;
  if (m->ka > 64) return set_err(TS_EUNSUPPORTED, "tf32 many-chain logistic path: num_features <= 62");
  TS_CUDA(cudaMalloc((void**)&m->xaug, (size_t)m->n_rows * m->ka * sizeof(float)));
  k_build_xaug<<<1184, 256>>>(x_dev, y_dev, m->n_rows, m->p, m->ka, m->xaug);
  TS_CUDA(cudaGetLastError());
  return TS_OK;
}

int launch_logistic_many(const ts_model* m, int nslots, OpArgs& A, int n_chains, cudaStream_t st) {
  if (A.op != OP_RUN) return launch_lm_chunk(m, nslots, A, 1, 0, st);
  int dev = 0, nsm = 0;
  TS_CUDA(cudaGetDevice(&dev));
  TS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int cap = nsm * kLmCW;
  for (int c0 = 0; c0 < n_chains; c0 += cap) {
    const int rc = launch_lm_chunk(m, nslots, A, n_chains - c0 < cap ? n_chains - c0 : cap, c0, st);
    if (rc) return rc;
  }
  return TS_OK;
}

}  // namespace ts_internal
