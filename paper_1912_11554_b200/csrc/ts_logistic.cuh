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
// Cross-CTA reduction: each CTA adds its (p+2)-vector of partial sums to a
// global accumulator as exact fixed-point int64 pairs (red.add; integer sums
// are order-independent, so the result is deterministic), one grid barrier,
// then every CTA reads the identical totals and runs the (replicated) tree
// logic without a second barrier.
#pragma once
#include <stdint.h>
#include "ts_team.cuh"

namespace ts {

struct WarpPipe {
  unsigned long long issued;    // tiles issued into the ring (periodic sequence index)
  unsigned long long consumed;  // tiles consumed
  // narrow pass (p <= 64): ring positions carried across passes (no
  // divisions on the per-pass entry path) and the warp's static tile range
  int cs, cpar, ctj;            // consumer: ring slot, mbarrier parity, periodic tile index
  int ps, pj;                   // producer: ring slot, periodic tile index
  int first, count, keep;       // first tile, tiles per pass, tiles fetched L2::evict_last
  int pad_[4];
};
static_assert(sizeof(WarpPipe) == 64, "WarpPipe is budgeted at 64 bytes per ring (launch_block_logistic)");

struct LogisticArgs {
  const float* xt;          // tiled X, ntiles * 32 * p floats
  const uint8_t* yt;        // labels, ntiles * 32 (padding rows 0)
  int64_t n_rows;
  int p;
  int64_t ntiles;
  double* pbuf;             // 3 rotating accumulators x kFxCopies copies of (p+2) fixed-point int64 pairs + flag
  unsigned long long* bar;  // grid barrier counter (zeroed before launch)
  int fp64;                 // precision policy
  int pmax;                 // compile-time feature capacity of the pass (8/32/56/64)
  // shared-memory pipeline of this CTA (set by the kernel)
  unsigned char* stages;    // [nwarps][nstage][stage_bytes]
  uint64_t* mbar;           // [nwarps][nstage]
  WarpPipe* pipe;           // [nwarps]
  int nstage;
  int stage_bytes;
  int exact_cvt;            // X holds fp32 subnormals (informational)
  int wide;                 // p > 64: 8-row row-major tiles (logistic_cta_pass_wide)
  double* slotws;           // wide p: NodeStore slot vectors in global memory [grid][5*nslots][D]
  unsigned long long* prof; // optional: CTA-0 cycle counters [prior, pass, barrier, reduce] (profiling)
  // row sharding across GPUs (ts_peer_mailbox_*): world > 0 enables the exchange
  int world, rank;
  unsigned long long* mail[8];    // every rank's mailbox, mapped into this process (mail_layout below)
  unsigned long long* mail_epoch; // this rank's exchange counter, persistent across launches
  unsigned long long xbase;       // *mail_epoch at kernel start
  unsigned long long* dump;       // optional: raw local totals of the first pass (ts_logistic_partial_sums)
  // this CTA within its rank: index, CTA count, and the rank's row range in
  // units of tiles (p <= 64) or of kWideGroup-tile groups (wide); set per CTA
  int cta, ncta;
  int64_t u_lo, u_hi;
  // test mode: `vranks` row-sharded ranks emulated inside one launch (groups
  // of CTAs exchanging through vmail), see ts_model_set_virtual_ranks
  int vranks;
  unsigned long long* vmail;
  int keep_pct;  // % of each warp's tiles fetched with L2::evict_last (resident across passes), rest evict_first
  int icvt;  // fp64 wide pass: 1 = odd features converted on the integer pipe (default), 0 = all F2F, 2 = all ALU
  const float* th32;  // FP32 narrow pass: theta as floats [pmax + 1] (smem, written by the driver before each pass)
  unsigned int* err;               // sticky synchronisation-timeout flag of the model (SpinGuard)
  unsigned long long spin_ns;      // wait limit
  int fault;                       // fault injection (tests): 1 = CTA 1 never arrives at the grid barrier
  int llmode;                      // FP32 narrow pass: log-likelihood term precision (logistic_cta_pass LL)
  int xd;                          // X stored as fp64 (wide layout, logistic_cta_pass_wide XD)
  const double* thd;  // FP64 narrow pass: theta as doubles [pmax + 1], zero-padded, 16-B aligned (smem, written by the driver)
  int fxc;            // cross-CTA accumulator copies in use (1..kFxCopies)
  int xh;                          // p <= 64 half-row layouts: 1 X fp64 (logistic_cta_pass_x64h), 2 X fp32 paired (logistic_cta_pass_pair)
};

// Mailbox of one rank: kMailFlags words of flags (flag[src] = 1 + the last
// exchange index src published here), then 3 rotating slots x world x
// (2*(p+2)+2) words of fixed-point totals.
constexpr int kMailFlags = 16;
__host__ __device__ inline int64_t mail_words(int p, int world) {
  return kMailFlags + 3 * (int64_t)world * (2 * (int64_t)(p + 2) + 2);
}

// Cross-CTA accumulators (LogisticArgs::pbuf): 3 rotating buffers per rank;
// a buffer holds up to kFxCopies copies of the (p+2) fixed-point pairs + flag,
// each padded to its own 1-KB block; CTA c adds into copy c % fxc (fewer
// red.adds per address, spread over more L2 slices) and a reader sums the
// copies (integers: the order does not matter).  fxc = 2 by default
// (launch_block_logistic: the read-back grows with the copies).
constexpr int kFxCopies = 8;
__host__ __device__ inline int64_t fx_copy_stride(int p) { return (2 * (int64_t)(p + 2) + 2 + 127) / 128 * 128; }
__host__ __device__ inline int64_t fx_buf_words(int p) { return kFxCopies * fx_copy_stride(p); }
__host__ __device__ inline int64_t fx_rank_words(int p) { return 3 * fx_buf_words(p); }

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
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Fixed-point pair of a double (all reductions across warps, CTAs and GPUs
// add these integers, so totals do not depend on the order of arrival):
//   v ~= hi * 2^-10 + lo * 2^-61,  hi = round(v * 2^10),  |lo| <= 2^50,
// both rounded to nearest-even with the 1.5*2^52 magic constant (two FMAs
// and integer subtractions, no float->int64 conversion instructions, which
// are multi-cycle on the XU pipe).  v - hi*2^-10 is exact, so rounding below
// 2^-61 is the only error.  Valid for |v| < 2^40 (false otherwise or if v is
// not finite).  Canonical pair: lo in [0, 2^51) (fx_canon), where a pair's
// words are exact doubles.
constexpr int kFxLoBits = 51;
constexpr unsigned long long kFxLoMask = (1ULL << kFxLoBits) - 1;  // one hi unit = 2^51 lo units
__device__ __forceinline__ bool fx_split(double v, long long& hi, long long& lo) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52
  if (!(fabs(v) < 1099511627776.0)) { hi = 0; lo = 0; return false; }
  const double t = __fma_rn(v, 1024.0, magic);
  hi = __double_as_longlong(t) - __double_as_longlong(magic);
  const double rem = __fma_rn(-__dsub_rn(t, magic), 1.0 / 1024.0, v);
  lo = __double_as_longlong(__fma_rn(rem, 2305843009213693952.0, magic)) - __double_as_longlong(magic);
  return true;
}
// canonical form of a (hi, signed lo) sum: lo in [0, 2^51)
__device__ __forceinline__ void fx_canon(unsigned long long& hi, unsigned long long& lo) {
  hi += (unsigned long long)((long long)lo >> kFxLoBits);
  lo &= kFxLoMask;
}
__device__ __forceinline__ double fx_join(long long hi, unsigned long long lo_canon) {
  return (double)hi * (1.0 / 1024.0) + (double)lo_canon * (1.0 / 2305843009213693952.0);
}

// Bounded spin.  Every inter-CTA / inter-GPU wait (grid barrier, peer
// mailbox, served flag) polls through a SpinGuard: a wait longer than `limit`
// ns (%globaltimer) sets *err (sticky, per model) and gives up; once *err is
// set every later wait gives up at once.  A kernel whose peer CTA or rank
// never arrives therefore still terminates, and the host raises RuntimeError
// (run status TS_STATUS_SYNC_TIMEOUT / ts_model_error) instead of the GPU
// hanging.  The clock is read every 64 polls only.
struct SpinGuard {
  unsigned int* err;
  unsigned long long limit, t0;
  unsigned int n;
  __device__ __forceinline__ SpinGuard(unsigned int* e, unsigned long long lim) : err(e), limit(lim), t0(0), n(0) {}
  // true: stop waiting
  __device__ __forceinline__ bool expired() {
    if (err == nullptr) return false;
    if ((++n & 63u) != 1u) return false;
    if (*reinterpret_cast<volatile unsigned int*>(err) != 0u) return true;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (n == 1u) { t0 = t; return false; }
    if (t - t0 > limit) { atomicOr(err, 1u); return true; }
    return false;
  }
};

// ------------------------------------------------------------- worker group
// Warp 0 of each CTA drives the chain; warps 1.. stream the data.  The pass
// code below runs on the worker warps only and synchronises with named
// barrier 1; barriers 2/3 hand a pass from the driver to the workers and back.
__device__ __forceinline__ int wk_tid() { return (int)threadIdx.x - 32; }
__device__ __forceinline__ int wk_threads() { return (int)blockDim.x - 32; }
__device__ __forceinline__ int wk_warp() { return (int)(threadIdx.x >> 5) - 1; }
__device__ __forceinline__ int wk_nwarps() { return (int)(blockDim.x >> 5) - 1; }
__device__ __forceinline__ void wk_sync() { asm volatile("bar.sync 1, %0;" ::"r"(wk_threads()) : "memory"); }
__device__ __forceinline__ void cta_bar(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"((int)blockDim.x) : "memory"); }
__device__ __forceinline__ void cta_arrive(int id) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"((int)blockDim.x) : "memory"); }

// ------------------------------------------------------------- tile pipeline
// Ring-position arithmetic: 32-bit div/mod while the counters fit (64-bit
// division is a long emulated sequence on the per-pass entry path).
__device__ __forceinline__ uint32_t umod(unsigned long long a, uint32_t b) {
  return (a >> 32) ? (uint32_t)(a % b) : (uint32_t)a % b;
}
__device__ __forceinline__ uint32_t udiv(unsigned long long a, uint32_t b) {
  return (a >> 32) ? (uint32_t)(a / b) : (uint32_t)a / b;
}
struct WarpTiles {
  int64_t first;  // first tile of this warp
  int64_t count;  // number of tiles (stride nwarps)
  int nwarps;
};

__device__ __forceinline__ WarpTiles warp_tiles(const LogisticArgs& a, int warp, int nwarps) {
  const int64_t G = a.ncta, span = a.u_hi - a.u_lo;
  const int64_t t_begin = a.u_lo + (span * (int64_t)a.cta) / G;
  const int64_t t_end = a.u_lo + (span * ((int64_t)a.cta + 1)) / G;
  WarpTiles w;
  w.first = t_begin + warp;
  w.count = (t_end - w.first + nwarps - 1) / nwarps;
  if (w.count < 0) w.count = 0;
  w.nwarps = nwarps;
  return w;
}
__device__ __forceinline__ WarpTiles warp_tiles(const LogisticArgs& a) { return warp_tiles(a, wk_warp(), wk_nwarps()); }

// Kernel prologue (worker warps): mbarriers and pipe counters.
static __device__ void logistic_pipeline_init(const LogisticArgs& a) {
  const int rings = wk_nwarps();
  if (a.wide) {
    uint32_t* z = reinterpret_cast<uint32_t*>(a.stages);
    const int nw = rings * a.nstage * a.stage_bytes / 4;
    for (int i = wk_tid(); i < nw; i += wk_threads()) z[i] = 0u;
  }
  for (int i = wk_tid(); i < rings * a.nstage; i += wk_threads()) mbar_init(a.mbar + i, 1);
  for (int i = wk_tid(); i < rings; i += wk_threads()) {
    WarpPipe& q = a.pipe[i];
    q.issued = 0; q.consumed = 0;
    q.cs = 0; q.cpar = 0; q.ctj = 0; q.ps = 0; q.pj = 0;
    if (!a.wide) {
      const WarpTiles wt = warp_tiles(a, i, rings);
      q.first = (int)wt.first;
      q.count = (int)wt.count;
      q.keep = (int)(wt.count * a.keep_pct / 100);
    } else {
      q.first = 0; q.count = 0; q.keep = 0;
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  wk_sync();
}

// Kernel epilogue (worker warps): wait for the tiles the producer prefetched
// for a pass that never came, so no bulk copy targets the shared memory of an
// exited CTA.
static __device__ void logistic_pipeline_drain(const LogisticArgs& a) {
  const int warp = wk_warp();
  const WarpTiles wt = warp_tiles(a);
  if (wt.count > 0) {
    const unsigned long long c = a.pipe[warp].consumed, iss = a.pipe[warp].issued;
    for (unsigned long long seq = c; seq < iss; ++seq)
      mbar_wait(a.mbar + warp * a.nstage + (int)(seq % a.nstage), (uint32_t)((seq / a.nstage) & 1ULL));
  }
  wk_sync();
}

// Lane's row of a tile in shared memory -> x[0..PMAX) (zeros past p), y.
// PE > 0 fixes p at compile time (branch-free body for the benchmark shape).
// `sb` points into the dynamic shared-memory symbol, so these are LDS (not
// generic loads with 64-bit addresses).
template <int PMAX, int PE>
__device__ __forceinline__ void row_from_stage(const unsigned char* sb, int p_rt, int lane, float (&x)[PMAX], uint8_t& y) {
  const int p = PE > 0 ? PE : p_rt;
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
// a / b for b in [1, 3]: MUFU reciprocal + one Newton correction of the
// quotient (within an ulp, no IEEE-division slow-path checks)
__device__ __forceinline__ float div_pos_f(float a, float b) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b));
  const float q = a * r;
  return __fmaf_rn(__fmaf_rn(-b, q, a), r, q);
}

// exp(x) for x <= 0 in float without the MUFU ex2 (whose error is biased:
// ~0.16 ulp on average over covtype's rows, i.e. 1.7e-3 nats summed over
// 581,012 rows): x log2(e) in two parts, 2^f on [-1/2, 1/2] by its Taylor
// polynomial of degree 9 (truncation < 1e-11 relative), 2^j by exponent
// arithmetic.  Round-to-nearest errors only, which average out over rows.
__device__ __forceinline__ float exp_neg_f(float x) {
  if (x < -87.0f) return 0.0f;
  const float j = rintf(x * 1.44269504088896341f);
  float f = __fmaf_rn(x, 1.44269502162933349609375f, -j);
  f = __fmaf_rn(x, 1.925963033500011e-08f, f);
  // 2^f = e^(f ln 2): c_k = ln2^k / k!
  float p = 1.0178086009239699e-07f;
  p = __fmaf_rn(p, f, 1.3215486790144307e-06f);
  p = __fmaf_rn(p, f, 1.5252733804059841e-05f);
  p = __fmaf_rn(p, f, 1.5403530393381609e-04f);
  p = __fmaf_rn(p, f, 1.3333558146428443e-03f);
  p = __fmaf_rn(p, f, 9.6181291076284772e-03f);
  p = __fmaf_rn(p, f, 5.5504108664821580e-02f);
  p = __fmaf_rn(p, f, 2.4022650695910071e-01f);
  p = __fmaf_rn(p, f, 6.9314718055994531e-01f);
  p = __fmaf_rn(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((int)j << 23));
}
// log1p(e) for e in [0, 1] in float: 2 atanh(s), s = e / (2 + e) <= 1/3,
// series in s^2 to s^18 (truncation < 2e-10 relative); no MUFU lg2.
// (also valid for e in [-1/2, 0], s in [-1/3, 0] (2 + e in [1.5, 3]): the pass evaluates
// log1p(e) - log 2 = log1p((e - 1) / 2), exactly 0 at e = 1, i.e. eta = 0)
__device__ __forceinline__ float log1p_unit_f(float e) {
  const float s = div_pos_f(e, 2.0f + e);
  const float s2 = s * s;
  float q = 1.0f / 19.0f;
  q = __fmaf_rn(q, s2, 1.0f / 17.0f);
  q = __fmaf_rn(q, s2, 1.0f / 15.0f);
  q = __fmaf_rn(q, s2, 1.0f / 13.0f);
  q = __fmaf_rn(q, s2, 1.0f / 11.0f);
  q = __fmaf_rn(q, s2, 1.0f / 9.0f);
  q = __fmaf_rn(q, s2, 1.0f / 7.0f);
  q = __fmaf_rn(q, s2, 1.0f / 5.0f);
  q = __fmaf_rn(q, s2, 1.0f / 3.0f);
  q = __fmaf_rn(q, s2, 1.0f);
  return 2.0f * s * q;
}

// fp32 -> fp64 on the integer pipe for normal numbers and zeros (X without
// fp32 subnormals, LogisticArgs::exact_cvt == 0): sign | (exponent + 896) |
// mantissa, in 5 integer operations, no XU conversion
__device__ __forceinline__ double f2d_int(float f) {
  const uint32_t u = __float_as_uint(f);
  const uint32_t hi = ((uint32_t)((int32_t)u >> 3) & 0x8fffffffu) + ((u << 1) ? 0x38000000u : 0u);
  return __hiloint2double((int)hi, (int)(u << 29));
}

// X element -> double in the FP64 narrow pass.  ICVT 0: XU conversions
// (F2F.F64.F32, ~12 cycles per warp instruction per SM: the scarce pipe);
// 1: every 4th element of eta on the XU, the rest and the gradient's on the
// integer ALU (f2d_int); 2: all on the ALU.  1/2 need X without fp32
// subnormals and non-finite values (LogisticArgs::exact_cvt == 0).
template <int ICVT>
__device__ __forceinline__ double cvt_x(float v, int k) {
  if constexpr (ICVT == 0) return (double)v;
  else if constexpr (ICVT == 2) return f2d_int(v);
  else return (k & 3) == 0 ? (double)v : f2d_int(v);
}
__device__ __forceinline__ double2 lds_d2(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}

template <int PMAX, bool FP64, int PE, int LL = 6, int ICVT = 0>
__device__ __noinline__ void logistic_cta_pass(const LogisticArgs& a, const double* __restrict__ theta_s, double* wred,
                                                  double* red_out) {
  extern __shared__ __align__(16) unsigned char ts_dyn_smem[];
  const int lane = threadIdx.x & 31, warp = wk_warp(), nwarps = wk_nwarps();
  const int p = PE > 0 ? PE : a.p;
  constexpr int NA = PMAX + 2;
  // features the loops touch: p itself when it is a compile-time constant
  // (no FMAs on the zero padding), else the padded capacity
  constexpr int KX = PE > 0 ? PE : PMAX;
  WarpPipe& pipe = a.pipe[warp];
  const int count = pipe.count;  // tiles of this warp per pass (static, logistic_pipeline_init)
  const bool prof = a.prof != nullptr && blockIdx.x == 0 && wk_tid() == 0;
  long long pc0 = prof ? clock64() : 0, pc1;
  // loop-invariant launch state in registers: the pipeline's asm statements
  // clobber memory, which would otherwise re-read these fields of `a` (local
  // memory) on every tile
  const int nstage = a.nstage;
  const int stage_bytes = a.stage_bytes;
  const uint32_t ring_off = (uint32_t)(a.stages - ts_dyn_smem) + (uint32_t)(warp * nstage * stage_bytes);
  uint64_t* const bars = a.mbar + warp * nstage;

  using acc_t = typename std::conditional<FP64, double, float>::type;
  acc_t acc[PMAX + 1];
  // log-likelihood terms accumulate in double in both policies: in the FP32
  // policy the per-row term y*eta - (max(eta,0) + log1p(exp(-|eta|))) is
  // evaluated in double from the float eta: float rounding of the term is
  // correlated across rows (identical at q = 0, where every term is log 2),
  // so N float roundings added up to 0.09 nats at 581,012 rows (q = 0) and
  // 2e-3 at the mode; in double |dU| stays below 1e-3 nats
  // (tests/test_gpu_covtype_fp32.py)
  double accl = 0.0;
#pragma unroll
  for (int j = 0; j <= PMAX; ++j) acc[j] = 0;

  float th32[PMAX];
  float thb32 = 0.f;
  const float* thlo = nullptr;  // LL = 5: theta - float(theta) (smem, broadcast loads)
  if constexpr (!FP64) {
    // theta as floats, broadcast with LDS.128: prepared by the driver warp
    // before the post (a.th32), else rounded here once per CTA
    // (addressed through the dynamic-smem symbol: LDS, not generic loads)
    const float* t32 = a.th32 ? reinterpret_cast<const float*>(ts_dyn_smem + (reinterpret_cast<const unsigned char*>(a.th32) - ts_dyn_smem)) : nullptr;
    if (t32 == nullptr || a.pmax != PMAX) {
      float* w32 = reinterpret_cast<float*>(wred);  // wred is free until the end
      for (int j = wk_tid(); j <= PMAX; j += wk_threads()) {
        const double v = (j < p) ? theta_s[j] : (j == PMAX ? theta_s[p] : 0.0);
        w32[j] = (float)v;
        w32[64 + j] = (float)(v - (double)(float)v);
      }
      wk_sync();
      t32 = w32;
    }
#pragma unroll
    for (int j = 0; j < PMAX; j += 4) {
      const float4 v = reinterpret_cast<const float4*>(t32)[j / 4];
      th32[j] = v.x; th32[j + 1] = v.y; th32[j + 2] = v.z; th32[j + 3] = v.w;
    }
    thb32 = t32[PMAX];
    if constexpr (LL == 5) thlo = t32 + 64;
    if (a.th32 == nullptr || a.pmax != PMAX) wk_sync();
  }

  // FP64: theta as doubles through the dynamic-smem symbol (LDS)
  const double* thd = nullptr;
  if constexpr (FP64) thd = reinterpret_cast<const double*>(ts_dyn_smem + (reinterpret_cast<const unsigned char*>(a.thd) - ts_dyn_smem));
  if (count > 0) {
    const unsigned long long c0 = pipe.consumed;
    unsigned long long issued = pipe.issued;
    // 32-bit tile bookkeeping (a warp owns < 2^31 tiles)
    const int tfirst = pipe.first, tstride = nwarps;
    // valid rows of tile t: 32 below the last (partial) tile
    const int nfull = (int)(a.n_rows >> 5), rem = (int)(a.n_rows & 31);
    // producer state, kept in registers by every lane (lane 0 issues)
    const uint32_t xb = 128u * (uint32_t)p;
    const float* const xfirst = a.xt + (int64_t)tfirst * 32 * p;
    const uint8_t* const yfirst = a.yt + (int64_t)tfirst * 32;
    const int64_t xstep = (int64_t)tstride * 32 * p, ystep = (int64_t)tstride * 32;
    const int keep = pipe.keep;
    const uint64_t pol = policy_evict_first(), pol_keep = policy_evict_last();
    int ps = pipe.ps, pj = pipe.pj;
    const float* pxs = xfirst + (int64_t)pj * xstep;
    const uint8_t* pys = yfirst + (int64_t)pj * ystep;
    auto issue = [&]() {
      if (lane == 0) {
        uint64_t* bar = bars + ps;
        unsigned char* dst = ts_dyn_smem + ring_off + (uint32_t)(ps * stage_bytes);
        const uint64_t pl = pj < keep ? pol_keep : pol;
        mbar_expect_tx(bar, xb + 32u);
        bulk_g2s(dst, pxs, xb, bar, pl);
        bulk_g2s(dst + xb, pys, 32u, bar, pl);
      }
      if (++ps == nstage) ps = 0;
      if (++pj == count) { pj = 0; pxs = xfirst; pys = yfirst; }
      else { pxs += xstep; pys += ystep; }
    };
    while (issued < c0 + (unsigned long long)nstage) { issue(); ++issued; }
    // ring position and periodic tile index, advanced incrementally
    int s = pipe.cs, tj = pipe.ctj;
    uint32_t parity = (uint32_t)pipe.cpar;
    if (prof) { pc1 = clock64(); a.prof[4] += pc1 - pc0; pc0 = pc1; }
    for (int j = 0; j < count; ++j) {
      mbar_wait(bars + s, parity);
      const unsigned char* sb = ts_dyn_smem + ring_off + (uint32_t)(s * stage_bytes);
      float x[PMAX];
      uint8_t yb;
      row_from_stage<PMAX, PE>(sb, p, lane, x, yb);
      __syncwarp();
      // stage s is free again: keep the producer NSTAGE tiles ahead (wrapping
      // into the next pass; X is read-only for the whole kernel)
      issue();
      ++issued;
      const int t = tfirst + tj * tstride;
      const bool valid = lane < (t < nfull ? 32 : rem);
      if (++s == nstage) { s = 0; parity ^= 1u; }
      if (++tj == count) tj = 0;
      if constexpr (FP64) {
        // x stays in float registers and is converted where it is used (cvt_x:
        // mostly on the integer ALU, the XU's F2F being the scarce pipe);
        // keeping 54 converted doubles live for the gradient spilled.  theta:
        // broadcast LDS.128 from the driver's zero-padded copy (thd).  The
        // arithmetic (4 FMA chains, then the gradient FMAs) is unchanged.
        double e0 = thd[PMAX], e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll
        for (int k = 0; k < KX; k += 4) {
          const double2 ta = lds_d2(thd + k), tb = lds_d2(thd + k + 2);
          e0 = __fma_rn(cvt_x<ICVT>(x[k], k), ta.x, e0);
          if (k + 1 < KX) e1 = __fma_rn(cvt_x<ICVT>(x[k + 1], k + 1), ta.y, e1);
          if (k + 2 < KX) e2 = __fma_rn(cvt_x<ICVT>(x[k + 2], k + 2), tb.x, e2);
          if (k + 3 < KX) e3 = __fma_rn(cvt_x<ICVT>(x[k + 3], k + 3), tb.y, e3);
        }
        const double eta = (e0 + e1) + (e2 + e3);
        const double e = exp(-fabs(eta));
        const double l = fmax(eta, 0.0) + log1p(e);
        const double sig = __ddiv_rn(eta >= 0.0 ? 1.0 : e, 1.0 + e);
        const double yv = (double)yb;
        const double resid = valid ? yv - sig : 0.0;
        accl += valid ? (yv * eta - l) : 0.0;
#pragma unroll
        for (int k = 0; k < KX; ++k) acc[k] = __fma_rn(resid, cvt_x<ICVT == 0 ? 0 : 2>(x[k], k), acc[k]);
        acc[PMAX] += resid;
      } else {
        float e0 = thb32, e1 = 0.f, e2 = 0.f, e3 = 0.f;
#pragma unroll
        for (int k = 0; k < KX; k += 4) {
          e0 = __fmaf_rn(x[k], th32[k], e0);
          if (k + 1 < KX) e1 = __fmaf_rn(x[k + 1], th32[k + 1], e1);
          if (k + 2 < KX) e2 = __fmaf_rn(x[k + 2], th32[k + 2], e2);
          if (k + 3 < KX) e3 = __fmaf_rn(x[k + 3], th32[k + 3], e3);
        }
        float eta = (e0 + e1) + (e2 + e3);
        if constexpr (LL == 5) {
          // theta's float rounding is common to every row: with the data
          // Hessian ~ 0.2 N it shifted the gradient by ~1e-3 at covtype size.
          // X theta_lo restores it (two more FMA chains, broadcast loads).
          float c0 = thlo[PMAX], c1 = 0.f;
#pragma unroll
          for (int k = 0; k < PMAX; k += 4) {
            const float4 tl = reinterpret_cast<const float4*>(thlo)[k / 4];
            c0 = __fmaf_rn(x[k], tl.x, c0);
            c1 = __fmaf_rn(x[k + 1], tl.y, c1);
            c0 = __fmaf_rn(x[k + 2], tl.z, c0);
            c1 = __fmaf_rn(x[k + 3], tl.w, c1);
          }
          eta += c0 + c1;
        }
        const float e = (LL >= 5) ? exp_neg_f(-fabsf(eta)) : expf(-fabsf(eta));
        // the row's log-likelihood term from the float eta, summed in double
        // (see accl).  LL 6 (default): e without the MUFU (exp_neg_f) and
        // log1p(e) = log 2 + log1p((e - 1)/2) by the atanh series - float
        // round-to-nearest errors only, which average out over rows, and
        // exact at eta = 0; 5: 6 + the theta_lo correction of eta above; 0:
        // expf + log1pf (biased: 2e-3 nats at covtype's mode); 2: exp and
        // log1p in double (A/B reference, +25% pass time).
        double l;
        if constexpr (LL == 0) l = (double)(fmaxf(eta, 0.f) + log1pf(e));
        else if constexpr (LL == 2) l = (double)fmaxf(eta, 0.f) + log1p(exp(-(double)fabsf(eta)));
        else l = (double)fmaxf(eta, 0.f) + ((double)log1p_unit_f(0.5f * (e - 1.0f)) + 0.69314718055994531);
        const float sig = (LL >= 5) ? div_pos_f(eta >= 0.f ? 1.f : e, 1.f + e) : __fdiv_rn(eta >= 0.f ? 1.f : e, 1.f + e);
        const float yv = (float)yb;
        const float resid = valid ? yv - sig : 0.f;
        accl += valid ? ((yb ? (double)eta : 0.0) - l) : 0.0;
#pragma unroll
        for (int k = 0; k < KX; ++k) acc[k] = __fmaf_rn(resid, x[k], acc[k]);
        acc[PMAX] += resid;
      }
    }
    __syncwarp();
    if (lane == 0) {
      pipe.consumed = c0 + (unsigned long long)count;
      pipe.issued = issued;
      pipe.cs = s; pipe.cpar = (int)parity; pipe.ctj = tj;
      pipe.ps = ps; pipe.pj = pj;
    }
    __syncwarp();
  }

  if (prof) { pc1 = clock64(); a.prof[5] += pc1 - pc0; pc0 = pc1; }
  // Warp reduce-scatter (fixed order): NP column sums over 32 lanes in
  // sum(NP/2^k) shuffles instead of 5*NP; lane ends with NP/32 columns.
  constexpr int NP = (NA <= 16) ? 16 : (NA <= 32 ? 32 : (NA <= 64 ? 64 : 128));
  acc_t v[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) v[j] = (j <= PMAX) ? acc[j <= PMAX ? j : PMAX] : (j == PMAX + 1 && FP64 ? (acc_t)accl : (acc_t)0);
  int colbase = 0;
  int cnt = NP;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool upper = (lane & off) != 0;
    if (cnt >= 2) {
      const int n = cnt / 2;
#pragma unroll
      for (int i = 0; i < NP / 2; ++i) {
        if (i < n) {
          const acc_t send = upper ? v[i] : v[n + i];
          const acc_t keep = upper ? v[n + i] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      if (upper) colbase += n;
      cnt = n;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    }
  }
  // lane holds columns colbase .. colbase+cnt-1 (duplicates across lanes when NP < 64)
#pragma unroll
  for (int i = 0; i < NP / 32 + 1; ++i) {
    if (i < cnt && colbase + i < NA && (NP >= 32 || (lane % (32 / NP)) == 0) && (FP64 || colbase + i != PMAX + 1))
      wred[warp * NA + colbase + i] = (double)v[i];
  }
  if constexpr (!FP64) {  // the double log-likelihood sum: its own fixed-order tree
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) accl += __shfl_xor_sync(0xffffffffu, accl, off);
    if (lane == 0) wred[warp * NA + PMAX + 1] = accl;
  }
  if (prof) { pc1 = clock64(); a.prof[6] += pc1 - pc0; pc0 = pc1; }
  wk_sync();
  // CTA reduction in warp order; output index: [0,p) features, p bias, p+1 loglik
  for (int d = wk_tid(); d < p + 2; d += wk_threads()) {
    const int j = (d < p) ? d : (d == p ? PMAX : PMAX + 1);
    double s = 0.0;
    for (int w = 0; w < nwarps; ++w) s += wred[w * NA + j];
    red_out[d] = s;
  }
  if (prof) { pc1 = clock64(); a.prof[7] += pc1 - pc0; }
}

// ------------------------------------------------------ fp64 storage, p <= 64
// Precision "fp64x" with p <= 64 (data that are not fp32-exact, kept in
// double as the reference's LogisticRegressionData does, models.py:43-64):
// 16-row tiles; lane L = 16 h + r holds row r's features [h H, h H + H),
// H = ceil(p / 2), lane-contiguously in groups of 2 doubles (LDS.128,
// conflict-free), then the 16 labels: one TMA bulk copy of 512 G + 16 bytes
// per tile (G = ceil(H / 2) groups; covtype: 7,184 B for 16 rows, +3.7% over
// 8 p bytes per row).  Each lane forms half of eta, one shuffle adds the
// halves, both halves evaluate the row and accumulate the gradient of their
// own features: 27 doubles of x and 27 accumulators per lane at p = 54 (the
// 32-row layout would need 54 + 55 live doubles and spills).
__host__ __device__ inline int x64h_half(int p) { return (p + 1) / 2; }
__host__ __device__ inline int x64h_groups(int p) { return (x64h_half(p) + 1) / 2; }
__host__ __device__ inline int64_t x64h_tile_bytes(int p) { return (int64_t)x64h_groups(p) * 512 + 16; }
__host__ __device__ inline int x64h_stage_bytes(int p) { return (int)((x64h_tile_bytes(p) + 127) / 128 * 128); }
constexpr int kX64hPmax = 64;  // thd capacity (zero padding between p and 64, bias at 64)

// HE > 0: compile-time H (covtype: 27); else runtime H <= 32
template <int HE>
__device__ __noinline__ void logistic_cta_pass_x64h(const LogisticArgs& a, const double* __restrict__ theta_s,
                                                    double* wred, double* red_out) {
  extern __shared__ __align__(16) unsigned char ts_dyn_smem[];
  constexpr int KX = HE > 0 ? ((HE + 1) & ~1) : 32;  // x values per lane (whole groups)
  constexpr int NA = kX64hPmax + 2;
  const int lane = threadIdx.x & 31, warp = wk_warp(), nwarps = wk_nwarps();
  const int p = a.p;
  const int H = HE > 0 ? HE : x64h_half(p);
  const int G = (H + 1) >> 1;
  const int h = lane >> 4, r = lane & 15;
  const int f0 = h * H;
  WarpPipe& pipe = a.pipe[warp];
  const int count = pipe.count;
  const bool prof = a.prof != nullptr && blockIdx.x == 0 && wk_tid() == 0;
  long long pc0 = prof ? clock64() : 0, pc1;
  const int nstage = a.nstage;
  const int stage_bytes = a.stage_bytes;
  const uint32_t ring_off = (uint32_t)(a.stages - ts_dyn_smem) + (uint32_t)(warp * nstage * stage_bytes);
  uint64_t* const bars = a.mbar + warp * nstage;
  // this lane's theta (zero past its features: thd is zero-padded to 64)
  const double* thd = reinterpret_cast<const double*>(ts_dyn_smem + (reinterpret_cast<const unsigned char*>(a.thd) - ts_dyn_smem));
  double th[KX];
#pragma unroll
  for (int k = 0; k < KX; ++k) th[k] = (k < H && f0 + k < p) ? thd[f0 + k] : 0.0;
  const double thb = thd[kX64hPmax];
  double acc[KX];
#pragma unroll
  for (int k = 0; k < KX; ++k) acc[k] = 0.0;
  double accb = 0.0, accl = 0.0;
  if (count > 0) {
    const unsigned long long c0 = pipe.consumed;
    unsigned long long issued = pipe.issued;
    const int tfirst = pipe.first, tstride = nwarps;
    const int nfull = (int)(a.n_rows >> 4), rem = (int)(a.n_rows & 15);
    const uint32_t tb = (uint32_t)x64h_tile_bytes(p);
    const unsigned char* const xfirst = reinterpret_cast<const unsigned char*>(a.xt) + (int64_t)tfirst * tb;
    const int64_t xstep = (int64_t)tstride * tb;
    const int keep = pipe.keep;
    const uint64_t pol = policy_evict_first(), pol_keep = policy_evict_last();
    int ps = pipe.ps, pj = pipe.pj;
    const unsigned char* pxs = xfirst + (int64_t)pj * xstep;
    auto issue = [&]() {
      if (lane == 0) {
        uint64_t* bar = bars + ps;
        unsigned char* dst = ts_dyn_smem + ring_off + (uint32_t)(ps * stage_bytes);
        mbar_expect_tx(bar, tb);
        bulk_g2s(dst, pxs, tb, bar, pj < keep ? pol_keep : pol);
      }
      if (++ps == nstage) ps = 0;
      if (++pj == count) { pj = 0; pxs = xfirst; }
      else pxs += xstep;
    };
    while (issued < c0 + (unsigned long long)nstage) { issue(); ++issued; }
    int s = pipe.cs, tj = pipe.ctj;
    uint32_t parity = (uint32_t)pipe.cpar;
    if (prof) { pc1 = clock64(); a.prof[4] += pc1 - pc0; pc0 = pc1; }
    for (int j = 0; j < count; ++j) {
      mbar_wait(bars + s, parity);
      const unsigned char* sb = ts_dyn_smem + ring_off + (uint32_t)(s * stage_bytes);
      double x[KX];
#pragma unroll
      for (int g = 0; g < KX / 2; ++g) {
        if (HE > 0 || g < G) {
          const double2 v = reinterpret_cast<const double2*>(sb)[g * 32 + lane];
          x[2 * g] = v.x; x[2 * g + 1] = v.y;
        } else {
          x[2 * g] = 0.0; x[2 * g + 1] = 0.0;
        }
      }
      const double yv = (double)sb[512 * G + r];
      __syncwarp();
      issue();
      ++issued;
      const int t = tfirst + tj * tstride;
      const bool valid = r < (t < nfull ? 16 : rem);
      if (++s == nstage) { s = 0; parity ^= 1u; }
      if (++tj == count) tj = 0;
      double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll
      for (int k = 0; k < KX; k += 4) {
        e0 = __fma_rn(x[k], th[k], e0);
        if (k + 1 < KX) e1 = __fma_rn(x[k + 1], th[k + 1], e1);
        if (k + 2 < KX) e2 = __fma_rn(x[k + 2], th[k + 2], e2);
        if (k + 3 < KX) e3 = __fma_rn(x[k + 3], th[k + 3], e3);
      }
      const double part = (e0 + e1) + (e2 + e3);
      const double other = __shfl_xor_sync(0xffffffffu, part, 16);
      // the same association in both halves: (lower + upper) + bias
      const double eta = (h ? other + part : part + other) + thb;
      const double e = exp(-fabs(eta));
      const double l = fmax(eta, 0.0) + log1p(e);
      const double sig = __ddiv_rn(eta >= 0.0 ? 1.0 : e, 1.0 + e);
      const double resid = valid ? yv - sig : 0.0;
      if (h == 0) {
        accl += valid ? (yv * eta - l) : 0.0;
        accb += resid;
      }
#pragma unroll
      for (int k = 0; k < KX; ++k) acc[k] = __fma_rn(resid, x[k], acc[k]);
    }
    __syncwarp();
    if (lane == 0) {
      pipe.consumed = c0 + (unsigned long long)count;
      pipe.issued = issued;
      pipe.cs = s; pipe.cpar = (int)parity; pipe.ctj = tj;
      pipe.ps = ps; pipe.pj = pj;
    }
    __syncwarp();
  }
  if (prof) { pc1 = clock64(); a.prof[5] += pc1 - pc0; pc0 = pc1; }
  // sums over the 16 rows of each half (fixed shuffle tree), lane 0 / 16 write
#pragma unroll
  for (int k = 0; k < KX; ++k) {
    double v = acc[k];
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (r == 0 && k < H && f0 + k < p) wred[warp * NA + f0 + k] = v;
  }
#pragma unroll
  for (int off = 8; off >= 1; off >>= 1) {
    accb += __shfl_xor_sync(0xffffffffu, accb, off);
    accl += __shfl_xor_sync(0xffffffffu, accl, off);
  }
  if (lane == 0) { wred[warp * NA + kX64hPmax] = accb; wred[warp * NA + kX64hPmax + 1] = accl; }
  if (prof) { pc1 = clock64(); a.prof[6] += pc1 - pc0; pc0 = pc1; }
  wk_sync();
  for (int d = wk_tid(); d < p + 2; d += wk_threads()) {
    const int jj = (d < p) ? d : (d == p ? kX64hPmax : kX64hPmax + 1);
    double sum = 0.0;
    for (int w = 0; w < nwarps; ++w) sum += wred[w * NA + jj];
    red_out[d] = sum;
  }
  if (prof) { pc1 = clock64(); a.prof[7] += pc1 - pc0; }
}

// ------------------------------------------- fp64 policy on fp32 X, p <= 64
// Paired half-row tiles (LogisticArgs::xh == 2): a 32-row tile holds two
// 16-row blocks in the half-row layout above with groups of 4 floats (block
// A = rows 0-15, B = rows 16-31), then the 32 labels in row order
// (covtype: 7,200 B per 32 rows, +4.2% over 4 p 32 + 32).  Lane 16 h + r
// forms half of eta for row r of both blocks (theta in 28 registers), one
// shuffle per block joins the halves, and then lane L evaluates the
// exp / log1p / division of tile row L alone -- each row's transcendental
// work done once, not twice as with one block per stage -- and two
// shuffles hand the residuals back to the half-row lanes for the gradient.
// Against the 32-row layout (54 x, 55 accumulators, theta by LDS per row)
// this halves the instructions per row.
__host__ __device__ inline int pair_groups(int p) { return (x64h_half(p) + 3) / 4; }
__host__ __device__ inline int64_t pair_tile_bytes(int p) { return 2 * (int64_t)pair_groups(p) * 512 + 32; }
__host__ __device__ inline int pair_stage_bytes(int p) { return (int)((pair_tile_bytes(p) + 127) / 128 * 128); }

template <int HE>
__device__ __noinline__ void logistic_cta_pass_pair(const LogisticArgs& a, const double* __restrict__ theta_s,
                                                    double* wred, double* red_out) {
  extern __shared__ __align__(16) unsigned char ts_dyn_smem[];
  constexpr int KX = HE > 0 ? ((HE + 3) / 4) * 4 : 32;  // x values per lane per block (whole groups)
  constexpr int NA = kX64hPmax + 2;
  const int lane = threadIdx.x & 31, warp = wk_warp(), nwarps = wk_nwarps();
  const int p = a.p;
  const int H = HE > 0 ? HE : x64h_half(p);
  const int G = (H + 3) / 4;
  const int h = lane >> 4, r = lane & 15;
  const int f0 = h * H;
  WarpPipe& pipe = a.pipe[warp];
  const int count = pipe.count;
  const bool prof = a.prof != nullptr && blockIdx.x == 0 && wk_tid() == 0;
  long long pc0 = prof ? clock64() : 0, pc1;
  const int nstage = a.nstage;
  const int stage_bytes = a.stage_bytes;
  const uint32_t ring_off = (uint32_t)(a.stages - ts_dyn_smem) + (uint32_t)(warp * nstage * stage_bytes);
  uint64_t* const bars = a.mbar + warp * nstage;
  const double* thd = reinterpret_cast<const double*>(ts_dyn_smem + (reinterpret_cast<const unsigned char*>(a.thd) - ts_dyn_smem));
  // theta per half, 16-B aligned and zero past each half's features: thh[h][32]
  // (after the driver's zero-padded copy in red_s); broadcast LDS.128 in the
  // loop instead of 56 registers (which spilled)
  double* thh = const_cast<double*>(thd) + 66;
  for (int i = wk_tid(); i < 64; i += wk_threads()) {
    const int hh = i >> 5, k = i & 31;
    thh[i] = (k < H && hh * H + k < p) ? thd[hh * H + k] : 0.0;
  }
  wk_sync();
  const uint32_t th_addr = smem_u32(thh + 32 * h);
  const double thb = thd[kX64hPmax];
  double acc[KX];
#pragma unroll
  for (int k = 0; k < KX; ++k) acc[k] = 0.0;
  double accb = 0.0, accl = 0.0;
  const int blk = G * 512;  // bytes per 16-row block
  if (count > 0) {
    const unsigned long long c0 = pipe.consumed;
    unsigned long long issued = pipe.issued;
    const int tfirst = pipe.first, tstride = nwarps;
    const int nfull = (int)(a.n_rows >> 5), rem = (int)(a.n_rows & 31);
    const uint32_t tb = (uint32_t)pair_tile_bytes(p);
    const unsigned char* const xfirst = reinterpret_cast<const unsigned char*>(a.xt) + (int64_t)tfirst * tb;
    const int64_t xstep = (int64_t)tstride * tb;
    const int keep = pipe.keep;
    const uint64_t pol = policy_evict_first(), pol_keep = policy_evict_last();
    int ps = pipe.ps, pj = pipe.pj;
    const unsigned char* pxs = xfirst + (int64_t)pj * xstep;
    auto issue = [&]() {
      if (lane == 0) {
        uint64_t* bar = bars + ps;
        unsigned char* dst = ts_dyn_smem + ring_off + (uint32_t)(ps * stage_bytes);
        mbar_expect_tx(bar, tb);
        bulk_g2s(dst, pxs, tb, bar, pj < keep ? pol_keep : pol);
      }
      if (++ps == nstage) ps = 0;
      if (++pj == count) { pj = 0; pxs = xfirst; }
      else pxs += xstep;
    };
    while (issued < c0 + (unsigned long long)nstage) { issue(); ++issued; }
    int s = pipe.cs, tj = pipe.ctj;
    uint32_t parity = (uint32_t)pipe.cpar;
    if (prof) { pc1 = clock64(); a.prof[4] += pc1 - pc0; pc0 = pc1; }
    for (int j = 0; j < count; ++j) {
      mbar_wait(bars + s, parity);
      const unsigned char* sb = ts_dyn_smem + ring_off + (uint32_t)(s * stage_bytes);
      float xa[KX], xb[KX];
#pragma unroll
      for (int g = 0; g < KX / 4; ++g) {
        if (HE > 0 || g < G) {
          const float4 va = reinterpret_cast<const float4*>(sb)[g * 32 + lane];
          const float4 vb = reinterpret_cast<const float4*>(sb + blk)[g * 32 + lane];
          xa[4 * g] = va.x; xa[4 * g + 1] = va.y; xa[4 * g + 2] = va.z; xa[4 * g + 3] = va.w;
          xb[4 * g] = vb.x; xb[4 * g + 1] = vb.y; xb[4 * g + 2] = vb.z; xb[4 * g + 3] = vb.w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) { xa[4 * g + u] = 0.f; xb[4 * g + u] = 0.f; }
        }
      }
      const double yv = (double)sb[2 * blk + lane];  // label of tile row `lane`
      __syncwarp();
      issue();
      ++issued;
      const int t = tfirst + tj * tstride;
      const bool valid = lane < (t < nfull ? 32 : rem);
      if (++s == nstage) { s = 0; parity ^= 1u; }
      if (++tj == count) tj = 0;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
#pragma unroll
      for (int k = 0; k < KX; k += 4) {
        double2 t01, t23;  // volatile loads: not hoisted into 56 registers
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(t01.x), "=d"(t01.y) : "r"(th_addr + 8u * k));
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(t23.x), "=d"(t23.y) : "r"(th_addr + 8u * (k + 2)));
        a0 = __fma_rn((double)xa[k], t01.x, a0);
        a1 = __fma_rn((double)xa[k + 1], t01.y, a1);
        a2 = __fma_rn((double)xa[k + 2], t23.x, a2);
        a3 = __fma_rn((double)xa[k + 3], t23.y, a3);
        b0 = __fma_rn((double)xb[k], t01.x, b0);
        b1 = __fma_rn((double)xb[k + 1], t01.y, b1);
        b2 = __fma_rn((double)xb[k + 2], t23.x, b2);
        b3 = __fma_rn((double)xb[k + 3], t23.y, b3);
      }
      const double pa = (a0 + a1) + (a2 + a3), pb = (b0 + b1) + (b2 + b3);
      const double oa = __shfl_xor_sync(0xffffffffu, pa, 16), ob = __shfl_xor_sync(0xffffffffu, pb, 16);
      // the same association in both halves: (lower + upper) + bias
      const double eta_a = (h ? oa + pa : pa + oa) + thb, eta_b = (h ? ob + pb : pb + ob) + thb;
      // lane L evaluates tile row L: block A's row L (L < 16), block B's row L - 16
      const double eta = h ? eta_b : eta_a;
      const double e = exp(-fabs(eta));
      const double l = fmax(eta, 0.0) + log1p(e);
      const double sig = __ddiv_rn(eta >= 0.0 ? 1.0 : e, 1.0 + e);
      const double resid = valid ? yv - sig : 0.0;
      accl += valid ? (yv * eta - l) : 0.0;
      accb += resid;
      const double ra = __shfl_sync(0xffffffffu, resid, r), rb = __shfl_sync(0xffffffffu, resid, 16 + r);
#pragma unroll
      for (int k = 0; k < KX; ++k) {
        acc[k] = __fma_rn(ra, (double)xa[k], acc[k]);
        acc[k] = __fma_rn(rb, (double)xb[k], acc[k]);
      }
    }
    __syncwarp();
    if (lane == 0) {
      pipe.consumed = c0 + (unsigned long long)count;
      pipe.issued = issued;
      pipe.cs = s; pipe.cpar = (int)parity; pipe.ctj = tj;
      pipe.ps = ps; pipe.pj = pj;
    }
    __syncwarp();
  }
  if (prof) { pc1 = clock64(); a.prof[5] += pc1 - pc0; pc0 = pc1; }
  // gradient: sums over the 16 rows of each half (fixed shuffle tree), lane 0 / 16 write
#pragma unroll
  for (int k = 0; k < KX; ++k) {
    double v = acc[k];
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (r == 0 && k < H && f0 + k < p) wred[warp * NA + f0 + k] = v;
  }
  // residual and log-likelihood: one row per lane, sums over all 32 lanes
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    accb += __shfl_xor_sync(0xffffffffu, accb, off);
    accl += __shfl_xor_sync(0xffffffffu, accl, off);
  }
  if (lane == 0) { wred[warp * NA + kX64hPmax] = accb; wred[warp * NA + kX64hPmax + 1] = accl; }
  if (prof) { pc1 = clock64(); a.prof[6] += pc1 - pc0; pc0 = pc1; }
  wk_sync();
  for (int d = wk_tid(); d < p + 2; d += wk_threads()) {
    const int jj = (d < p) ? d : (d == p ? kX64hPmax : kX64hPmax + 1);
    double sum = 0.0;
    for (int w = 0; w < nwarps; ++w) sum += wred[w * NA + jj];
    red_out[d] = sum;
  }
  if (prof) { pc1 = clock64(); a.prof[7] += pc1 - pc0; }
}

// ---------------------------------------------------------------- wide p
// p in (64, kWideMax]: a tile is kWideRows = 8 rows in the input's row-major
// order followed by 16 bytes holding the 8 labels (+ 8 zero bytes): one TMA
// bulk copy of 32p+16 bytes.  kWideGroup = 4 consecutive tiles (32 rows)
// form a group, the unit of work assignment and of exact accumulation: each
// worker warp owns whole groups (periodic sequence, run-ahead producer as for
// p <= 64) and streams their tiles through its own ring.
//
// Per tile, in two halves of 4 rows: lane l holds features l, l+32, ... of
// each row in registers (conflict-free LDS from the row-major stage), forms 4
// partial dot products, and a reduce-scatter over the warp (6 shuffles for 4
// rows) leaves each lane with the full sum of one row; that lane evaluates
// the row's sigmoid / log1pexp, 4 shuffles broadcast the residuals, and the
// gradient contributions accumulate per lane from the same registers.  No
// CTA synchronisation inside the pass; each X element is read from shared
// memory (and in the FP64 policy converted to double) exactly once.
//
// Exactness: a group's partial sums (fp32 or fp64 in the policy's type) are
// converted to fixed-point pairs (fx_split) and added as integers, so the
// totals do not depend on which warp, CTA or GPU processed a group: row
// shards aligned to groups reproduce the single-GPU totals bit for bit.
constexpr int kWideMax = 256;
constexpr int kWideRows = 8;
constexpr int kWideGroup = 4;
constexpr int kWideTotWords = 2 * (kWideMax + 2) + 2;  // CTA totals at the start of wred (16-B multiple)
// wred doubles the wide pass needs: totals + lane-private accumulator slots
__host__ __device__ inline int wide_scratch_doubles(int worker_warps) {
  return kWideTotWords + worker_warps * (kWideMax / 32 + 2) * 32 * 2;
}
// esz: bytes per X element (4: fp32 storage; 8: fp64 storage, "fp64x")
__host__ __device__ inline int64_t wide_tile_bytes(int p, int esz = 4) { return kWideRows * esz * (int64_t)p + 16; }
__host__ __device__ inline int wide_kl(int p, int esz) { return (esz == 8 && p <= 64) ? 2 : (p <= 128 ? 4 : 8); }
// ring stage: the tile plus zeroed slack covering the pass's unconditional
// reads (row 7, features up to 32*KL - 1), 128-byte multiple
__host__ __device__ inline int wide_stage_bytes(int p, int esz = 4) {
  const int kl = wide_kl(p, esz);
  int64_t b = wide_tile_bytes(p, esz);
  const int64_t reach = esz * (int64_t)((kWideRows - 1) * p + 32 * kl);
  if (reach > b) b = reach;
  return (int)((b + 127) / 128 * 128);
}

struct WideProducer {
  const unsigned char* src;    // next tile to issue
  const unsigned char* first;  // this warp's first tile
  int64_t gstep;               // bytes from one of this warp's groups to the next
  int64_t gj, count;           // group index within the warp's sequence, group count
  int k;                       // tile within the group
  int s, nstage;
  uint32_t tb, ring, bars;     // tile bytes; shared addresses of the ring and its mbarriers
  uint32_t stage_bytes;
  uint64_t pol;

  __device__ __forceinline__ void init(const LogisticArgs& a, const WarpTiles& wt, unsigned long long issued) {
    const int warp = wk_warp();
    nstage = a.nstage;
    stage_bytes = (uint32_t)a.stage_bytes;
    ring = smem_u32(a.stages) + (uint32_t)(warp * nstage) * stage_bytes;
    bars = smem_u32(a.mbar + warp * nstage);
    s = (int)(umod(issued, nstage));
    count = wt.count;
    const unsigned long long i = umod(issued, (uint32_t)(count * kWideGroup));
    gj = (int64_t)(i / kWideGroup);
    k = (int)(i % kWideGroup);
    tb = (uint32_t)wide_tile_bytes(a.p, a.xd ? 8 : 4);
    first = reinterpret_cast<const unsigned char*>(a.xt) + wt.first * kWideGroup * (int64_t)tb;
    gstep = (int64_t)wt.nwarps * kWideGroup * tb;
    src = first + gj * gstep + (int64_t)k * tb;
    pol = policy_evict_first();
  }
  __device__ __forceinline__ void issue() {
    const uint32_t bar = bars + 8u * (uint32_t)s;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tb) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            ring + (uint32_t)s * stage_bytes),
        "l"(src), "r"(tb), "r"(bar), "l"(pol)
        : "memory");
    if (++s == nstage) s = 0;
    if (++k == kWideGroup) {
      k = 0;
      if (++gj == count) { gj = 0; src = first; }
      else src += gstep - (int64_t)(kWideGroup - 1) * tb;
    } else {
      src += tb;
    }
  }
};

// KL = features per lane (p <= 32 KL); ICVT: 1 odd m / 2 all on the ALU;
// XD: X stored as fp64 (the "fp64x" policy: data that are not fp32-exact)
template <bool FP64, int KL, int ICVT = 0, bool XD = false>
__device__ __noinline__ void logistic_cta_pass_wide(const LogisticArgs& a, const double* __restrict__ theta_s,
                                                    double* wred, double* red_out) {
  using acc_t = typename std::conditional<FP64, double, float>::type;
  extern __shared__ __align__(16) unsigned char ts_dyn_smem[];
  constexpr int R = 4;  // rows per half tile
  const int lane = threadIdx.x & 31, warp = wk_warp();
  const int p = a.p;
  const int64_t n_rows = a.n_rows;
  const int nstage = a.nstage;
  const int stage_bytes = a.stage_bytes;
  // work assignment in groups of kWideGroup tiles
  WarpTiles wt;
  {
    const int nwarps = wk_nwarps();
    const int64_t G = a.ncta, ng = a.u_hi - a.u_lo;
    const int64_t g_begin = a.u_lo + (ng * (int64_t)a.cta) / G, g_end = a.u_lo + (ng * ((int64_t)a.cta + 1)) / G;
    wt.first = g_begin + warp;
    wt.count = (g_end - wt.first + nwarps - 1) / nwarps;
    if (wt.count < 0) wt.count = 0;
    wt.nwarps = nwarps;
  }
  const bool prof = a.prof != nullptr && blockIdx.x == 0 && wk_tid() == 0;
  long long pc0 = prof ? clock64() : 0, pc1;

  bool fvalid[KL];
  acc_t th[KL];
#pragma unroll
  for (int m = 0; m < KL; ++m) {
    fvalid[m] = lane + 32 * m < p;
    th[m] = fvalid[m] ? (acc_t)theta_s[lane + 32 * m] : (acc_t)0;
  }
  const acc_t thb = (acc_t)theta_s[p];
  // exact fixed-point accumulators: [0, KL) features lane + 32 m, KL the
  // residual sum, KL + 1 the log-likelihood (nonzero on lanes 0, 8, 16, 24)
  // (lane-private slots in shared memory: [warp][NF][32 lanes] (hi, signed lo)
  // pairs, touched once per group, so they cost no registers in the loop)
  constexpr int NF = KL + 2;
  bool bad = false;
  unsigned long long* tot = reinterpret_cast<unsigned long long*>(wred);  // CTA totals [2*(p+2)] + flag
  ulonglong2* fx = reinterpret_cast<ulonglong2*>(wred + kWideTotWords) + (warp * NF) * 32 + lane;
#pragma unroll
  for (int m = 0; m < NF; ++m) fx[32 * m] = make_ulonglong2(0ULL, 0ULL);
  for (int i = wk_tid(); i < 2 * (p + 2) + 1; i += wk_threads()) tot[i] = 0ULL;
  wk_sync();
  // after the reduce-scatter, lane holds row (bit 4, bit 3) of a half tile
  const int my_r = ((lane >> 3) & 2) | ((lane >> 3) & 1);
  const bool up16 = (lane & 16) != 0, up8 = (lane & 8) != 0;

  if (wt.count > 0) {
    WarpPipe& pipe = a.pipe[warp];
    const unsigned long long c0 = pipe.consumed;
    unsigned long long issued = pipe.issued;
    const int64_t ntile_w = wt.count * kWideGroup;  // tiles of this warp per pass
    WideProducer prod;
    if (lane == 0) {
      prod.init(a, wt, issued);
      while (issued < c0 + (unsigned long long)nstage) { prod.issue(); ++issued; }
    }
    int s = (int)(umod(c0, nstage));
    uint32_t parity = udiv(c0, nstage) & 1u;
    const unsigned long long i0 = umod(c0, (uint32_t)ntile_w);
    int64_t gj = (int64_t)(i0 / kWideGroup);
    int k = (int)(i0 % kWideGroup);
    const uint32_t ring_off = (uint32_t)(a.stages - ts_dyn_smem) + (uint32_t)(warp * nstage * stage_bytes);
    uint64_t* bars = a.mbar + warp * nstage;
    // group-level partial sums in the policy's type (folded exactly per group)
    acc_t gacc[NF];
#pragma unroll
    for (int m = 0; m < NF; ++m) gacc[m] = 0;
    if (prof) { pc1 = clock64(); a.prof[4] += pc1 - pc0; pc0 = pc1; }
    for (int64_t j = 0; j < ntile_w; ++j) {
      mbar_wait(bars + s, parity);
      const unsigned char* sb = ts_dyn_smem + ring_off + (uint32_t)(s * stage_bytes);
      using xel_t = typename std::conditional<XD, double, float>::type;
      const xel_t* xs = reinterpret_cast<const xel_t*>(sb);
      const int64_t row0 = ((wt.first + gj * wt.nwarps) * kWideGroup + k) * kWideRows;
#pragma unroll
      for (int g = 0; g < kWideRows; g += R) {
        acc_t xv[R][KL];
        // unconditional loads: features past p read the next row / the
        // label bytes / the stage's zeroed slack (finite values, see
        // wide_stage_bytes); they meet theta = 0 in eta and their gradient
        // slots are dropped at the fold
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const xel_t* xr = xs + (g + r) * p + lane;
#pragma unroll
          for (int m = 0; m < KL; ++m) {
            if constexpr (FP64 && ICVT > 0 && !XD) xv[r][m] = (ICVT == 2 || (m & 1)) ? (acc_t)f2d_int(xr[32 * m]) : (acc_t)xr[32 * m];
            else xv[r][m] = (acc_t)xr[32 * m];
          }
        }
        const int yr = g + my_r;
        const acc_t yv = (acc_t)sb[kWideRows * (int)sizeof(xel_t) * p + yr];
        if (g + R == kWideRows) {
          // the stage is fully read: refill it (wrapping into the next pass)
          __syncwarp();
          if (lane == 0) { prod.issue(); ++issued; }
        }
        acc_t e[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          acc_t a0 = 0, a1 = 0;
#pragma unroll
          for (int m = 0; m < KL; m += 2) {
            if constexpr (FP64) {
              a0 = __fma_rn(xv[r][m], th[m], a0);
              a1 = __fma_rn(xv[r][m + 1], th[m + 1], a1);
            } else {
              a0 = __fmaf_rn(xv[r][m], th[m], a0);
              a1 = __fmaf_rn(xv[r][m + 1], th[m + 1], a1);
            }
          }
          e[r] = a0 + a1;
        }
        // reduce-scatter of 4 row sums over the warp (fixed order)
        acc_t k0 = up16 ? e[2] : e[0], k1 = up16 ? e[3] : e[1];
        k0 += __shfl_xor_sync(0xffffffffu, up16 ? e[0] : e[2], 16);
        k1 += __shfl_xor_sync(0xffffffffu, up16 ? e[1] : e[3], 16);
        acc_t kk = up8 ? k1 : k0;
        kk += __shfl_xor_sync(0xffffffffu, up8 ? k0 : k1, 8);
        kk += __shfl_xor_sync(0xffffffffu, kk, 4);
        kk += __shfl_xor_sync(0xffffffffu, kk, 2);
        kk += __shfl_xor_sync(0xffffffffu, kk, 1);
        const acc_t eta = kk + thb;
        const bool valid = row0 + yr < n_rows;
        acc_t resid, llt;
        if constexpr (FP64) {
          const double ex = exp(-fabs(eta));
          const double l = fmax(eta, 0.0) + log1p(ex);
          const double sig = __ddiv_rn(eta >= 0.0 ? 1.0 : ex, 1.0 + ex);
          resid = valid ? yv - sig : 0.0;
          llt = valid ? (yv * eta - l) : 0.0;
        } else {
          // branch-free fast intrinsics (FP32 policy tolerance)
          const float ex = __expf(-fabsf(eta));
          const float op = 1.f + ex;
          const float l = fmaxf(eta, 0.f) + __logf(op);
          const float sig = __fdividef(eta >= 0.f ? 1.f : ex, op);
          resid = valid ? yv - sig : 0.f;
          llt = valid ? __fmaf_rn(yv, eta, -l) : 0.f;
        }
        if ((lane & 7) == 0) { gacc[KL] += resid; gacc[KL + 1] += llt; }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const acc_t rr = __shfl_sync(0xffffffffu, resid, ((r >> 1) << 4) | ((r & 1) << 3));
#pragma unroll
          for (int m = 0; m < KL; ++m) {
            if constexpr (FP64) gacc[m] = __fma_rn(rr, xv[r][m], gacc[m]);
            else gacc[m] = __fmaf_rn(rr, xv[r][m], gacc[m]);
          }
        }
      }
      if (++s == nstage) { s = 0; parity ^= 1u; }
      if (++k == kWideGroup) {  // group done: exact fold
        k = 0;
        if (++gj == wt.count) gj = 0;
#pragma unroll
        for (int m = 0; m < NF; ++m) {
          long long h, l;
          const bool keep = m >= KL || fvalid[m < KL ? m : 0];
          bad |= !fx_split(keep ? (double)gacc[m] : 0.0, h, l);
          ulonglong2 v = fx[32 * m];
          v.x += (unsigned long long)h;
          v.y += (unsigned long long)l;
          fx_canon(v.x, v.y);
          fx[32 * m] = v;
          gacc[m] = 0;
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      pipe.consumed = c0 + (unsigned long long)ntile_w;
      pipe.issued = issued;
    }
    __syncwarp();
  }
  if (prof) { pc1 = clock64(); a.prof[5] += pc1 - pc0; pc0 = pc1; }
  // CTA totals: shared-memory integer atomics (order-free)
#pragma unroll
  for (int m = 0; m < KL; ++m) {
    if (fvalid[m]) {
      const ulonglong2 v = fx[32 * m];
      atomicAdd(tot + 2 * (lane + 32 * m), v.x);
      atomicAdd(tot + 2 * (lane + 32 * m) + 1, v.y);
    }
  }
  if ((lane & 7) == 0) {
    const ulonglong2 b = fx[32 * KL], l = fx[32 * (KL + 1)];
    atomicAdd(tot + 2 * p, b.x);
    atomicAdd(tot + 2 * p + 1, b.y);
    atomicAdd(tot + 2 * p + 2, l.x);
    atomicAdd(tot + 2 * p + 3, l.y);
  }
  if (bad) atomicOr(tot + 2 * (p + 2), 1ULL);
  if (prof) { pc1 = clock64(); a.prof[7] += pc1 - pc0; }
}

static __device__ __forceinline__ void logistic_cta_dispatch(const LogisticArgs& a, const double* theta, double* wred,
                                                             double* red_s) {
  if (a.xh == 1) {  // fp64 storage, p <= 64
    if (a.p == 54) logistic_cta_pass_x64h<27>(a, theta, wred, red_s);
    else logistic_cta_pass_x64h<0>(a, theta, wred, red_s);
    return;
  }
  if (a.xh == 2) {  // fp64 policy on fp32 X, p <= 64: paired half-row tiles
    if (a.p == 54) logistic_cta_pass_pair<27>(a, theta, wred, red_s);
    else logistic_cta_pass_pair<0>(a, theta, wred, red_s);
    return;
  }
  if (a.wide) {
    if (a.xd) {  // fp64 X storage (always the fp64 policy)
      if (a.p <= 64) logistic_cta_pass_wide<true, 2, 0, true>(a, theta, wred, red_s);
      else if (a.p <= 128) logistic_cta_pass_wide<true, 4, 0, true>(a, theta, wred, red_s);
      else logistic_cta_pass_wide<true, 8, 0, true>(a, theta, wred, red_s);
      return;
    }
    if (a.p <= 128) {
      if (a.fp64) logistic_cta_pass_wide<true, 4>(a, theta, wred, red_s);
      else logistic_cta_pass_wide<false, 4>(a, theta, wred, red_s);
    } else {
      if (a.fp64 && !a.exact_cvt && a.icvt == 1) logistic_cta_pass_wide<true, 8, 1>(a, theta, wred, red_s);
      else if (a.fp64 && !a.exact_cvt && a.icvt == 2) logistic_cta_pass_wide<true, 8, 2>(a, theta, wred, red_s);
      else if (a.fp64) logistic_cta_pass_wide<true, 8>(a, theta, wred, red_s);
      else logistic_cta_pass_wide<false, 8>(a, theta, wred, red_s);
    }
    return;
  }
  if (a.p == 54) {  // covtype's feature count: compile-time row layout
    if (a.fp64 && !a.exact_cvt && a.icvt == 1) logistic_cta_pass<56, true, 54, 6, 1>(a, theta, wred, red_s);
    else if (a.fp64 && !a.exact_cvt && a.icvt == 2) logistic_cta_pass<56, true, 54, 6, 2>(a, theta, wred, red_s);
    else if (a.fp64) logistic_cta_pass<56, true, 54>(a, theta, wred, red_s);
    else if (a.llmode == 0) logistic_cta_pass<56, false, 54, 0>(a, theta, wred, red_s);
    else if (a.llmode == 2) logistic_cta_pass<56, false, 54, 2>(a, theta, wred, red_s);
    else if (a.llmode == 5) logistic_cta_pass<56, false, 54, 5>(a, theta, wred, red_s);
    else logistic_cta_pass<56, false, 54, 6>(a, theta, wred, red_s);
    return;
  }
  switch (a.pmax * 2 + (a.fp64 ? 1 : 0)) {
    case 16: logistic_cta_pass<8, false, 0>(a, theta, wred, red_s); break;
    case 17:
      if (!a.exact_cvt && a.icvt) logistic_cta_pass<8, true, 0, 6, 2>(a, theta, wred, red_s);
      else logistic_cta_pass<8, true, 0>(a, theta, wred, red_s);
      break;
    case 64: logistic_cta_pass<32, false, 0>(a, theta, wred, red_s); break;
    case 65:
      if (!a.exact_cvt && a.icvt) logistic_cta_pass<32, true, 0, 6, 1>(a, theta, wred, red_s);
      else logistic_cta_pass<32, true, 0>(a, theta, wred, red_s);
      break;
    case 112: logistic_cta_pass<56, false, 0>(a, theta, wred, red_s); break;
    case 113:
      if (!a.exact_cvt && a.icvt) logistic_cta_pass<56, true, 0, 6, 1>(a, theta, wred, red_s);
      else logistic_cta_pass<56, true, 0>(a, theta, wred, red_s);
      break;
    case 128: logistic_cta_pass<64, false, 0>(a, theta, wred, red_s); break;
    case 129:
      if (!a.exact_cvt && a.icvt) logistic_cta_pass<64, true, 0, 6, 1>(a, theta, wred, red_s);
      else logistic_cta_pass<64, true, 0>(a, theta, wred, red_s);
      break;
    default: break;
  }
}

// Full logistic evaluation over the grid for q (vector qid): leaves U in
// red_s (U = red_s[1] - red_s[0]) and the gradient in vector gid.  `epoch`
// counts grid barriers already passed by this kernel (identical in every
// CTA).  Called by the WORKER warps of the CTA.
// (theta and g: contiguous vectors in shared memory)
static __device__ void logistic_eval_grid(const LogisticArgs& a, const double* theta, double* g, double* wred,
                                          double* red_s, unsigned long long& epoch) {
  const int p = a.p;
  const int P2 = p + 2;
  const int64_t G = a.ncta;  // CTAs of this rank
  const bool prof = a.prof != nullptr && blockIdx.x == 0 && wk_tid() == 0;
  long long c0 = prof ? clock64() : 0, c1;
  // TS_PROF per-CTA skew: [24 + 2 b] += pass ns, [25 + 2 b] += barrier-wait ns (globaltimer)
  const bool skew = a.prof != nullptr && wk_tid() == 0;
  unsigned long long g0 = 0, g1 = 0, g2 = 0;
  if (skew) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));

  logistic_cta_dispatch(a, theta, wred, red_s);
  wk_sync();
  if (prof) { c1 = clock64(); a.prof[1] += c1 - c0; c0 = c1; }
  if (skew) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  // Cross-CTA sum by exact fixed-point atomics into accumulator buffer
  // epoch % 3 (see fx_split): integer addition is associative, so the result
  // is independent of the order in which CTAs arrive -- deterministic.
  unsigned long long* accb = reinterpret_cast<unsigned long long*>(a.pbuf);
  const int64_t bstride = 2 * (int64_t)P2 + 2;  // words of one set of totals (mailbox slots)
  const int64_t cstride = fx_copy_stride(p), bufw = fx_buf_words(p);
  unsigned long long* const curb = accb + (int64_t)(epoch % 3ULL) * bufw;  // this pass's buffer
  const int ncopy = a.fxc;  // copies in use (<= kFxCopies; buffers are sized for kFxCopies)
  unsigned long long* cur = curb + (int64_t)(a.cta % ncopy) * cstride;  // this CTA's copy
  // total of word w over the copies (after the barrier)
  auto total = [&](int w) {
    unsigned long long v = 0;
#pragma unroll
    for (int c = 0; c < kFxCopies; ++c)
      if (c < ncopy) v += __ldcg(curb + c * cstride + w);
    return v;
  };
  if (a.wide) {  // the wide pass leaves exact fixed-point CTA totals in wred
    const unsigned long long* tot = reinterpret_cast<const unsigned long long*>(wred);
    for (int d = wk_tid(); d < P2; d += wk_threads()) {
      unsigned long long hi = tot[2 * d], lo = tot[2 * d + 1];
      fx_canon(hi, lo);
      red_add_u64(cur + 2 * d, hi);
      red_add_u64(cur + 2 * d + 1, lo);
    }
    if (wk_tid() == 0 && tot[2 * P2] != 0ULL) red_add_u64(cur + 2 * P2, 1ULL);
  } else {
    for (int d = wk_tid(); d < P2; d += wk_threads()) {
      long long hi, lo;
      const bool ok = fx_split(red_s[d], hi, lo);
      red_add_u64(cur + 2 * d, (unsigned long long)hi);
      red_add_u64(cur + 2 * d + 1, (unsigned long long)lo);
      if (!ok) red_add_u64(cur + 2 * P2, 1ULL);  // non-finite / out-of-range partial
    }
  }
  wk_sync();
  if (wk_tid() == 0) {
    if (G > 1 && !(a.fault == 1 && a.cta == 1)) red_release_add_u64(a.bar, 1ULL);
    // prior term 0.5 |theta|^2 (kernels.py:92-95), computed by the thread
    // that waits at the barrier anyway (left to right, bias first)
    double pr = 0.5 * theta[p] * theta[p];
    for (int d = 0; d < p; ++d) pr += 0.5 * theta[d] * theta[d];
    red_s[1] = pr;
    if (G > 1) {
      const unsigned long long target = (epoch + 1) * (unsigned long long)G;
      SpinGuard sg(a.err, a.spin_ns);
      // relaxed polling, then one acquire load (instead of a full fence)
      while (ld_relaxed_u64(a.bar) < target) {
        if (sg.expired()) break;
      }
      (void)ld_acquire_u64(a.bar);
    }
  }
  wk_sync();
  // buffer (epoch+2)%3 was last read before this barrier by every CTA and is
  // next accumulated after the following barrier: CTA 0 clears it now.
  {  // every CTA clears its share (a CTA-0-only clear made CTA 0 the last to start the next pass)
    unsigned long long* nxt = accb + (int64_t)((epoch + 2) % 3ULL) * bufw;
    const int64_t used = (int64_t)ncopy * cstride;
    for (int64_t i = (int64_t)a.cta * wk_threads() + wk_tid(); i < used; i += (int64_t)G * wk_threads()) nxt[i] = 0ULL;
  }
  epoch += 1;
  if (prof) { c1 = clock64(); a.prof[2] += c1 - c0; c0 = c1; }
  if (skew && blockIdx.x < 2048) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g2));
    a.prof[24 + 2 * blockIdx.x] += g1 - g0;
    a.prof[25 + 2 * blockIdx.x] += g2 - g1;
  }

  if (a.dump && epoch == 1 && blockIdx.x == 0)  // test hook: this GPU's totals of the first pass
    for (int i = wk_tid(); i < 2 * P2 + 1; i += wk_threads()) a.dump[i] = total(i);

  if (a.world > 0) {
    // Row sharding across GPUs: CTA 0 pushes this GPU's totals into slot
    // x % 3 of every rank's mailbox (NVLink stores to peer memory), then
    // raises its flag there; every CTA waits for all `world` flags of pass x
    // and adds the copies -- integer sums, so every rank gets the same bits.
    // A slot is rewritten 3 passes later, when every rank has consumed it.
    const int W = a.world;
    const unsigned long long x = a.xbase + (epoch - 1);
    const int64_t slot = (int64_t)(x % 3ULL);
    const int nwords = 2 * P2 + 1;
    if (a.cta == 0) {
      for (int i = wk_tid(); i < W * nwords; i += wk_threads()) {
        const int r = i / nwords, w = i - r * nwords;
        unsigned long long v;
        if (w < 2 * P2) {  // canonical pair
          unsigned long long hi = total(w & ~1), lo = total(w | 1);
          fx_canon(hi, lo);
          v = (w & 1) ? lo : hi;
        } else {
          v = total(w);
        }
        a.mail[r][kMailFlags + (slot * W + a.rank) * bstride + w] = v;
      }
      __threadfence_system();
      wk_sync();
      if (wk_tid() < W) st_release_sys_u64(a.mail[wk_tid()] + a.rank, x + 1);
    }
    const unsigned long long* box = a.mail[a.rank];
    if (wk_tid() < W) {  // relaxed polling, then one acquire (each acquire load invalidates L1)
      SpinGuard sg(a.err, a.spin_ns);
      while (ld_relaxed_sys_u64(box + wk_tid()) < x + 1) {
        if (sg.expired()) break;
      }
      (void)ld_acquire_sys_u64(box + wk_tid());
    }
    wk_sync();
    const unsigned long long* sl = box + kMailFlags + slot * W * bstride;
    unsigned long long badw = 0;
    for (int r = 0; r < W; ++r) badw |= __ldcg(sl + r * bstride + 2 * P2);
    for (int d = wk_tid(); d < P2; d += wk_threads()) {
      unsigned long long hi = 0, lo = 0;
      for (int r = 0; r < W; ++r) {
        hi += __ldcg(sl + r * bstride + 2 * d);
        lo += __ldcg(sl + r * bstride + 2 * d + 1);
      }
      fx_canon(hi, lo);  // both words exact in double
      const double s = badw ? __longlong_as_double(0x7ff8000000000000LL) : fx_join((long long)hi, lo);
      if (d <= p) g[d] = theta[d] - s;
      else red_s[0] = s;
    }
  } else {
    const bool bad = total(2 * P2) != 0ULL;
    for (int d = wk_tid(); d < P2; d += wk_threads()) {
      unsigned long long hi = total(2 * d), lo = total(2 * d + 1);
      fx_canon(hi, lo);  // both words exact in double
      const double s = bad ? __longlong_as_double(0x7ff8000000000000LL) : fx_join((long long)hi, lo);
      if (d <= p) g[d] = theta[d] - s;
      else red_s[0] = s;  // sum of log-likelihood terms
    }
  }
  if (prof) { c1 = clock64(); a.prof[3] += c1 - c0; }
}

}  // namespace ts
