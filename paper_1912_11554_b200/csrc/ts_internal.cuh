// Internal declarations shared by the translation units of the engine.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <string>
#include <type_traits>

#include "ts_engine.cuh"
#include "ts_logistic.cuh"
#include "ts_models.cuh"
#include "../../include/turnstile_b200.h"

// Device model handle behind the opaque ts_model of the C ABI.
struct ts_model {
  int kind;
  int dim;
  int device;
  double* params;  // device
  int n_params;
  // logistic
  float* xt;
  uint8_t* yt;
  int64_t n_rows;
  int p;
  int64_t ntiles;
  double* pbuf;
  unsigned long long* bar;
  int fp64;
  int grid;
  int pmax;
  unsigned long long* prof;  // transient: phase counters for ts_eval_bench
  int exact_cvt;             // X holds fp32 subnormals (fp64 pass uses F2F)
  int wide;                  // 64 < p <= 256, or X in fp64: 8-row row-major tiles (ts_logistic.cuh)
  int xd;                    // X stored as fp64 (TS_PREC_FP64X)
  double* slotws;            // wide: per-CTA NodeStore slot vectors (grown on demand)
  size_t slotws_size;        // doubles
  // row sharding across GPUs (ts_peer_mailbox_*)
  int world, rank;
  unsigned long long* mail_local;  // this rank's mailbox (+ exchange counter after it)
  unsigned long long* mail[TS_MAX_PEERS];
  unsigned long long* dump;        // transient: ts_logistic_partial_sums output
  int vranks;                      // test mode: row-sharded ranks emulated in one launch
  unsigned long long* vmail;       // their mailboxes
  size_t vmail_words;
  // dense Gaussian (TS_DENSE_GAUSS): params = A (dim x dim, fp64), a32 = tf32-rounded copy
  float* a32;
  unsigned char* dws;  // lockstep workspaces (grown on demand)
  size_t dws_size;
  unsigned int* errw;  // sticky device error word: bit 0 = a synchronisation wait timed out (SpinGuard)
  // logistic, TF32 policy: many chains sharing X on the tensor cores (ts_k_logistic_many.cu)
  int many;
  int ka;        // columns of xaug = p + 2 rounded up to 8
  float* xaug;   // [n_rows][ka] = X | 1 | y | 0
};

namespace ts_internal {
using namespace ts;

int set_err(int code, const char* msg);

// Limit of every inter-CTA / inter-GPU wait (SpinGuard): TS_SPIN_TIMEOUT_S
// seconds (default 30).
inline unsigned long long spin_limit_ns() {
  double s = 30.0;
  if (const char* e = getenv("TS_SPIN_TIMEOUT_S")) s = atof(e);
  if (!(s > 0)) s = 30.0;
  return (unsigned long long)(s * 1e9);
}


// ------------------------------------------------------------------ op args
enum OpCode : int { OP_POTGRAD = 0, OP_LEAPFROG = 1, OP_TREE = 2, OP_TRANSITION = 3, OP_STEPSEARCH = 4, OP_RUN = 5, OP_EVALBENCH = 6,
                    OP_HMC = 7 };

struct OpArgs {
  int op;
  const double* z_in;
  double* z_out;
  const double* inv;
  SamplerCfg cfg;
  int depth;
  double eps;
  double h_ref;
  uint64_t key_hi, key_lo;
  const double* inj;
  TraceBuf trace;
  int has_trace;
  int n_points;
  // run
  RunCfg rc;
  const uint64_t* chain_keys;  // [C][2]
  int n_chains;
  double* samples;  // [C][S][D]
  double* stats;    // [C][W+S][5]
  double* adapt;    // [C][2+W+D]
  int32_t* status;  // [C]
  int64_t* evals;   // [C]
  unsigned long long* prof;  // TS_PROF cycle counters (chain 0), or null
};

struct SmallW {
  static constexpr bool kAsync = false;
  static constexpr bool kVecOps = false;  // Engine: 16-byte warp vector paths (large-D models only)
  SmallModel m;
  template <class Team>
  __device__ double eval(const Team& T, const VecStore& S, int q, int g) { return small_model_eval(T, m, S, q, g); }
};

// Logistic model on a persistent grid.  In each CTA the driver warp runs the
// chain (WarpTeam) and the other warps serve data passes: eval() posts a
// command word in shared memory and joins the pass with them.
struct LogisticW {
  LogisticArgs a;
  VecStore S;  // the chain's vectors (driver side of post)
  double* wred;
  double* red_s;
  int* cmd;  // smem: [0] 1 = evaluate / 0 = exit, [1] q vector id, [2] gradient vector id
  unsigned long long epoch;
  static constexpr bool kAsync = true;
  static constexpr bool kVecOps = false;
  // driver warp: post a pass (non-blocking arrive on barrier 2) ...
  __device__ void post(int q, int g) {
    if (threadIdx.x == 0) { cmd[0] = 1; cmd[1] = q; cmd[2] = g; }
    if (a.th32 != nullptr) {
      // theta rounded to float for the FP32 pass, by the driver lanes (the
      // workers then start streaming without a conversion round and two syncs)
      const double* th = S.v(q);
      float* t32 = const_cast<float*>(a.th32);
      for (int j = (int)(threadIdx.x & 31); j <= a.pmax; j += 32) {
        const double v = (j < a.p) ? th[j] : (j == a.pmax ? th[a.p] : 0.0);
        const float h = (float)v;
        t32[j] = h;
        t32[64 + j] = (float)(v - (double)h);  // lo part: eta = X theta_hi + X theta_lo (logistic_cta_pass)
      }
      __syncwarp();
    }
    if (a.thd != nullptr) {  // FP64 narrow pass: theta as zero-padded doubles
      const double* th = S.v(q);
      double* td = const_cast<double*>(a.thd);
      for (int j = (int)(threadIdx.x & 31); j <= a.pmax; j += 32)
        td[j] = (j < a.p) ? th[j] : (j == a.pmax ? th[a.p] : 0.0);
      __syncwarp();
    }
    cta_arrive(2);  // publishes q and the command to the worker warps
  }
  // ... and collect it (barrier 3: gradient written to vector g, U in red_s)
  __device__ double wait() {
    cta_bar(3);
    return red_s[1] - red_s[0];
  }
  template <class Team>
  __device__ double eval(const Team&, const VecStore&, int q, int g) {
    post(q, g);
    return wait();
  }
  // worker warps; `sa`: this CTA's copy of the launch state in shared memory
  // (a local-memory copy is re-read on every pass and misses in the L1 that
  // the TMA ring leaves over: ~0.8 us per pass of serialized misses)
  __device__ void serve(const VecStore& S, const LogisticArgs& sa) {
    for (;;) {
      cta_bar(2);
      if (cmd[0] == 0) break;
      logistic_eval_grid(sa, S, cmd[1], cmd[2], wred, red_s, epoch);
      cta_arrive(3);
    }
  }
  __device__ void release_workers() {  // driver warp, once at the end
    if (threadIdx.x == 0) cmd[0] = 0;
    cta_arrive(2);
  }
};

// Run one parity/production op for the engine E (vectors already allocated).
template <class Team, class Model>
__device__ void do_op(Engine<Team, Model>& E, const OpArgs& A, int chain, bool writer) {
  const int D = E.D;
  const int64_t s = E.ds();
  const int rk = E.T.rank(), sz = E.T.size();
  // mass matrix
  {
    double* inv = E.v(V_INV);
    for (int d = rk; d < D; d += sz) inv[d * s] = A.inv[d];
    E.T.sync();
    E.refresh_mstd();
  }
  E.tr = (A.has_trace && writer) ? const_cast<TraceBuf*>(&A.trace) : nullptr;
  E.n_evals = 0;
  E.n_wasted = 0;
  E.cfg = A.cfg;
  switch (A.op) {
    case OP_POTGRAD: {
      for (int k = 0; k < A.n_points; ++k) {
        double* q = E.v(V_CQ);
        for (int d = rk; d < D; d += sz) q[d * s] = A.z_in[(int64_t)k * D + d];
        E.T.sync();
        const double u = E.M.eval(E.T, E.S, V_CQ, V_CG);
        E.T.sync();
        if (writer) {
          const double* g = E.v(V_CG);
          double* o = A.z_out + (int64_t)k * (D + 1);
          if (E.T.leader()) o[0] = u;
          for (int d = rk; d < D; d += sz) o[1 + d] = g[d * s];
        }
      }
      break;
    }
    case OP_EVALBENCH: {
      double* q = E.v(V_CQ);
      for (int d = rk; d < D; d += sz) q[d * s] = A.z_in[d];
      double u = 0.0;
      unsigned long long t0 = 0, t1 = 0;
      E.T.sync();
      if (writer && E.T.leader()) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (int k = 0; k < A.n_points; ++k) u = E.eval(V_CQ, V_CG);
      if (writer && E.T.leader()) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        A.z_out[0] = u;
        A.z_out[1] = (double)(t1 - t0);
      }
      break;
    }
    case OP_LEAPFROG: {
      double* q = E.v(V_CQ); double* r = E.v(V_CR); double* g = E.v(V_CG);
      for (int d = rk; d < D; d += sz) { q[d * s] = A.z_in[d]; r[d * s] = A.z_in[D + d]; g[d * s] = A.z_in[2 * D + d]; }
      E.cur_U = A.z_in[3 * D];
      E.leapfrog(A.eps);
      if (writer) {
        for (int d = rk; d < D; d += sz) { A.z_out[d] = q[d * s]; A.z_out[D + d] = r[d * s]; A.z_out[2 * D + d] = g[d * s]; }
        if (E.T.leader()) A.z_out[3 * D] = E.cur_U;
      }
      break;
    }
    case OP_TREE: {
      double* q = E.v(V_CQ); double* r = E.v(V_CR); double* g = E.v(V_CG);
      for (int d = rk; d < D; d += sz) { q[d * s] = A.z_in[d]; r[d * s] = A.z_in[D + d]; g[d * s] = A.z_in[2 * D + d]; }
      E.cur_U = A.z_in[3 * D];
      double h_ref = A.h_ref;
      const TreeOut t = E.build_tree(A.depth, A.eps, h_ref, Key{A.key_hi, A.key_lo});
      if (writer) {
        const int ids[8] = {V_FQ, V_FR, V_CQ, V_CR, V_CG, V_TPQ, V_TPG, V_MSUM};
        for (int k = 0; k < 8; ++k) {
          const double* vv = E.v(ids[k]);
          for (int d = rk; d < D; d += sz) A.z_out[(int64_t)k * D + d] = vv[d * s];
        }
        if (E.T.leader()) {
          double* o = A.z_out + 8 * (int64_t)D;
          o[0] = t.lw; o[1] = t.sum_metro; o[2] = t.count; o[3] = t.stop == kStopTurn; o[4] = t.stop == kStopDiv;
          o[5] = t.pU; o[6] = t.pH; o[7] = t.pidx; o[8] = t.fU; o[9] = E.cur_U;
        }
      }
      break;
    }
    case OP_TRANSITION: {
      double* q = E.v(V_Q0); double* g = E.v(V_G0);
      for (int d = rk; d < D; d += sz) { q[d * s] = A.z_in[d]; g[d * s] = A.z_in[2 * D + d]; }
      E.U0 = A.z_in[3 * D];
      const Stats st = E.transition(Key{A.key_hi, A.key_lo}, A.inj, 1);
      if (writer) {
        for (int d = rk; d < D; d += sz) { A.z_out[d] = q[d * s]; A.z_out[D + d] = g[d * s]; }
        if (E.T.leader()) {
          double* o = A.z_out + 2 * (int64_t)D;
          o[0] = E.U0; o[1] = st.depth; o[2] = st.leapfrogs; o[3] = st.diverged; o[4] = st.accept; o[5] = st.energy;
          o[6] = E.p_tree; o[7] = E.p_leaf;
        }
      }
      break;
    }
    case OP_HMC: {
      double* q = E.v(V_Q0); double* g = E.v(V_G0);
      for (int d = rk; d < D; d += sz) { q[d * s] = A.z_in[d]; g[d * s] = A.z_in[2 * D + d]; }
      E.U0 = A.z_in[3 * D];
      bool acc = false;
      const Stats st = E.hmc(Key{A.key_hi, A.key_lo}, A.inj, 1, A.depth, acc);
      if (writer) {
        for (int d = rk; d < D; d += sz) { A.z_out[d] = q[d * s]; A.z_out[D + d] = g[d * s]; }
        if (E.T.leader()) {
          double* o = A.z_out + 2 * (int64_t)D;
          o[0] = E.U0; o[1] = st.depth; o[2] = st.leapfrogs; o[3] = st.diverged; o[4] = st.accept; o[5] = st.energy;
          o[6] = acc ? 1.0 : 0.0;
        }
      }
      break;
    }
    case OP_STEPSEARCH: {
      double* q = E.v(V_Q0); double* g = E.v(V_G0);
      for (int d = rk; d < D; d += sz) { q[d * s] = A.z_in[d]; g[d * s] = A.z_in[2 * D + d]; }
      E.U0 = A.z_in[3 * D];
      const double eps = E.find_step_size(Key{A.key_hi, A.key_lo}, A.eps, A.inj, 1);
      if (writer && E.T.leader()) A.z_out[0] = eps;
      break;
    }
    case OP_RUN: {
      const int W = A.rc.num_warmup, S = A.rc.num_samples;
      RunOut ro;
      ro.samples = A.samples + (int64_t)chain * (S + (A.rc.keep_warmup ? W : 0)) * D;
      ro.s_stride = D;
      ro.d_stride = 1;
      ro.stats = A.stats + (int64_t)chain * (W + S) * 5;
      ro.adapt = A.adapt + (int64_t)chain * (2 + W + D);
      ro.status = A.status + chain;
      ro.evals = A.evals ? A.evals + chain : nullptr;
      const Key ck{A.chain_keys[2 * chain], A.chain_keys[2 * chain + 1]};
      run_chain(E, ck, A.rc, ro, writer);
      break;
    }
  }
}

// BlockTeam: vectors in shared memory.  smem = vecs | team scratch(64) | model scratch
template <class MW>
__global__ void __launch_bounds__(256, 1) k_block_op(MW mw, int D, int nslots, int model_scratch, OpArgs A) {
  extern __shared__ double smem[];
  const int nv = num_vecs(nslots);
  const bool writer = blockIdx.x == 0;
  const int chain = (A.op == OP_RUN) ? A.n_points : 0;  // grid mode: one chain per launch
  VecStore S;
  S.base = smem;
  S.vstride = D;
  S.dstride = 1;
  if constexpr (std::is_same<MW, SmallW>::value) {
    Engine<BlockTeam, MW> E;
    E.T.scratch = smem + (int64_t)nv * D;
    E.ss = reinterpret_cast<SlotScalars*>(smem + (int64_t)nv * D + 64);
    E.M = mw;
    E.D = D;
    E.S = S;
    // small models: one CTA per chain for runs (chain = launch offset + CTA)
    if (A.op == OP_RUN) do_op(E, A, A.n_points + (int)blockIdx.x, true);
    else do_op(E, A, chain, writer);
  } else {
    // wide-p models keep the NodeStore slot vectors in a per-CTA global
    // workspace (their data pass is long; shared memory goes to the ring)
    const int nvs = mw.a.slotws ? (int)V_SLOT0 : nv;
    if (mw.a.slotws) {
      S.slots = mw.a.slotws + (int64_t)blockIdx.x * kSlotVecs * nslots * D;
      S.slot0 = V_SLOT0;
    }
    mw.wred = smem + (((int64_t)nvs * D + kTeamScratch + 1) & ~(int64_t)1);  // 16-byte aligned
    mw.red_s = mw.wred + model_scratch;
    mw.cmd = reinterpret_cast<int*>(smem + (int64_t)nvs * D);   // team scratch area
    mw.epoch = 0;
    {
      // this CTA's rank-local index and the rank's row range
      const int64_t units = mw.a.wide ? mw.a.ntiles / kWideGroup : mw.a.ntiles;
      if (mw.a.vranks > 1) {  // test mode: ranks emulated by groups of CTAs
        const int V = mw.a.vranks, Gc = (int)gridDim.x / V, vg = (int)blockIdx.x / Gc;
        mw.a.cta = (int)blockIdx.x % Gc;
        mw.a.ncta = Gc;
        mw.a.u_lo = units * vg / V;
        mw.a.u_hi = units * (vg + 1) / V;
        mw.a.world = V;
        mw.a.rank = vg;
        const int64_t mwords = mail_words(mw.a.p, V);
        for (int r = 0; r < V; ++r) mw.a.mail[r] = mw.a.vmail + r * mwords;
        mw.a.mail_epoch = mw.a.vmail + V * mwords;
        mw.a.pbuf += (int64_t)vg * fx_rank_words(mw.a.p);
        mw.a.bar += 16 * vg;
      } else {
        mw.a.cta = (int)blockIdx.x;
        mw.a.ncta = (int)gridDim.x;
        mw.a.u_lo = 0;
        mw.a.u_hi = units;
      }
    }
    // exchange index base (row sharding): the pass count of earlier launches
    if (mw.a.world > 0) mw.a.xbase = __ldcg(mw.a.mail_epoch);
    // TMA pipeline region: stages (128-B aligned) | mbarriers | per-ring counters;
    // one ring per worker warp
    const int rings = (int)(blockDim.x >> 5) - 1;
    // float copy of theta for the FP32 narrow pass (written by the driver in post)
    mw.a.th32 = (!mw.a.fp64 && !mw.a.wide) ? reinterpret_cast<const float*>(mw.red_s + ((mw.a.p + 3) & ~1)) : nullptr;
    mw.a.thd = (mw.a.fp64 && !mw.a.wide) ? mw.red_s + ((mw.a.p + 3) & ~1) : nullptr;
    mw.S = S;
    uintptr_t pb = reinterpret_cast<uintptr_t>(mw.red_s + mw.a.p + 2 + (kWideMax + 8) / 2);
    pb = (pb + 127) & ~(uintptr_t)127;
    mw.a.stages = reinterpret_cast<unsigned char*>(pb);
    mw.a.mbar = reinterpret_cast<uint64_t*>(pb + (size_t)rings * mw.a.nstage * mw.a.stage_bytes);
    mw.a.pipe = reinterpret_cast<WarpPipe*>(mw.a.mbar + rings * mw.a.nstage);
    if ((threadIdx.x >> 5) == 0) {
      // driver warp: the whole NUTS state machine, warp-synchronous
      Engine<WarpTeam, MW> E;
      E.M = mw;
      E.D = D;
      E.S = S;
      E.prof = (blockIdx.x == 0) ? mw.a.prof : nullptr;
      E.prof_last = 0;
      E.tr = nullptr;
      E.ss = reinterpret_cast<SlotScalars*>(smem + (int64_t)nvs * D + 64);
      __syncwarp();
      do_op(E, A, chain, writer);
      E.M.release_workers();
    } else {
      __shared__ __align__(16) unsigned char sh_args[sizeof(LogisticArgs)];
      LogisticArgs& sa = *reinterpret_cast<LogisticArgs*>(sh_args);
      if (wk_tid() == 0) sa = mw.a;
      wk_sync();
      logistic_pipeline_init(sa);
      mw.serve(S, sa);
      logistic_pipeline_drain(sa);
      if (mw.a.world > 0 && blockIdx.x == 0 && wk_tid() == 0) *mw.a.mail_epoch = mw.a.xbase + mw.epoch;
    }
  }
}


int launch_thread(const SmallModel& sm, int D, int C, int nslots, OpArgs& A, cudaStream_t st);
int launch_block_small(const SmallModel& sm, int D, int nslots, OpArgs& A, int C, cudaStream_t st);
int launch_warp_small(const SmallModel& sm, int D, int nslots, OpArgs& A, int C, cudaStream_t st);
int launch_block_logistic(const ts_model* m, int nslots, OpArgs& A, cudaStream_t st);
int launch_dense(const ts_model* m, int nslots, OpArgs& A, int n_chains, cudaStream_t st);
int launch_logistic_many(const ts_model* m, int nslots, OpArgs& A, int n_chains, cudaStream_t st);
int build_logistic_xaug(ts_model* m, const float* x_dev, const uint8_t* y_dev);

}  // namespace ts_internal

#define TS_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      char b_[512];                                                                \
      snprintf(b_, sizeof b_, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return ts_internal::set_err(TS_ECUDA, b_);                                   \
    }                                                                              \
  } while (0)
