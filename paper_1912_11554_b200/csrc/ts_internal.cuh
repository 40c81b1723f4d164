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
  int xh;                    // p <= 64 half-row tiles: 1 fp64 X (logistic_cta_pass_x64h), 2 fp32 X paired (fp64 policy)
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
//
// Trajectories (narrow p): within one doubling the leapfrog steps do not
// depend on the tree decisions, only on when the tree stops, so the worker
// warps run the leapfrog chain themselves -- drift, pass, kick -- and put each
// leaf (q, r, g, U) into a ring of kTrajRing shared-memory slots; the driver
// consumes leaf n (NodeStore bookkeeping, U-turn checks) while the workers
// stream leaf n+1.  Gate: the workers start leaf m >= 2 only after the driver
// approved leaf m-2 (traj_approve), so every CTA runs exactly the same passes
// (the decisions are replicated) and at most one pass is wasted when a tree
// stops (the speculative leaf n+1, as with post/wait).  The arithmetic is
// Engine::advance_drift's, element by element, so the leaves are identical.
constexpr int kTrajRing = 4;
// Handshake (shared memory).  Leaves and approvals are numbered globally
// over the launch; leaf L completes phase L>>1 of done[L&1], approval A
// (leaf A's verdict: 1 continue, 0 stop) phase A>>1 of appr[A&1].  Neither
// side can run two phases ahead on one barrier (leaf m+2 needs leaf m's
// approval, which needs leaf m), so parity waits are exact; the waits are
// hardware-suspended (mbarrier.try_wait), not polling loops that would take
// issue slots from the streaming warps.
struct TrajCtl {
  uint64_t done[2];
  uint64_t appr[2];
  int verdict[2];
  int nleaves;
  int src_q, src_r, src_g;
  int lbase, abase;  // global numbers of this trajectory's leaf 0 / approval 0
  double eps;
};
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "TC_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra TC_WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// asynchronous models without worker-run trajectories
struct NoTraj {
  __device__ __forceinline__ bool traj_ok() const { return false; }
  __device__ void traj_start(int, int, int, double, int) {}
  __device__ const double* traj_wait(int) { return nullptr; }
  __device__ void traj_approve(int) {}
  __device__ int traj_stop(int) { return 0; }
};
struct LogisticW {
  LogisticArgs a;
  VecStore S;  // the chain's vectors (driver side of post)
  double* wred;
  double* red_s;
  int* cmd;  // smem: [0] 1 = evaluate / 2 = trajectory / 0 = exit, [1] q vector id, [2] gradient vector id
  TrajCtl* tc;   // smem (team scratch, after cmd)
  double* ring;  // smem: kTrajRing slots of (q, r, g: D doubles each; U), null when trajectories are off
  unsigned long long epoch;
  int nleaf, nappr;  // driver copy: leaves waited for / approvals issued so far (global numbers)
  int tl, ta, tn;    // driver: this trajectory's leaf 0 / approval 0 numbers, leaves
  static constexpr bool kAsync = true;
  static constexpr bool kVecOps = false;
  __device__ __forceinline__ int slot_doubles() const { return 3 * (a.p + 1) + 2; }
  // theta -> the pass's copies (fp32 hi/lo or padded fp64), element j of q,
  // for the threads given by (j0, stride)
  __device__ __forceinline__ void stage_theta(const double* th, int j0, int stride) const {
    if (a.th32 != nullptr) {
      float* t32 = const_cast<float*>(a.th32);
      for (int j = j0; j <= a.pmax; j += stride) {
        const double v = (j < a.p) ? th[j] : (j == a.pmax ? th[a.p] : 0.0);
        const float h = (float)v;
        t32[j] = h;
        t32[64 + j] = (float)(v - (double)h);  // lo part: eta = X theta_hi + X theta_lo (logistic_cta_pass)
      }
    }
    if (a.thd != nullptr) {  // FP64 narrow pass: theta as zero-padded doubles
      double* td = const_cast<double*>(a.thd);
      for (int j = j0; j <= a.pmax; j += stride) td[j] = (j < a.p) ? th[j] : (j == a.pmax ? th[a.p] : 0.0);
    }
  }
  // driver warp: post a pass (non-blocking arrive on barrier 2) ...
  __device__ void post(int q, int g) {
    if (threadIdx.x == 0) { cmd[0] = 1; cmd[1] = q; cmd[2] = g; }
    // theta staged by the driver lanes (the workers then start streaming
    // without a conversion round and two syncs)
    stage_theta(S.v(q), (int)(threadIdx.x & 31), 32);
    __syncwarp();
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

  // ------------------------------------------------ trajectories (driver side)
  __device__ __forceinline__ bool traj_ok() const { return ring != nullptr; }
  __device__ __forceinline__ double* traj_slot(int n) const { return ring + (n % kTrajRing) * slot_doubles(); }
  // leaves 0 .. nleaves-1 of a doubling from (q, r, g) with step eps (nleaves >= 2)
  __device__ void traj_start(int q, int r, int g, double eps, int nleaves) {
    tl = nleaf; ta = nappr; tn = nleaves;
    if ((threadIdx.x & 31) == 0) {
      tc->src_q = q; tc->src_r = r; tc->src_g = g;
      tc->eps = eps;
      tc->nleaves = nleaves;
      tc->lbase = tl;
      tc->abase = ta;
      cmd[0] = 2;
    }
    __syncwarp();
    cta_arrive(2);
  }
  // wait for leaf n (in order); returns its slot (q | r | g | U)
  __device__ const double* traj_wait(int n) {
    const int L = nleaf++;
    tc_wait(&tc->done[L & 1], (uint32_t)((L >> 1) & 1));
    return traj_slot(n);
  }
  __device__ void traj_verdict(int v) {
    const int A = nappr++;
    if ((threadIdx.x & 31) == 0) {
      tc->verdict[A & 1] = v;
      tc_arrive(&tc->appr[A & 1]);
    }
    __syncwarp();
  }
  __device__ void traj_approve(int) { traj_verdict(1); }  // leaf n did not stop the tree
  // the tree stopped at leaf n: returns 1 if the speculative leaf n+1 ran
  // (waited for and discarded), else 0
  __device__ int traj_stop(int n) {
    traj_verdict(0);
    if (n + 1 < tn) {  // leaf n+1 was approved (via leaf n-1) or is leaf 1
      (void)traj_wait(n + 1);
      return 1;
    }
    return 0;
  }

  // ------------------------------------------------ worker warps
  // trajectory loop: leaf m = drift from leaf m-1 (or the start point), pass, kick
  __device__ void serve_traj(const VecStore& S, const LogisticArgs& sa) {
    const int D = sa.p + 1;
    const int nl = tc->nleaves;
    const int lbase = tc->lbase, abase = tc->abase;
    const double eps = tc->eps;
    const double half = __dmul_rn(0.5, eps);
    const double* inv = S.v(V_INV);
    const double* q0 = S.v(tc->src_q);
    const double* r0 = S.v(tc->src_r);
    const double* g0 = S.v(tc->src_g);
    const int t = wk_tid(), nt = wk_threads();
    // TS_PROF (CTA 0): [17] gate wait, [18] per-leaf work outside the pass, [19] leaves
    const bool pf = sa.prof != nullptr && blockIdx.x == 0 && t == 0;
    long long pc = pf ? clock64() : 0;
    // drift of one component into slot (sq, sr) from (q, r, g), staged for the pass
    auto drift = [&](double* sq, double* sr, int d, double qv, double rv, double gv) {
      const double rh = __dsub_rn(rv, __dmul_rn(half, gv));
      sr[d] = rh;
      const double qd = __dadd_rn(qv, __dmul_rn(eps, __dmul_rn(inv[d], rh)));
      sq[d] = qd;
      const int j = d < sa.p ? d : sa.pmax;  // the bias goes to slot pmax (stage_theta's layout)
      if (sa.th32 != nullptr) {
        float* t32 = const_cast<float*>(sa.th32);
        const float h = (float)qd;
        t32[j] = h;
        t32[64 + j] = (float)(qd - (double)h);
      }
      if (sa.thd != nullptr) const_cast<double*>(sa.thd)[j] = qd;
    };
    // leaf 0: drift from the start point; zero padding between p and pmax
    {
      double* sq = traj_slot(0);
      for (int d = t; d < D; d += nt) drift(sq, sq + D, d, q0[d], r0[d], g0[d]);
      for (int j = sa.p + t; j < sa.pmax; j += nt) {
        if (sa.th32 != nullptr) { const_cast<float*>(sa.th32)[j] = 0.f; const_cast<float*>(sa.th32)[64 + j] = 0.f; }
        if (sa.thd != nullptr) const_cast<double*>(sa.thd)[j] = 0.0;
      }
      wk_sync();
    }
    for (int m = 0; m < nl; ++m) {
      double* sq = traj_slot(m);
      double* sr = sq + D;
      double* sg = sq + 2 * D;
      if (pf) sa.prof[18] += clock64() - pc;
      logistic_eval_grid(sa, sq, sg, wred, red_s, epoch);
      if (pf) pc = clock64();
      // kick of leaf m (Engine::advance_leaf: r = r_half - half * g; thread d
      // wrote g[d]) fused with the drift of leaf m+1 into the next slot (free:
      // its previous leaf m-3 was consumed before leaf m-1 passed its gate);
      // if the tree stops at leaf m-1 the drift is simply never streamed
      const bool next = m + 1 < nl;
      double* nq = traj_slot(m + 1);
      for (int d = t; d < D; d += nt) {
        const double gd = sg[d];
        const double rd = __dsub_rn(sr[d], __dmul_rn(half, gd));
        sr[d] = rd;
        if (next) drift(nq, nq + D, d, sq[d], rd, gd);
      }
      // U by the thread that wrote the log-likelihood total red_s[0] (the
      // final loop of logistic_eval_grid: d = p + 1); the prior red_s[1] was
      // written before that loop's barrier
      if (t == (sa.p + 1) % nt) sq[3 * D] = red_s[1] - red_s[0];
      wk_sync();
      if (t == 0) tc_arrive(&tc->done[(lbase + m) & 1]);
      if (pf) sa.prof[19] += 1;
      if (next && m + 1 >= 2) {  // gate of leaf m+1: leaf m-1's verdict
        const long long g0c = pf ? clock64() : 0;
        const int A = abase + m - 1;
        tc_wait(&tc->appr[A & 1], (uint32_t)((A >> 1) & 1));
        if (pf) { const long long g1 = clock64(); sa.prof[17] += g1 - g0c; pc += g1 - g0c; }
        if (!tc->verdict[A & 1]) break;  // the tree stopped
      }
    }
  }
  // `sa`: this CTA's copy of the launch state in shared memory (a
  // local-memory copy is re-read on every pass and misses in the L1 that the
  // TMA ring leaves over: ~0.8 us per pass of serialized misses)
  __device__ void serve(const VecStore& S, const LogisticArgs& sa) {
    for (;;) {
      cta_bar(2);
      const int c = cmd[0];
      if (c == 0) break;
      if (c == 2) {
        serve_traj(S, sa);
        continue;
      }
      logistic_eval_grid(sa, S.v(cmd[1]), S.v(cmd[2]), wred, red_s, epoch);
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
    mw.tc = reinterpret_cast<TrajCtl*>(mw.cmd + 16);
    mw.ring = nullptr;
    if (!mw.a.wide) {  // trajectory ring (LogisticW::serve_traj)
      pb = (pb + 15) & ~(uintptr_t)15;
      mw.ring = reinterpret_cast<double*>(pb);
      pb += (size_t)kTrajRing * mw.slot_doubles() * sizeof(double);
    }
    pb = (pb + 127) & ~(uintptr_t)127;
    mw.a.stages = reinterpret_cast<unsigned char*>(pb);
    mw.a.mbar = reinterpret_cast<uint64_t*>(pb + (size_t)rings * mw.a.nstage * mw.a.stage_bytes);
    mw.a.pipe = reinterpret_cast<WarpPipe*>(mw.a.mbar + rings * mw.a.nstage);
    // trajectory handshake barriers (one arrival per phase); both sides number
    // leaves and approvals from 0
    mw.nleaf = 0; mw.nappr = 0; mw.tl = 0; mw.ta = 0; mw.tn = 0;
    if (threadIdx.x == 0) {
      for (int i = 0; i < 2; ++i) { mbar_init(&mw.tc->done[i], 1); mbar_init(&mw.tc->appr[i], 1); }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
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
