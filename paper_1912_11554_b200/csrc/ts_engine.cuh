// Device NUTS engine: leapfrog, iterative tree builder, doubling transition,
// step-size search, warmup adaptation and the whole per-chain run loop.
//
// Every function restates a reference routine (file:line in turnstile/):
//   leapfrog              integrator.py:90-103, kernels.py:148-165
//   hamiltonian           integrator.py:82-87,  kernels.py:125-130
//   build_tree            tree.py:344-453 (+ _merge 140-156, _logaddexp 131-137,
//                         merge_out 395-400, _leaf_summary 262-280)
//   transition            sampler.py:83-148 (biased progressive, outer U-turn)
//   find_step_size        adapt.py:172-204
//   dual averaging        adapt.py:28-70, Welford adapt.py:73-108,
//   warmup driver         adapt.py:207-236, chains.py:98-163
// Floating-point expressions keep the reference's association and use
// explicit _rn intrinsics (the file is also compiled with -fmad=false), so
// a ThreadTeam chain of a small model reproduces the reference bit for bit
// up to the last-ulp behaviour of exp/log1p.
#pragma once
#include <stddef.h>
#include <math.h>
#include <stdint.h>
#include "ts_rng.cuh"
#include "ts_libm.cuh"
#include "ts_team.cuh"

namespace ts {

enum Vid : int {
  V_INV = 0, V_Q0, V_G0, V_R0,        // current state z0 (position, gradient), momentum
  V_LQ, V_LR, V_LG,                   // trajectory left end (earliest in time)
  V_RQ, V_RR, V_RG,                   // trajectory right end (latest in time)
  V_PQ, V_PG,                         // transition proposal
  V_RHO,                              // transition momentum sum
  V_CQ, V_CR, V_CG, V_CUM,            // current leaf z_cur, running momentum prefix sum
  V_FQ, V_FR, V_CUMF,                 // running subtree: first leaf and its prefix sum
  V_TPQ, V_TPG,                       // running subtree proposal
  V_MSUM,                             // tree momentum sum (output of build_tree)
  V_WMEAN, V_WM2,                     // Welford accumulator
  V_NQ, V_NR, V_NG,                   // speculative next leaf (drifted q, r_half, gradient)
  V_MSTD,                             // momentum_std = 1/sqrt(inv), refreshed at every mass install
  V_SLOT0                             // NodeStore slots: 5 vectors each
};
constexpr int kSlotVecs = 5;  // FQ, FR, CUMF, PQ, PG
constexpr int kMaxSlots = 30;  // treemath.MAX_TREE_DEPTH_LIMIT
__host__ __device__ inline int num_vecs(int nslots) { return V_SLOT0 + kSlotVecs * nslots; }
// shared-memory scratch of a team (doubles): 64 for reductions / commands,
// then the NodeStore scalars (kMaxSlots SlotScalars)
constexpr int kTeamScratch = 64 + (kMaxSlots * 56 + 7) / 8;
__device__ __forceinline__ int slot_vec(int s, int k) { return V_SLOT0 + kSlotVecs * s + k; }

// Warp vector helpers for warp-owned large-D vectors in global memory (the
// batched dense model).  Loads are ld.global.cg (L2 only): the vectors
// stream through once per leaf and would otherwise evict the chain warps'
// local memory (engine state) from L1 (ld.global.L1::no_allocate measured
// slower: 8.06 -> 7.09 M chain-leapfrog/s).
//
// Warp copy of n2 double2 (lane-strided, 8 loads in flight per lane).  A
// separate function: its registers stay out of the engine's allocation.
static __device__ __noinline__ void warp_copy2(double2* __restrict__ a, const double2* __restrict__ b, int n2) {
  for (int base = (int)(threadIdx.x & 31); base < n2; base += 32 * 8) {
    double2 t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (base + 32 * u < n2) t[u] = __ldcg(b + base + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (base + 32 * u < n2) a[base + 32 * u] = t[u];
  }
}

// Elementwise leaf updates for warp-owned large-D vectors: 16-byte accesses,
// two double2 per operand in flight per lane in an unpredicated main loop
// plus a tail (the earlier four / eight-wide predicated loops spilled their
// arrays to local memory inside the loop); per-component arithmetic is the
// same as the scalar loops (so results are identical), and per lane the
// elements are visited in ascending order (reduction order unchanged).
#define TS_WARP_LOOP2(N2, BODY)                               \
  {                                                           \
    int i_ = (int)(threadIdx.x & 31);                         \
    const int nfull_ = (N2) & ~63;                            \
    _Pragma("unroll 1") for (; i_ < nfull_; i_ += 64) { BODY(i_, i_ + 32) } \
    _Pragma("unroll 1") for (; i_ < (N2); i_ += 32) { BODY(i_, -1) }        \
  }
static __device__ __noinline__ void warp_drift2(double2* __restrict__ nq, double2* __restrict__ nr,
                                                const double2* __restrict__ q, const double2* __restrict__ r,
                                                const double2* __restrict__ g, const double2* __restrict__ inv,
                                                double half, double eps, int n2) {
  auto one = [&](int i, double2 tq, double2 tr, double2 tg, double2 ti) {
    double2 rh, nqv;
    rh.x = __dsub_rn(tr.x, __dmul_rn(half, tg.x));
    rh.y = __dsub_rn(tr.y, __dmul_rn(half, tg.y));
    nqv.x = __dadd_rn(tq.x, __dmul_rn(eps, __dmul_rn(ti.x, rh.x)));
    nqv.y = __dadd_rn(tq.y, __dmul_rn(eps, __dmul_rn(ti.y, rh.y)));
    nr[i] = rh;
    nq[i] = nqv;
  };
#define TS_BODY(I, J)                                                                                          \
  const double2 q0 = __ldcg(q + I), r0 = __ldcg(r + I), g0 = __ldcg(g + I), v0 = __ldcg(inv + I);            \
  if (J >= 0) {                                                                                                \
    const double2 q1 = __ldcg(q + J), r1 = __ldcg(r + J), g1 = __ldcg(g + J), v1 = __ldcg(inv + J);          \
    one(I, q0, r0, g0, v0);                                                                                    \
    one(J, q1, r1, g1, v1);                                                                                    \
  } else {                                                                                                     \
    one(I, q0, r0, g0, v0);                                                                                    \
  }
  TS_WARP_LOOP2(n2, TS_BODY)
#undef TS_BODY
}
static __device__ __noinline__ void warp_advance2(double2* __restrict__ q, double2* __restrict__ r,
                                                  double2* __restrict__ g, const double2* __restrict__ nq,
                                                  const double2* __restrict__ nr, const double2* __restrict__ ng,
                                                  double half, int n2) {
  auto one = [&](int i, double2 tq, double2 tr, double2 tg) {
    double2 rv;
    rv.x = __dsub_rn(tr.x, __dmul_rn(half, tg.x));
    rv.y = __dsub_rn(tr.y, __dmul_rn(half, tg.y));
    q[i] = tq;
    g[i] = tg;
    r[i] = rv;
  };
#define TS_BODY(I, J)                                                                 \
  const double2 q0 = __ldcg(nq + I), r0 = __ldcg(nr + I), g0 = __ldcg(ng + I);      \
  if (J >= 0) {                                                                       \
    const double2 q1 = __ldcg(nq + J), r1 = __ldcg(nr + J), g1 = __ldcg(ng + J);    \
    one(I, q0, r0, g0);                                                               \
    one(J, q1, r1, g1);                                                               \
  } else {                                                                            \
    one(I, q0, r0, g0);                                                               \
  }
  TS_WARP_LOOP2(n2, TS_BODY)
#undef TS_BODY
}
static __device__ __noinline__ void warp_add2(double2* __restrict__ c, const double2* __restrict__ r, int n2) {
  auto one = [&](int i, double2 tc, double2 tr) { c[i] = make_double2(__dadd_rn(tc.x, tr.x), __dadd_rn(tc.y, tr.y)); };
#define TS_BODY(I, J)                                          \
  const double2 c0 = __ldcg(c + I), r0 = __ldcg(r + I);       \
  if (J >= 0) {                                                \
    const double2 c1 = __ldcg(c + J), r1 = __ldcg(r + J);     \
    one(I, c0, r0);                                            \
    one(J, c1, r1);                                            \
  } else {                                                     \
    one(I, c0, r0);                                            \
  }
  TS_WARP_LOOP2(n2, TS_BODY)
#undef TS_BODY
}
// per-lane partial of kinetic_energy_impl over warp-owned vectors (lane's
// components in order 2k, 2k+1 of each of its double2 slots)
static __device__ __noinline__ double warp_kinetic2(const double2* __restrict__ r, const double2* __restrict__ inv, int n2) {
  double acc = 0.0;
  auto one = [&](double2 tr, double2 ti) {
    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(0.5, tr.x), tr.x), ti.x));
    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(0.5, tr.y), tr.y), ti.y));
  };
#define TS_BODY(I, J)                                          \
  const double2 r0 = __ldcg(r + I), v0 = __ldcg(inv + I);     \
  if (J >= 0) {                                                \
    const double2 r1 = __ldcg(r + J), v1 = __ldcg(inv + J);   \
    one(r0, v0);                                               \
    one(r1, v1);                                               \
  } else {                                                     \
    one(r0, v0);                                               \
  }
  TS_WARP_LOOP2(n2, TS_BODY)
#undef TS_BODY
  return acc;
}
// generalized U-turn dots of the running subtree with rho = (cum - cum_first) + r_first
// formed on the fly: per-lane partials a = sum rho inv rl, b = sum rho inv rr
static __device__ __noinline__ double2 warp_gen_uturn2(const double2* __restrict__ cum, const double2* __restrict__ cf,
                                                    const double2* __restrict__ fr, const double2* __restrict__ inv,
                                                    const double2* __restrict__ rr, int n2) {
  double a = 0.0, b = 0.0;
  for (int base = (int)(threadIdx.x & 31); base < n2; base += 32 * 4) {
    double2 tc[4], tf[4], trf[4], ti[4], trr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (base + 32 * u < n2) {
        tc[u] = __ldcg(cum + base + 32 * u); tf[u] = __ldcg(cf + base + 32 * u); trf[u] = __ldcg(fr + base + 32 * u);
        ti[u] = __ldcg(inv + base + 32 * u); trr[u] = __ldcg(rr + base + 32 * u);
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (base + 32 * u < n2) {
        const double wx = __dmul_rn(__dadd_rn(__dsub_rn(tc[u].x, tf[u].x), trf[u].x), ti[u].x);
        const double wy = __dmul_rn(__dadd_rn(__dsub_rn(tc[u].y, tf[u].y), trf[u].y), ti[u].y);
        a = __dadd_rn(a, __dmul_rn(wx, trf[u].x));
        b = __dadd_rn(b, __dmul_rn(wx, trr[u].x));
        a = __dadd_rn(a, __dmul_rn(wy, trf[u].y));
        b = __dadd_rn(b, __dmul_rn(wy, trr[u].y));
      }
  }
  return make_double2(a, b);  // (a, b) partials in registers (an array argument lived in local memory)
}
__device__ __forceinline__ bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
// One pass over a leaf for warp-owned large-D vectors (batched models):
// advance_leaf (kick of leaf n from its pass), add_cum, the kinetic-energy
// partial of leaf n (same lane order as warp_kinetic2), drift_next (leaf
// n+1) and the request row for leaf n+1 (tf32 floats, or doubles).  Every
// element gets the same arithmetic as the separate loops.  ST: the leaf's
// NodeStore copies written from the same registers (leaf_book's copies,
// which would re-read the vectors in another pass): 5 = even leaf into its
// slot (q, r, cum, proposal q, proposal g -> st[0..4]), 2 = odd leaf into
// the running proposal (st[0] = q, st[1] = g), 0 = none.
// Operands of warp_leaf_fused, in shared memory (one record per chain warp,
// written by the engine before the call): passed as one pointer instead of
// 18 arguments, which spilled past the ABI's register arguments onto the
// stack and were re-read from local memory every iteration.
#ifndef TS_LEAF_INLINE
#define TS_LEAF_INLINE __forceinline__
#endif
struct LeafVecs {
  double2* q;
  double2* r;
  double2* g;
  double2* nq;
  double2* nr;
  const void* grow;
  const double2* inv;
  double2* cum;
  void* row;
  double2* st[5];
  double half, eps;
  int n2;
  int pad_;
};
// pointer field `off` (bytes) of a shared-memory record, re-read at every
// use (volatile): short live ranges instead of 14 pointers held across the
// loop, which the register allocator spilled to local memory
template <class P>
__device__ __forceinline__ P* lds_ptr(uint32_t rec, uint32_t off) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(rec + off));
  return reinterpret_cast<P*>(v);
}
#ifndef TS_PF_DIST
#define TS_PF_DIST 192  // double2 elements ahead (three iterations of the two-wide loop; 64 / 192 / none: 9.40 / 9.52 / 9.35 M)
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
template <bool F64ROW, int ST>
static __device__ TS_LEAF_INLINE double2 warp_leaf_fused(const LeafVecs* __restrict__ L) {
  // grow: the served gradient row (fp32 tf32-GEMM output, or doubles);
  // returns this lane's (kinetic partial, q . g partial) (U = q'Aq / 2 = q . g / 2).
  // Two elements per lane in flight, no predicated arrays, operand pointers
  // re-read from the shared record at each use: the four-wide form with 18
  // pointer arguments spilled its loads and pointers to local memory on
  // every iteration (64 us per 1000-D leaf).  Per lane the elements are
  // still visited in ascending order (the kinetic-energy / U partial sums
  // keep warp_kinetic2's order).
  const uint32_t rec = static_cast<uint32_t>(__cvta_generic_to_shared(L));
  const double half = L->half, eps = L->eps;
  const int n2 = L->n2;
  constexpr uint32_t oQ = offsetof(LeafVecs, q), oR = offsetof(LeafVecs, r), oG = offsetof(LeafVecs, g),
                     oNQ = offsetof(LeafVecs, nq), oNR = offsetof(LeafVecs, nr), oGR = offsetof(LeafVecs, grow),
                     oINV = offsetof(LeafVecs, inv), oCUM = offsetof(LeafVecs, cum), oROW = offsetof(LeafVecs, row),
                     oST = offsetof(LeafVecs, st);
  double kin = 0.0, ud = 0.0;
  auto load_g = [&](int i) -> double2 {
    if constexpr (F64ROW) {
      return __ldcg(lds_ptr<const double2>(rec, oGR) + i);
    } else {
      const float2 f = __ldcg(lds_ptr<const float2>(rec, oGR) + i);
      return make_double2((double)f.x, (double)f.y);
    }
  };
  auto body = [&](int i, double2 tq, double2 tr, double2 tg, double2 ti, double2 tc) {
    double2 rr, rh, nqv, cv;
    rr.x = __dsub_rn(tr.x, __dmul_rn(half, tg.x));
    rr.y = __dsub_rn(tr.y, __dmul_rn(half, tg.y));
    lds_ptr<double2>(rec, oQ)[i] = tq;
    lds_ptr<double2>(rec, oG)[i] = tg;
    lds_ptr<double2>(rec, oR)[i] = rr;
    ud = __dadd_rn(ud, __dmul_rn(tq.x, tg.x));
    ud = __dadd_rn(ud, __dmul_rn(tq.y, tg.y));
    cv.x = __dadd_rn(tc.x, rr.x);
    cv.y = __dadd_rn(tc.y, rr.y);
    lds_ptr<double2>(rec, oCUM)[i] = cv;
    if constexpr (ST == 5) {
      lds_ptr<double2>(rec, oST)[i] = tq;
      lds_ptr<double2>(rec, oST + 8)[i] = rr;
      lds_ptr<double2>(rec, oST + 16)[i] = cv;
      lds_ptr<double2>(rec, oST + 24)[i] = tq;
      lds_ptr<double2>(rec, oST + 32)[i] = tg;
    }
    if constexpr (ST == 2) {
      lds_ptr<double2>(rec, oST)[i] = tq;
      lds_ptr<double2>(rec, oST + 8)[i] = tg;
    }
    kin = __dadd_rn(kin, __dmul_rn(__dmul_rn(__dmul_rn(0.5, rr.x), rr.x), ti.x));
    kin = __dadd_rn(kin, __dmul_rn(__dmul_rn(__dmul_rn(0.5, rr.y), rr.y), ti.y));
    rh.x = __dsub_rn(rr.x, __dmul_rn(half, tg.x));
    rh.y = __dsub_rn(rr.y, __dmul_rn(half, tg.y));
    nqv.x = __dadd_rn(tq.x, __dmul_rn(eps, __dmul_rn(ti.x, rh.x)));
    nqv.y = __dadd_rn(tq.y, __dmul_rn(eps, __dmul_rn(ti.y, rh.y)));
    lds_ptr<double2>(rec, oNR)[i] = rh;
    lds_ptr<double2>(rec, oNQ)[i] = nqv;
    if constexpr (F64ROW) {
      lds_ptr<double2>(rec, oROW)[i] = nqv;
    } else {
      uint32_t a, b;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(a) : "f"((float)nqv.x));
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"((float)nqv.y));
      lds_ptr<float2>(rec, oROW)[i] = make_float2(__uint_as_float(a), __uint_as_float(b));
    }
  };
  auto ld = [&](uint32_t off, int i) -> double2 { return __ldcg(lds_ptr<const double2>(rec, off) + i); };
  int i = (int)(threadIdx.x & 31);
  const int nfull = n2 & ~63;
  for (; i < nfull; i += 64) {
    const int j = i + 32;
#ifndef TS_NO_L2_PREFETCH
    // the NodeStore workspaces exceed L2, so these streams come from DRAM:
    // pull the elements of the iteration after next into L2 (no registers)
    if (i + TS_PF_DIST < n2) {
      prefetch_l2(lds_ptr<const double2>(rec, oNQ) + i + TS_PF_DIST);
      prefetch_l2(lds_ptr<const double2>(rec, oNR) + i + TS_PF_DIST);
      prefetch_l2(lds_ptr<const double2>(rec, oINV) + i + TS_PF_DIST);
      prefetch_l2(lds_ptr<const double2>(rec, oCUM) + i + TS_PF_DIST);
    }
#endif
    const double2 q0 = ld(oNQ, i), r0 = ld(oNR, i), i0 = ld(oINV, i), c0 = ld(oCUM, i), g0 = load_g(i);
    const double2 q1 = ld(oNQ, j), r1 = ld(oNR, j), i1 = ld(oINV, j), c1 = ld(oCUM, j), g1 = load_g(j);
    body(i, q0, r0, g0, i0, c0);
    body(j, q1, r1, g1, i1, c1);
  }
  for (; i < n2; i += 32) {
    const double2 q0 = ld(oNQ, i), r0 = ld(oNR, i), i0 = ld(oINV, i), c0 = ld(oCUM, i), g0 = load_g(i);
    body(i, q0, r0, g0, i0, c0);
  }
  return make_double2(kin, ud);  // (kinetic-energy partial, this lane's part of q . g)
}
// K vector copies in one pass (K = 2, 3 or 5 pairs): U x double2 per operand
// in flight per lane (4 for K <= 3, 2 for K = 5) in an unpredicated main
// loop plus a one-element tail
template <int K, int U>
static __device__ __noinline__ void warp_copy_multi(double2* __restrict__ d0, const double2* __restrict__ s0,
                                                    double2* __restrict__ d1, const double2* __restrict__ s1,
                                                    double2* __restrict__ d2, const double2* __restrict__ s2,
                                                    double2* __restrict__ d3, const double2* __restrict__ s3,
                                                    double2* __restrict__ d4, const double2* __restrict__ s4, int n2) {
  int i = (int)(threadIdx.x & 31);
  const int nfull = n2 - n2 % (32 * U);
#pragma unroll 1
  for (; i < nfull; i += 32 * U) {
    double2 t[K][U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      t[0][u] = __ldcg(s0 + i + 32 * u);
      t[1][u] = __ldcg(s1 + i + 32 * u);
      if constexpr (K > 2) t[2][u] = __ldcg(s2 + i + 32 * u);
      if constexpr (K > 3) { t[3][u] = __ldcg(s3 + i + 32 * u); t[4][u] = __ldcg(s4 + i + 32 * u); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      d0[i + 32 * u] = t[0][u];
      d1[i + 32 * u] = t[1][u];
      if constexpr (K > 2) d2[i + 32 * u] = t[2][u];
      if constexpr (K > 3) { d3[i + 32 * u] = t[3][u]; d4[i + 32 * u] = t[4][u]; }
    }
  }
#pragma unroll 1
  for (; i < n2; i += 32) {
    const double2 x0 = __ldcg(s0 + i), x1 = __ldcg(s1 + i);
    double2 x2, x3, x4;
    if constexpr (K > 2) x2 = __ldcg(s2 + i);
    if constexpr (K > 3) { x3 = __ldcg(s3 + i); x4 = __ldcg(s4 + i); }
    d0[i] = x0;
    d1[i] = x1;
    if constexpr (K > 2) d2[i] = x2;
    if constexpr (K > 3) { d3[i] = x3; d4[i] = x4; }
  }
}

enum Stop : int { kStopNone = 0, kStopTurn = 1, kStopDiv = 2 };

// trace event kinds (int32 x5 per event: kind, a, b, c, e)
enum TraceKind : int {
  kEvWrite = 1,      // (n, slot, -)
  kEvCheck = 2,      // (n, slot, stored leaf)
  kEvTreeEnd = 3,    // (depth j, leapfrogs, stop*16 + go_right, max occupied slots)
  kEvProposal = 4,   // (tree j, leaf index, accepted by outer step)
  kEvOuter = 5,      // (j, turned, -)
};

struct TraceBuf {
  int32_t* ev;      // [cap][5]
  int cap;
  double* leaf_lw;  // [lw_cap]
  int lw_cap;
  int32_t* counts;  // [0] = events written, [1] = leaf lws written, [2] = max occupied slots
};

struct SamplerCfg {
  double step;
  int max_depth;
  int generalized;
  double threshold;
};

struct SlotScalars {
  double lw, metro, pU, pH, fU;
  int count, pidx, leaf;
};
static_assert(sizeof(SlotScalars) == 56, "kTeamScratch assumes 56-byte slot records");

struct TreeOut {
  double lw, sum_metro, pU, pH, fU;
  int count, stop, pidx;
};

struct Stats {
  int depth, leapfrogs, diverged;
  double accept, energy;
};

__device__ __forceinline__ double kInf() { return __longlong_as_double(0x7ff0000000000000LL); }

// tree._logaddexp (tree.py:131-137)
template <bool EXACT>
__device__ __forceinline__ double logaddexp_inner(double a, double b) {
  if (a == -kInf()) return b;
  if (b == -kInf()) return a;
  double hi = a, lo = b;
  if (!(a >= b)) { hi = b; lo = a; }
  return __dadd_rn(hi, x_log1p<EXACT>(x_exp<EXACT>(__dsub_rn(lo, hi))));
}
// numpy npy_logaddexp (used at sampler.py:129)
template <bool EXACT>
__device__ __forceinline__ double logaddexp_np(double x, double y) {
  if (x == y) return __dadd_rn(x, 0.693147180559945309417232121458176568);
  const double tmp = __dsub_rn(x, y);
  if (tmp > 0) return __dadd_rn(x, x_log1p<EXACT>(x_exp<EXACT>(-tmp)));
  if (tmp <= 0) return __dadd_rn(y, x_log1p<EXACT>(x_exp<EXACT>(tmp)));
  return tmp;
}

template <class Team, class Model>
struct Engine {
  Team T;
  Model M;
  VecStore S;
  int D;
  SamplerCfg cfg;
  TraceBuf* tr;  // null unless tracing (leader writes)
  int occupied_mask;

  // replicated scalars
  double U0;            // potential at z0
  double cur_U;         // potential at z_cur
  double LU, RU;        // potentials at the trajectory ends
  double pU, pH;        // transition proposal potential / energy
  int p_tree, p_leaf;   // transition proposal provenance (trace only)
  // running subtree scalars
  double r_lw, r_metro, r_pU, r_pH, r_fU;
  int r_count, r_pidx;
  // NodeStore scalars: per-thread local array for ThreadTeam; shared memory
  // for CTA/warp teams (every team thread writes the identical value), which
  // keeps them out of the local-memory path when shared memory crowds L1.
  SlotScalars* ss;
  // running subtree's first leaf / prefix sum live in NodeStore slot f_alias
  // (instead of V_FQ/V_FR/V_CUMF) after a merge; materialised at tree end
  int f_alias = -1;
  unsigned long long n_evals;
  unsigned long long n_wasted;  // speculative passes discarded (tree stopped early)
  double pending_u;
  unsigned long long* prof = nullptr;  // CTA 0 / thread 0 only (profiling builds of a run)
  long long prof_last = 0;
  long long prof_post = 0;
  long long prof_w0 = 0, prof_w1 = 0;  // dense fused-leaf phase stamps ([24] wait, [25] pass, [26] bookkeeping, [27] leaves)

  // CTA/warp teams keep vectors contiguous in shared memory (unit component
  // stride, 32-bit offsets); thread teams interleave chains in global memory.
  __device__ __forceinline__ double* v(int id) const {
    if constexpr (Team::kUnitStride) {
      if (S.slots != nullptr && id >= S.slot0) return S.slots + (id - S.slot0) * (int)S.vstride;
      return S.base + id * (int)S.vstride;
    } else {
      return S.base + (int64_t)id * S.vstride;  // thread teams never use the slot region
    }
  }
  __device__ __forceinline__ int64_t ds() const {
    if constexpr (Team::kUnitStride) return 1;
    else return S.dstride;
  }

  // ---------------------------------------------------------------- trace
  __device__ void ev(int kind, int a, int b, int c, int e = 0) {
    if (tr == nullptr || !T.leader()) return;
    int n = tr->counts[0];
    if (n < tr->cap) {
      int32_t* p = tr->ev + 5 * n;
      p[0] = kind; p[1] = a; p[2] = b; p[3] = c; p[4] = e;
    }
    tr->counts[0] = n + 1;
  }
  __device__ void ev_lw(double lw) {
    if (tr == nullptr || !T.leader()) return;
    int n = tr->counts[1];
    if (n < tr->lw_cap) tr->leaf_lw[n] = lw;
    tr->counts[1] = n + 1;
  }

  // ------------------------------------------------------- vector helpers
  __device__ __forceinline__ void copy(int dst, int src) {
    double* a = v(dst);
    const double* b = v(src);
    if constexpr (Team::kWarp && Team::kUnitStride && Model::kVecOps) {
      // warp-owned contiguous vectors (large D in global memory): 16-byte
      // accesses, 8 in flight per lane, so a copy costs ~D/512 round trips
      if (((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0 && (D & 1) == 0 && D >= 128) {
        warp_copy2(reinterpret_cast<double2*>(a), reinterpret_cast<const double2*>(b), D >> 1);
        return;
      }
    }
    const int64_t s = ds();
    for (int d = T.rank(); d < D; d += T.size()) a[d * s] = b[d * s];
  }
  // 3 or 5 copies (d3 < 0: three); one fused pass for large-D warp vectors
  __device__ void copy_group(int d0, int s0, int d1, int s1, int d2, int s2, int d3 = -1, int s3 = -1, int d4 = -1,
                             int s4 = -1) {
    if constexpr (Team::kWarp && Team::kUnitStride && Model::kVecOps) {
      // k = 2 when the third pair repeats the second (the proposal copies)
      const int k = d3 >= 0 ? 5 : ((d2 == d1 && s2 == s1) ? 2 : 3);
      double* a[5] = {v(d0), v(d1), v(d2), k > 3 ? v(d3) : v(d0), k > 3 ? v(d4) : v(d0)};
      const double* b[5] = {v(s0), v(s1), v(s2), k > 3 ? v(s3) : v(s0), k > 3 ? v(s4) : v(s0)};
      bool ok = D >= 128 && (D & 1) == 0;
#pragma unroll
      for (int i = 0; i < 5; ++i) ok = ok && al16(a[i]) && al16(b[i]);
      if (ok) {
        double2* A0 = reinterpret_cast<double2*>(a[0]); double2* A1 = reinterpret_cast<double2*>(a[1]);
        double2* A2 = reinterpret_cast<double2*>(a[2]); double2* A3 = reinterpret_cast<double2*>(a[3]);
        double2* A4 = reinterpret_cast<double2*>(a[4]);
        const double2* B0 = reinterpret_cast<const double2*>(b[0]); const double2* B1 = reinterpret_cast<const double2*>(b[1]);
        const double2* B2 = reinterpret_cast<const double2*>(b[2]); const double2* B3 = reinterpret_cast<const double2*>(b[3]);
        const double2* B4 = reinterpret_cast<const double2*>(b[4]);
        if (k == 2) warp_copy_multi<2, 4>(A0, B0, A1, B1, A1, B1, A1, B1, A1, B1, D >> 1);
        else if (k == 3) warp_copy_multi<3, 4>(A0, B0, A1, B1, A2, B2, A2, B2, A2, B2, D >> 1);
        else warp_copy_multi<5, 2>(A0, B0, A1, B1, A2, B2, A3, B3, A4, B4, D >> 1);
        return;
      }
    }
    // one loop, all loads of an element before its stores (the groups never
    // copy into a vector another member of the group reads)
    double* a0 = v(d0); double* a1 = v(d1); double* a2 = v(d2);
    const double* b0 = v(s0); const double* b1 = v(s1); const double* b2 = v(s2);
    const int64_t s = ds();
    if (d3 < 0) {
      for (int d = T.rank(); d < D; d += T.size()) {
        const double x0 = b0[d * s], x1 = b1[d * s], x2 = b2[d * s];
        a0[d * s] = x0; a1[d * s] = x1; a2[d * s] = x2;
      }
      return;
    }
    double* a3 = v(d3); double* a4 = v(d4);
    const double* b3 = v(s3); const double* b4 = v(s4);
    for (int d = T.rank(); d < D; d += T.size()) {
      const double x0 = b0[d * s], x1 = b1[d * s], x2 = b2[d * s], x3 = b3[d * s], x4 = b4[d * s];
      a0[d * s] = x0; a1[d * s] = x1; a2[d * s] = x2; a3[d * s] = x3; a4[d * s] = x4;
    }
  }
  // momentum_std (sampler.py:95 draws r0 = N(0,1) * mass.momentum_std)
  __device__ void refresh_mstd() {
    const double* inv = v(V_INV);
    double* m = v(V_MSTD);
    const int64_t s = ds();
    for (int d = T.rank(); d < D; d += T.size()) m[d * s] = __ddiv_rn(1.0, __dsqrt_rn(inv[d * s]));
    T.sync();
  }
  __device__ __forceinline__ void fill(int dst, double x) {
    double* a = v(dst);
    const int64_t s = ds();
    for (int d = T.rank(); d < D; d += T.size()) a[d * s] = x;
  }

  // model evaluation at vector qid -> U (non-finite -> +inf), gradient -> gid
  __device__ double eval(int qid, int gid) {
    post_eval(qid, gid);
    return wait_eval();
  }
  // Asynchronous form (grid mode: the worker warps stream while the driver
  // continues); synchronous models evaluate in post and return in wait.
  __device__ void post_eval(int qid, int gid) {
    T.sync();
    if (prof != nullptr && T.leader()) {  // profiling: [9] cycles between passes
      const long long c0 = clock64();
      if (prof_last) prof[9] += c0 - prof_last;
      prof_post = c0;
    }
    if constexpr (Model::kAsync) M.post(qid, gid);
    else pending_u = M.eval(T, S, qid, gid);
  }
  __device__ double wait_eval() {
    double u;
    if constexpr (Model::kAsync) u = M.wait();
    else u = pending_u;
    T.sync();
    if (prof != nullptr && T.leader()) {  // [8] cycles from post to result, [10] passes
      const long long c1 = clock64();
      prof[8] += c1 - prof_post;
      prof[10] += 1;
      prof_last = c1;
    }
    n_evals += 1;
    return isfinite(u) ? u : kInf();
  }

  // kinetic_energy_impl (kernels.py:125-130): sum 0.5 r r inv, left to right
  __device__ double kinetic(int rid) {
    const double* r = v(rid);
    const double* inv = v(V_INV);
    if constexpr (Team::kWarp && Team::kUnitStride && Model::kVecOps) {
      if (D >= 128 && (D & 1) == 0 && al16(r) && al16(inv))
        return T.sum(warp_kinetic2(reinterpret_cast<const double2*>(r), reinterpret_cast<const double2*>(inv), D >> 1));
    }
    const int64_t s = ds();
    double acc = 0.0;
    for (int d = T.rank(); d < D; d += T.size()) {
      const double x = r[d * s];
      acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(0.5, x), x), inv[d * s]));
    }
    return T.sum(acc);
  }
  // hamiltonian (integrator.py:82-87)
  __device__ double hamiltonian(double U, int rid) {
    if (!isfinite(U)) return kInf();
    const double h = __dadd_rn(U, kinetic(rid));
    return isfinite(h) ? h : kInf();
  }

  // uturn_dots (kernels.py:132-139): (sum rho inv rl < 0) or (sum rho inv rr < 0)
  __device__ bool uturn_dots(int rho_id, int rl_id, int rr_id) {
    const double* rho = v(rho_id);
    const double* inv = v(V_INV);
    const double* rl = v(rl_id);
    const double* rr = v(rr_id);
    const int64_t s = ds();
    double a = 0.0, b = 0.0;
    for (int d = T.rank(); d < D; d += T.size()) {
      const double w = __dmul_rn(rho[d * s], inv[d * s]);
      a = __dadd_rn(a, __dmul_rn(w, rl[d * s]));
      b = __dadd_rn(b, __dmul_rn(w, rr[d * s]));
    }
    T.sum2(a, b);
    return a < 0.0 || b < 0.0;
  }

  // leapfrog on (CQ, CR, CG, cur_U) in place (integrator.py:90-103)
  __device__ void leapfrog(double eps) {
    const double half = __dmul_rn(0.5, eps);
    double* q = v(V_CQ);
    double* r = v(V_CR);
    const double* g = v(V_CG);
    const double* inv = v(V_INV);
    const int64_t s = ds();
    for (int d = T.rank(); d < D; d += T.size()) {
      const double rh = __dsub_rn(r[d * s], __dmul_rn(half, g[d * s]));
      r[d * s] = rh;
      q[d * s] = __dadd_rn(q[d * s], __dmul_rn(eps, __dmul_rn(inv[d * s], rh)));
    }
    cur_U = eval(V_CQ, V_CG);
    for (int d = T.rank(); d < D; d += T.size()) r[d * s] = __dsub_rn(r[d * s], __dmul_rn(half, g[d * s]));
  }

  // ------------------------------------------------------- tree builder
  // with_first = false: the caller merges a stored subtree next, which
  // replaces first / cum_first, so only the proposal is materialised
  __device__ int fq_id() const { return f_alias < 0 ? (int)V_FQ : slot_vec(f_alias, 0); }
  __device__ int fr_id() const { return f_alias < 0 ? (int)V_FR : slot_vec(f_alias, 1); }
  __device__ int cumf_id() const { return f_alias < 0 ? (int)V_CUMF : slot_vec(f_alias, 2); }
  __device__ void running_from_leaf(int n, double lw, double metro, double h, bool with_first = true,
                                    bool copy_proposal = true) {
    if (with_first) {
      copy_group(V_FQ, V_CQ, V_FR, V_CR, V_CUMF, V_CUM, V_TPQ, V_CQ, V_TPG, V_CG);
      f_alias = -1;
    } else if (copy_proposal) {
      copy_group(V_TPQ, V_CQ, V_TPG, V_CG, V_TPG, V_CG);
    }
    r_lw = lw; r_metro = metro; r_count = 1; r_pU = cur_U; r_pH = h; r_pidx = n; r_fU = cur_U;
  }

  // running = _merge(summaries[s], running, u)   (tree.py:140-156)
  __device__ void merge_slot(int s, double u) {
    const SlotScalars& L = ss[s];
    const double lw = logaddexp_inner<Team::kExactMath>(L.lw, r_lw);
    const double p_right = (r_lw == -kInf()) ? 0.0 : x_exp<Team::kExactMath>(__dsub_rn(r_lw, lw));
    if (!(u < p_right)) {
      copy_group(V_TPQ, slot_vec(s, 3), V_TPG, slot_vec(s, 4), V_TPG, slot_vec(s, 4));
      r_pU = L.pU; r_pH = L.pH; r_pidx = L.pidx;
    }
    // first / cum_first come from the left (stored) subtree: alias, no copy
    f_alias = s;
    r_fU = L.fU;
    r_lw = lw;
    r_count = L.count + r_count;
    r_metro = __dadd_rn(L.metro, r_metro);
  }

  __device__ void merge_out(int start, Stream& draws) {
    for (int s = start - 1; s >= 0; --s) merge_slot(s, draws.next_double());
  }

  // U-turn test of the running subtree (tree.py:436-446)
  __device__ bool running_turning(bool forward) {
    const int64_t s = ds();
    if (cfg.generalized) {
      // rho = (cum_last - cum_first) + first.r  -> V_MSUM as scratch
      double* rho = v(V_MSUM);
      const double* cum = v(V_CUM);
      const double* cf = v(cumf_id());
      const double* fr = v(fr_id());
      if constexpr (Team::kWarp && Team::kUnitStride && Model::kVecOps) {
        const double* inv = v(V_INV);
        const double* cr = v(V_CR);
        if (D >= 128 && (D & 1) == 0 && al16(cum) && al16(cf) && al16(fr) && al16(inv) && al16(cr)) {
          const double2 ab = warp_gen_uturn2(reinterpret_cast<const double2*>(cum), reinterpret_cast<const double2*>(cf),
                                             reinterpret_cast<const double2*>(fr), reinterpret_cast<const double2*>(inv),
                                             reinterpret_cast<const double2*>(cr), D >> 1);
          double a = ab.x, b = ab.y;
          T.sum2(a, b);
          return a < 0.0 || b < 0.0;
        }
      }
      for (int d = T.rank(); d < D; d += T.size()) rho[d * s] = __dadd_rn(__dsub_rn(cum[d * s], cf[d * s]), fr[d * s]);
      return uturn_dots(V_MSUM, fr_id(), V_CR);
    }
    double* dq = v(V_MSUM);
    const double* lq = v(V_CQ);
    const double* fq = v(fq_id());
    if (forward) {
      for (int d = T.rank(); d < D; d += T.size()) dq[d * s] = __dsub_rn(lq[d * s], fq[d * s]);
      return uturn_dots(V_MSUM, fr_id(), V_CR);
    }
    for (int d = T.rank(); d < D; d += T.size()) dq[d * s] = __dsub_rn(fq[d * s], lq[d * s]);
    return uturn_dots(V_MSUM, V_CR, fr_id());
  }

  // leaf energy bookkeeping shared by both branches
  __device__ void leaf_energy(double h_ref, double& h, double& delta) {
    h = hamiltonian(cur_U, V_CR);
    delta = __dsub_rn(h, h_ref);
  }

  __device__ void add_cum() {
    double* c = v(V_CUM);
    const double* r = v(V_CR);
    if constexpr (Team::kWarp && Team::kUnitStride && Model::kVecOps) {
      if (D >= 128 && (D & 1) == 0 && al16(c) && al16(r)) {
        warp_add2(reinterpret_cast<double2*>(c), reinterpret_cast<const double2*>(r), D >> 1);
        return;
      }
    }
    const int64_t s = ds();
    for (int d = T.rank(); d < D; d += T.size()) c[d * s] = __dadd_rn(c[d * s], r[d * s]);
  }

  // Split leapfrog for the speculative pipeline: drift from the current leaf
  // into (NQ, NR = r_half); after the pass, the new leaf becomes current and
  // gets its kick (same arithmetic as leapfrog()).
  __device__ void drift_next(double eps) {
    const double half = __dmul_rn(0.5, eps);
    const double* q = v(V_CQ);
    const double* r = v(V_CR);
    const double* g = v(V_CG);
    double* nq = v(V_NQ);
    double* nr = v(V_NR);
    const double* inv = v(V_INV);
    if constexpr (Team::kWarp && Team::kUnitStride && Model::kVecOps) {
      if (D >= 128 && (D & 1) == 0 && al16(q) && al16(r) && al16(g) && al16(nq) && al16(nr) && al16(inv)) {
        warp_drift2(reinterpret_cast<double2*>(nq), reinterpret_cast<double2*>(nr), reinterpret_cast<const double2*>(q),
                    reinterpret_cast<const double2*>(r), reinterpret_cast<const double2*>(g),
                    reinterpret_cast<const double2*>(inv), half, eps, D >> 1);
        return;
      }
    }
    const int64_t s = ds();
    for (int d = T.rank(); d < D; d += T.size()) {
      const double rh = __dsub_rn(r[d * s], __dmul_rn(half, g[d * s]));
      nr[d * s] = rh;
      nq[d * s] = __dadd_rn(q[d * s], __dmul_rn(eps, __dmul_rn(inv[d * s], rh)));
    }
  }
  __device__ void advance_leaf(double eps, double u) {
    const double half = __dmul_rn(0.5, eps);
    double* q = v(V_CQ);
    double* r = v(V_CR);
    double* g = v(V_CG);
    const double* nq = v(V_NQ);
    const double* nr = v(V_NR);
    const double* ng = v(V_NG);
    cur_U = u;
    if constexpr (Team::kWarp && Team::kUnitStride && Model::kVecOps) {
      if (D >= 128 && (D & 1) == 0 && al16(q) && al16(r) && al16(g) && al16(nq) && al16(nr) && al16(ng)) {
        warp_advance2(reinterpret_cast<double2*>(q), reinterpret_cast<double2*>(r), reinterpret_cast<double2*>(g),
                      reinterpret_cast<const double2*>(nq), reinterpret_cast<const double2*>(nr),
                      reinterpret_cast<const double2*>(ng), half, D >> 1);
        return;
      }
    }
    const int64_t s = ds();
    for (int d = T.rank(); d < D; d += T.size()) {
      const double gg = ng[d * s];
      q[d * s] = nq[d * s];
      g[d * s] = gg;
      r[d * s] = __dsub_rn(nr[d * s], __dmul_rn(half, gg));
    }
  }

  // advance_leaf(eps, u) followed by drift_next(eps) in one pass over the
  // vectors (same arithmetic, element by element)
  __device__ void advance_drift(double eps, double u) {
    const double half = __dmul_rn(0.5, eps);
    double* q = v(V_CQ);
    double* r = v(V_CR);
    double* g = v(V_CG);
    double* nq = v(V_NQ);
    double* nr = v(V_NR);
    const double* ng = v(V_NG);
    const double* inv = v(V_INV);
    cur_U = u;
    if constexpr (Team::kWarp && Team::kUnitStride && Model::kVecOps) {
      if (D >= 128 && (D & 1) == 0 && al16(q) && al16(r) && al16(g) && al16(nq) && al16(nr) && al16(ng) && al16(inv)) {
        warp_advance2(reinterpret_cast<double2*>(q), reinterpret_cast<double2*>(r), reinterpret_cast<double2*>(g),
                      reinterpret_cast<const double2*>(nq), reinterpret_cast<const double2*>(nr),
                      reinterpret_cast<const double2*>(ng), half, D >> 1);
        warp_drift2(reinterpret_cast<double2*>(nq), reinterpret_cast<double2*>(nr), reinterpret_cast<const double2*>(q),
                    reinterpret_cast<const double2*>(r), reinterpret_cast<const double2*>(g),
                    reinterpret_cast<const double2*>(inv), half, eps, D >> 1);
        return;
      }
    }
    const int64_t s = ds();
    for (int d = T.rank(); d < D; d += T.size()) {
      const double gg = ng[d * s];
      const double qq = nq[d * s];
      const double rr = __dsub_rn(nr[d * s], __dmul_rn(half, gg));
      q[d * s] = qq;
      g[d * s] = gg;
      r[d * s] = rr;
      const double rh = __dsub_rn(rr, __dmul_rn(half, gg));
      nr[d * s] = rh;
      nq[d * s] = __dadd_rn(qq, __dmul_rn(eps, __dmul_rn(inv[d * s], rh)));
    }
  }

  // Bookkeeping of leaf n (tree.py:403-450): divergence exit, even-leaf store
  // at slot popcount(n), odd-leaf merges + U-turn checks down to i_min.
  // prestored: the leaf pass already wrote the even leaf's slot / the odd
  // leaf's running proposal (warp_leaf_fused ST)
  __device__ int leaf_book(unsigned long long n, double h, double delta, Stream& draws, bool forward,
                           bool prestored = false) {
    const double thr = cfg.threshold;
    const int pc = __popcll(n);
    if (!(isfinite(delta) && delta <= thr)) {
      const double metro = isfinite(delta) ? x_exp<Team::kExactMath>(-delta) : 0.0;
      ev_lw(-kInf());
      running_from_leaf((int)n, -kInf(), metro, h);
      merge_out(pc, draws);
      return kStopDiv;
    }
    const double lw = -h;
    const double metro = delta > 0 ? x_exp<Team::kExactMath>(-delta) : 1.0;
    ev_lw(lw);
    if ((n & 1ULL) == 0) {
      const int slot = pc;
      if (!prestored)
        copy_group(slot_vec(slot, 0), V_CQ, slot_vec(slot, 1), V_CR, slot_vec(slot, 2), V_CUM, slot_vec(slot, 3), V_CQ,
                   slot_vec(slot, 4), V_CG);
      SlotScalars& L = ss[slot];
      L.lw = lw; L.metro = metro; L.pU = cur_U; L.pH = h; L.fU = cur_U;
      L.count = 1; L.pidx = (int)n; L.leaf = (int)n;
      occupied_mask |= 1 << slot;
      ev(kEvWrite, (int)n, slot, 0);
      return kStopNone;
    }
    int slot = pc - 1;
    const int i_min = slot - __popcll(((n + 1) & ~n) - 1) + 1;
    running_from_leaf((int)n, lw, metro, h, false, !prestored);  // odd n: at least one merge follows
    while (slot >= i_min) {
      ev(kEvCheck, (int)n, slot, ss[slot].leaf);
      merge_slot(slot, draws.next_double());
      if (running_turning(forward)) {
        merge_out(slot, draws);
        return kStopTurn;
      }
      --slot;
    }
    // summaries[i_min] = running: first/cum_first already equal slot i_min's
    copy_group(slot_vec(i_min, 3), V_TPQ, slot_vec(i_min, 4), V_TPG, slot_vec(i_min, 4), V_TPG);
    SlotScalars& L = ss[i_min];
    L.lw = r_lw; L.metro = r_metro; L.pU = r_pU; L.pH = r_pH; L.count = r_count; L.pidx = r_pidx;
    return kStopNone;
  }

  // build_tree_iterative (tree.py:344-453).  Input: frontier in CQ/CR/CG/cur_U.
  // Output: running subtree (FQ/FR/CUMF + TPQ/TPG + r_* scalars), last leaf in
  // CQ/CR/CG/cur_U, momentum sum in V_MSUM.
  // (noinline: separate register allocation per phase keeps the chain state
  // out of local memory, which shares the L1 left over by the TMA stages)
  __device__ __noinline__ TreeOut build_tree(int depth, double eps, double h_ref, Key key) {
    if constexpr (!Model::kAsync) {
      // Synchronous (small) models: run the tree on a private copy of the
      // engine.  Its address never escapes, so the engine's fields stay in
      // registers instead of being reloaded from the stack after every
      // vector store (which may alias it through a generic pointer).
      Engine L = *this;
      const TreeOut o = L.build_tree_body(depth, eps, h_ref, key);
      *this = L;
      return o;
    } else {
      return build_tree_body(depth, eps, h_ref, key);
    }
  }
  __device__ __forceinline__ TreeOut build_tree_body(int depth, double eps, double h_ref, Key key) {
    Stream draws;
    draws.init(key);
    occupied_mask = 0;
    fill(V_CUM, 0.0);
    const double thr = cfg.threshold;
    const bool forward = eps > 0;
    (void)thr;
    int stop = kStopNone;
    if (depth == 0) {
      leapfrog(eps);
      add_cum();
      double h, delta;
      leaf_energy(h_ref, h, delta);
      const bool div = !isfinite(delta) || delta > thr;
      const double lw = div ? -kInf() : -h;
      const double metro = !isfinite(delta) ? 0.0 : (delta > 0 ? x_exp<Team::kExactMath>(-delta) : 1.0);
      ev_lw(lw);
      running_from_leaf(0, lw, metro, h);
      stop = div ? kStopDiv : kStopNone;
    } else {
      const unsigned long long nleaves = 1ULL << depth;
      if constexpr (Model::kAsync) {
       if (M.traj_ok()) {
        // The workers run the leapfrog chain (LogisticW::serve_traj): leaf n
        // arrives in a ring slot while leaf n+1 streams; this warp only does
        // the bookkeeping and gates the chain (at most one wasted pass).
        M.traj_start(V_CQ, V_CR, V_CG, eps, (int)nleaves);
        double* cq = v(V_CQ);
        double* cr = v(V_CR);
        double* cg = v(V_CG);
        // TS_PROF (CTA 0): [20] driver waiting for leaves, [21] bookkeeping per leaf, [22] leaves
        const bool tpf = prof != nullptr && T.leader();
        for (unsigned long long n = 0; n < nleaves; ++n) {
          const long long w0 = tpf ? clock64() : 0;
          const double* sl = M.traj_wait((int)n);
          const long long w1 = tpf ? clock64() : 0;
          if (tpf) { prof[20] += w1 - w0; prof[22] += 1; }
          for (int d = T.rank(); d < D; d += T.size()) {
            const double a0 = sl[d], a1 = sl[D + d], a2 = sl[2 * D + d];
            cq[d] = a0; cr[d] = a1; cg[d] = a2;
          }
          const double u = sl[3 * D];
          cur_U = isfinite(u) ? u : kInf();
          n_evals += 1;
          T.sync();
          add_cum();
          double h, delta;
          leaf_energy(h_ref, h, delta);
          stop = leaf_book(n, h, delta, draws, forward);
          if (stop != kStopNone) {
            const int w = M.traj_stop((int)n);
            n_evals += w;
            n_wasted += w;
            break;
          }
          M.traj_approve((int)n);
          if (tpf) prof[21] += clock64() - w1;
        }
       } else {
        // Speculative pipelining (grid mode): as soon as leaf n's gradient is
        // back, drift to leaf n+1 and post its data pass to the worker warps,
        // then do leaf n's bookkeeping while they stream.  If the bookkeeping
        // stops the tree (U-turn / divergence), the posted pass is waited for
        // and discarded; the last leaf of a tree is never speculated.
        drift_next(eps);
        post_eval(V_NQ, V_NG);
        for (unsigned long long n = 0; n < nleaves; ++n) {
          const bool spec = n + 1 < nleaves;
          bool fusable = false;
          if constexpr (Team::kWarp && Team::kUnitStride && Model::kVecOps) fusable = spec && D >= 128 && (D & 1) == 0;
          double u = 0.0;
          bool waited = false;
          if constexpr (Team::kWarp && Team::kUnitStride && Model::kVecOps) {
            if (fusable) {
              if (prof != nullptr && T.leader()) prof_w0 = clock64();
              M.wait_poll();  // the fused pass reads the gradient row itself and forms U
              if (prof != nullptr && T.leader()) { prof_w1 = clock64(); prof[24] += prof_w1 - prof_w0; prof[27] += 1; }
              n_evals += 1;
              waited = true;
            }
          }
          if (!waited) u = wait_eval();
          double h, delta;
          bool fused = false;
          if constexpr (Team::kWarp && Team::kUnitStride && Model::kVecOps) {
            // batched large-D model: kick, prefix sum, kinetic energy, U,
            // next drift, the request row and the NodeStore copies in one
            // pass over the vectors
            if (fusable) {
              const double half = __dmul_rn(0.5, eps);
              void* row = M.request_row();
              double2* q2 = reinterpret_cast<double2*>(v(V_CQ));
              double2* r2 = reinterpret_cast<double2*>(v(V_CR));
              double2* g2 = reinterpret_cast<double2*>(v(V_CG));
              double2* nq2 = reinterpret_cast<double2*>(v(V_NQ));
              double2* nr2 = reinterpret_cast<double2*>(v(V_NR));
              const void* ng2 = M.grad_row();
              const double2* inv2 = reinterpret_cast<const double2*>(v(V_INV));
              double2* c2 = reinterpret_cast<double2*>(v(V_CUM));
              // leaf_book's NodeStore copies written by the same pass
              LeafVecs* lv = M.leaf_vecs();
              if (T.leader()) {
                lv->q = q2; lv->r = r2; lv->g = g2; lv->nq = nq2; lv->nr = nr2; lv->grow = ng2; lv->inv = inv2;
                lv->cum = c2; lv->row = row; lv->half = half; lv->eps = eps; lv->n2 = D >> 1;
                if ((n & 1ULL) == 0) {
                  const int sl = __popcll(n);
#pragma unroll
                  for (int k = 0; k < 5; ++k) lv->st[k] = reinterpret_cast<double2*>(v(slot_vec(sl, k)));
                } else {
                  lv->st[0] = reinterpret_cast<double2*>(v(V_TPQ));
                  lv->st[1] = reinterpret_cast<double2*>(v(V_TPG));
                }
              }
              __syncwarp();
              double2 ku;
              if ((n & 1ULL) == 0) ku = M.fp64 ? warp_leaf_fused<true, 5>(lv) : warp_leaf_fused<false, 5>(lv);
              else ku = M.fp64 ? warp_leaf_fused<true, 2>(lv) : warp_leaf_fused<false, 2>(lv);
              const double kin = ku.x, ud = ku.y;
              T.sync();
              if (prof != nullptr && T.leader()) { const long long c = clock64(); prof[28] += c - prof_w1; prof_w1 = c; }
              M.post_written(V_NQ, V_NG);
              if (prof != nullptr && T.leader()) { const long long c = clock64(); prof[29] += c - prof_w1; prof[25] += c - prof_w1; prof_w1 = c; }
              // both warp reductions in one interleaved shuffle tree (same
              // tree order per value as T.sum)
              double uds = ud, ke = kin;
              T.sum2(uds, ke);
              {
                const double uu = 0.5 * uds;  // DenseW::wait's U, formed in the pass
                cur_U = isfinite(uu) ? uu : kInf();
              }
              if (!isfinite(cur_U)) h = kInf();
              else {
                h = __dadd_rn(cur_U, ke);
                if (!isfinite(h)) h = kInf();
              }
              delta = __dsub_rn(h, h_ref);
              fused = true;
              if (prof != nullptr && T.leader()) { prof_w0 = clock64(); prof[25] += prof_w0 - prof_w1; prof[30] += prof_w0 - prof_w1; }
            }
          }
          if (!fused) {
            if (spec) {
              // leaf n's kick fused with leaf n+1's drift: the next pass is
              // posted after one vector loop; leaf n's energy, prefix sum and
              // bookkeeping overlap with it
              advance_drift(eps, u);
              post_eval(V_NQ, V_NG);
            } else {
              advance_leaf(eps, u);
            }
            add_cum();
            leaf_energy(h_ref, h, delta);
          }
          stop = leaf_book(n, h, delta, draws, forward, fused);
          if (fused && prof != nullptr && T.leader()) prof[26] += clock64() - prof_w0;
          if (stop != kStopNone) {
            if (spec) { (void)wait_eval(); n_wasted += 1; }
            break;
          }
        }
       }
      } else {
        for (unsigned long long n = 0; n < nleaves; ++n) {
          leapfrog(eps);
          add_cum();
          double h, delta;
          leaf_energy(h_ref, h, delta);
          stop = leaf_book(n, h, delta, draws, forward);
          if (stop != kStopNone) break;
        }
      }
    }
    if (f_alias >= 0) {  // the tree's first leaf / prefix sum into V_FQ/V_FR/V_CUMF
      copy_group(V_FQ, slot_vec(f_alias, 0), V_FR, slot_vec(f_alias, 1), V_CUMF, slot_vec(f_alias, 2));
      f_alias = -1;
    }
    // momentum_sum = (cum_last - cum_first) + first.r   (tree.py:283-294)
    {
      double* ms = v(V_MSUM);
      const double* cum = v(V_CUM);
      const double* cf = v(V_CUMF);
      const double* fr = v(V_FR);
      const int64_t s = ds();
      for (int d = T.rank(); d < D; d += T.size()) ms[d * s] = __dadd_rn(__dsub_rn(cum[d * s], cf[d * s]), fr[d * s]);
    }
    if (tr != nullptr && T.leader()) tr->counts[2] = __popc(occupied_mask);
    TreeOut o;
    o.lw = r_lw; o.sum_metro = r_metro; o.pU = r_pU; o.pH = r_pH; o.fU = r_fU;
    o.count = r_count; o.stop = stop; o.pidx = r_pidx;
    return o;
  }

  // ------------------------------------------------------- transition
  // Momentum refresh r0 = N(0,1) * momentum_std (sampler.py:95); normals from
  // fold(key, 0) (or injected, std normal, component-major with stride inj_ds).
  __device__ void draw_momentum(int rid, Key nkey, const double* inj, int64_t inj_ds) {
    double* r = v(rid);
    const double* mstd = v(V_MSTD);  // 1/sqrt(inv), exactly as computed per draw before
    const int64_t s = ds();
    if (inj != nullptr) {
      for (int d = T.rank(); d < D; d += T.size()) r[d * s] = __dmul_rn(inj[d * inj_ds], mstd[d * s]);
      return;
    }
    if constexpr (Team::kWarp) {
      // Warp-parallel ziggurat: lane l tries normal (done + l) on stream word
      // (w + l), i.e. assuming the preceding normals of the chunk each took
      // one word (the ziggurat fast path, ~99%).  The first lane that falls
      // off the fast path is resolved with the sequential generator, and the
      // chunk restarts after it: the values are exactly numpy's sequence.
      const int lane = T.rank();
      uint64_t w = 0;  // next unread word of the stream
      int done = 0;
      while (done < D) {
        const uint64_t my = w + lane;
        uint64_t c[4] = {my / 4 + 1, 0, 0, 1};
        if (c[0] == 0) c[1] = 1;
        philox4x64_10(c, nkey.hi, nkey.lo);
        const int o = (int)(my & 3);
        uint64_t rr = o == 0 ? c[0] : (o == 1 ? c[1] : (o == 2 ? c[2] : c[3]));
        const int idx = (int)(rr & 0xff);
        rr >>= 8;
        const int sign = (int)(rr & 1);
        const uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
        double z = __dmul_rn((double)rabs, TS_ZIG_WI[idx]);
        if (sign) z = -z;
        const bool fast = rabs < TS_ZIG_KI[idx];
        const int want = min(32, D - done);
        const unsigned slow = __ballot_sync(0xffffffffu, !fast) & (want == 32 ? 0xffffffffu : ((1u << want) - 1u));
        const int nfast = slow ? __ffs(slow) - 1 : want;
        if (lane < nfast) r[(done + lane) * s] = __dmul_rn(z, mstd[(done + lane) * s]);
        done += nfast;
        w += (uint64_t)nfast;
        if (slow) {  // normal `done` leaves the fast path: replay it sequentially
          Stream ns;
          ns.init(nkey);
          ns.c0 = w / 4;
          for (int k = 0; k < (int)(w & 3); ++k) (void)ns.next_u64();
          if ((w & 3) == 0) ns.pos = 4;
          const double zs = ns.normal();
          if (lane == 0) r[done * s] = __dmul_rn(zs, mstd[done * s]);
          w = (ns.pos == 4) ? ns.c0 * 4 : (ns.c0 - 1) * 4 + (uint64_t)ns.pos;
          done += 1;
        }
      }
      __syncwarp();
      return;
    }
    Stream ns;
    ns.init(nkey);
    for (int d = 0; d < D; ++d) {
      const double z = ns.normal();
      if ((d % T.size()) == T.rank()) r[d * s] = __dmul_rn(z, mstd[d * s]);
    }
  }

  // nuts_transition_from (sampler.py:83-148): z0 = (Q0, G0, U0) -> proposal
  // sampler.hmc_transition (sampler.py:163-203): fixed-length HMC baseline.
  // State in (Q0, G0, U0); momentum from fold(key, 0), accept uniform from
  // fold(key, 1).  On acceptance (Q0, G0, U0) move to the trajectory end.
  __device__ __noinline__ Stats hmc(Key key, const double* inj, int64_t inj_ds, int num_steps, bool& accepted) {
    draw_momentum(V_R0, key_fold(key, 0), inj, inj_ds);
    const double h0 = hamiltonian(U0, V_R0);
    copy(V_CQ, V_Q0); copy(V_CR, V_R0); copy(V_CG, V_G0); cur_U = U0;
    int steps = 0;
    for (int i = 0; i < num_steps; ++i) {
      leapfrog(cfg.step);
      steps += 1;
      if (!isfinite(cur_U)) break;
    }
    const double h1 = hamiltonian(cur_U, V_CR);
    const double delta = __dsub_rn(h1, h0);
    const double p_accept = (isfinite(delta) && delta > 0) ? x_exp<Team::kExactMath>(-delta) : (isfinite(delta) ? 1.0 : 0.0);
    Stream gen;
    gen.init(key_fold(key, 1));
    accepted = gen.next_double() < p_accept;
    if (accepted) { copy(V_Q0, V_CQ); copy(V_G0, V_CG); U0 = cur_U; }
    Stats st;
    st.depth = 0;
    st.leapfrogs = steps;
    st.diverged = !isfinite(delta) || delta > cfg.threshold;
    st.accept = p_accept;
    st.energy = accepted ? h1 : h0;
    return st;
  }

  __device__ __noinline__ Stats transition(Key key, const double* inj, int64_t inj_ds) {
    if constexpr (!Model::kAsync) {
      // synchronous models: the whole transition (trees inlined) on a
      // register-resident copy of the engine, as in build_tree
      Engine L = *this;
      const Stats st = L.transition_body(key, inj, inj_ds);
      *this = L;
      return st;
    } else {
      return transition_body(key, inj, inj_ds);
    }
  }
  __device__ __forceinline__ Stats transition_body(Key key, const double* inj, int64_t inj_ds) {
    // profiling (CTA 0 driver lane 0): [12] transition prologue, [13] between
    // trees, [14] trees, [15] transitions
    const bool tp = prof != nullptr && T.leader();
    long long t_last = tp ? clock64() : 0;
    if (tp) prof[15] += 1;
    draw_momentum(V_R0, key_fold(key, 0), inj, inj_ds);
    if (tp) prof[16] += clock64() - t_last;
    const double h0 = hamiltonian(U0, V_R0);
    Stream gen;
    gen.init(key_fold(key, 1));
    copy_group(V_LQ, V_Q0, V_LR, V_R0, V_LG, V_G0, V_RQ, V_Q0, V_RR, V_R0);
    copy_group(V_RG, V_G0, V_PQ, V_Q0, V_PG, V_G0, V_RHO, V_R0, V_RHO, V_R0);
    LU = U0; RU = U0; pU = U0; pH = h0; p_tree = -1; p_leaf = -1;
    double lw = -h0;
    int leapfrogs = 0;
    double sum_metro = 0.0;
    bool diverged = false;
    int depth_reached = 0;
    for (int j = 0; j < cfg.max_depth; ++j) {
      const bool go_right = gen.next_double() < 0.5;
      const double eps = go_right ? cfg.step : -cfg.step;
      if (go_right) { copy_group(V_CQ, V_RQ, V_CR, V_RR, V_CG, V_RG); cur_U = RU; }
      else { copy_group(V_CQ, V_LQ, V_CR, V_LR, V_CG, V_LG); cur_U = LU; }
      if (tp) { const long long c = clock64(); prof[j == 0 ? 12 : 13] += c - t_last; prof[14] += 1; }
      TreeOut t;
      if constexpr (!Model::kAsync) t = build_tree_body(j, eps, h0, key_fold(key, 2 + (uint64_t)j));
      else t = build_tree(j, eps, h0, key_fold(key, 2 + (uint64_t)j));
      if (tp) t_last = clock64();
      leapfrogs += t.count;
      sum_metro = __dadd_rn(sum_metro, t.sum_metro);
      ev(kEvTreeEnd, j, t.count, t.stop * 16 + (go_right ? 1 : 0), __popc(occupied_mask));
      if (t.stop != kStopNone) {
        diverged = diverged || (t.stop == kStopDiv);
        depth_reached = j;
        break;
      }
      const double u = gen.next_double();
      const bool take = (t.lw >= lw) || (u < x_exp<Team::kExactMath>(__dsub_rn(t.lw, lw)));
      if (take) {
        copy_group(V_PQ, V_TPQ, V_PG, V_TPG, V_PG, V_TPG); pU = t.pU; pH = t.pH; p_tree = j; p_leaf = t.pidx;
      }
      ev(kEvProposal, j, t.pidx, take ? 1 : 0);
      lw = logaddexp_np<Team::kExactMath>(lw, t.lw);
      {
        double* rho = v(V_RHO);
        const double* ms = v(V_MSUM);
        const int64_t s = ds();
        for (int d = T.rank(); d < D; d += T.size()) rho[d * s] = __dadd_rn(rho[d * s], ms[d * s]);
      }
      if (go_right) { copy_group(V_RQ, V_CQ, V_RR, V_CR, V_RG, V_CG); RU = cur_U; }
      else { copy_group(V_LQ, V_CQ, V_LR, V_CR, V_LG, V_CG); LU = cur_U; }
      depth_reached = j + 1;
      bool turned;
      if (cfg.generalized) {
        turned = uturn_dots(V_RHO, V_LR, V_RR);
      } else {
        double* dq = v(V_MSUM);
        const double* rq = v(V_RQ);
        const double* lq = v(V_LQ);
        const int64_t s = ds();
        for (int d = T.rank(); d < D; d += T.size()) dq[d * s] = __dsub_rn(rq[d * s], lq[d * s]);
        turned = uturn_dots(V_MSUM, V_LR, V_RR);
      }
      ev(kEvOuter, j, turned ? 1 : 0, 0);
      if (turned) break;
    }
    Stats st;
    st.depth = depth_reached;
    st.leapfrogs = leapfrogs;
    st.diverged = diverged ? 1 : 0;
    st.accept = leapfrogs ? __ddiv_rn(sum_metro, (double)leapfrogs) : 0.0;
    st.energy = pH;
    copy_group(V_Q0, V_PQ, V_G0, V_PG, V_G0, V_PG); U0 = pU;
    return st;
  }

  // ------------------------------------------------------- step-size search
  __device__ double accept_prob(double h0, double eps) {
    copy(V_CQ, V_Q0); copy(V_CR, V_R0); copy(V_CG, V_G0); cur_U = U0;
    leapfrog(eps);
    const double h1 = hamiltonian(cur_U, V_CR);
    if (!isfinite(h1)) return 0.0;
    const double x = __dsub_rn(h0, h1);
    return x_exp<Team::kExactMath>(x < 0.0 ? x : 0.0);
  }
  // find_reasonable_step_size (adapt.py:172-204); z0 in Q0/G0/U0
  __device__ __noinline__ double find_step_size(Key key, double init, const double* inj, int64_t inj_ds) {
    const double target = 0.5;
    // rng.generator() of the given key directly (not a fold)
    draw_momentum(V_R0, key, inj, inj_ds);
    const double h0 = hamiltonian(U0, V_R0);
    double eps = init;
    const int direction = accept_prob(h0, eps) > target ? 1 : -1;
    for (int it = 0; it < 64; ++it) {
      const double eps_next = __dmul_rn(eps, direction == 1 ? 2.0 : 0.5);
      if (!(1e-10 < eps_next && eps_next < 1e7)) break;
      const double prob = accept_prob(h0, eps_next);
      if ((direction == 1 && prob <= target) || (direction == -1 && prob > target))
        return direction == -1 ? eps_next : eps;
      eps = eps_next;
    }
    return eps;
  }
};

// ------------------------------------------------------------------- run
struct RunCfg {
  int num_warmup;
  int num_samples;
  double target_accept;
  double base_step;
  int has_sampler;  // RunConfig.sampler is not None (chains.py:137-143)
  int keep_warmup;  // 1: RunOut.samples holds W + S draws, the warmup draws first (adaptation replay tests)
  SamplerCfg sampler;
  const uint8_t* schedule;    // [W]: bit0 in a covariance window, bit1 window end
  const double* da_weight;    // [W]: t ** -kappa for t = 1..W
};

struct RunOut {
  double* samples;   // [S][D] for this chain (component stride ds_out)
  int64_t s_stride;  // stride between draws
  int64_t d_stride;  // stride between components
  double* stats;     // [(W+S)][5]
  double* adapt;     // [2 + W + D]: eps0, final step, step trace, inv mass
  int32_t* status;   // 0 ok, 1 invalid mass matrix install
  int64_t* evals;    // model evaluations (passes over the data) of this chain
};

// run_chain (chains.py:98-163) for the chain owning key `ck`.
template <class Team, class Model>
__device__ void run_chain(Engine<Team, Model>& E, Key ck, const RunCfg& rc, const RunOut& out, bool writer) {
  const int D = E.D;
  const int W = rc.num_warmup, S = rc.num_samples;
  const int64_t s = E.ds();
  // q0 ~ U(-2, 2)^D from fold(0) (chains.py:107)
  {
    Stream us;
    us.init(key_fold(ck, 0));
    double* q = E.v(V_Q0);
    for (int d = 0; d < D; ++d) {
      const double u = us.next_double();
      if ((d % E.T.size()) == E.T.rank()) q[d * s] = __dadd_rn(-2.0, __dmul_rn(4.0, u));
    }
  }
  E.U0 = E.eval(V_Q0, V_G0);
  int status = 0;
  double step;
  if (W > 0) {
    const double eps0 = E.find_step_size(key_fold(ck, 1), rc.base_step, nullptr, 0);
    if (writer && E.T.leader()) out.adapt[0] = eps0;
    // DualAveragingState.init (adapt.py:44-50)
    const double mu = x_log<Team::kExactMath>(__dmul_rn(10.0, eps0));
    double log_eps = x_log<Team::kExactMath>(eps0), log_eps_bar = 0.0, h_bar = 0.0;
    const double gamma = 0.05, t0 = 10.0, delta = rc.target_accept;
    int wcount = 0;
    E.fill(V_WMEAN, 0.0);
    E.fill(V_WM2, 0.0);
    for (int i = 0; i < W; ++i) {
      E.cfg.step = x_exp<Team::kExactMath>(log_eps);
      if (writer && E.T.leader()) out.adapt[2 + i] = E.cfg.step;
      const Stats st = E.transition(key_fold(ck, 10 + (uint64_t)i), nullptr, 0);
      if (writer && E.T.leader()) {
        double* o = out.stats + (int64_t)i * 5;
        o[0] = st.depth; o[1] = st.leapfrogs; o[2] = st.diverged; o[3] = st.accept; o[4] = st.energy;
      }
      // da_update (adapt.py:60-70) with the clipped acceptance (adapt.py:227)
      {
        const double a = fmin(1.0, fmax(0.0, st.accept));
        const int t = i + 1;
        const double frac = __ddiv_rn(1.0, __dadd_rn((double)t, t0));
        h_bar = __dadd_rn(__dmul_rn(__dsub_rn(1.0, frac), h_bar), __dmul_rn(frac, __dsub_rn(delta, a)));
        log_eps = __dsub_rn(mu, __dmul_rn(__ddiv_rn(__dsqrt_rn((double)t), gamma), h_bar));
        const double w = rc.da_weight[i];
        log_eps_bar = __dadd_rn(__dmul_rn(w, log_eps), __dmul_rn(__dsub_rn(1.0, w), log_eps_bar));
      }
      if (writer && rc.keep_warmup) {
        const double* q = E.v(V_Q0);
        for (int d = E.T.rank(); d < D; d += E.T.size()) out.samples[(int64_t)i * out.s_stride + d * out.d_stride] = q[d * s];
      }
      const uint8_t flag = rc.schedule[i];
      if (flag & 1) {  // welford_update (adapt.py:86-94)
        wcount += 1;
        double* mean = E.v(V_WMEAN);
        double* m2 = E.v(V_WM2);
        const double* x = E.v(V_Q0);
        for (int d = E.T.rank(); d < D; d += E.T.size()) {
          const double dl = __dsub_rn(x[d * s], mean[d * s]);
          const double nm = __dadd_rn(mean[d * s], __ddiv_rn(dl, (double)wcount));
          mean[d * s] = nm;
          m2[d * s] = __dadd_rn(m2[d * s], __dmul_rn(dl, __dsub_rn(x[d * s], nm)));
        }
      }
      if ((flag & 2) && wcount >= 2) {  // install regularized variance (adapt.py:104-108, 228-232)
        double* inv = E.v(V_INV);
        double* mean = E.v(V_WMEAN);
        double* m2 = E.v(V_WM2);
        const double n = (double)wcount;
        double bad = 0.0;
        for (int d = E.T.rank(); d < D; d += E.T.size()) {
          const double var = __ddiv_rn(m2[d * s], (double)(wcount - 1));
          const double nv = __dadd_rn(__dmul_rn(__ddiv_rn(n, __dadd_rn(n, 5.0)), var),
                                      __dmul_rn(__ddiv_rn(5.0, __dadd_rn(n, 5.0)), 1e-3));
          if (!(isfinite(nv) && nv > 0.0)) bad = 1.0;
          inv[d * s] = nv;
          mean[d * s] = 0.0;
          m2[d * s] = 0.0;
        }
        wcount = 0;
        if (E.T.sum(bad) != 0.0) { status = 1; break; }
        E.refresh_mstd();
      }
    }
    step = x_exp<Team::kExactMath>(log_eps_bar);
  } else {
    step = rc.base_step;
    if (!rc.has_sampler) step = E.find_step_size(key_fold(ck, 1), 1.0, nullptr, 0);
    if (writer && E.T.leader()) out.adapt[0] = step;
  }
  if (writer && E.T.leader()) { out.adapt[1] = step; out.status[0] = status; }
  if (status != 0) return;
  E.cfg.step = step;
  const int64_t s0 = rc.keep_warmup ? W : 0;
  for (int i = 0; i < S; ++i) {
    const Stats st = E.transition(key_fold(ck, 10 + (uint64_t)(W + i)), nullptr, 0);
    if (writer) {
      const double* q = E.v(V_Q0);
      for (int d = E.T.rank(); d < D; d += E.T.size())
        out.samples[(s0 + i) * out.s_stride + d * out.d_stride] = q[d * s];
      if (E.T.leader()) {
        double* o = out.stats + (int64_t)(W + i) * 5;
        o[0] = st.depth; o[1] = st.leapfrogs; o[2] = st.diverged; o[3] = st.accept; o[4] = st.energy;
      }
    }
  }
  if (writer) {
    const double* inv = E.v(V_INV);
    for (int d = E.T.rank(); d < D; d += E.T.size()) out.adapt[2 + W + d] = inv[d * s];
    if (E.T.leader() && out.evals) out.evals[0] = (int64_t)E.n_evals;
    if (E.T.leader() && E.prof) E.prof[11] = E.n_wasted;
  }
}

}  // namespace ts
