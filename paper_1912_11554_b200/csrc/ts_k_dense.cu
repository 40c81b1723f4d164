// Many-chain dense-Gaussian model and its tcgen05
// TF32 GEMM.  This translation unit holds the tensor-map plumbing, the GEMM
// probe (ts_gemm_tf32_probe, used by the parity tests) and the persistent
// lockstep kernel (k_dense_op, see ts_dense.cuh).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>
#include "ts_internal.cuh"
#include "ts_umma.cuh"

namespace ts_internal {

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Row-major fp32 matrix rows x cols (cols % 4 == 0) as a 2-D tensor map with
// boxes of box_rows x kUmmaBK and the 128-byte swizzle (K-major UMMA layout);
// out-of-range boxes read zeros.
int make_tmap_f32(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int box_rows) {
  auto enc = get_encode();
  if (!enc) return set_err(TS_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if (cols % 4 != 0) return set_err(TS_EINVAL, "tensor map: row length must be a multiple of 4 floats");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {(cuuint32_t)kUmmaBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(TS_ECUDA, "cuTensorMapEncodeTiled failed");
  return TS_OK;
}

// GEMM probe: GT[n][m] = sum_k A[m][k] XT[n][k], one CTA (4 warps) per tile.
__global__ void __launch_bounds__(128, 1)
    k_umma_probe(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, float* GT, int M,
                 int N, int K) {
  extern __shared__ __align__(1024) unsigned char dsm[];
  UmmaGemm g;
  g.init(dsm);
  if (threadIdx.x == 0) { u_prefetch_tmap(&tmA); u_prefetch_tmap(&tmB); }
  const int mt = (M + kUmmaBM - 1) / kUmmaBM, nt = (N + kUmmaBN - 1) / kUmmaBN;
  const int nkb = (K + kUmmaBK - 1) / kUmmaBK;
  for (int tile = blockIdx.x; tile < mt * nt; tile += gridDim.x) {
    const int m0 = (tile % mt) * kUmmaBM, n0 = (tile / mt) * kUmmaBN;
    g.tile(&tmA, &tmB, m0, n0, nkb, GT, M, M - m0 < kUmmaBM ? M - m0 : kUmmaBM, N - n0 < kUmmaBN ? N - n0 : kUmmaBN);
  }
  g.release();
}

// ------------------------------------------------------------------ batched model
// Dense Gaussian U(x) = 1/2 x^T A x, gradient A x, for C chains at once.
// CTA = 4 GEMM warps (warps 0..3) + kDenseCW chain warps; each chain warp
// runs one chain (Engine<WarpTeam>, vectors in a global workspace).
//
// The GEMM warps of all CTAs run a continuous sequence of batched steps,
// decoupled from the chains: a chain posts a request (its position row in
// XT, then posted[c] = seq with release semantics) and spins on served[c].
// Each step, every CTA snapshots which of its chains have a request
// outstanding (posted > served), the GEMM warps meet at a grid barrier,
// compute GT = X A^T for the N-tiles holding outstanding requests (tcgen05
// TF32, or SIMT fp64 in the parity policy), storing only outstanding
// columns, meet again, and release served[c].  A chain's row is stable from
// its post until it is served, and GT[c] is written only while c is
// outstanding, so reads and writes never race.  Chains therefore never
// wait for the slowest chain (no lockstep): a request waits at most one
// step (~GEMM + 2 grid barriers).
constexpr int kDenseCW = 8;  // chain warps per CTA (at most; DenseArgs::cpc of them run chains)

__device__ __forceinline__ void st_release_gpu_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ float tf32r(double x) {
  uint32_t v;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(v) : "f"((float)x));
  return __uint_as_float(v);
}

// Request-row write of one chain (warp), 4 components per lane and step, two
// steps per iteration in an unpredicated main loop (a separate function: the
// engine's registers stay out of the loop, which spilled to local memory
// when inlined)
static __device__ __noinline__ void dense_write_row_tf32(float4* __restrict__ row, const double2* __restrict__ q2, int n4) {
  auto one = [&](int i) {
    const double2 a = q2[2 * i], b = q2[2 * i + 1];
    row[i] = make_float4(tf32r(a.x), tf32r(a.y), tf32r(b.x), tf32r(b.y));
  };
  int i = (int)(threadIdx.x & 31);
#pragma unroll 1
  for (; i + 32 < n4; i += 64) {
    const double2 a0 = q2[2 * i], b0 = q2[2 * i + 1];
    const double2 a1 = q2[2 * (i + 32)], b1 = q2[2 * (i + 32) + 1];
    row[i] = make_float4(tf32r(a0.x), tf32r(a0.y), tf32r(b0.x), tf32r(b0.y));
    row[i + 32] = make_float4(tf32r(a1.x), tf32r(a1.y), tf32r(b1.x), tf32r(b1.y));
  }
#pragma unroll 1
  for (; i < n4; i += 32) one(i);
}
struct DenseW : NoTraj {
  static constexpr bool kAsync = true;
  static constexpr bool kVecOps = true;  // D ~ 1000 vectors in global memory
  int D;
  int fp64;
  float* xt;        // [Cpad][D] tf32-rounded positions (TF32 policy)
  double* xt64;     // [Cpad][D] positions (FP64 policy)
  const float* gt;  // [Cpad][D] gradients
  const double* gt64;
  unsigned long long* posted;  // [Cpad] request sequence numbers
  unsigned long long* served;  // [Cpad]
  unsigned long long seq;
  int chain;
  unsigned int* err;
  unsigned long long spin_ns;
  VecStore S;
  int pq, pg;
  LeafVecs* lv;  // this chain warp's fused-leaf operand record (shared memory)
  __device__ LeafVecs* leaf_vecs() const { return lv; }

  __device__ void post(int q, int g) {
    pq = q;
    pg = g;
    const int lane = threadIdx.x & 31;
    const double* qv = S.v(q);
    if (fp64) {
      double* row = xt64 + (int64_t)chain * D;
      for (int d = lane; d < D; d += 32) row[d] = qv[d];
    } else {
      dense_write_row_tf32(reinterpret_cast<float4*>(xt + (int64_t)chain * D), reinterpret_cast<const double2*>(qv), D >> 2);
    }
    // the GEMM reads the row through the async (TMA) proxy in another CTA
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence();
    __syncwarp();
    seq += 1;
    if (lane == 0) st_release_gpu_u64(posted + chain, seq);
  }
  // the engine's fused leaf pass: wait for the step, then read the row itself
  __device__ void wait_poll() {
    if ((threadIdx.x & 31) == 0) {
      SpinGuard sg(err, spin_ns);
      while (ld_relaxed_u64(served + chain) < seq) {
        if (sg.expired()) break;
      }
      (void)ld_acquire_u64(served + chain);
    }
    __syncwarp();
  }
  __device__ const void* grad_row() const {
    return fp64 ? (const void*)(gt64 + (int64_t)chain * D) : (const void*)(gt + (int64_t)chain * D);
  }
  __device__ double wait() {
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
      // relaxed polling (an acquire load per iteration would invalidate the
      // SM's L1 every time), then one acquire
      SpinGuard sg(err, spin_ns);
      while (ld_relaxed_u64(served + chain) < seq) {
        if (sg.expired()) break;
      }
      (void)ld_acquire_u64(served + chain);
    }
    __syncwarp();
    const double* qv = S.v(pq);
    double* gv = S.v(pg);
    double acc = 0.0;
    if (fp64) {
      const double* row = gt64 + (int64_t)chain * D;
      for (int d = lane; d < D; d += 32) {
        const double g = __ldcg(row + d);
        gv[d] = g;
        acc = __dadd_rn(acc, __dmul_rn(qv[d], g));
      }
    } else {
      const float4* row = reinterpret_cast<const float4*>(gt + (int64_t)chain * D);
      const double2* q2 = reinterpret_cast<const double2*>(qv);
      double2* g2 = reinterpret_cast<double2*>(gv);
      const int n4 = D >> 2;
      for (int base = lane; base < n4; base += 32 * 4) {
        float4 f[4];
        double2 a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (base + 32 * u < n4) {
            f[u] = __ldcg(row + base + 32 * u);
            a[u] = q2[2 * (base + 32 * u)];
            b[u] = q2[2 * (base + 32 * u) + 1];
          }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (base + 32 * u < n4) {
            const double2 g0 = make_double2((double)f[u].x, (double)f[u].y);
            const double2 g1 = make_double2((double)f[u].z, (double)f[u].w);
            g2[2 * (base + 32 * u)] = g0;
            g2[2 * (base + 32 * u) + 1] = g1;
            acc = __dadd_rn(acc, __dmul_rn(a[u].x, g0.x));
            acc = __dadd_rn(acc, __dmul_rn(a[u].y, g0.y));
            acc = __dadd_rn(acc, __dmul_rn(b[u].x, g1.x));
            acc = __dadd_rn(acc, __dmul_rn(b[u].y, g1.y));
          }
      }
    }
    __syncwarp();
    return 0.5 * WarpTeam().sum(acc);
  }
  template <class Team>
  __device__ double eval(const Team&, const VecStore&, int q, int g) {
    post(q, g);
    return wait();
  }
  // the engine's fused leaf pass writes the request row itself
  __device__ void* request_row() const {
    return fp64 ? (void*)(xt64 + (int64_t)chain * D) : (void*)(xt + (int64_t)chain * D);
  }
  __device__ void post_written(int q, int g) {
    pq = q;
    pg = g;
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence();
    __syncwarp();
    seq += 1;
    if ((threadIdx.x & 31) == 0) st_release_gpu_u64(posted + chain, seq);
  }
};

struct DenseArgs {
  int D, C, Cpad, fp64, nv;
  int cpc;    // chains per CTA (<= kDenseCW): C spread over every SM (1024 chains: 7 x 147 CTAs, not 8 x 128)
  int chain0;  // first chain of this launch (runs with more chains than one grid holds are chunked)
  float* xt;
  double* xt64;
  float* gt;
  double* gt64;
  const double* a64;        // [D][D] (FP64 policy)
  double* ws;               // chain workspaces [C][nv][D]
  unsigned long long* bar;  // grid barrier counter (zeroed before launch)
  int* done;                // finished chain warps (zeroed before launch)
  unsigned long long* prof;  // optional (TS_PROF): CTA-0 ns [snapshot+barrier, GEMM, release], steps, busy steps
  unsigned long long* posted;   // [Cpad] (zeroed before launch)
  unsigned long long* served;   // [Cpad]
  unsigned long long* pending;  // [2][Cpad] request served by the step of that parity (0 = none)
  unsigned long long* npend;    // [4] outstanding requests of the step (step & 3), [4..6) all-done flags (step & 1)
  unsigned int* err;            // sticky synchronisation-timeout flag of the model (SpinGuard)
  unsigned long long spin_ns;
  unsigned int* ncnt;           // [2][N-tiles] finished M-tiles of each N-tile per step parity (early release)
  int early;                    // 1: the last M-tile of an N-tile releases its chains (no release barrier)
};

__device__ __forceinline__ void gemm_grid_barrier(unsigned long long* bar, unsigned long long& epoch, unsigned int* err,
                                                  unsigned long long spin_ns) {
  asm volatile("bar.sync 4, 128;" ::: "memory");  // every GEMM thread's stores precede the release
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long target = (epoch + 1) * (unsigned long long)gridDim.x;
    red_release_add_u64(bar, 1ULL);
    SpinGuard sg(err, spin_ns);
    while (ld_relaxed_u64(bar) < target) {
      if (sg.expired()) break;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  epoch += 1;
  asm volatile("bar.sync 4, 128;" ::: "memory");
}

// SIMT fp64 tile (parity policy): thread = row m, 16 chains at a time, k in
// order, multiply then add (oracle/turnstile_oracle.py restates it bit for bit)
__device__ void dense_tile_fp64(const DenseArgs& a, const unsigned long long* pend, int m0, int n0) {
  const int m = m0 + (int)threadIdx.x;
  if (m >= a.D) return;
  const double* arow = a.a64 + (int64_t)m * a.D;
  for (int nb = 0; nb < kUmmaBN; nb += 16) {
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0;
    const int nmax = (a.Cpad - (n0 + nb)) < 16 ? (a.Cpad - (n0 + nb)) : 16;
    if (nmax <= 0) break;
    for (int k = 0; k < a.D; ++k) {
      const double av = arow[k];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < nmax) acc[j] = __dadd_rn(acc[j], __dmul_rn(av, __ldcg(a.xt64 + (int64_t)(n0 + nb + j) * a.D + k)));
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < nmax && __ldcg(pend + n0 + nb + j) != 0ULL) a.gt64[(int64_t)(n0 + nb + j) * a.D + m] = acc[j];
  }
}

__global__ void __launch_bounds__(128 + 32 * kDenseCW, 1)
    k_dense_op(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX, DenseArgs a,
               int nslots, OpArgs A) {
  extern __shared__ __align__(1024) unsigned char dsm[];
  volatile int* flag = reinterpret_cast<volatile int*>(dsm + kUmmaSmemBytes);
  SlotScalars* ss_all = reinterpret_cast<SlotScalars*>(dsm + kUmmaSmemBytes + 64);
  LeafVecs* lv_all = reinterpret_cast<LeafVecs*>(dsm + kUmmaSmemBytes + 64 + kDenseCW * kMaxSlots * sizeof(SlotScalars));
  const int warp = threadIdx.x >> 5;
  if (warp < 4) {
    // ---------------- GEMM warps
    UmmaGemm g;
    if (!a.fp64) {
      g.init(dsm);
      if (threadIdx.x == 0) { u_prefetch_tmap(&tmA); u_prefetch_tmap(&tmX); }
    }
    const int t = threadIdx.x;
    const int mt = (a.D + kUmmaBM - 1) / kUmmaBM, nt = a.Cpad / kUmmaBN;
    const int nkb = (a.D + kUmmaBK - 1) / kUmmaBK;
    const int total = (int)gridDim.x * kDenseCW;
    const int my_chain = blockIdx.x * a.cpc + t;  // t < cpc: this CTA's chain t
    unsigned long long srv = 0;                      // requests of my_chain served so far
    unsigned long long epoch = 0;
    const bool prof = a.prof != nullptr && blockIdx.x == 0 && t == 0;
    unsigned long long tp0 = 0, tp1 = 0, busy = 0;
    if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp0));
    for (int step = 0;; ++step) {
      // snapshot: requests outstanding now are served by this step
      unsigned long long mine = 0;
      if (t < a.cpc) {
        const unsigned long long p = ld_acquire_u64(a.posted + my_chain);
        mine = p > srv ? p : 0ULL;
        a.pending[(step & 1) * a.Cpad + my_chain] = mine;
        if (mine) atomicAdd(a.npend + (step & 3), 1ULL);
      }
      // the exit decision must be the same in every CTA: CTA 0 samples the
      // finished-chain count BEFORE the barrier (chains keep finishing
      // asynchronously, so reading it after the barrier could differ per CTA)
      if (t == 0 && blockIdx.x == 0)
        a.npend[4 + (step & 1)] = (*reinterpret_cast<volatile int*>(a.done) >= total) ? 1ULL : 0ULL;
      gemm_grid_barrier(a.bar, epoch, a.err, a.spin_ns);
      if (t == 0) {
        const unsigned long long np = ld_relaxed_u64(a.npend + (step & 3));
        const bool all_done = ld_relaxed_u64(a.npend + 4 + (step & 1)) != 0ULL;
        *flag = (np == 0ULL && all_done) ? 0 : (np ? 1 : 2);
        // slot of step + 2: last read after the barrier of step - 2, so every
        // CTA is done with it; with the per-N-tile release a fast CTA can reach
        // the next snapshot before CTA 0 gets here, hence four slots
        if (blockIdx.x == 0) a.npend[(step + 2) & 3] = 0ULL;
      }
      asm volatile("bar.sync 4, 128;" ::: "memory");
      const int f = *flag;
      if (f == 0) break;
      if (prof) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1));
        a.prof[0] += tp1 - tp0;
        tp0 = tp1;
      }
      const unsigned long long* pend = a.pending + (step & 1) * a.Cpad;
      if (f == 1) {  // at least one request in the grid
        if (t == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
        for (int tile = blockIdx.x; tile < mt * nt; tile += gridDim.x) {
          const int m0 = (tile % mt) * kUmmaBM, n0 = (tile / mt) * kUmmaBN;
          // skip N-tiles without outstanding requests (uniform over the 128 threads)
          int any = 0;
          for (int j = t; j < kUmmaBN; j += 128) any |= __ldcg(pend + n0 + j) != 0ULL;
          any = gemm_sync_or(any);
          if (!any) continue;
          if (a.fp64) dense_tile_fp64(a, pend, m0, n0);
          else
            g.tile(&tmA, &tmX, m0, n0, nkb, a.gt, a.D, a.D - m0 < kUmmaBM ? a.D - m0 : kUmmaBM, kUmmaBN, pend + n0);
          if (a.early) {
            // the CTA finishing the last M-tile of this N-tile releases its
            // requested chains (every M-tile CTA fenced its gradient stores
            // before counting; the counter is reset for step + 2)
            asm volatile("bar.sync 4, 128;" ::: "memory");
            __shared__ int last;
            if (t == 0) {
              __threadfence();
              unsigned int* cnt = a.ncnt + (step & 1) * nt + tile / mt;
              const unsigned int old = atomicAdd(cnt, 1u);
              last = (old + 1u == (unsigned int)mt);
              if (last) {
                __threadfence();
                *cnt = 0u;
              }
            }
            asm volatile("bar.sync 4, 128;" ::: "memory");
            if (last && t < kUmmaBN) {
              const unsigned long long pv = __ldcg(pend + n0 + t);
              if (pv != 0ULL) st_release_gpu_u64(a.served + n0 + t, pv);
            }
          }
        }
        busy += 1;
      }
      if (prof) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1));
        a.prof[1] += tp1 - tp0;
        tp0 = tp1;
      }
      if (a.early) {
        // released per N-tile above; the next snapshot only needs this
        // CTA's view of what it has served
        if (t < a.cpc && mine) srv = mine;
      } else {
        gemm_grid_barrier(a.bar, epoch, a.err, a.spin_ns);  // all gradient tiles written
        if (t < a.cpc && mine) {
          srv = mine;
          st_release_gpu_u64(a.served + my_chain, mine);
        }
      }
      if (prof) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1));
        a.prof[2] += tp1 - tp0;
        a.prof[3] += 1;
        tp0 = tp1;
      }
    }
    if (prof) a.prof[4] = busy;
    if (!a.fp64) g.release();
    return;
  }
  // ---------------- chain warps
  const int cw = warp - 4;
  const int chain = blockIdx.x * a.cpc + cw;
  const int n_active = (A.op == OP_RUN) ? a.C : 1;
  if (cw < a.cpc && chain < n_active) {
    DenseW M;
    M.D = a.D;
    M.fp64 = a.fp64;
    M.xt = a.xt; M.xt64 = a.xt64; M.gt = a.gt; M.gt64 = a.gt64;
    M.posted = a.posted;
    M.served = a.served;
    M.seq = 0;
    M.chain = chain;
    M.err = a.err;
    M.spin_ns = a.spin_ns;
    M.lv = lv_all + cw;
    Engine<WarpTeam, DenseW> E;
    E.D = a.D;
    E.S.base = a.ws + (int64_t)chain * a.nv * a.D;
    E.S.vstride = a.D;
    E.S.dstride = 1;
    M.S = E.S;
    E.M = M;
    E.prof = (A.prof != nullptr && chain == 0) ? A.prof : nullptr;  // TS_PROF: chain 0's leaf phases
    E.prof_last = 0;
    E.tr = nullptr;
    E.ss = ss_all + cw * kMaxSlots;
    __syncwarp();
    do_op(E, A, A.op == OP_RUN ? a.chain0 + chain : 0, chain == 0 || A.op == OP_RUN);
  }
  __syncwarp();
  __threadfence();
  if ((threadIdx.x & 31) == 0) atomicAdd(a.done, 1);
}

static int launch_dense_chunk(const ts_model* m, int nslots, OpArgs& A, int C, int chain0, cudaStream_t st);

int launch_dense(const ts_model* m, int nslots, OpArgs& A, int n_chains, cudaStream_t st) {
  if (A.op != OP_RUN) return launch_dense_chunk(m, nslots, A, 1, 0, st);
  // one co-resident grid holds (CTAs per SM x SMs) x kDenseCW chains; larger
  // runs go in chunks (each chain is a pure function of its key)
  int dev = 0, nsm = 0, occ = 0;
  TS_CUDA(cudaGetDevice(&dev));
  TS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const size_t smem = kUmmaSmemBytes + 64 + kDenseCW * (kMaxSlots * sizeof(SlotScalars) + sizeof(LeafVecs));
  TS_CUDA(cudaFuncSetAttribute(k_dense_op, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  TS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dense_op, 128 + 32 * kDenseCW, smem));
  const int cap = occ * nsm * kDenseCW;
  if (cap < 1) return set_err(TS_EUNSUPPORTED, "dense model kernel cannot be resident");
  for (int c0 = 0; c0 < n_chains; c0 += cap) {
    const int rc = launch_dense_chunk(m, nslots, A, n_chains - c0 < cap ? n_chains - c0 : cap, c0, st);
    if (rc) return rc;
  }
  return TS_OK;
}

static int launch_dense_chunk(const ts_model* m, int nslots, OpArgs& A, int C, int chain0, cudaStream_t st) {
  ts_model* mm = const_cast<ts_model*>(m);
  const int D = m->dim;
  int dev0 = 0, nsm0 = 148;
  TS_CUDA(cudaGetDevice(&dev0));
  TS_CUDA(cudaDeviceGetAttribute(&nsm0, cudaDevAttrMultiProcessorCount, dev0));
  // chains per CTA: the fewest that fit C on one CTA per SM, so every SM runs chains
  int cpc = (C + nsm0 - 1) / nsm0;
  if (cpc > kDenseCW) cpc = kDenseCW;
  if (cpc < 1) cpc = 1;
  const int grid = (C + cpc - 1) / cpc;
  const int Cpad = ((grid * cpc + kUmmaBN - 1) / kUmmaBN) * kUmmaBN;
  const int nv = num_vecs(nslots);
  int dev = 0, nsm = 0;
  TS_CUDA(cudaGetDevice(&dev));
  TS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const size_t smem = kUmmaSmemBytes + 64 + kDenseCW * (kMaxSlots * sizeof(SlotScalars) + sizeof(LeafVecs));
  auto kern = k_dense_op;
  TS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  TS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128 + 32 * kDenseCW, smem));
  if ((int64_t)occ * nsm < grid) return set_err(TS_EUNSUPPORTED, "dense model: too many chains for one co-resident grid");
  // workspaces (grown on demand, owned by the model)
  const size_t need = (size_t)Cpad * D * (m->fp64 ? 16 : 8) + (size_t)C * nv * D * 8 + 64 + (size_t)Cpad * 32 + 64 +
                     2 * (size_t)(Cpad / kUmmaBN) * sizeof(unsigned int) + 16;  // + flags, N-tile counters
  if (mm->dws_size < need) {
    if (mm->dws) cudaFree(mm->dws);
    mm->dws = nullptr;
    mm->dws_size = 0;
    TS_CUDA(cudaMalloc((void**)&mm->dws, need));
    mm->dws_size = need;
    TS_CUDA(cudaMemset(mm->dws, 0, need));
  }
  DenseArgs a;
  memset(&a, 0, sizeof a);
  a.D = D; a.C = C; a.Cpad = Cpad; a.fp64 = m->fp64; a.nv = nv; a.chain0 = chain0; a.cpc = cpc;
  unsigned char* p = mm->dws;
  a.bar = reinterpret_cast<unsigned long long*>(p);
  a.done = reinterpret_cast<int*>(p + 8);
  p += 64;
  if (m->fp64) {
    a.xt64 = reinterpret_cast<double*>(p); p += (size_t)Cpad * D * 8;
    a.gt64 = reinterpret_cast<double*>(p); p += (size_t)Cpad * D * 8;
  } else {
    a.xt = reinterpret_cast<float*>(p); p += (size_t)Cpad * D * 4;
    a.gt = reinterpret_cast<float*>(p); p += (size_t)Cpad * D * 4;
  }
  a.ws = reinterpret_cast<double*>(p);
  p += (size_t)C * nv * D * 8;
  a.posted = reinterpret_cast<unsigned long long*>(p);
  a.served = a.posted + Cpad;
  a.pending = a.served + Cpad;
  a.npend = a.pending + 2 * Cpad;
  a.ncnt = reinterpret_cast<unsigned int*>(a.npend + 8);
  // per-N-tile release instead of the release barrier: correct (same chains
  // bit for bit) but slower, 9.33 -> 8.36 M chain-leapfrog/s: steps get
  // shorter (23 vs 30 us) yet serve fewer requests each, and the gradient
  // wait per leaf does not drop; TS_DENSE_EARLY=1 for A/B
  a.early = 0;
  if (const char* e = getenv("TS_DENSE_EARLY")) a.early = atoi(e) != 0;
  a.a64 = m->params;
  a.err = m->errw;
  a.spin_ns = spin_limit_ns();
  CUtensorMap ta, tx;
  memset(&ta, 0, sizeof ta);
  memset(&tx, 0, sizeof tx);
  if (!m->fp64) {
    int rc = make_tmap_f32(&ta, m->a32, D, D, kUmmaBM);
    if (rc) return rc;
    rc = make_tmap_f32(&tx, a.xt, Cpad, D, kUmmaBN);
    if (rc) return rc;
  }
  TS_CUDA(cudaMemsetAsync(mm->dws, 0, 64, st));
  TS_CUDA(cudaMemsetAsync(a.posted, 0, ((size_t)Cpad * 4 + 8) * sizeof(unsigned long long) + 2 * (size_t)(Cpad / kUmmaBN) * sizeof(unsigned int), st));
  const bool prof = getenv("TS_PROF") != nullptr;  // profiling aid: CTA-0 step phases to stderr
  if (prof) a.prof = reinterpret_cast<unsigned long long*>(mm->dws + 16);  // 5 words in the zeroed header
  int ns = nslots;
  void* args[] = {&ta, &tx, &a, &ns, &A};
  TS_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3((unsigned)grid), dim3(128 + 32 * kDenseCW), args, smem, st));
  if (prof) {
    unsigned long long h[5];
    TS_CUDA(cudaMemcpyAsync(h, a.prof, sizeof h, cudaMemcpyDeviceToHost, st));
    TS_CUDA(cudaStreamSynchronize(st));
    const double n = h[3] ? (double)h[3] : 1.0;
    fprintf(stderr, "TS_PROF dense steps=%llu (with requests %llu) us/step: snapshot+barrier %.2f  GEMM %.2f  release barrier %.2f\n",
            h[3], h[4], h[0] / n / 1e3, h[1] / n / 1e3, h[2] / n / 1e3);
  }
  return TS_OK;
}

}  // namespace ts_internal

using namespace ts_internal;

extern "C" int ts_gemm_tf32_probe(const float* a_dev, const float* xt_dev, float* gt_dev, int M, int N, int K, int grid,
                                  void* stream) {
  if (!a_dev || !xt_dev || !gt_dev || M < 1 || N < 1 || K < 1) return set_err(TS_EINVAL, "bad GEMM probe arguments");
  CUtensorMap ta, tb;
  int rc = make_tmap_f32(&ta, a_dev, M, K, kUmmaBM);
  if (rc) return rc;
  rc = make_tmap_f32(&tb, xt_dev, N, K, kUmmaBN);
  if (rc) return rc;
  const int tiles = ((M + kUmmaBM - 1) / kUmmaBM) * ((N + kUmmaBN - 1) / kUmmaBN);
  if (grid <= 0 || grid > tiles) grid = tiles;
  TS_CUDA(cudaFuncSetAttribute(k_umma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, kUmmaSmemBytes));
  k_umma_probe<<<grid, 128, kUmmaSmemBytes, (cudaStream_t)stream>>>(ta, tb, gt_dev, M, N, K);
  TS_CUDA(cudaGetLastError());
  return TS_OK;
}
