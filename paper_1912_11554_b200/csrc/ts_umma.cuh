// 5th-generation tensor-core (tcgen05) GEMM tile for sm_100a, TF32 inputs,
// FP32 accumulation in tensor memory.
//
// Used by the many-chain dense-Gaussian model: one
// lockstep step evaluates the gradients of every chain at once,
//   GT[n][m] = sum_k A[m][k] * XT[n][k]      (G = A X, chain-major output)
// where A (Mp x Kp) is the fixed precision matrix and XT (Np x Kp) holds the
// chains' positions, one row per chain (K-major for both operands).
//
// Per output tile (BM = 128 rows of A x BN = 64 chains):
//   * one producer thread streams 32-column k-blocks of A and XT into a
//     STAGES-deep shared-memory ring with 2-D TMA (128-byte swizzle, the
//     canonical K-major UMMA layout), completion on a "full" mbarrier;
//   * one MMA thread issues 4 tcgen05.mma.kind::tf32 (K = 8 each) per
//     k-block into a 128 x 64 fp32 accumulator in TMEM and frees the stage
//     with tcgen05.commit on its "empty" mbarrier;
//   * after the last k-block a commit signals the 4 epilogue warps, which
//     read the accumulator with tcgen05.ld (warp w owns TMEM lanes 32w..)
//     and store GT rows with coalesced writes.
#pragma once
#include <stdint.h>

namespace ts {

constexpr int kUmmaBM = 128;
constexpr int kUmmaBN = 64;  // chains per tile (128 measured slower: fewer CTAs share the step)
constexpr int kUmmaBK = 32;  // fp32/tf32 elements per k-block = one 128-B swizzle row
#ifndef TS_UMMA_STAGES
#define TS_UMMA_STAGES 4
#endif
constexpr int kUmmaStages = TS_UMMA_STAGES;  // 2: 8.5 M, 4: 9.6 M, 8: 8.2 M chain-leapfrog/s (shared memory vs the chains' L1)
constexpr int kUmmaABytes = kUmmaBM * kUmmaBK * 4;  // 16 KB
constexpr int kUmmaBBytes = kUmmaBN * kUmmaBK * 4;  // 8 KB
constexpr int kUmmaStageBytes = kUmmaABytes + kUmmaBBytes;
static_assert(kUmmaBN <= 128, "the stored-column mask gives one chain per GEMM thread");
// shared memory of the GEMM: 1024-B aligned ring + mbarriers (full, empty, accum) + TMEM address
constexpr int kUmmaSmemBytes = kUmmaStages * kUmmaStageBytes + 1024 + 256;

__device__ __forceinline__ uint32_t u_smem(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void u_mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void u_mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void u_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "UWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra UWAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// 2-D TMA tile load: box at (c0 = inner/k, c1 = row) of the tensor map
__device__ __forceinline__ void u_tma_load_2d(uint32_t dst, const void* tmap, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(tmap), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void u_prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups
// 1024 B apart (SBO), LBO unused (16 B), version 1 (sm_100).
__device__ __forceinline__ uint64_t u_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
// Instruction descriptor: D f32, A/B tf32, both K-major, N and M.
__host__ __device__ constexpr uint32_t u_idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void u_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void u_mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void u_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void u_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// warp-wide TMEM allocation (power of two >= 32 columns); address to *dst_smem
__device__ __forceinline__ void u_tmem_alloc(uint32_t dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void u_tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread
__device__ __forceinline__ void u_tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// OR-reduction barrier over the 128 GEMM threads (named barrier 4)
__device__ __forceinline__ int gemm_sync_or(int v) {
  int r;
  asm volatile(
      "{\n"
      ".reg .pred p, q;\n"
      "setp.ne.s32 p, %1, 0;\n"
      "bar.red.or.pred q, 4, 128, p;\n"
      "selp.s32 %0, 1, 0, q;\n"
      "}\n"
      : "=r"(r)
      : "r"(v)
      : "memory");
  return r;
}

// Persistent-GEMM state of one CTA's 4 GEMM warps (warps 0..3 of the CTA).
struct UmmaGemm {
  unsigned char* ring;  // 1024-B aligned: kUmmaStages x (A tile | B tile)
  uint32_t full0, empty0, accum;  // mbarrier shared addresses (full[s] = full0 + 8 s)
  uint32_t tmem;                  // TMEM accumulator base (kUmmaBN columns)
  uint32_t kb_issued;             // k-blocks loaded so far (ring position, persists across tiles)
  uint32_t kb_mma;                // k-blocks consumed by the MMA thread
  uint32_t tiles_done;            // accumulator phases

  // carve the shared region (>= kUmmaSmemBytes); called by all 128 GEMM threads
  __device__ void init(unsigned char* smem_region) {
    uintptr_t p = reinterpret_cast<uintptr_t>(smem_region);
    p = (p + 1023) & ~(uintptr_t)1023;
    ring = reinterpret_cast<unsigned char*>(p);
    const uint32_t b = u_smem(ring + kUmmaStages * kUmmaStageBytes);
    full0 = b;
    empty0 = b + 8 * kUmmaStages;
    accum = b + 16 * kUmmaStages;
    const uint32_t tslot = accum + 8;
    const int t = threadIdx.x;
    if (t == 0) {
      for (int s = 0; s < kUmmaStages; ++s) { u_mbar_init(full0 + 8 * s, 1); u_mbar_init(empty0 + 8 * s, 1); }
      u_mbar_init(accum, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (t < 32) u_tmem_alloc(tslot, kUmmaBN);
    u_fence_before();
    asm volatile("bar.sync 4, 128;" ::: "memory");
    u_fence_after();
    uint32_t tv;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tv) : "r"(tslot));
    tmem = tv;
    kb_issued = kb_mma = 0;
    tiles_done = 0;
  }
  __device__ void release() {
    asm volatile("bar.sync 4, 128;" ::: "memory");
    if (threadIdx.x < 32) u_tmem_dealloc(tmem, kUmmaBN);
  }

  // One 128 x kUmmaBN output tile: rows m0.., chains n0..; nkb k-blocks.
  // Output GT[(n0 + j) * ldo + m0 + i] for i < m_valid, j < n_valid.
  // pend (optional): output column j is stored only if pend[j] != 0.
  __device__ void tile(const void* tmA, const void* tmB, int m0, int n0, int nkb, float* GT, int64_t ldo, int m_valid,
                       int n_valid, const unsigned long long* pend = nullptr) {
    const int t = threadIdx.x;
    const uint32_t idesc = u_idesc_tf32(kUmmaBM, kUmmaBN);
    if (t == 0) {
      // producer: all k-blocks of the tile, STAGES ahead of the MMA thread
      for (int kb = 0; kb < nkb; ++kb, ++kb_issued) {
        const int s = (int)(kb_issued % kUmmaStages);
        const uint32_t use = kb_issued / kUmmaStages;
        if (use > 0) u_mbar_wait(empty0 + 8 * s, (use - 1) & 1);
        const uint32_t a_dst = u_smem(ring + s * kUmmaStageBytes);
        u_mbar_expect_tx(full0 + 8 * s, kUmmaStageBytes);
        u_tma_load_2d(a_dst, tmA, kb * kUmmaBK, m0, full0 + 8 * s);
        u_tma_load_2d(a_dst + kUmmaABytes, tmB, kb * kUmmaBK, n0, full0 + 8 * s);
      }
    } else if (t == 32) {
      // MMA issuer
      for (int kb = 0; kb < nkb; ++kb, ++kb_mma) {
        const int s = (int)(kb_mma % kUmmaStages);
        u_mbar_wait(full0 + 8 * s, (kb_mma / kUmmaStages) & 1);
        u_fence_after();
        const uint32_t a_addr = u_smem(ring + s * kUmmaStageBytes);
        const uint64_t ad = u_desc_sw128(a_addr), bd = u_desc_sw128(a_addr + kUmmaABytes);
#pragma unroll
        for (int kk = 0; kk < kUmmaBK / 8; ++kk)  // K = 8 tf32 = 32 B per instruction
          u_mma_tf32(tmem, ad + (uint64_t)(2 * kk), bd + (uint64_t)(2 * kk), idesc, (kb | kk) != 0);
        u_mma_commit(empty0 + 8 * s);  // frees the stage when these MMAs have read it
      }
      u_mma_commit(accum);  // accumulator complete
    } else {
      // the other lanes of warps 0 / 1 keep the MMA issue path warp-uniform-free
      (void)idesc;
    }
    __syncwarp();
    // stored-column mask (one bit per chain of the tile) while the MMAs run
    const uint32_t smask = accum + 16;  // 4 words after the TMEM address slot
    if (pend != nullptr) {
      const bool want = t < n_valid && __ldcg(pend + t) != 0ULL;
      const uint32_t b = __ballot_sync(0xffffffffu, want);
      if ((t & 31) == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(smask + 4 * (t >> 5)), "r"(b) : "memory");
      asm volatile("bar.sync 4, 128;" ::: "memory");
    }
    // epilogue: all 4 warps
    u_mbar_wait(accum, tiles_done & 1);
    u_fence_after();
    ++tiles_done;
    const int w = t >> 5, lane = t & 31;
    const int row = w * 32 + lane;
#pragma unroll
    for (int c = 0; c < kUmmaBN; c += 16) {
      float v[16];
      u_tmem_ld16(tmem + ((uint32_t)(w * 32) << 16) + (uint32_t)c, v);
      uint32_t mw = 0xffffffffu;
      if (pend != nullptr) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(mw) : "r"(smask + 4 * (c >> 5)));
      mw >>= (c & 31);
      if (row < m_valid) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c + j < n_valid && ((mw >> j) & 1u)) GT[(int64_t)(n0 + c + j) * ldo + m0 + row] = v[j];
      }
    }
    u_fence_before();
    asm volatile("bar.sync 4, 128;" ::: "memory");  // accumulator free for the next tile
    u_fence_after();
  }
};

}  // namespace ts
