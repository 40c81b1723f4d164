// BlockTeam kernel for small models (one CTA per chain; parity/testing layout).
#include <stdio.h>
#include "ts_internal.cuh"

namespace ts_internal {

int launch_block_small(const SmallModel& sm, int D, int nslots, OpArgs& A, int C, cudaStream_t st) {
  SmallW mw;
  mw.m = sm;
  const size_t smem = ((size_t)num_vecs(nslots) * D + kTeamScratch) * sizeof(double);
  auto kern = k_block_op<SmallW>;
  TS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<A.op == OP_RUN ? (C > 0 ? C : 1) : 1, 256, smem, st>>>(mw, D, nslots, 0, A);
  TS_CUDA(cudaGetLastError());
  return TS_OK;
}

// WarpTeam kernel for small models: one warp per chain, its vectors in shared
// memory.  Latency per leapfrog falls with D-wide vector ops done by 32 lanes
// and reductions by shuffle trees, and many chains per SM hide the rest;
// rounding differs from the one-chain-per-thread layout only at ulp level.
__global__ void __launch_bounds__(256) k_warp_small(SmallModel m, int D, int C, int nslots, int wpb, OpArgs A) {
  extern __shared__ double smem[];
  const int w = (int)(threadIdx.x >> 5);
  const int chain = (int)blockIdx.x * wpb + w;
  if (w >= wpb || chain >= C) return;  // warp-uniform
  const int nv = num_vecs(nslots);
  double* base = smem + (size_t)w * ((size_t)nv * D + kTeamScratch);
  Engine<WarpTeam, SmallW> E;
  E.M.m = m;
  E.D = D;
  E.S.base = base;
  E.S.vstride = D;
  E.S.dstride = 1;
  E.ss = reinterpret_cast<SlotScalars*>(base + (size_t)nv * D + 64);
  E.prof = chain == 0 ? A.prof : nullptr;
  E.prof_last = 0;
  E.tr = nullptr;
  __syncwarp();
  do_op(E, A, A.op == OP_RUN ? chain : 0, A.op == OP_RUN || chain == 0);
}

int launch_warp_small(const SmallModel& sm, int D, int nslots, OpArgs& A, int C, cudaStream_t st) {
  const size_t per_warp = ((size_t)num_vecs(nslots) * D + kTeamScratch) * sizeof(double);
  int wpb = (int)((200 * 1024) / per_warp);
  if (wpb > 8) wpb = 8;
  if (wpb < 1) return set_err(TS_EUNSUPPORTED, "warp layout: model too large for shared memory");
  const int chains = A.op == OP_RUN ? (C > 0 ? C : 1) : 1;
  const size_t smem = per_warp * wpb;
  TS_CUDA(cudaFuncSetAttribute(k_warp_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_warp_small<<<(chains + wpb - 1) / wpb, 32 * wpb, smem, st>>>(sm, D, chains, nslots, wpb, A);
  TS_CUDA(cudaGetLastError());
  return TS_OK;
}

}  // namespace ts_internal
