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

}  // namespace ts_internal
