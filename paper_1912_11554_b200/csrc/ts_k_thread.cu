// ThreadTeam kernel: one chain (or one parity op) per thread, small models.
#include <stdio.h>
#include "ts_internal.cuh"

namespace ts_internal {

// ThreadTeam: workspace ws[(id*D + d)*C + c]
__global__ void __launch_bounds__(128) k_thread_op(SmallModel m, int D, int C, double* ws, int nslots, OpArgs A) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  Engine<ThreadTeam, SmallW> E;
  SlotScalars ss_local[kMaxSlots];
  E.ss = ss_local;
  E.M.m = m;
  E.D = D;
  E.S.base = ws + c;
  E.S.vstride = (int64_t)D * C;
  E.S.dstride = C;
  do_op(E, A, c, true);
}

int launch_thread(const SmallModel& sm, int D, int C, int nslots, OpArgs& A, cudaStream_t st) {
  double* ws = nullptr;
  const size_t bytes = (size_t)num_vecs(nslots) * D * C * sizeof(double);
  TS_CUDA(cudaMallocAsync((void**)&ws, bytes, st));
  const int tpb = 32;
  k_thread_op<<<(C + tpb - 1) / tpb, tpb, 0, st>>>(sm, D, C, ws, nslots, A);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(ws, st);
  if (e != cudaSuccess) return set_err(TS_ECUDA, cudaGetErrorString(e));
  return TS_OK;
}

}  // namespace ts_internal
