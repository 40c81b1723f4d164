// BlockTeam kernel for the logistic model: cooperative persistent grid.
#include <stdio.h>
#include <stdlib.h>
#include "ts_internal.cuh"

namespace ts_internal {

int launch_block_logistic(const ts_model* m, int nslots, OpArgs& A, cudaStream_t st) {
  const int PMAX = m->pmax;
  LogisticW mw;
  mw.a.xt = m->xt; mw.a.yt = m->yt; mw.a.n_rows = m->n_rows; mw.a.p = m->p; mw.a.ntiles = m->ntiles;
  mw.a.pbuf = m->pbuf; mw.a.bar = m->bar; mw.a.fp64 = m->fp64; mw.a.pmax = m->pmax;
  mw.wred = nullptr; mw.red_s = nullptr; mw.epoch = 0;
  const int threads = 256;
  const int nwarps = threads / 32;
  int scratch = (nwarps * (PMAX + 2) + 1) & ~1;
  if (scratch < threads) scratch = threads;
  if (scratch < m->p + 2) scratch = m->p + 2;
  const int D = m->dim;
  const size_t base = ((size_t)num_vecs(nslots) * D + kTeamScratch + 2 + scratch + (m->p + 2)) * sizeof(double) + 128;
  int dev = 0, nsm = 0, smem_max = 0;
  TS_CUDA(cudaGetDevice(&dev));
  TS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  TS_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  // per-warp TMA ring: as many stages (<= 4) as shared memory allows
  const int stage_bytes = ((128 * m->p + 32) + 127) / 128 * 128;
  // Two stages per worker warp: enough bytes in flight to saturate HBM, and
  // the rest of the 256 KB L1/shared array stays L1 for the engine's stack.
  int nstage = 2;
  if (const char* e = getenv("TS_NSTAGE")) nstage = atoi(e) < 1 ? 1 : (atoi(e) > 4 ? 4 : atoi(e));  // profiling
  auto need = [&](int ns) { return base + (size_t)nwarps * ns * (stage_bytes + 8) + nwarps * 16; };
  while (nstage > 1 && need(nstage) > (size_t)smem_max) --nstage;
  if (need(nstage) > (size_t)smem_max)
    return set_err(TS_EUNSUPPORTED, "logistic model: shared memory too small for D / max_tree_depth");
  mw.a.nstage = nstage;
  mw.a.stage_bytes = stage_bytes;
  mw.a.l2_keep_tiles = 0;
  mw.a.prof = m->prof;
  mw.a.l2_prefetch = 0;
  mw.a.exact_cvt = m->exact_cvt;
  if (const char* e = getenv("TS_L2_PREFETCH")) mw.a.l2_prefetch = atoi(e);
  if (const char* e = getenv("TS_L2_KEEP_FRAC")) mw.a.l2_keep_tiles = (int)(atof(e) * (double)m->ntiles);
  const size_t smem = need(nstage);
  auto kern = k_block_op<LogisticW>;
  TS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  TS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
  if (occ < 1) return set_err(TS_EUNSUPPORTED, "logistic kernel cannot be resident (shared memory / registers)");
  int64_t grid = (int64_t)nsm * occ;
  if (m->grid > 0 && m->grid < grid) grid = m->grid;
  if (grid > m->ntiles) grid = m->ntiles;
  if (grid < 1) grid = 1;
  TS_CUDA(cudaMemsetAsync(m->bar, 0, sizeof(unsigned long long), st));
  // component-major partial slots are padded to 16 CTAs; padding must read 0
  const size_t gpad = ((size_t)grid + 15) / 16 * 16;
  TS_CUDA(cudaMemsetAsync(m->pbuf, 0, 2 * gpad * (m->p + 2) * sizeof(double), st));
  int Dv = D, ns = nslots, sc = scratch;
  void* args[] = {&mw, &Dv, &ns, &sc, &A};
  TS_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3((unsigned)grid), dim3(threads), args, smem, st));
  return TS_OK;
}


}  // namespace ts_internal
