// Launcher of the logistic model's cooperative persistent grid (k_block_op<LogisticW>).
//
// Shared memory per CTA:
//   engine vectors (all, or only the hot ones for wide p) | team scratch |
//   model scratch (wred) | CTA partial sums | TMA ring(s) | mbarriers | ring counters
// One ring of `nstage` tiles per worker warp: 32-row tiles for p <= 64,
// 8-row tiles (32p+16 bytes) for 64 < p <= 256 (wide), where the NodeStore
// slot vectors also move to a per-CTA global workspace.
#include <stdio.h>
#include <stdlib.h>
#include "ts_internal.cuh"

namespace ts_internal {

int launch_block_logistic(const ts_model* m, int nslots, OpArgs& A, cudaStream_t st) {
  LogisticW mw;
  memset(&mw, 0, sizeof mw);
  mw.a.xt = m->xt; mw.a.yt = m->yt; mw.a.n_rows = m->n_rows; mw.a.p = m->p; mw.a.ntiles = m->ntiles;
  mw.a.pbuf = m->pbuf; mw.a.bar = m->bar; mw.a.fp64 = m->fp64; mw.a.pmax = m->pmax;
  mw.a.wide = m->wide;
  mw.a.xd = m->xd;
  mw.a.xh = m->xh;
  mw.a.prof = m->prof;
  mw.a.exact_cvt = m->exact_cvt;
  mw.a.dump = m->dump;
  mw.a.vranks = m->vranks;
  mw.a.err = m->errw;
  mw.a.spin_ns = spin_limit_ns();
  if (const char* e = getenv("TS_FAULT_INJECT")) mw.a.fault = atoi(e);  // tests of the bounded waits only
  // cross-CTA accumulator copies: 2 (covtype, same box: pass 19.08 / 19.08 /
  // 19.38 / 20.00 us and run 21.8 / 22.4 / 23.2 us per leapfrog with 1/2/4/8
  // copies: more copies spread the atomics but lengthen the read-back);
  // TS_FX_COPIES=1/2/4/8 for A/B
  mw.a.fxc = 2;
  if (const char* e = getenv("TS_FX_COPIES")) { const int c = atoi(e); mw.a.fxc = (c == 1 || c == 2 || c == 4) ? c : kFxCopies; }
  mw.a.llmode = 6;
  if (const char* e = getenv("TS_LLMODE")) mw.a.llmode = atoi(e);  // A/B of the fp32 log-likelihood precision
  // fp64 wide pass: half of the fp32->fp64 conversions on the integer pipe
  // (XU-bound otherwise; 2.77 -> 2.61 ms per 8Mx255 pass); the narrow pass
  // measured best with XU conversions (covtype: 32.8 us vs 37.9 with every
  // 4th / 36.0 with no element on the XU); TS_ICVT=0/1/2 for A/B
  mw.a.icvt = m->wide ? 1 : 0;
  // L2 residency: the first 70% of each warp's tiles are fetched with
  // L2::evict_last and the rest evict_first, so ~88 MB of X stays in L2
  // across passes (covtype pass 23.8 -> 21.8 us; 90% thrashes: 24.4 us).
  // The fp64 policy is XU-bound (conversions), not DRAM-bound: no split.
  // TS_L2_KEEP=<pct> overrides for A/B.
  mw.a.keep_pct = m->fp64 ? 0 : 70;
  if (const char* e = getenv("TS_L2_KEEP")) mw.a.keep_pct = atoi(e) < 0 ? 0 : (atoi(e) > 100 ? 100 : atoi(e));
  if (const char* e = getenv("TS_ICVT")) mw.a.icvt = atoi(e);
  if (m->world > 0) {
    mw.a.world = m->world;
    mw.a.rank = m->rank;
    for (int r = 0; r < m->world; ++r) mw.a.mail[r] = m->mail[r];
    mw.a.mail_epoch = m->mail_local + mail_words(m->p, m->world);
  }
  const int threads = 256;
  const int nwarps = threads / 32;
  const int D = m->dim;
  int scratch = m->wide ? wide_scratch_doubles(nwarps - 1) : (nwarps * (m->pmax + 2) + 1) & ~1;
  if (scratch < threads) scratch = threads;
  if (scratch < m->p + 2) scratch = m->p + 2;
  const int nv_smem = m->wide ? (int)V_SLOT0 : num_vecs(nslots);
  const size_t ring = m->wide ? 0 : ((size_t)kTrajRing * (3 * (m->p + 1) + 2) * sizeof(double) + 16);  // LogisticW::ring
  const size_t base = ((size_t)nv_smem * D + kTeamScratch + 2 + scratch + (m->p + 2) + (kWideMax + 8) / 2) * sizeof(double) + 128 + ring;
  int dev = 0, nsm = 0, smem_max = 0;
  TS_CUDA(cudaGetDevice(&dev));
  TS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  TS_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int stage_bytes = m->wide ? wide_stage_bytes(m->p, m->xd ? 8 : 4)
                          : (m->xh == 1 ? x64h_stage_bytes(m->p)
                             : m->xh == 2 ? pair_stage_bytes(m->p) : (int)((128 * (int64_t)m->p + 32 + 127) / 128 * 128));
  // Two stages per worker warp are enough bytes in flight to saturate HBM
  // and leave the rest of the L1/shared array to the engine's stack.
  const int rings = nwarps - 1;  // worker warps
  int nstage = 2;
  if (const char* e = getenv("TS_NSTAGE")) nstage = atoi(e) < 1 ? 1 : (atoi(e) > 4 ? 4 : atoi(e));  // profiling
  auto need = [&](int ns) { return base + (size_t)rings * ns * (stage_bytes + 8) + rings * sizeof(WarpPipe); };
  while (nstage > 1 && need(nstage) > (size_t)smem_max) --nstage;
  if (need(nstage) > (size_t)smem_max)
    return set_err(TS_EUNSUPPORTED, "logistic model: shared memory too small for D / max_tree_depth");
  mw.a.nstage = nstage;
  mw.a.stage_bytes = stage_bytes;
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
  if (m->vranks > 1) {  // emulated ranks: equal CTA groups, one mailbox set per launch
    grid = grid / m->vranks * m->vranks;
    if (grid < m->vranks) return set_err(TS_EUNSUPPORTED, "too few CTAs for the emulated ranks");
    ts_model* mm = const_cast<ts_model*>(m);
    const size_t words = (size_t)m->vranks * mail_words(m->p, m->vranks) + 16;
    if (mm->vmail_words < words) {
      if (mm->vmail) cudaFree(mm->vmail);
      mm->vmail = nullptr;
      mm->vmail_words = 0;
      TS_CUDA(cudaMalloc((void**)&mm->vmail, words * sizeof(unsigned long long)));
      mm->vmail_words = words;
    }
    TS_CUDA(cudaMemsetAsync(mm->vmail, 0, words * sizeof(unsigned long long), st));
    mw.a.vmail = mm->vmail;
  }
  if (m->wide) {  // per-CTA NodeStore slot vectors in global memory
    ts_model* mm = const_cast<ts_model*>(m);
    const size_t need_ws = (size_t)grid * kSlotVecs * (nslots < 1 ? 1 : nslots) * D;
    if (mm->slotws_size < need_ws) {
      if (mm->slotws) cudaFree(mm->slotws);
      mm->slotws = nullptr;
      mm->slotws_size = 0;
      TS_CUDA(cudaMalloc((void**)&mm->slotws, need_ws * sizeof(double)));
      mm->slotws_size = need_ws;
    }
    mw.a.slotws = mm->slotws;
  }
  const int nranks = m->vranks > 1 ? m->vranks : 1;
  TS_CUDA(cudaMemsetAsync(m->bar, 0, 16 * nranks * sizeof(unsigned long long), st));
  // rotating fixed-point accumulators start at zero (fx_rank_words per rank)
  TS_CUDA(cudaMemsetAsync(m->pbuf, 0, nranks * (size_t)fx_rank_words(m->p) * sizeof(unsigned long long), st));
  int Dv = D, ns = nslots, sc = scratch;
  void* args[] = {&mw, &Dv, &ns, &sc, &A};
  TS_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3((unsigned)grid), dim3(threads), args, smem, st));
  return TS_OK;
}

}  // namespace ts_internal
