// C-ABI of the B200 turnstile engine (declared in include/turnstile_b200.h).
//
// Kernels:
//   k_thread_op  - ThreadTeam: one chain (or one parity op) per thread, small
//                  models, vectors in a chain-interleaved global workspace.
//   k_block_op   - BlockTeam: one replica of the chain per CTA; with the
//                  logistic model the CTAs form a cooperative persistent grid
//                  that evaluates each potential together (one grid barrier
//                  per leapfrog) and run the tree logic redundantly.
#include <stdio.h>
#include <stdlib.h>
#include "ts_internal.cuh"

using namespace ts;
using namespace ts_internal;

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;
namespace ts_internal {
int set_err(int code, const char* msg) {
  g_last_error = msg;
  return code;
}
}  // namespace ts_internal

extern "C" const char* ts_last_error(void) { return g_last_error.c_str(); }
extern "C" int ts_abi_version(void) { return TS_ABI_VERSION; }

// Re-tile X into 32-row tiles (padding rows are zero with label 0),
// feature-group-major inside a tile (lane-contiguous rows for LDS.128).
__global__ void k_retile(const float* __restrict__ x, const uint8_t* __restrict__ y, int64_t n, int p, int64_t ntiles,
                         float* __restrict__ xt, uint8_t* __restrict__ yt, int* __restrict__ has_subnormal) {
  const int64_t total = ntiles * 32 * (int64_t)p;
  int sub = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / p;
    const int j = (int)(i % p);
    const int64_t t = row >> 5;
    const int lane = (int)(row & 31);
    const int g = j >> 2;
    const int w = (p - 4 * g) < 4 ? (p - 4 * g) : 4;
    const int64_t dst = t * 32 * (int64_t)p + 128 * (int64_t)g + (int64_t)lane * w + (j & 3);
    const float v = row < n ? x[row * p + j] : 0.f;
    const unsigned a = __float_as_uint(v) & 0x7fffffffu;
    sub |= (a != 0u && a < 0x00800000u) || a >= 0x7f800000u;  // subnormal or non-finite: no integer fp64 conversion
    xt[dst] = v;
    if (j == 0) yt[row] = row < n ? y[row] : 0;
  }
  if (__syncthreads_or(sub) && threadIdx.x == 0) atomicOr(has_subnormal, 1);
}

// fp64 storage, p <= 64 (ts_logistic.cuh, logistic_cta_pass_x64h): 16-row
// tiles, lane 16 h + r = row r's features [h H, h H + H) in lane-contiguous
// pairs of doubles, then the 16 labels; padding (odd H / odd p, rows past n)
// stays zero from the memset.
__global__ void k_retile_x64h(const double* __restrict__ x, const uint8_t* __restrict__ y, int64_t n, int p,
                              int64_t ntiles, unsigned char* __restrict__ xt) {
  const int H = x64h_half(p), G = x64h_groups(p);
  const int64_t tb = x64h_tile_bytes(p);
  const int64_t total = ntiles * 16 * (int64_t)p;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / p;
    const int j = (int)(i % p);
    const int64_t t = row >> 4;
    const int r = (int)(row & 15);
    const int h = j >= H ? 1 : 0;
    const int k = j - h * H;
    unsigned char* tile = xt + t * tb;
    reinterpret_cast<double*>(tile)[((k >> 1) * 32 + 16 * h + r) * 2 + (k & 1)] = row < n ? x[row * p + j] : 0.0;
    if (j == 0) tile[512 * G + r] = row < n ? y[row] : 0;
  }
}

// Paired half-row layout (fp64 policy on fp32 X, p <= 64;
// ts_logistic.cuh, logistic_cta_pass_pair): 32-row tiles of two 16-row
// half-row blocks (groups of 4 floats), then the 32 labels in row order;
// padding stays zero from the memset.
__global__ void k_retile_pair(const float* __restrict__ x, const uint8_t* __restrict__ y, int64_t n, int p,
                              int64_t ntiles, unsigned char* __restrict__ xt) {
  const int H = x64h_half(p), G = pair_groups(p);
  const int64_t tb = pair_tile_bytes(p);
  const int64_t total = ntiles * 32 * (int64_t)p;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / p;
    const int j = (int)(i % p);
    const int64_t t = row >> 5;
    const int rr = (int)(row & 31), b = rr >> 4, r = rr & 15;
    const int h = j >= H ? 1 : 0;
    const int k = j - h * H;
    unsigned char* tile = xt + t * tb;
    reinterpret_cast<float*>(tile + (int64_t)b * G * 512)[((k >> 2) * 32 + 16 * h + r) * 4 + (k & 3)] =
        row < n ? x[row * p + j] : 0.f;
    if (j == 0) tile[2 * G * 512 + rr] = row < n ? y[row] : 0;
  }
}

// Wide p (64 < p <= 256): tiles of kWideRows = 8 rows, row-major, each
// followed by 16 label bytes (8 labels + 8 zeros): 32p + 16 bytes per tile,
// one TMA bulk copy (ts_logistic.cuh, logistic_cta_pass_wide).
// T = double: the fp64-storage layout ("fp64x"), 64p + 16 bytes per tile.
template <class T>
__global__ void k_retile_wide(const T* __restrict__ x, const uint8_t* __restrict__ y, int64_t n, int p,
                              int64_t ntiles, unsigned char* __restrict__ xt, int* __restrict__ has_subnormal) {
  const int64_t total = ntiles * kWideRows * (int64_t)p;
  const int64_t tb = wide_tile_bytes(p, (int)sizeof(T));
  const int64_t lab = kWideRows * (int64_t)sizeof(T) * p;
  int sub = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / p;
    const int j = (int)(i % p);
    const int64_t t = row / kWideRows;
    const int r = (int)(row % kWideRows);
    const T v = row < n ? x[row * p + j] : (T)0;
    if (sizeof(T) == 4) {
      const unsigned a = __float_as_uint((float)v) & 0x7fffffffu;
      sub |= (a != 0u && a < 0x00800000u) || a >= 0x7f800000u;
    }
    unsigned char* tile = xt + t * tb;
    reinterpret_cast<T*>(tile)[r * p + j] = v;
    if (j == 0) {
      tile[lab + r] = row < n ? y[row] : 0;
      tile[lab + kWideRows + r] = 0;
    }
  }
  if (__syncthreads_or(sub) && threadIdx.x == 0) atomicOr(has_subnormal, 1);
}

static int pick_pmax(int p) {
  if (p <= 8) return 8;
  if (p <= 32) return 32;
  if (p <= 56) return 56;
  if (p <= 64) return 64;
  if (p <= kWideMax) return kWideMax;  // wide pass
  return 0;
}

// ------------------------------------------------------------------ helpers
constexpr int kProfWords = 24 + 2 * 2048;  // TS_PROF counters + per-CTA skew slots
static int check_cfg(const ts_sampler_cfg* c) {
  if (!c) return set_err(TS_EINVAL, "null sampler config");
  if (!(c->step_size > 0) || !isfinite(c->step_size)) return set_err(TS_EINVAL, "step_size must be positive and finite");
  if (c->max_tree_depth < 1 || c->max_tree_depth > 30) return set_err(TS_EINVAL, "max_tree_depth must be in [1, 30]");
  if (c->criterion != TS_GENERALIZED && c->criterion != TS_CLASSIC) return set_err(TS_EINVAL, "unknown criterion");
  if (!(c->divergence_threshold > 0)) return set_err(TS_EINVAL, "divergence_threshold must be positive");
  return TS_OK;
}

static SamplerCfg to_cfg(const ts_sampler_cfg* c) {
  SamplerCfg s;
  s.step = c->step_size;
  s.max_depth = c->max_tree_depth;
  s.generalized = c->criterion == TS_GENERALIZED;
  s.threshold = c->divergence_threshold;
  return s;
}

static int launch(const ts_model* m, int nslots, OpArgs& A, int n_threads_chains, ts_exec_mode mode, cudaStream_t st) {
  if (nslots < 1) nslots = 1;
  if (nslots > kMaxSlots) return set_err(TS_EINVAL, "tree depth exceeds device slot limit (30)");
  if (m->kind == TS_LOGISTIC) {
    if (m->many) return launch_logistic_many(m, nslots, A, n_threads_chains, st);
    if (!m->pmax) return set_err(TS_EUNSUPPORTED, "logistic feature count > 256 not supported on this path");
    return launch_block_logistic(m, nslots, A, st);
  }
  if (m->kind == TS_DENSE_GAUSS) return launch_dense(m, nslots, A, n_threads_chains, st);
  SmallModel sm;
  sm.kind = m->kind;
  sm.dim = m->dim;
  sm.params = m->params;
  const int D = m->dim;
  if (mode == TS_EXEC_BLOCK) return launch_block_small(sm, D, nslots, A, n_threads_chains, st);
  if (mode == TS_EXEC_WARP) return launch_warp_small(sm, D, nslots, A, n_threads_chains, st);
  return launch_thread(sm, D, n_threads_chains, nslots, A, st);
}

// ------------------------------------------------------------------ C ABI
extern "C" int ts_model_create(int kind, int dim, const double* params, int n_params, const void* x_dev,
                               const uint8_t* y_dev, int64_t n_rows, int n_feat, int precision, ts_model** out) {
  if (!out) return set_err(TS_EINVAL, "null output handle");
  *out = nullptr;
  if (dim < 1) return set_err(TS_EINVAL, "model dimension must be positive");
  ts_model* m = new ts_model();
  memset(m, 0, sizeof(*m));
  m->kind = kind;
  m->dim = dim;
  cudaGetDevice(&m->device);
  auto fail = [&](int code, const char* msg) {
    if (m->errw) cudaFree(m->errw);
    if (m->xaug) cudaFree(m->xaug);
    if (m->params) cudaFree(m->params);
    if (m->xt) cudaFree(m->xt);
    if (m->yt) cudaFree(m->yt);
    if (m->pbuf) cudaFree(m->pbuf);
    if (m->bar) cudaFree(m->bar);
    delete m;
    return set_err(code, msg);
  };
  switch (kind) {
    case TS_STD_NORMAL:
      break;
    case TS_GAUSSIAN:
      if (n_params != dim || !params) return fail(TS_EINVAL, "gaussian needs dim inverse variances");
      break;
    case TS_FUNNEL:
      if (dim < 2) return fail(TS_EINVAL, "funnel needs the scale coordinate plus at least one other");
      break;
    case TS_DENSE_GAUSS: {
      if (n_params != dim * dim || !params) return fail(TS_EINVAL, "dense_gauss needs A[dim][dim]");
      m->fp64 = precision == TS_PREC_FP64;
      if (!m->fp64 && dim % 4 != 0) return fail(TS_EUNSUPPORTED, "dense_gauss TF32 path needs dim % 4 == 0");
      // tf32-rounded copy of A for the tensor-core path (round to nearest, ties away)
      float* h = (float*)malloc((size_t)dim * dim * sizeof(float));
      if (!h) return fail(TS_ECUDA, "host allocation failed");
      for (int64_t i = 0; i < (int64_t)dim * dim; ++i) {
        float f = (float)params[i];
        uint32_t b;
        memcpy(&b, &f, 4);
        if ((b & 0x7f800000u) != 0x7f800000u) b = (b + 0x1000u) & 0xffffe000u;
        memcpy(&f, &b, 4);
        h[i] = f;
      }
      cudaError_t e = cudaMalloc((void**)&m->a32, (size_t)dim * dim * sizeof(float));
      if (e == cudaSuccess) e = cudaMemcpy(m->a32, h, (size_t)dim * dim * sizeof(float), cudaMemcpyHostToDevice);
      free(h);
      if (e != cudaSuccess) return fail(TS_ECUDA, "dense_gauss upload failed");
      break;
    }
    case TS_EIGHT_SCHOOLS:
      if (dim < 3 || n_params != 2 * (dim - 2) || !params) return fail(TS_EINVAL, "eight_schools needs y[J], sigma[J] with dim = J + 2");
      break;
    case TS_LOGISTIC: {
      if (n_feat < 1 || dim != n_feat + 1) return fail(TS_EINVAL, "logistic dim must equal num_features + 1");
      if (n_rows < 1 || !x_dev || !y_dev) return fail(TS_EINVAL, "logistic needs at least one data row");
      if (precision == TS_PREC_TF32) {  // many chains sharing X on the tensor cores
        m->many = 1;
        m->n_rows = n_rows;
        m->p = n_feat;
        const int rc = build_logistic_xaug(m, static_cast<const float*>(x_dev), y_dev);
        if (rc) {
          const std::string why = ts_last_error();
          return fail(rc, why.c_str());
        }
        if (cudaDeviceSynchronize() != cudaSuccess) return fail(TS_ECUDA, "augmented X build failed");
        break;
      }
      m->pmax = pick_pmax(n_feat);
      if (!m->pmax) return fail(TS_EUNSUPPORTED, "logistic feature count > 256 not supported on this path");
      m->xd = precision == TS_PREC_FP64X;  // X stored as fp64
      m->wide = n_feat > 64;
      // p <= 64 in fp64 arithmetic: half-row tiles (1: X fp64, 16-row tiles;
      // 2: X fp32, paired 32-row tiles)
      m->xh = m->wide ? 0 : (m->xd ? 1 : (precision == TS_PREC_FP64 ? 2 : 0));
      if (m->xd) m->pmax = m->wide ? kWideMax : kX64hPmax;
      if (m->xh) m->pmax = kX64hPmax;
      m->n_rows = n_rows;
      m->p = n_feat;
      // wide: whole groups of kWideGroup tiles (32 rows), padding rows zero with label 0
      m->ntiles = m->wide ? (n_rows + kWideRows * kWideGroup - 1) / (kWideRows * kWideGroup) * kWideGroup
                          : (m->xh == 1 ? (n_rows + 15) / 16 : (n_rows + 31) / 32);
      m->fp64 = precision == TS_PREC_FP64 || m->xd;
      const size_t xbytes = m->wide ? (size_t)m->ntiles * wide_tile_bytes(n_feat, m->xd ? 8 : 4)
                                    : (m->xh == 1 ? (size_t)m->ntiles * x64h_tile_bytes(n_feat)
                                       : m->xh == 2 ? (size_t)m->ntiles * pair_tile_bytes(n_feat)
                                             : (size_t)m->ntiles * 32 * n_feat * sizeof(float));
      if (cudaMalloc((void**)&m->xt, xbytes) != cudaSuccess) return fail(TS_ECUDA, "cudaMalloc X failed");
      // wide tiles carry their labels; the separate label array is then unused
      if (cudaMalloc((void**)&m->yt, (m->wide || m->xh) ? 16 : (size_t)m->ntiles * 32) != cudaSuccess) return fail(TS_ECUDA, "cudaMalloc y failed");
      // grid-barrier counters: one cache line per (emulated) rank, up to 8
      if (cudaMalloc((void**)&m->bar, 16 * 8 * sizeof(unsigned long long)) != cudaSuccess) return fail(TS_ECUDA, "cudaMalloc barrier failed");
      if (cudaMemset(m->bar, 0, 16 * 8 * sizeof(unsigned long long)) != cudaSuccess) return fail(TS_ECUDA, "memset barrier failed");
      // the barrier word doubles as the "X has fp32 subnormals" flag during re-tiling
      if (m->xh) {
        if (cudaMemset(m->xt, 0, xbytes) != cudaSuccess) return fail(TS_ECUDA, "memset X failed");
        if (m->xh == 1)
          k_retile_x64h<<<1184, 256>>>(static_cast<const double*>(x_dev), y_dev, n_rows, n_feat, m->ntiles,
                                       reinterpret_cast<unsigned char*>(m->xt));
        else
          k_retile_pair<<<1184, 256>>>(static_cast<const float*>(x_dev), y_dev, n_rows, n_feat, m->ntiles,
                                       reinterpret_cast<unsigned char*>(m->xt));
      } else if (m->xd)
        k_retile_wide<double><<<1184, 256>>>(static_cast<const double*>(x_dev), y_dev, n_rows, n_feat, m->ntiles,
                                             reinterpret_cast<unsigned char*>(m->xt), reinterpret_cast<int*>(m->bar));
      else if (m->wide)
        k_retile_wide<float><<<1184, 256>>>(static_cast<const float*>(x_dev), y_dev, n_rows, n_feat, m->ntiles,
                                            reinterpret_cast<unsigned char*>(m->xt), reinterpret_cast<int*>(m->bar));
      else
        k_retile<<<1184, 256>>>(static_cast<const float*>(x_dev), y_dev, n_rows, n_feat, m->ntiles, m->xt, m->yt,
                                reinterpret_cast<int*>(m->bar));
      if (cudaGetLastError() != cudaSuccess) return fail(TS_ECUDA, "retile launch failed");
      unsigned long long flag = 0;
      if (cudaMemcpy(&flag, m->bar, sizeof flag, cudaMemcpyDeviceToHost) != cudaSuccess) return fail(TS_ECUDA, "retile failed");
      m->exact_cvt = flag != 0;
      int nsm = 148;
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m->device);
      const size_t pb = (size_t)TS_MAX_PEERS * fx_rank_words(n_feat);  // up to 8 (emulated) ranks
      if (cudaMalloc((void**)&m->pbuf, pb * sizeof(double)) != cudaSuccess) return fail(TS_ECUDA, "cudaMalloc partials failed");
      if (cudaMemset(m->pbuf, 0, pb * sizeof(double)) != cudaSuccess) return fail(TS_ECUDA, "memset partials failed");
      if (cudaDeviceSynchronize() != cudaSuccess) return fail(TS_ECUDA, "retile failed");
      break;
    }
    default:
      return fail(TS_EINVAL, "unknown model kind");
  }
  if (n_params > 0 && params && kind != TS_LOGISTIC) {
    if (cudaMalloc((void**)&m->params, n_params * sizeof(double)) != cudaSuccess) return fail(TS_ECUDA, "cudaMalloc params failed");
    if (cudaMemcpy(m->params, params, n_params * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(TS_ECUDA, "params upload failed");
    m->n_params = n_params;
  }
  if (cudaMalloc((void**)&m->errw, 16) != cudaSuccess || cudaMemset(m->errw, 0, 16) != cudaSuccess)
    return fail(TS_ECUDA, "cudaMalloc error word failed");
  *out = m;
  return TS_OK;
}

extern "C" int ts_model_destroy(ts_model* m) {
  if (!m) return TS_OK;
  if (m->params) cudaFree(m->params);
  if (m->xt) cudaFree(m->xt);
  if (m->yt) cudaFree(m->yt);
  if (m->pbuf) cudaFree(m->pbuf);
  if (m->bar) cudaFree(m->bar);
  if (m->slotws) cudaFree(m->slotws);
  if (m->a32) cudaFree(m->a32);
  if (m->dws) cudaFree(m->dws);
  for (int r = 0; r < m->world; ++r)
    if (m->mail[r] && m->mail[r] != m->mail_local) cudaIpcCloseMemHandle(m->mail[r]);
  if (m->mail_local) cudaFree(m->mail_local);
  if (m->vmail) cudaFree(m->vmail);
  if (m->errw) cudaFree(m->errw);
  if (m->xaug) cudaFree(m->xaug);
  delete m;
  return TS_OK;
}

extern "C" int ts_model_error(const ts_model* m, int* code) {
  if (!m || !code) return set_err(TS_EINVAL, "null argument");
  unsigned int w = 0;
  TS_CUDA(cudaMemcpy(&w, m->errw, sizeof w, cudaMemcpyDeviceToHost));
  *code = w ? TS_STATUS_SYNC_TIMEOUT : TS_OK;
  return TS_OK;
}

// Stream-ordered: a run whose kernel gave up on a wait reports it per chain.
__global__ void k_fold_timeout(const unsigned int* errw, int32_t* status, int n) {
  if (*errw == 0u) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) status[i] = TS_STATUS_SYNC_TIMEOUT;
}

extern "C" int ts_model_set_grid(ts_model* m, int grid) {
  if (!m) return set_err(TS_EINVAL, "null model");
  m->grid = grid;
  return TS_OK;
}

extern "C" int ts_model_dim(const ts_model* m) { return m ? m->dim : -1; }

static OpArgs base_args(int op) {
  OpArgs A;
  memset(&A, 0, sizeof A);
  A.op = op;
  return A;
}

extern "C" int ts_potential_grad(const ts_model* m, const double* q_dev, int n_points, double* out_dev, void* stream) {
  if (!m || !q_dev || !out_dev) return set_err(TS_EINVAL, "null argument");
  if (n_points < 1) return TS_OK;
  OpArgs A = base_args(OP_POTGRAD);
  A.z_in = q_dev; A.z_out = out_dev; A.n_points = n_points;
  // inv is read by do_op; use a dummy ones vector
  double* ones = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  TS_CUDA(cudaMallocAsync((void**)&ones, m->dim * sizeof(double), st));
  TS_CUDA(cudaMemsetAsync(ones, 0, m->dim * sizeof(double), st));
  A.inv = ones;
  int rc = launch(m, 1, A, 1, TS_EXEC_THREAD, st);
  cudaFreeAsync(ones, st);
  return rc;
}

// ------------------------------------------------------------------ row sharding
extern "C" int ts_peer_mailbox_create(ts_model* m, int rank, int world, void* ipc_handle_out) {
  if (!m || !ipc_handle_out) return set_err(TS_EINVAL, "null argument");
  if (m->kind != TS_LOGISTIC) return set_err(TS_EINVAL, "row sharding applies to the logistic model only");
  if (world < 1 || world > TS_MAX_PEERS || rank < 0 || rank >= world) return set_err(TS_EINVAL, "rank/world out of range");
  if (m->mail_local) return set_err(TS_EINVAL, "mailbox already created");
  const size_t words = (size_t)mail_words(m->p, world) + 16;  // + exchange counter (own cache line)
  TS_CUDA(cudaMalloc((void**)&m->mail_local, words * sizeof(unsigned long long)));
  TS_CUDA(cudaMemset(m->mail_local, 0, words * sizeof(unsigned long long)));
  cudaIpcMemHandle_t h;
  TS_CUDA(cudaIpcGetMemHandle(&h, m->mail_local));
  memcpy(ipc_handle_out, &h, sizeof h);
  m->rank = rank;
  m->mail[rank] = m->mail_local;
  m->world = -world;  // connected by ts_peer_mailbox_connect
  return TS_OK;
}

extern "C" int ts_peer_mailbox_connect(ts_model* m, const void* ipc_handles) {
  if (!m || !ipc_handles) return set_err(TS_EINVAL, "null argument");
  if (m->world >= 0 || !m->mail_local) return set_err(TS_EINVAL, "call ts_peer_mailbox_create first (once)");
  const int world = -m->world;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  for (int r = 0; r < world; ++r) {
    if (r == m->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)ipc_handles + 64 * r, 64);
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      for (int k = 0; k < r; ++k)
        if (k != m->rank && m->mail[k]) { cudaIpcCloseMemHandle(m->mail[k]); m->mail[k] = nullptr; }
      cudaGetLastError();
      return set_err(TS_ECUDA, "cudaIpcOpenMemHandle failed (peer GPU not reachable?)");
    }
    m->mail[r] = (unsigned long long*)p;
  }
  m->world = world;
  return TS_OK;
}

extern "C" int ts_model_set_virtual_ranks(ts_model* m, int vranks) {
  if (!m) return set_err(TS_EINVAL, "null model");
  if (m->kind != TS_LOGISTIC) return set_err(TS_EINVAL, "logistic model only");
  if (vranks < 1 || vranks > TS_MAX_PEERS) return set_err(TS_EINVAL, "vranks must be in [1, 8]");
  if (m->world != 0) return set_err(TS_EINVAL, "model already joined a multi-GPU group");
  m->vranks = vranks;
  return TS_OK;
}

extern "C" int ts_logistic_partial_sums(const ts_model* m, const double* q_dev, uint64_t* words_dev, void* stream) {
  if (!m || !q_dev || !words_dev) return set_err(TS_EINVAL, "null argument");
  if (m->kind != TS_LOGISTIC) return set_err(TS_EINVAL, "logistic model only");
  if (m->world > 0) return set_err(TS_EINVAL, "partial sums of a connected model would take part in the exchange");
  cudaStream_t st = (cudaStream_t)stream;
  double* out = nullptr;
  TS_CUDA(cudaMallocAsync((void**)&out, (m->dim + 1) * sizeof(double), st));
  ts_model* mm = const_cast<ts_model*>(m);
  mm->dump = reinterpret_cast<unsigned long long*>(words_dev);
  const int rc = ts_potential_grad(m, q_dev, 1, out, stream);
  mm->dump = nullptr;
  cudaFreeAsync(out, st);
  return rc;
}

extern "C" int ts_eval_bench(const ts_model* m, const double* q_dev, int repeats, double* out_dev, void* stream) {
  if (!m || !q_dev || !out_dev) return set_err(TS_EINVAL, "null argument");
  OpArgs A = base_args(OP_EVALBENCH);
  A.z_in = q_dev; A.z_out = out_dev; A.n_points = repeats;
  double* ones = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  TS_CUDA(cudaMallocAsync((void**)&ones, m->dim * sizeof(double), st));
  TS_CUDA(cudaMemsetAsync(ones, 0, m->dim * sizeof(double), st));
  A.inv = ones;
  // out_dev[2..5] (as u64): CTA-0 cycle counters of the logistic pass phases
  TS_CUDA(cudaMemsetAsync(out_dev, 0, 10 * sizeof(double), st));
  const_cast<ts_model*>(m)->prof = reinterpret_cast<unsigned long long*>(out_dev + 2);
  int rc = launch(m, 1, A, 1, TS_EXEC_BLOCK, st);
  const_cast<ts_model*>(m)->prof = nullptr;
  cudaFreeAsync(ones, st);
  return rc;
}

extern "C" int ts_leapfrog(const ts_model* m, const double* inv_dev, const double* z_in, double eps, double* z_out,
                           int exec_mode, void* stream) {
  if (!m || !inv_dev || !z_in || !z_out) return set_err(TS_EINVAL, "null argument");
  OpArgs A = base_args(OP_LEAPFROG);
  A.z_in = z_in; A.z_out = z_out; A.inv = inv_dev; A.eps = eps;
  return launch(m, 1, A, 1, (ts_exec_mode)exec_mode, (cudaStream_t)stream);
}

extern "C" int ts_build_tree(const ts_model* m, const ts_sampler_cfg* cfg, const double* inv_dev, const double* z_in,
                             int depth, double eps, double h_ref, uint64_t key_hi, uint64_t key_lo, double* tree_out,
                             int32_t* trace_ev, int trace_cap, double* leaf_lw, int lw_cap, int32_t* trace_counts,
                             int exec_mode, void* stream) {
  if (!m || !inv_dev || !z_in || !tree_out) return set_err(TS_EINVAL, "null argument");
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (depth < 0) return set_err(TS_EINVAL, "depth must be non-negative");
  if (depth > cfg->max_tree_depth) return set_err(TS_EINVAL, "depth exceeds max_tree_depth");
  if (depth > 30) return set_err(TS_EINVAL, "depth exceeds the hard limit 30");
  OpArgs A = base_args(OP_TREE);
  A.z_in = z_in; A.z_out = tree_out; A.inv = inv_dev; A.cfg = to_cfg(cfg);
  A.depth = depth; A.eps = eps; A.h_ref = h_ref; A.key_hi = key_hi; A.key_lo = key_lo;
  if (trace_ev && trace_counts) {
    A.has_trace = 1;
    A.trace.ev = trace_ev; A.trace.cap = trace_cap; A.trace.leaf_lw = leaf_lw; A.trace.lw_cap = leaf_lw ? lw_cap : 0;
    A.trace.counts = trace_counts;
  }
  return launch(m, depth, A, 1, (ts_exec_mode)exec_mode, (cudaStream_t)stream);
}

extern "C" int ts_transition(const ts_model* m, const ts_sampler_cfg* cfg, const double* inv_dev, const double* z_in,
                             const double* normals_or_null, uint64_t key_hi, uint64_t key_lo, double* out,
                             int32_t* trace_ev, int trace_cap, int32_t* trace_counts, int exec_mode, void* stream) {
  if (!m || !inv_dev || !z_in || !out) return set_err(TS_EINVAL, "null argument");
  int rc = check_cfg(cfg);
  if (rc) return rc;
  OpArgs A = base_args(OP_TRANSITION);
  A.z_in = z_in; A.z_out = out; A.inv = inv_dev; A.cfg = to_cfg(cfg);
  A.key_hi = key_hi; A.key_lo = key_lo; A.inj = normals_or_null;
  if (trace_ev && trace_counts) {
    A.has_trace = 1;
    A.trace.ev = trace_ev; A.trace.cap = trace_cap; A.trace.counts = trace_counts;
  }
  return launch(m, cfg->max_tree_depth - 1, A, 1, (ts_exec_mode)exec_mode, (cudaStream_t)stream);
}

extern "C" int ts_hmc_transition(const ts_model* m, const ts_sampler_cfg* cfg, const double* inv_dev, const double* z_in,
                                 const double* normals_or_null, uint64_t key_hi, uint64_t key_lo, int num_steps,
                                 double* out, int exec_mode, void* stream) {
  if (!m || !inv_dev || !z_in || !out) return set_err(TS_EINVAL, "null argument");
  if (num_steps < 1) return set_err(TS_EINVAL, "num_steps must be >= 1");
  int rc = check_cfg(cfg);
  if (rc) return rc;
  OpArgs A = base_args(OP_HMC);
  A.z_in = z_in; A.z_out = out; A.inv = inv_dev; A.cfg = to_cfg(cfg);
  A.key_hi = key_hi; A.key_lo = key_lo; A.inj = normals_or_null; A.depth = num_steps;
  return launch(m, 1, A, 1, (ts_exec_mode)exec_mode, (cudaStream_t)stream);
}

extern "C" int ts_find_step_size(const ts_model* m, const double* inv_dev, const double* z_in, const double* normals_or_null,
                                 uint64_t key_hi, uint64_t key_lo, double init, double* out, int exec_mode, void* stream) {
  if (!m || !inv_dev || !z_in || !out) return set_err(TS_EINVAL, "null argument");
  OpArgs A = base_args(OP_STEPSEARCH);
  A.z_in = z_in; A.z_out = out; A.inv = inv_dev; A.eps = init;
  A.key_hi = key_hi; A.key_lo = key_lo; A.inj = normals_or_null;
  return launch(m, 1, A, 1, (ts_exec_mode)exec_mode, (cudaStream_t)stream);
}

extern "C" int ts_run_chains(const ts_model* m, const ts_run_cfg* rc, const uint64_t* chain_keys_dev, int n_chains,
                             const double* inv0_dev, const uint8_t* schedule_dev, const double* da_weight_dev,
                             double* samples, double* stats, double* adapt, int32_t* status, int64_t* evals, int exec_mode,
                             void* stream) {
  if (!m || !rc || !chain_keys_dev || !inv0_dev || !samples || !stats || !adapt || !status)
    return set_err(TS_EINVAL, "null argument");
  int r = check_cfg(&rc->sampler);
  if (r) return r;
  if (n_chains < 1) return set_err(TS_EINVAL, "num_chains must be >= 1");
  if (rc->num_samples < 1) return set_err(TS_EINVAL, "num_samples must be >= 1");
  if (rc->num_warmup != 0 && rc->num_warmup < 20) return set_err(TS_EINVAL, "num_warmup must be 0 (off) or at least 20");
  if (rc->num_warmup > 0 && (!schedule_dev || !da_weight_dev)) return set_err(TS_EINVAL, "warmup needs schedule and weights");
  OpArgs A = base_args(OP_RUN);
  A.inv = inv0_dev;
  A.cfg = to_cfg(&rc->sampler);
  A.rc.num_warmup = rc->num_warmup;
  A.rc.num_samples = rc->num_samples;
  A.rc.target_accept = rc->target_accept;
  A.rc.base_step = rc->sampler.step_size;
  A.rc.has_sampler = rc->has_sampler;
  A.rc.keep_warmup = rc->keep_warmup ? 1 : 0;
  A.rc.sampler = A.cfg;
  A.rc.schedule = schedule_dev;
  A.rc.da_weight = da_weight_dev;
  A.chain_keys = chain_keys_dev;
  A.n_chains = n_chains;
  A.samples = samples; A.stats = stats; A.adapt = adapt; A.status = status; A.evals = evals;
  cudaStream_t st = (cudaStream_t)stream;
  const int nslots = rc->sampler.max_tree_depth - 1;
  // TS_PROF=1: chain-0 cycle counters of the run, printed to stderr (profiling
  // aid; logistic runs and warp-team small-model runs)
  // (allocated per call on the launch stream: no buffer shared across devices or threads)
  unsigned long long* prof_buf = nullptr;
  const bool prof = getenv("TS_PROF") != nullptr &&
                    (m->kind == TS_LOGISTIC || m->kind == TS_DENSE_GAUSS || exec_mode == TS_EXEC_WARP);
  if (prof) {
    TS_CUDA(cudaMallocAsync((void**)&prof_buf, kProfWords * sizeof(unsigned long long), st));
    TS_CUDA(cudaMemsetAsync(prof_buf, 0, kProfWords * sizeof(unsigned long long), st));
  }
  auto fold_timeout = [&]() -> int {
    k_fold_timeout<<<1, 256, 0, st>>>(m->errw, status, n_chains);
    TS_CUDA(cudaGetLastError());
    return TS_OK;
  };
  if (m->kind != TS_LOGISTIC || m->many) {
    A.prof = prof ? prof_buf : nullptr;
    int e = launch(m, nslots, A, n_chains, (ts_exec_mode)exec_mode, st);
    if (!e) e = fold_timeout();
    if (e || !prof) {
      if (prof_buf) cudaFreeAsync(prof_buf, st);
      return e;
    }
  } else {
    if (prof) const_cast<ts_model*>(m)->prof = prof_buf;
    for (int c = 0; c < n_chains; ++c) {
      A.n_points = c;
      int e = launch(m, nslots, A, 1, TS_EXEC_BLOCK, st);
      if (e) {
        const_cast<ts_model*>(m)->prof = nullptr;
        if (prof_buf) cudaFreeAsync(prof_buf, st);
        return e;
      }
    }
    const int e = fold_timeout();
    if (e) return e;
  }
  {
    if (prof) {
      const_cast<ts_model*>(m)->prof = nullptr;
      static unsigned long long h[kProfWords];
      TS_CUDA(cudaMemcpyAsync(h, prof_buf, sizeof h, cudaMemcpyDeviceToHost, st));
      TS_CUDA(cudaStreamSynchronize(st));
      const double n = h[10] ? (double)h[10] : 1.0;
      fprintf(stderr,
              "TS_PROF evals=%llu wasted=%llu cycles/eval: post-to-result %.0f (pass %.0f [entry %.0f loop %.0f "
              "warpred %.0f ctared %.0f] barrier %.0f reduce %.0f) result-to-next-post %.0f\n",
              h[10], h[11], h[8] / n, h[1] / n, h[4] / n, h[5] / n, h[6] / n, h[7] / n, h[2] / n, h[3] / n, h[9] / n);
      const double nt = h[14] ? (double)h[14] : 1.0, nx = h[15] ? (double)h[15] : 1.0;
      fprintf(stderr, "TS_PROF transitions=%llu trees=%llu cycles: prologue/transition %.0f (momentum %.0f)  between-trees/tree %.0f\n",
              h[15], h[14], h[12] / nx, h[16] / nx, h[13] / nt);
      if (h[22] || h[19]) {
        const double nl = h[22] ? (double)h[22] : 1.0, nw = h[19] ? (double)h[19] : 1.0;
        fprintf(stderr, "TS_PROF trajectories: driver %llu leaves, wait %.0f + bookkeeping %.0f cycles/leaf; workers %llu leaves, "
                "gate wait %.0f + leaf work outside the pass %.0f cycles/leaf\n", h[22], h[20] / nl, h[21] / nl, h[19],
                h[17] / nw, h[18] / nw);
      }
      if (m->kind == TS_DENSE_GAUSS && h[27]) {
        const double nl = (double)h[27];
        fprintf(stderr, "TS_PROF dense chain 0: %llu fused leaves, cycles/leaf: gradient wait %.0f, fused pass %.0f, "
                "bookkeeping %.0f\n", h[27], h[24] / nl, (h[25] + h[28]) / nl, h[26] / nl);
        fprintf(stderr, "TS_PROF dense chain 0 pass split: vector loop %.0f, post (fences + flag) %.0f, sums %.0f\n",
                h[28] / nl, h[29] / nl, h[30] / nl);
      }
      if (m->kind == TS_LOGISTIC && m->many && h[24 + 8]) {
        const double nt = h[24 + 7] ? (double)h[24 + 7] : 1.0, nc = (double)h[24 + 8];
        fprintf(stderr, "TS_PROF many-chain: %llu chain tiles, %.1f row tiles each; cycles per row tile: X wait %.0f, "
                "GEMM2 wait %.0f, SIMT X pass %.0f, GEMM1 %.0f, epilogue1 %.0f, ll reduce %.0f; per chain tile: "
                "epilogue2+atomics %.0f\n", h[24 + 8], nt / nc, h[24] / nt, h[25] / nt, h[26] / nt, h[27] / nt,
                h[28] / nt, h[29] / nt, h[30] / nc);
      }
      if (m->kind == TS_LOGISTIC && !m->many && h[10]) {  // per-CTA pass / barrier-wait skew
        double pmin = 1e300, pmax = 0, psum = 0, wsum = 0;
        int nb = 0, slow = -1;
        for (int b = 0; b < 2048 && h[24 + 2 * b]; ++b, ++nb) {
          const double pp = (double)h[24 + 2 * b] / n, ww = (double)h[25 + 2 * b] / n;
          psum += pp; wsum += ww;
          if (pp < pmin) pmin = pp;
          if (pp > pmax) { pmax = pp; slow = b; }
        }
        if (nb) {
          fprintf(stderr, "TS_PROF per-CTA ns/pass over %d CTAs: pass mean %.0f min %.0f max %.0f (CTA %d), barrier wait mean %.0f\n",
                  nb, psum / nb, pmin, pmax, slow, wsum / nb);
          fprintf(stderr, "TS_PROF pass ns by CTA:");
          for (int b = 0; b < nb; ++b) fprintf(stderr, " %.0f", (double)h[24 + 2 * b] / n);
          fprintf(stderr, "\n");
        }
      }
      cudaFreeAsync(prof_buf, st);
    }
    return TS_OK;
  }
}

// ------------------------------------------------------------------ rng probe
// Device streams for parity tests: kind 0 = random() doubles, 1 = standard
// normals, 2 = fold(i) keys for i = 0..n-1 (hi, lo as raw bits in doubles).
__global__ void k_rng_probe(uint64_t hi, uint64_t lo, int kind, int n, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Stream s;
  s.init(Key{hi, lo});
  for (int i = 0; i < n; ++i) {
    if (kind == 0) out[i] = s.next_double();
    else if (kind == 1) out[i] = s.normal();
    else {
      Key k = key_fold(Key{hi, lo}, (uint64_t)i);
      out[2 * i] = __longlong_as_double((long long)k.hi);
      out[2 * i + 1] = __longlong_as_double((long long)k.lo);
    }
  }
}

// glibc-exact exp / log1p and the correctly rounded log of the engine (ts_libm.cuh)
__global__ void k_libm_probe(int kind, const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = kind == 0 ? ts::lm_exp(x[i]) : (kind == 1 ? ts::lm_log1p(x[i]) : ts::lm_log(x[i]));
}
extern "C" int ts_libm_probe(int kind, const double* x_dev, double* y_dev, int64_t n, void* stream) {
  if (!x_dev || !y_dev || n < 0 || kind < 0 || kind > 2) return set_err(TS_EINVAL, "bad libm probe arguments");
  if (n == 0) return TS_OK;
  k_libm_probe<<<592, 256, 0, (cudaStream_t)stream>>>(kind, x_dev, y_dev, n);
  TS_CUDA(cudaGetLastError());
  return TS_OK;
}

extern "C" int ts_rng_probe(uint64_t key_hi, uint64_t key_lo, int kind, int n, double* out_dev, void* stream) {
  if (!out_dev || n < 0 || kind < 0 || kind > 2) return set_err(TS_EINVAL, "bad rng probe arguments");
  k_rng_probe<<<1, 32, 0, (cudaStream_t)stream>>>(key_hi, key_lo, kind, n, out_dev);
  TS_CUDA(cudaGetLastError());
  return TS_OK;
}
