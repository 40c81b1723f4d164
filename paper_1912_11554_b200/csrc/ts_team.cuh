// Teams: the set of threads that jointly own one chain's D-vectors.
//
// A chain's vectors (position, momentum, gradient, prefix sums, the
// iterative builder's slot store R, ...) are distributed over the team:
// component d belongs to thread (d % SIZE) of the team.  Every thread keeps
// an identical replica of all scalar state (energies, log weights, counters,
// Philox streams), so control flow is replicated and only dot products and
// the model evaluation communicate.
//
//  * BlockTeam  - one CTA per chain replica; vectors in shared memory.
//                 Used for the data-parallel models (logistic regression),
//                 where a grid of CTAs evaluates one potential together.
//  * ThreadTeam - one thread per chain; vectors in a global workspace laid
//                 out component-major / chain-minor so a warp of chains
//                 touches consecutive addresses.  Used for many-chain runs
//                 of small models.
//
// Reductions: ThreadTeam sums left to right (the reference numba loop order,
// kernels.py:44-146), so small models are bitwise identical to the
// reference.  BlockTeam uses a fixed shuffle tree, deterministic but in a
// different order (ulp-level differences only).
#pragma once
#include <stdint.h>

namespace ts {

struct VecStore {
  double* base;    // element (id, d) at base + id*vstride + d*dstride
  int64_t vstride;
  int64_t dstride;
  double* slots = nullptr;  // optional second region for vector ids >= slot0
  int slot0 = 0;
  __device__ __forceinline__ double* v(int id) const {
    if (slots != nullptr && id >= slot0) return slots + (int64_t)(id - slot0) * vstride;
    return base + (int64_t)id * vstride;
  }
  __device__ __forceinline__ double& at(int id, int d) const { return v(id)[(int64_t)d * dstride]; }
};

struct ThreadTeam {
  // exp / log1p / log with glibc's results (ts_libm.cuh): the thread team
  // keeps the reference's operation order, so whole chains are bitwise the
  // reference's; the warp / CTA teams reduce in another order anyway and use
  // CUDA's functions (1 ulp, faster)
  static constexpr bool kExactMath = true;
  static constexpr bool kBlock = false;
  static constexpr bool kUnitStride = false;  // chains interleaved in global memory
  static constexpr bool kWarp = false;
  __device__ __forceinline__ int rank() const { return 0; }
  __device__ __forceinline__ int size() const { return 1; }
  __device__ __forceinline__ bool leader() const { return true; }
  __device__ __forceinline__ void sync() const {}
  __device__ __forceinline__ double sum(double x) const { return x; }
  __device__ __forceinline__ void sum2(double& a, double& b) const {}
};

// One warp owns the chain (driver warp of a persistent data-parallel CTA):
// reductions are shuffle trees to lane 0 plus a broadcast, so every lane
// holds the bitwise-identical value and no CTA barrier is involved.
struct WarpTeam {
  static constexpr bool kExactMath = false;
  static constexpr bool kBlock = false;
  static constexpr bool kUnitStride = true;  // vectors contiguous in shared memory
  static constexpr bool kWarp = true;
  __device__ __forceinline__ int rank() const { return threadIdx.x & 31; }
  __device__ __forceinline__ int size() const { return 32; }
  __device__ __forceinline__ bool leader() const { return (threadIdx.x & 31) == 0; }
  __device__ __forceinline__ void sync() const { __syncwarp(); }
  __device__ __forceinline__ double sum(double x) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = __dadd_rn(x, __shfl_down_sync(0xffffffffu, x, o));
    return __shfl_sync(0xffffffffu, x, 0);
  }
  __device__ __forceinline__ void sum2(double& a, double& b) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, o));
      b = __dadd_rn(b, __shfl_down_sync(0xffffffffu, b, o));
    }
    a = __shfl_sync(0xffffffffu, a, 0);
    b = __shfl_sync(0xffffffffu, b, 0);
  }
};

// Deterministic CTA-wide reduction.  `scratch` holds >= 2*32 doubles.
struct BlockTeam {
  static constexpr bool kExactMath = false;
  static constexpr bool kBlock = true;
  static constexpr bool kUnitStride = true;
  static constexpr bool kWarp = false;
  double* scratch;
  __device__ __forceinline__ int rank() const { return threadIdx.x; }
  __device__ __forceinline__ int size() const { return blockDim.x; }
  __device__ __forceinline__ bool leader() const { return threadIdx.x == 0; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }

  __device__ __forceinline__ static double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
  }
  __device__ double sum(double x) const {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    x = warp_sum(x);
    __syncthreads();  // previous users of scratch are done
    if (lane == 0) scratch[w] = x;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s = __dadd_rn(s, scratch[i]);
    return s;
  }
  __device__ void sum2(double& a, double& b) const {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    a = warp_sum(a);
    b = warp_sum(b);
    __syncthreads();
    if (lane == 0) { scratch[w] = a; scratch[32 + w] = b; }
    __syncthreads();
    double sa = 0.0, sb = 0.0;
    for (int i = 0; i < nw; ++i) { sa = __dadd_rn(sa, scratch[i]); sb = __dadd_rn(sb, scratch[32 + i]); }
    a = sa; b = sb;
  }
};

}  // namespace ts
