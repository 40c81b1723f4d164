// Device counter-based randomness reproducing the reference's numpy streams.
//
// Reference: turnstile/rng.py:36-73 (RngKey over numpy Philox4x64-10).
//  * numpy's Philox pre-increments counter word 0 before each 4-word block
//    and hands the block out word by word;
//  * Generator.random()        = (u64 >> 11) * 2^-53           (tree.py:235-244, sampler.py:111,126)
//  * Generator.uniform(lo, hi) = lo + (hi - lo) * random()     (chains.py:107)
//  * Generator.standard_normal = numpy's 256-layer ziggurat    (sampler.py:95, adapt.py:186)
//  * RngKey.fold(i)  = first two words of Philox(key, ctr=(i, i>>64, 0, 3))  (rng.py:259-264)
//  * RngKey.generator() starts the stream at ctr=(0, 0, 0, 1)               (rng.py:266-276)
// Every thread of a team runs its own replica of a stream, so draws are
// identical across the team without any communication.
#pragma once
#include <stdint.h>
#include "ts_ziggurat_tables.h"

namespace ts {

struct Key {
  uint64_t hi, lo;
};

__device__ __forceinline__ void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t lo0 = M0 * c[0], hi0 = __umul64hi(M0, c[0]);
    uint64_t lo1 = M1 * c[2], hi1 = __umul64hi(M1, c[2]);
    uint64_t n0 = hi1 ^ c[1] ^ k0;
    uint64_t n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += W0; k1 += W1;
  }
}

// RngKey.fold(index): numpy receives counter (i, 0, 0, 3) and pre-increments.
__device__ __forceinline__ Key key_fold(Key k, uint64_t index) {
  uint64_t c[4] = {index + 1, (index + 1 == 0) ? 1ULL : 0ULL, 0, 3};
  philox4x64_10(c, k.hi, k.lo);
  return Key{c[0], c[1]};
}

// The draw stream of a key (RngKey.generator()).
struct Stream {
  uint64_t k0, k1;
  uint64_t c0, c1;  // words 2,3 of the counter stay (0, 1)
  uint64_t b0, b1, b2, b3;  // current block (scalars, not an array: stays in registers)
  int pos;

  __device__ __forceinline__ void init(Key k) {
    k0 = k.hi; k1 = k.lo; c0 = 0; c1 = 0; pos = 4;
    b0 = b1 = b2 = b3 = 0;
  }
  __device__ __forceinline__ uint64_t next_u64() {
    if (pos < 4) {
      const uint64_t v = pos == 1 ? b1 : (pos == 2 ? b2 : (pos == 3 ? b3 : b0));
      ++pos;
      return v;
    }
    c0 += 1;
    if (c0 == 0) c1 += 1;
    uint64_t c[4] = {c0, c1, 0, 1};
    philox4x64_10(c, k0, k1);
    b0 = c[0]; b1 = c[1]; b2 = c[2]; b3 = c[3];
    pos = 1;
    return b0;
  }
  __device__ __forceinline__ double next_double() {
    return (double)(next_u64() >> 11) * (1.0 / 9007199254740992.0);
  }
  // numpy random_standard_normal (ziggurat, 256 layers)
  __device__ double normal() {
    const double R = 3.6541528853610088;
    const double INV_R = 0.27366123732975828;
    for (;;) {
      uint64_t r = next_u64();
      int idx = (int)(r & 0xff);
      r >>= 8;
      int sign = (int)(r & 0x1);
      uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      double x = __dmul_rn((double)rabs, TS_ZIG_WI[idx]);
      if (sign) x = -x;
      if (rabs < TS_ZIG_KI[idx]) return x;
      if (idx == 0) {
        for (;;) {
          double xx = -INV_R * log1p(-next_double());
          double yy = -log1p(-next_double());
          if (yy + yy > xx * xx) return ((rabs >> 8) & 0x1) ? -(R + xx) : R + xx;
        }
      } else {
        if (__dadd_rn(__dmul_rn(__dsub_rn(TS_ZIG_FI[idx - 1], TS_ZIG_FI[idx]), next_double()),
                      TS_ZIG_FI[idx]) < exp(-0.5 * x * x))
          return x;
      }
    }
  }
};

// _DrawStream (tree.py:221-244) consumes the same values as scalar draws,
// so a plain Stream is the device equivalent.

}  // namespace ts
