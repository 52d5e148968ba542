// Philox4x64-10 counter-based RNG, bit-exact with the reference
// (rng.py:24-63, Random123 network; numpy.random.Philox emits the same words
// after its counter pre-increment, tests/test_rng.py:14-37).
//
// Key = (seed, stream_id), counter = (block, 0, 0, 0).  Draw k of a stream is
// word k&3 of block k>>2 (rng.py:1-13, 122-140).  In the filter loop the
// stream id is the particle *slot* j and block t feeds step t: word 0 = state
// innovation, 1 = sigma2 draw, 2 = tau2 draw, 3 = resampling uniform
// (filtering.py:221-224).
#pragma once
#include "common.cuh"

namespace pf {

struct Philox4 {
  uint64_t w[4];
};

PF_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
}

// Ten rounds with counter (c0,0,0,0); the zero words let the first round
// skip two multiplies' worth of inputs but the network is unchanged.
PF_HD Philox4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                            uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(M0, c0, hi0, lo0);
    mulhilo64(M1, c2, hi1, lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0;
    uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += W0;
    k1 += W1;
  }
  Philox4 o;
  o.w[0] = c0;
  o.w[1] = c1;
  o.w[2] = c2;
  o.w[3] = c3;
  return o;
}

PF_HD Philox4 philox_block(uint64_t seed, uint64_t stream, uint64_t block) {
  return philox4x64_10(block, 0, 0, 0, seed, stream);
}

// (w >> 12 + 0.5) * 2^-52, exactly (rng.py:113-119).  Built without an
// int->double conversion: 1 + k 2^-52 is exact, and subtracting (1 - 2^-53)
// is exact by Sterbenz, giving (2k+1) 2^-53.
PF_HD double unit_open(uint64_t w) {
  union { uint64_t u; double d; } c;
  c.u = 0x3FF0000000000000ull | (w >> 12);
  return c.d - 0x1.fffffffffffffp-1;  // 1 - 2^-53
}

}  // namespace pf
