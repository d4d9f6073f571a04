// warp_bits.cuh -- warp-level bit-matrix helpers shared by the codec and the batch kernels.
#pragma once
#include <cstdint>

namespace fpm {

// 32x32 bit transpose across a warp: on entry lane r holds row r (bit c = M[r][c]); on exit lane c
// holds column c (bit r = M[r][c]).  Five exchange steps with the lane at distance s = 16..1: the
// byte-granular steps are one PRMT with a lane-dependent selector, the bit steps one rotate (left
// by s in the lower lane, right in the upper) and one masked merge (LOP3) -- 8 ALU ops + 5 SHFL.
struct Transpose32 {
  uint32_t sel16, sel8, amt[3], msk[3];
  __device__ explicit Transpose32(int lane) {
    sel16 = (lane & 16) ? 0x3276u : 0x5410u;
    sel8 = (lane & 8) ? 0x3715u : 0x6240u;
    const uint32_t m[3] = {0xF0F0F0F0u, 0xCCCCCCCCu, 0xAAAAAAAAu};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int sft = 4 >> k;
      const bool up = lane & sft;
      amt[k] = up ? 32 - sft : sft;
      msk[k] = up ? ~m[k] : m[k];
    }
  }
  __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
    x = __byte_perm(x, __shfl_xor_sync(0xFFFFFFFFu, x, 16), sel16);
    x = __byte_perm(x, __shfl_xor_sync(0xFFFFFFFFu, x, 8), sel8);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, 4 >> k);
      const uint32_t r = __funnelshift_l(y, y, amt[k]);
      x = (x & ~msk[k]) | (r & msk[k]);
    }
    return x;
  }
};

}  // namespace fpm
