// tower.cuh -- the product pipeline's internal tower representation R of GF(2^128) (fpm_tables.h
// TowerTables): 16 coordinates over the subfield GF(2^8) = span(v_0..v_7) of the Cantor basis,
// basis e_{8j+s} = x^j t^s, t^8 = t^4 + t^3 + t + 1.  Byte j of a uint4 is the coordinate of x^j.
//
// Why: a tile layer's twiddles are w(i, b) = Z ^ C2P(2b) with Z fixed per tile and, for b < 128,
// C2P(2b) in GF(2^8) (v_1..v_7 lie in the subfield).  w*u = Z*u ^ C2P(2b)*u: the first term is one M8
// table per tile layer (gf128.cuh layout; tables are GF(2)-linear maps, so any basis works), the
// second is a scalar product, which in R is 16 independent byte products -- bytewise xtime on
// packed words, ~170 ALU ops instead of the ~390-op Karatsuba gf_mul.  No reference counterpart:
// R never leaves the FFT (encode writes R through a transformed M8 table, decode reads it likewise).
#pragma once
#include <cstdint>

#include "gf128.cuh"
#include "gf64.cuh"

namespace fpm {

// t * y for four packed GF(2^8) coordinates (bytewise shift, reduce by 0x1B)
__device__ __forceinline__ uint32_t xt32(uint32_t y) {
  return ((y << 1) & 0xFEFEFEFEu) ^ (((y >> 7) & 0x01010101u) * 0x1Bu);
}
__device__ __forceinline__ uint4 xt(uint4 y) { return make_uint4(xt32(y.x), xt32(y.y), xt32(y.z), xt32(y.w)); }
__device__ __forceinline__ uint4 and4(uint4 a, uint32_t m) { return make_uint4(a.x & m, a.y & m, a.z & m, a.w & m); }

// u * d for a subfield scalar d (8-bit, t-basis), Horner from the top bit: 7 xtimes + 8 masked XORs.
__device__ __forceinline__ uint4 smul(uint4 u, uint32_t d) {
  uint4 acc = and4(u, 0u - ((d >> 7) & 1u));
#pragma unroll
  for (int s = 6; s >= 0; --s) acc = x4(xt(acc), and4(u, 0u - ((d >> s) & 1u)));
  return acc;
}

// u * d by byte permutes: "times d" is GF(2)-linear on each byte, so byte v maps to
// M(v & 7) ^ [v & 8] M(8) ^ M(v & 0x70) ^ [v & 0x80] M(0x80).  The eight products M(0..7) and
// M(0x00..0x70) sit in two register pairs, and one PRMT looks up four bytes at once: the selector
// nibbles are the low 3 bits of the four bytes (gathered in the order 0, 2, 1, 3 by u | u >> 12),
// the bit-3 terms come from PRMT sign replication.  ~16 instructions per 32-bit word instead of
// ~42 for the xtime chain.  SmulTab is the per-d table (8 words), built once per kernel for the
// 128 subfield twiddle parts d = R(C2P(2b)), b < 128.
struct SmulTab {
  uint32_t lo0, lo1;  // M(0..3), M(4..7)
  uint32_t hi0, hi1;  // M(0x00, 0x10, 0x20, 0x30), M(0x40, 0x50, 0x60, 0x70)
  uint32_t m8, m80;   // M(0x08), M(0x80), replicated to 4 bytes
};
// Shared-memory layout: the four table words of d at a[d] (16 B: eight consecutive d of a
// quarter-warp hit eight bank groups), the two sign-term words at b[d].
struct SmulTabs {
  uint4 a[128];
  uint2 b[128];
};
__device__ __forceinline__ SmulTab smul_tab(const SmulTabs& t, int d) {
  const uint4 a = t.a[d];
  const uint2 b = t.b[d];
  return SmulTab{a.x, a.y, a.z, a.w, b.x, b.y};
}
// PTX prmt in its default mode: a selector nibble with bit 3 set replicates the sign bit of the
// selected byte (__byte_perm ignores that bit, so this needs the instruction itself).
__device__ __forceinline__ uint32_t prmt_sign(uint32_t a, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(d) : "r"(a), "r"(sel));
  return d;
}
__device__ __forceinline__ uint32_t smul_w(uint32_t w, const SmulTab& t) {
  const uint32_t u = w & 0x07070707u, v = (w >> 4) & 0x07070707u;
  const uint32_t r = __byte_perm(t.lo0, t.lo1, u | (u >> 12)) ^ (prmt_sign(w << 4, 0xB9A8) & t.m8) ^
                     __byte_perm(t.hi0, t.hi1, v | (v >> 12)) ^ (prmt_sign(w, 0xB9A8) & t.m80);
  return __byte_perm(r, 0, 0x3120);  // bytes back from the (0, 2, 1, 3) order
}
__device__ __forceinline__ uint4 smul_t(uint4 u, const SmulTab& t) {
  return make_uint4(smul_w(u.x, t), smul_w(u.y, t), smul_w(u.z, t), smul_w(u.w, t));
}
__device__ __forceinline__ uint2 smul_t2(uint2 u, const SmulTab& t) { return make_uint2(smul_w(u.x, t), smul_w(u.y, t)); }
// SmulTabs of the powers t^s (t-basis byte 1 << s), s < 8: field constants of GF(2^8) mod 0x11B
// (independent of the embedding), so rows_r multiplies by t^s with one smul_t instead of s xtimes.
constexpr uint32_t gf8c(uint32_t a, uint32_t b) {
  uint32_t r = 0;
  for (int i = 0; i < 8; ++i) {
    if (b >> i & 1) r ^= a;
    a <<= 1;
    if (a & 0x100) a ^= 0x11B;
  }
  return r;
}
constexpr uint32_t gf8c4(uint32_t k0, uint32_t step, uint32_t d) {
  return gf8c(k0, d) | gf8c(k0 + step, d) << 8 | gf8c(k0 + 2 * step, d) << 16 | gf8c(k0 + 3 * step, d) << 24;
}
#define FPM_TPOW(s) {gf8c4(0, 1, 1u << s), gf8c4(4, 1, 1u << s), gf8c4(0, 16, 1u << s), gf8c4(64, 16, 1u << s)}, \
                    {gf8c(8, 1u << s) * 0x01010101u, gf8c(0x80, 1u << s) * 0x01010101u, 0u, 0u}
static __device__ const uint4 g_tpow[16] = {FPM_TPOW(0), FPM_TPOW(1), FPM_TPOW(2), FPM_TPOW(3),
                                            FPM_TPOW(4), FPM_TPOW(5), FPM_TPOW(6), FPM_TPOW(7)};
#undef FPM_TPOW
__device__ __forceinline__ SmulTab tpow_tab(int s) {
  const uint4 a = g_tpow[2 * s], b = g_tpow[2 * s + 1];
  return SmulTab{a.x, a.y, a.z, a.w, b.x, b.y};
}

// Rows of the M8 table of "multiply by w" (w in POLYNOMIAL representation) in R: row 8j+s =
// R(w x^j) * t^s.  Threads tid < 128 (four whole warps): thread (j, s) converts bits [16s, 16s+16)
// of w x^j with the to_r rows, the 8 partial sums of a j meet by shuffle-XOR, then times t^s.
// Writes rows[k + k/8] (m8 padding).  to_r: 128 rows, row k at index k + k/16 (TO_R_PAD) when
// staged in shared memory, so the 8 lanes (s = 0..7) of a quarter-warp read distinct bank groups.
__device__ __forceinline__ int to_r_pad(int k) { return k + (k >> 4); }
template <bool SMEM>
__device__ __forceinline__ void rows_r(uint4* __restrict__ rows, uint4 w, int tid, const uint4* __restrict__ to_r) {
  if (tid >= 128) return;
  const int j = tid >> 3, s = tid & 7;
  const uint4 p = gf_mul_xk(w, (unsigned)j);
  const uint32_t word = s < 2 ? p.x : s < 4 ? p.y : s < 6 ? p.z : p.w;
  const uint32_t bits = (word >> (16 * (s & 1))) & 0xFFFFu;
  uint4 acc = make_uint4(0, 0, 0, 0);
  const uint4* src = to_r + (SMEM ? to_r_pad(16 * s) : 16 * s);
#pragma unroll
  for (int b = 0; b < 16; ++b) acc = x4(acc, and4(SMEM ? src[b] : __ldg(src + b), 0u - ((bits >> b) & 1u)));
#pragma unroll
  for (int m = 1; m < 8; m <<= 1) {
    acc.x ^= __shfl_xor_sync(0xffffffffu, acc.x, m);
    acc.y ^= __shfl_xor_sync(0xffffffffu, acc.y, m);
    acc.z ^= __shfl_xor_sync(0xffffffffu, acc.z, m);
    acc.w ^= __shfl_xor_sync(0xffffffffu, acc.w, m);
  }
  rows[tid + (tid >> 3)] = smul_t(acc, tpow_tab(s));
}

// GF(2^64) (8 coordinates): rows of the G8 table of "multiply by w" (w polynomial) in R, row 8j+s =
// R(w x^j) * t^s, by threads tid < 64 (two whole warps): thread (j, s) converts bits [8s, 8s+8) of
// w x^j, shuffle-XOR over the 8 lanes of j, then s xtimes.  to_r: 64 rows at to_r64_pad(k)
// (the 8 lanes s = 0..7 read 8 distinct bank pairs).  Writes rows[k + k/8].
__device__ __forceinline__ int to_r64_pad(int k) { return k + (k >> 3); }
__device__ __forceinline__ void rows_r64(uint2* __restrict__ rows, uint2 w, int tid, const uint2* __restrict__ to_r) {
  if (tid >= 64) return;
  const int j = tid >> 3, s = tid & 7;
  const uint2 p = gf64_mul_xk(w, (unsigned)j);
  const uint32_t bits = ((s < 4 ? p.x : p.y) >> (8 * (s & 3))) & 0xFFu;
  uint2 acc = make_uint2(0, 0);
  const uint2* src = to_r + to_r64_pad(8 * s);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const uint32_t m = 0u - ((bits >> b) & 1u);
    acc.x ^= src[b].x & m;
    acc.y ^= src[b].y & m;
  }
#pragma unroll
  for (int m = 1; m < 8; m <<= 1) {
    acc.x ^= __shfl_xor_sync(0xffffffffu, acc.x, m);
    acc.y ^= __shfl_xor_sync(0xffffffffu, acc.y, m);
  }
  rows[tid + (tid >> 3)] = smul_t2(acc, tpow_tab(s));
}

// Rows of a constant linear map (to_r / to_poly) into the m8 row scratch.
__device__ __forceinline__ void rows_const(uint4* __restrict__ rows, const uint4* __restrict__ src, int tid) {
  if (tid < 128) rows[tid + (tid >> 3)] = __ldg(src + tid);
}

__device__ __forceinline__ uint32_t gf8_mul(uint32_t a, uint32_t b) {  // mod t^8 + t^4 + t^3 + t + 1
  uint32_t r = 0;
  for (int i = 0; i < 8; ++i) {
    if (b >> i & 1) r ^= a;
    a <<= 1;
    if (a & 0x100) a ^= 0x11B;
  }
  return r;
}
// Threads tid < 128 build the table of d = R(C2P(2 tid)) = sum over bits b of tid of tau byte b.
__device__ __forceinline__ void smul_tabs_build(SmulTabs& tabs, uint64_t tau, int tid) {
  if (tid < 128) {
    uint32_t d = 0;
#pragma unroll
    for (int b = 0; b < 7; ++b)
      if (tid >> b & 1) d ^= (uint32_t)(tau >> (8 * b)) & 0xFFu;
    SmulTab t;
    t.lo0 = t.lo1 = t.hi0 = t.hi1 = 0;
    for (int k = 0; k < 4; ++k) {
      t.lo0 |= gf8_mul(k, d) << (8 * k);
      t.lo1 |= gf8_mul(4 + k, d) << (8 * k);
      t.hi0 |= gf8_mul(k << 4, d) << (8 * k);
      t.hi1 |= gf8_mul((4 + k) << 4, d) << (8 * k);
    }
    t.m8 = gf8_mul(8, d) * 0x01010101u;
    t.m80 = gf8_mul(0x80, d) * 0x01010101u;
    tabs.a[tid] = make_uint4(t.lo0, t.lo1, t.hi0, t.hi1);
    tabs.b[tid] = make_uint2(t.m8, t.m80);
  }
}

}  // namespace fpm
