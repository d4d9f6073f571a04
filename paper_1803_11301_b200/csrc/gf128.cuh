// gf128.cuh -- GF(2^128) arithmetic for sm_100a (no carry-less multiply instruction on the GPU).
//
// Field: x^128 + x^7 + x^2 + x + 1 (reference proj/include/fpmul/gf.hpp:115-123), element layout
// uint4 {x,y,z,w} = 32-bit limbs, bit k of the element is bit (k%32) of limb k/32 -- byte-identical
// to the reference u128 {lo, hi} (gf.hpp:24-52) so device EvalVecs are reference EvalVecs.
//
// Multipliers, chosen per call site by measurement (profiles/):
//  * gf_mul():      generic a*b.  Karatsuba 128 -> 3x64 -> 9x32; each 32x32 carry-less product is
//                   16 IMAD.WIDE.U32 on "holed" operands (every 4th bit), whose digit sums stay < 16 so
//                   bit 4k+r of the integer product is the GF(2) coefficient; XOR-combine, mask.
//                   IMAD runs on the FMA pipe, the masks/XORs on the ALU pipe (~7-8 clk/mul/SM).
//  * M8 tables:     w*x for a twiddle w shared by a whole butterfly block: 16 byte-chunk tables of
//                   w*(v << 8c) in a lane-rotated layout (16 conflict-free LDS.128 per product).
//  * M4 tables:     8 twiddles at a time for blocks of 64..128 butterflies (32 lookups, 8 KiB each).
//  These replace PCLMULQDQ (reference gf_pclmul.cpp:25-30).
#pragma once
#include <cstdint>

namespace fpm {

__device__ __forceinline__ uint4 x4(uint4 a, uint4 b) { return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w); }
__device__ __forceinline__ uint4 xor3(uint4 a, uint4 b, uint4 c) {
  return make_uint4(a.x ^ b.x ^ c.x, a.y ^ b.y ^ c.y, a.z ^ b.z ^ c.z, a.w ^ b.w ^ c.w);
}
__device__ __forceinline__ bool is_zero(uint4 a) { return (a.x | a.y | a.z | a.w) == 0; }

// 32x32 -> 64 carry-less product via integer multiply with 4-bit holes.
__device__ __forceinline__ uint64_t clmul32(uint32_t a, uint32_t b) {
  const uint32_t m = 0x11111111u;
  const uint32_t a0 = a & m, a1 = a & (m << 1), a2 = a & (m << 2), a3 = a & (m << 3);
  const uint32_t b0 = b & m, b1 = b & (m << 1), b2 = b & (m << 2), b3 = b & (m << 3);
  const uint64_t r0 = (uint64_t)a0 * b0 ^ (uint64_t)a1 * b3 ^ (uint64_t)a2 * b2 ^ (uint64_t)a3 * b1;
  const uint64_t r1 = (uint64_t)a0 * b1 ^ (uint64_t)a1 * b0 ^ (uint64_t)a2 * b3 ^ (uint64_t)a3 * b2;
  const uint64_t r2 = (uint64_t)a0 * b2 ^ (uint64_t)a1 * b1 ^ (uint64_t)a2 * b0 ^ (uint64_t)a3 * b3;
  const uint64_t r3 = (uint64_t)a0 * b3 ^ (uint64_t)a1 * b2 ^ (uint64_t)a2 * b1 ^ (uint64_t)a3 * b0;
  const uint64_t M = 0x1111111111111111ull;
  return (r0 & M) | (r1 & (M << 1)) | (r2 & (M << 2)) | (r3 & (M << 3));
}

__device__ __forceinline__ void clmul64(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
  const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  const uint64_t p0 = clmul32(a0, b0), p2 = clmul32(a1, b1);
  const uint64_t p1 = clmul32(a0 ^ a1, b0 ^ b1) ^ p0 ^ p2;
  lo = p0 ^ (p1 << 32);
  hi = p2 ^ (p1 >> 32);
}

// Fold a 256-bit product r0..r3 (64-bit words) modulo x^128 + x^7 + x^2 + x + 1
// (the two-step fold of kernels.hpp:51-55 restated on 64-bit halves).
__device__ __forceinline__ uint4 gf_reduce(uint64_t r0, uint64_t r1, uint64_t r2, uint64_t r3) {
  const uint64_t o = (r3 >> 63) ^ (r3 >> 62) ^ (r3 >> 57);
  r2 ^= o;
  r1 ^= r3 ^ (r3 << 1) ^ (r3 << 2) ^ (r3 << 7);
  r0 ^= r2 ^ (r2 << 1) ^ (r2 << 2) ^ (r2 << 7);
  r1 ^= (r2 >> 63) ^ (r2 >> 62) ^ (r2 >> 57);
  return make_uint4((uint32_t)r0, (uint32_t)(r0 >> 32), (uint32_t)r1, (uint32_t)(r1 >> 32));
}

__device__ __forceinline__ uint4 gf_mul(uint4 a, uint4 b) {
  const uint64_t al = a.x | ((uint64_t)a.y << 32), ah = a.z | ((uint64_t)a.w << 32);
  const uint64_t bl = b.x | ((uint64_t)b.y << 32), bh = b.z | ((uint64_t)b.w << 32);
  uint64_t c0l, c0h, c2l, c2h, c1l, c1h;
  clmul64(al, bl, c0l, c0h);
  clmul64(ah, bh, c2l, c2h);
  clmul64(al ^ ah, bl ^ bh, c1l, c1h);
  c1l ^= c0l ^ c2l;
  c1h ^= c0h ^ c2h;
  return gf_reduce(c0l, c0h ^ c1l, c2l ^ c1h, c2h);
}

// ---------------------------------------------------------------- prepared-operand multiply
// gf_mul(w, x) splits both operands into the 9 Karatsuba 32-bit limbs and masks each limb four
// ways (4-bit holes).  When one twiddle w multiplies many x, its 9 x 4 masked limbs are computed
// once (GfPrep, 144 B) and the product costs only x's side: ~14% fewer ALU ops.
struct GfPrep {
  uint4 m[9];  // limb k (al.lo, al.hi, al.lo^hi, ah.lo, ..., (al^ah).lo^hi): {& M, & M<<1, & M<<2, & M<<3}
};
__device__ __forceinline__ uint4 mask4(uint32_t a) {
  const uint32_t m = 0x11111111u;
  return make_uint4(a & m, a & (m << 1), a & (m << 2), a & (m << 3));
}
__device__ __forceinline__ GfPrep gf_prep(uint4 w) {
  GfPrep p;
  const uint32_t l0 = w.x, l1 = w.y, h0 = w.z, h1 = w.w;
  const uint32_t s0 = l0 ^ h0, s1 = l1 ^ h1;
  p.m[0] = mask4(l0); p.m[1] = mask4(l1); p.m[2] = mask4(l0 ^ l1);
  p.m[3] = mask4(h0); p.m[4] = mask4(h1); p.m[5] = mask4(h0 ^ h1);
  p.m[6] = mask4(s0); p.m[7] = mask4(s1); p.m[8] = mask4(s0 ^ s1);
  return p;
}
__device__ __forceinline__ uint64_t clmul32_p(uint4 a, uint32_t b) {  // a = mask4(limb)
  const uint32_t m = 0x11111111u;
  const uint32_t b0 = b & m, b1 = b & (m << 1), b2 = b & (m << 2), b3 = b & (m << 3);
  const uint64_t r0 = (uint64_t)a.x * b0 ^ (uint64_t)a.y * b3 ^ (uint64_t)a.z * b2 ^ (uint64_t)a.w * b1;
  const uint64_t r1 = (uint64_t)a.x * b1 ^ (uint64_t)a.y * b0 ^ (uint64_t)a.z * b3 ^ (uint64_t)a.w * b2;
  const uint64_t r2 = (uint64_t)a.x * b2 ^ (uint64_t)a.y * b1 ^ (uint64_t)a.z * b0 ^ (uint64_t)a.w * b3;
  const uint64_t r3 = (uint64_t)a.x * b3 ^ (uint64_t)a.y * b2 ^ (uint64_t)a.z * b1 ^ (uint64_t)a.w * b0;
  const uint64_t M = 0x1111111111111111ull;
  return (r0 & M) | (r1 & (M << 1)) | (r2 & (M << 2)) | (r3 & (M << 3));
}
__device__ __forceinline__ void clmul64_p(uint4 a0, uint4 a1, uint4 a01, uint64_t b, uint64_t& lo, uint64_t& hi) {
  const uint32_t b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  const uint64_t p0 = clmul32_p(a0, b0), p2 = clmul32_p(a1, b1);
  const uint64_t p1 = clmul32_p(a01, b0 ^ b1) ^ p0 ^ p2;
  lo = p0 ^ (p1 << 32);
  hi = p2 ^ (p1 >> 32);
}
// == gf_mul(w, x) for p = gf_prep(w)
__device__ __forceinline__ uint4 gf_mul_prep(const GfPrep& p, uint4 x) {
  const uint64_t bl = x.x | ((uint64_t)x.y << 32), bh = x.z | ((uint64_t)x.w << 32);
  uint64_t c0l, c0h, c2l, c2h, c1l, c1h;
  clmul64_p(p.m[0], p.m[1], p.m[2], bl, c0l, c0h);
  clmul64_p(p.m[3], p.m[4], p.m[5], bh, c2l, c2h);
  clmul64_p(p.m[6], p.m[7], p.m[8], bl ^ bh, c1l, c1h);
  c1l ^= c0l ^ c2l;
  c1h ^= c0h ^ c2h;
  return gf_reduce(c0l, c0h ^ c1l, c2l ^ c1h, c2h);
}

// w * x^k mod P for 0 <= k < 128 (shift then fold), used to build table rows.
__device__ __forceinline__ uint4 gf_mul_xk(uint4 w, unsigned k) {
  uint64_t lo = w.x | ((uint64_t)w.y << 32), hi = w.z | ((uint64_t)w.w << 32);
  uint64_t r0, r1, r2, r3;
  if (k == 0) { r0 = lo; r1 = hi; r2 = 0; r3 = 0; }
  else if (k < 64) { r0 = lo << k; r1 = (hi << k) | (lo >> (64 - k)); r2 = hi >> (64 - k); r3 = 0; }
  else if (k == 64) { r0 = 0; r1 = lo; r2 = hi; r3 = 0; }
  else { const unsigned s = k - 64; r0 = 0; r1 = lo << s; r2 = (hi << s) | (lo >> (64 - s)); r3 = hi >> (64 - s); }
  return gf_reduce(r0, r1, r2, r3);
}

// ---------------------------------------------------------------- rotated 8-bit (M8) tables
// 16 byte-chunk tables of w*(v << 8c), 256 entries each, 64 KiB total, no replication: entry
// (c, v) lives at uint4 index (c >> 3) * 2048 + v * 8 + (c & 7), i.e. in 16-byte bank group c & 7.
// Lane q (= lane & 7) of a quarter-warp visits chunks in the rotated order (k + q) & 7, so at
// every lookup the 8 lanes of a quarter-warp hit 8 distinct bank groups: conflict-free LDS.128,
// 16 lookups per product (2 clk/mul/SM of shared-memory bandwidth).
constexpr int kM8Uint4 = 4096;

// Build by threads tid < 256: thread (c = tid & 15, s = tid >> 4) writes entries v = 16s..16s+15
// of chunk c -- the high nibble s once from rows 8c+4..8c+7, the 16 low-nibble combinations
// incrementally in registers; stores are conflict-free (a quarter-warp covers 8 bank groups).
// rows_scratch: 144 uint4 of shared memory (row k padded to k + k/8).
// Expansion of 128 rows (rows_scratch[k + k/8] = image of basis vector k) into the 16 chunk tables.
__device__ __forceinline__ void m8_expand(uint4* __restrict__ tab, const uint4* __restrict__ rows_scratch, int tid) {
  if (tid < 256) {  // larger CTAs: the other threads only join the barriers
  const int c = tid & 15, s = tid >> 4;
  uint4 r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = rows_scratch[9 * c + j];
  uint4 t[16];
  t[0] = make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (s >> j & 1) t[0] = x4(t[0], r[4 + j]);
#pragma unroll
  for (int u = 1; u < 16; ++u) t[u] = x4(t[u & (u - 1)], r[(u & 1) ? 0 : (u & 2) ? 1 : (u & 4) ? 2 : 3]);
  uint4* dst = tab + (c >> 3) * 2048 + 16 * s * 8 + (c & 7);
#pragma unroll
  for (int u = 0; u < 16; ++u) dst[u * 8] = t[u];
  }
}

__device__ __forceinline__ void m8_build(uint4* __restrict__ tab, uint4* __restrict__ rows_scratch, uint4 w, int tid) {
  if (tid < 128) rows_scratch[tid + (tid >> 3)] = gf_mul_xk(w, (unsigned)tid);
  __syncthreads();
  m8_expand(tab, rows_scratch, tid);
  __syncthreads();
}

__device__ __forceinline__ uint4 m8_mul(const uint4* __restrict__ tab, uint4 x, int q) {
  uint4 acc0 = make_uint4(0, 0, 0, 0), acc1 = make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = (k + q) & 7;                         // low chunks 0..7 live in x.x, x.y
    const uint32_t sel = 0x4440u | (uint32_t)(c & 3);  // PRMT: byte (c&3) -> low byte, zeros above
    const uint32_t lo = __byte_perm(c < 4 ? x.x : x.y, 0, sel);
    const uint32_t hi = __byte_perm(c < 4 ? x.z : x.w, 0, sel);  // chunk 8 + c
    acc0 = x4(acc0, tab[lo * 8 + c]);
    acc1 = x4(acc1, tab[2048 + hi * 8 + c]);
  }
  return x4(acc0, acc1);
}


// m8_mul with the lane rotation applied to the operand once: the 64-bit halves are rotated right by
// 8q bits, so lookup k reads byte k at a constant position (one PRMT) of chunk (k + q) & 7, and the
// entry address is base[k] + 128 * byte with base[k] = tab + ((k + q) & 7) (one IMAD).
struct M8Base {
  uint32_t b[8];  // shared-memory byte addresses of tab + ((k + q) & 7)
};
__device__ __forceinline__ M8Base m8_base(const uint4* tab, int q) {
  M8Base m;
  const uint32_t t = (uint32_t)__cvta_generic_to_shared(tab);
#pragma unroll
  for (int k = 0; k < 8; ++k) m.b[k] = t + 16u * (uint32_t)((k + q) & 7);
  return m;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
// off: byte offset of another table laid out after the one mb was made for (folded into the LDS).
__device__ __forceinline__ uint4 m8_mul_r(const M8Base& mb, uint4 x, int q, uint32_t off = 0) {
  // rotate (x.y:x.x) and (x.w:x.z) right by 8q bits
  const bool sw = q & 4;
  const uint32_t s = 8u * (uint32_t)(q & 3);
  const uint32_t a0 = sw ? x.y : x.x, a1 = sw ? x.x : x.y, b0 = sw ? x.w : x.z, b1 = sw ? x.z : x.w;
  const uint32_t lo0 = __funnelshift_r(a0, a1, s), lo1 = __funnelshift_r(a1, a0, s);
  const uint32_t hi0 = __funnelshift_r(b0, b1, s), hi1 = __funnelshift_r(b1, b0, s);
  uint4 acc0 = make_uint4(0, 0, 0, 0), acc1 = make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t sel = 0x4440u | (uint32_t)(k & 3);
    const uint32_t lo = __byte_perm(k < 4 ? lo0 : lo1, 0, sel);
    const uint32_t hi = __byte_perm(k < 4 ? hi0 : hi1, 0, sel);
    acc0 = x4(acc0, lds128(mb.b[k] + 128u * lo + off));
    acc1 = x4(acc1, lds128(mb.b[k] + 128u * hi + 2048u * 16u + off));
  }
  return x4(acc0, acc1);
}

// ---------------------------------------------------------------- rotated 4-bit tables, 8 at a time
// For tile layers whose twiddles are shared by only 2^5..2^7 butterflies: 32 nibble-chunk tables of
// w*(v << 4c), 8 KiB per twiddle, entry (c, v) at uint4 index v*32 + c (16-byte bank group c & 7);
// lane q visits chunks (k + q) & 31, so a quarter-warp's LDS.128 never conflicts.  Building 8
// tables costs what one M8 table does (4096 stores), lookups are 32 per product.
constexpr int kM4TabUint4 = 512;

// 256 threads build tables t = 0..7; thread (table t = tid >> 5, chunk tid & 31) passes w = w_t.
__device__ __forceinline__ void m4s_build8(uint4* __restrict__ tab, uint4 w, int tid) {
  const int t = tid >> 5, c = tid & 31;
  uint4 r[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) r[j] = gf_mul_xk(w, (unsigned)(4 * c + j));
  uint4* dst = tab + t * kM4TabUint4 + c;
  uint4 acc = make_uint4(0, 0, 0, 0);
  dst[0] = acc;
#pragma unroll
  for (int v = 1; v < 16; ++v) {  // gray-code walk: one XOR per entry
    const int g = v ^ (v >> 1);  // Gray code: step v flips bit ctz(v)
    acc = x4(acc, r[(v & 1) ? 0 : (v & 2) ? 1 : (v & 4) ? 2 : 3]);
    dst[g * 32] = acc;
  }
}

__device__ __forceinline__ uint4 m4s_mul(const uint4* __restrict__ tab, uint4 x, int q) {
  uint4 acc0 = make_uint4(0, 0, 0, 0), acc1 = make_uint4(0, 0, 0, 0);
  auto word = [&](int c) { return c < 16 ? (c < 8 ? x.x : x.y) : (c < 24 ? x.z : x.w); };
#pragma unroll
  for (int k = 0; k < 32; k += 2) {
    const int c0 = (k + q) & 31, c1 = (k + 1 + q) & 31;
    const uint32_t n0 = (word(c0) >> (4 * (c0 & 7))) & 15u, n1 = (word(c1) >> (4 * (c1 & 7))) & 15u;
    acc0 = x4(acc0, tab[n0 * 32 + c0]);
    acc1 = x4(acc1, tab[n1 * 32 + c1]);
  }
  return x4(acc0, acc1);
}

}  // namespace fpm
