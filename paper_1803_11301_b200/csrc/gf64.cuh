// gf64.cuh -- GF(2^64) arithmetic for sm_100a (the reference's auto-field pipeline, m = 64).
//
// Field: x^64 + x^4 + x^3 + x + 1 (reference proj/include/fpmul/gf.hpp:105-113).  Element layout
// uint2 {x, y} = 32-bit limbs of the reference u64, so device EvalVec<gf64>s are byte-identical to
// the reference's std::vector<FieldElem<gf64>>.
//
//  * gf64_mul():  generic a*b, Karatsuba 64 -> 3 x 32-bit carry-less products (the IMAD-holes
//                 clmul32 of gf128.cuh) and a two-step fold.
//  * G8 tables:   w*x for a twiddle w shared by a butterfly block: 8 byte-chunk tables of
//                 w*(v << 8c), stored twice (32 KiB): entry (c, v) copy h at uint2 index
//                 v*16 + 8h + c.  Lane L reads copy h = (L >> 3) & 1 and visits chunks in the order
//                 (k + L) & 7, so the 16 lanes of a half-warp hit 16 distinct 8-byte bank pairs:
//                 8 conflict-free LDS.64 per product.
#pragma once
#include <cstdint>

#include "gf128.cuh"

namespace fpm {

__device__ __forceinline__ uint2 x2(uint2 a, uint2 b) { return make_uint2(a.x ^ b.x, a.y ^ b.y); }
__device__ __forceinline__ uint64_t as_u64(uint2 a) { return a.x | ((uint64_t)a.y << 32); }
__device__ __forceinline__ uint2 as_u2(uint64_t v) { return make_uint2((uint32_t)v, (uint32_t)(v >> 32)); }

// lo + x^64 hi modulo x^64 + x^4 + x^3 + x + 1: x^64 hi = hi (x^4 + x^3 + x + 1); the bits that
// spill past x^63 (from hi's top 4 bits) are folded once more (kernels.hpp gf64 fold, restated).
__device__ __forceinline__ uint64_t gf64_reduce(uint64_t lo, uint64_t hi) {
  hi ^= (hi >> 60) ^ (hi >> 61) ^ (hi >> 63);
  return lo ^ hi ^ (hi << 1) ^ (hi << 3) ^ (hi << 4);
}

__device__ __forceinline__ uint2 gf64_mul(uint2 a, uint2 b) {
  uint64_t lo, hi;
  clmul64(as_u64(a), as_u64(b), lo, hi);
  return as_u2(gf64_reduce(lo, hi));
}

// Prepared operand (cf. gf128.cuh GfPrep): the 3 Karatsuba limbs of w, each masked four ways.
struct Gf64Prep {
  uint4 m[3];
};
__device__ __forceinline__ Gf64Prep gf64_prep(uint2 w) {
  Gf64Prep p;
  p.m[0] = mask4(w.x);
  p.m[1] = mask4(w.y);
  p.m[2] = mask4(w.x ^ w.y);
  return p;
}
__device__ __forceinline__ uint2 gf64_mul_prep(const Gf64Prep& p, uint2 x) {
  uint64_t lo, hi;
  clmul64_p(p.m[0], p.m[1], p.m[2], as_u64(x), lo, hi);
  return as_u2(gf64_reduce(lo, hi));
}

// w * x^k mod P for 0 <= k < 64 (table rows).
__device__ __forceinline__ uint2 gf64_mul_xk(uint2 w, unsigned k) {
  const uint64_t v = as_u64(w);
  return as_u2(k == 0 ? v : gf64_reduce(v << k, v >> (64 - k)));
}

constexpr int kG8Uint2 = 4096;  // 8 chunks x 256 values x 2 copies
constexpr int kG8Rows = 72;     // 64 rows, row k at k + k/8 (conflict-free row reads)

// Build by exactly 256 threads (thread c = tid & 7, s = tid >> 3 writes v = 8s .. 8s+7 of chunk c);
// rows_scratch: kG8Rows uint2 of shared memory.  Ends with a barrier.
// Expansion of the 64 rows (rows_scratch[k + k/8]) into the table; exactly 256 threads.
__device__ __forceinline__ void g8_expand(uint2* __restrict__ tab, const uint2* __restrict__ rows_scratch, int tid) {
  const int c = tid & 7, s = tid >> 3;
  uint2 r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = rows_scratch[9 * c + j];
  uint2 t[8];
  t[0] = make_uint2(0, 0);
#pragma unroll
  for (int j = 0; j < 5; ++j)
    if (s >> j & 1) t[0] = x2(t[0], r[3 + j]);
#pragma unroll
  for (int u = 1; u < 8; ++u) t[u] = x2(t[u & (u - 1)], r[(u & 1) ? 0 : (u & 2) ? 1 : 2]);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    uint2* e = tab + (8 * s + u) * 16 + c;
    e[0] = t[u];
    e[8] = t[u];
  }
}

__device__ __forceinline__ void g8_build(uint2* __restrict__ tab, uint2* __restrict__ rows_scratch, uint2 w, int tid) {
  if (tid < 64) rows_scratch[tid + (tid >> 3)] = gf64_mul_xk(w, (unsigned)tid);
  __syncthreads();
  g8_expand(tab, rows_scratch, tid);
  __syncthreads();
}

// x * w from the G8 table; lane = threadIdx.x & 31.
__device__ __forceinline__ uint2 g8_mul(const uint2* __restrict__ tab, uint2 x, int lane) {
  const int q = lane & 7, h8 = lane & 8;
  uint2 acc0 = make_uint2(0, 0), acc1 = make_uint2(0, 0);
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const int c0 = (k + q) & 7, c1 = (k + 1 + q) & 7;
    const uint32_t b0 = __byte_perm(c0 < 4 ? x.x : x.y, 0, 0x4440u | (uint32_t)(c0 & 3));
    const uint32_t b1 = __byte_perm(c1 < 4 ? x.x : x.y, 0, 0x4440u | (uint32_t)(c1 & 3));
    acc0 = x2(acc0, tab[b0 * 16 + h8 + c0]);
    acc1 = x2(acc1, tab[b1 * 16 + h8 + c1]);
  }
  return x2(acc0, acc1);
}

// g8_mul with the lane rotation applied to the operand once (cf. gf128.cuh m8_mul_r): x rotated
// right by 8q bits puts chunk (k + q) & 7 at byte k, so each lookup is one PRMT (constant selector)
// and one IMAD on a per-lane base address.
struct G8Base {
  uint32_t b[8];  // shared-memory byte address of entry (0, chunk (k + q) & 7, copy h)
};
__device__ __forceinline__ G8Base g8_base(const uint2* tab, int lane) {
  G8Base g;
  const uint32_t t = (uint32_t)__cvta_generic_to_shared(tab) + 8u * (uint32_t)(lane & 8);
#pragma unroll
  for (int k = 0; k < 8; ++k) g.b[k] = t + 8u * (uint32_t)((k + lane) & 7);
  return g;
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint2 g8_mul_r(const G8Base& gb, uint2 x, int lane, uint32_t off = 0) {
  const int q = lane & 7;
  const bool sw = q & 4;
  const uint32_t s = 8u * (uint32_t)(q & 3);
  const uint32_t a0 = sw ? x.y : x.x, a1 = sw ? x.x : x.y;
  const uint32_t r0 = __funnelshift_r(a0, a1, s), r1 = __funnelshift_r(a1, a0, s);
  uint2 acc0 = make_uint2(0, 0), acc1 = make_uint2(0, 0);
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const uint32_t b0 = __byte_perm(k < 4 ? r0 : r1, 0, 0x4440u | (uint32_t)(k & 3));
    const uint32_t b1 = __byte_perm(k < 4 ? r0 : r1, 0, 0x4440u | (uint32_t)((k + 1) & 3));
    acc0 = x2(acc0, lds64(gb.b[k] + 128u * b0 + off));
    acc1 = x2(acc1, lds64(gb.b[k + 1] + 128u * b1 + off));
  }
  return x2(acc0, acc1);
}

// ---------------------------------------------------------------- 4-bit tables, 16 at a time
// For tile layers whose twiddles are shared by only 2^4..2^7 butterflies: 16 nibble-chunk tables of
// w*(v << 4c), 2 KiB per twiddle, entry (c, v) at uint2 index v*16 + c (8-byte slot c of a 128-byte
// row); lane L visits chunks (k + L) & 15, so the 16 lanes of a half-warp hit 16 distinct slots:
// 16 conflict-free LDS.64 per product.
constexpr int kG4TabUint2 = 256;

// 256 threads build tables t = 0..15 (thread: table tid >> 4, chunk tid & 15; it passes w = w_t).
__device__ __forceinline__ void g4_build16(uint2* __restrict__ tab, uint2 w, int tid) {
  const int t = tid >> 4, c = tid & 15;
  uint2 r[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) r[j] = gf64_mul_xk(w, (unsigned)(4 * c + j));
  uint2* dst = tab + t * kG4TabUint2 + c;
  uint2 acc = make_uint2(0, 0);
  dst[0] = acc;
#pragma unroll
  for (int v = 1; v < 16; ++v) {  // gray-code walk
    const int g = v ^ (v >> 1);  // Gray code: step v flips bit ctz(v)
    acc = x2(acc, r[(v & 1) ? 0 : (v & 2) ? 1 : (v & 4) ? 2 : 3]);
    dst[g * 16] = acc;
  }
}

__device__ __forceinline__ uint2 g4_mul(const uint2* __restrict__ tab, uint2 x, int lane) {
  uint2 acc0 = make_uint2(0, 0), acc1 = make_uint2(0, 0);
#pragma unroll
  for (int k = 0; k < 16; k += 2) {
    const int c0 = (k + lane) & 15, c1 = (k + 1 + lane) & 15;
    const uint32_t n0 = ((c0 < 8 ? x.x : x.y) >> (4 * (c0 & 7))) & 15u;
    const uint32_t n1 = ((c1 < 8 ? x.x : x.y) >> (4 * (c1 & 7))) & 15u;
    acc0 = x2(acc0, tab[n0 * 16 + c0]);
    acc1 = x2(acc1, tab[n1 * 16 + c1]);
  }
  return x2(acc0, acc1);
}

}  // namespace fpm
