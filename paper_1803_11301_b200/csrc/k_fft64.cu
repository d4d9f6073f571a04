// k_fft64.cu -- LCH butterflies and pointwise products over GF(2^64) on sm_100a: the reference's
// auto-field pipeline (plan_mul picks m = 64 whenever the field supports the size, polymul.cpp:
// 203-205; run_pipeline<gf64>, polymul.cpp:78-135, 235).
//
// Same schedule as k_fft.cu (see there for the layer/twiddle algebra):
//     w(i, b) = C2P((base >> i) ^ 2b) = layer[i] ^ C2P(2b),  base = e_{l+32}  (butterfly.cpp:45-49)
// with 8-byte elements and 32 KiB G8 twiddle tables (gf64.cuh):
//  * fft64_top4_kernel: layers (i+1, i) per HBM round trip, three G8 tables per CTA.
//  * fft64_top_kernel:  one layer (odd top-layer count).
//  * fft64_tile_kernel / fft64_tile_fused_kernel: layers [0, T) in shared-memory tiles (generic
//    gf64_mul below layer 8, one G8 table at a time above); the fused one also does the pointwise
//    product with operand a and the inverse tile layers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "fpm_internal.h"
#include "gf64.cuh"
#include "tower.cuh"

namespace fpm {
namespace {

constexpr int kTileMax64 = 12;  // 2^12 x 8 B = 32 KiB tile

__device__ __forceinline__ uint2 c2p2_64(const uint2* __restrict__ c2p, uint64_t b) {  // C2P(2b)
  uint2 r = c2p[b & 511];
  if (b >> 9) r = x2(r, c2p[512 + ((b >> 9) & 511)]);
  if (b >> 18) r = x2(r, c2p[1024 + ((b >> 18) & 511)]);
  if (b >> 27) r = x2(r, c2p[1536 + ((b >> 27) & 511)]);
  return r;
}

__device__ __forceinline__ uint2 twiddle64(const TwiddleSrc64& tw, unsigned i, uint64_t b) {
  return x2(tw.layer[i], c2p2_64(tw.c2p, b));
}

// ------------------------------------------------------------------ one top layer
// R: elements in the tower representation (tower.cuh), the table built in R.
template <bool INV, bool R>
__global__ void __launch_bounds__(256) fft64_top_kernel(uint2* __restrict__ ev, unsigned i, int ppc, TwiddleSrc64 tw) {
  pdl_wait();
  extern __shared__ uint2 tab64[];  // kG8Uint2
  __shared__ uint2 rows[kG8Rows];
  __shared__ uint2 to_r[72];
  const uint64_t half = (uint64_t)1 << i;
  const uint64_t pair0 = (uint64_t)blockIdx.x * ppc;  // ppc <= 2^i: a CTA stays inside one block
  const uint64_t b = pair0 >> i;
  if (R) {
    if (threadIdx.x < 64) to_r[to_r64_pad(threadIdx.x)] = __ldg(tw.to_r + threadIdx.x);
    __syncthreads();
    rows_r64(rows, twiddle64(tw, i, b), threadIdx.x, to_r);
    __syncthreads();
    g8_expand(tab64, rows, threadIdx.x);
    __syncthreads();
  } else {
    g8_build(tab64, rows, twiddle64(tw, i, b), threadIdx.x);
  }
  const int lane = threadIdx.x & 31;
  uint2* base = ev + (b << (i + 1));
#pragma unroll 4
  for (int k = threadIdx.x; k < ppc; k += blockDim.x) {
    const uint64_t j = (pair0 & (half - 1)) + k;
    uint2 u0 = base[j], u1 = base[j + half];
    if (!INV) {
      u0 = x2(u0, g8_mul(tab64, u1, lane));
      u1 = x2(u1, u0);
    } else {
      u1 = x2(u1, u0);
      u0 = x2(u0, g8_mul(tab64, u1, lane));
    }
    base[j] = u0;
    base[j + half] = u1;
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ two top layers per pass
// 384 threads (three 128-thread table builders), two CTAs per SM: one CTA's table build overlaps
// the other's streaming.
constexpr int kTop4Threads64 = 384;
constexpr size_t kTop4Smem64 = (3 * (size_t)kG8Uint2 + 3 * kG8Rows + 72) * sizeof(uint2);  // + to_r (tower)

// ev2 (optional): the other operand at the same layers and twiddles (one set of tables for both).
template <bool INV, bool R>
__global__ void __launch_bounds__(kTop4Threads64, 2) fft64_top4_kernel(uint2* __restrict__ ev, unsigned i, int qpc,
                                                                       TwiddleSrc64 tw, uint2* __restrict__ ev2) {
  pdl_wait();
  extern __shared__ uint2 sm64[];
  uint2* t1 = sm64;                    // w(i+1, B); then w(i, 2B) at + kG8Uint2, w(i, 2B+1) at + 2 kG8Uint2
  uint2* rows = sm64 + 3 * kG8Uint2;   // 3 x kG8Rows
  uint2* to_r = rows + 3 * kG8Rows;    // tower: conversion rows, to_r64_pad layout
  const uint64_t h = (uint64_t)1 << i;
  const uint64_t quad0 = (uint64_t)blockIdx.x * qpc;  // qpc <= h
  const uint64_t B = quad0 >> i;
  const int tid = threadIdx.x, grp = tid >> 7, lt = tid & 127;
  // twiddle loads issued before the to_r staging barrier (one L2 round trip)
  const uint2 w = grp == 0 ? twiddle64(tw, i + 1, B) : twiddle64(tw, i, 2 * B + (grp - 1));
  if (R) {
    if (tid < 64) to_r[to_r64_pad(tid)] = __ldg(tw.to_r + tid);
    __syncthreads();
  }
  {
    uint2* tab = sm64 + grp * kG8Uint2;
    uint2* rs = rows + grp * kG8Rows;
    if (R) rows_r64(rs, w, lt, to_r);
    else if (lt < 64) rs[lt + (lt >> 3)] = gf64_mul_xk(w, (unsigned)lt);
    __syncthreads();
    const int c = lt & 7;
    uint2 r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = rs[9 * c + j];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int sv = (lt >> 3) + 16 * half;
      uint2 t[8];
      t[0] = make_uint2(0, 0);
#pragma unroll
      for (int j = 0; j < 5; ++j)
        if (sv >> j & 1) t[0] = x2(t[0], r[3 + j]);
#pragma unroll
      for (int u = 1; u < 8; ++u) t[u] = x2(t[u & (u - 1)], r[(u & 1) ? 0 : (u & 2) ? 1 : 2]);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        uint2* e = tab + (8 * sv + u) * 16 + c;
        e[0] = t[u];
        e[8] = t[u];
      }
    }
    __syncthreads();
  }
  const int lane = tid & 31;
  uint2* base = ev + (B << (i + 2));
  const uint64_t j0 = quad0 & (h - 1);
  // Each thread transforms two adjacent quads with 16-byte accesses (512 B per warp per quarter
  // stream: the eight streams of a CTA stay DRAM-page friendly).
  const G8Base gb = g8_base(t1, lane);
  constexpr uint32_t kA = kG8Uint2 * 8u, kB = 2u * kG8Uint2 * 8u;  // t0a, t0b after t1
  auto bfly = [&](uint2& a0, uint2& a1, uint2& a2, uint2& a3) {
    if (!INV) {
      a0 = x2(a0, g8_mul_r(gb, a2, lane));
      a1 = x2(a1, g8_mul_r(gb, a3, lane));
      a2 = x2(a2, a0);
      a3 = x2(a3, a1);
      a0 = x2(a0, g8_mul_r(gb, a1, lane, kA));
      a2 = x2(a2, g8_mul_r(gb, a3, lane, kB));
      a1 = x2(a1, a0);
      a3 = x2(a3, a2);
    } else {
      a1 = x2(a1, a0);
      a3 = x2(a3, a2);
      a0 = x2(a0, g8_mul_r(gb, a1, lane, kA));
      a2 = x2(a2, g8_mul_r(gb, a3, lane, kB));
      a2 = x2(a2, a0);
      a3 = x2(a3, a1);
      a0 = x2(a0, g8_mul_r(gb, a2, lane));
      a1 = x2(a1, g8_mul_r(gb, a3, lane));
    }
  };
  const int nq = ev2 ? 2 * qpc : qpc;
  const uint64_t off = (uint64_t)(base - ev) + j0;
#pragma unroll 1
  for (int k = 2 * tid; k < nq; k += 2 * kTop4Threads64) {
    uint4* p = reinterpret_cast<uint4*>((k < qpc ? ev + k : ev2 + (k - qpc)) + off);
    const uint64_t h2 = h / 2;
    uint4 v0 = p[0], v1 = p[h2], v2 = p[2 * h2], v3 = p[3 * h2];
    uint2 a0 = make_uint2(v0.x, v0.y), a1 = make_uint2(v1.x, v1.y), a2 = make_uint2(v2.x, v2.y),
          a3 = make_uint2(v3.x, v3.y);
    uint2 b0 = make_uint2(v0.z, v0.w), b1 = make_uint2(v1.z, v1.w), b2 = make_uint2(v2.z, v2.w),
          b3 = make_uint2(v3.z, v3.w);
    bfly(a0, a1, a2, a3);
    bfly(b0, b1, b2, b3);
    p[0] = make_uint4(a0.x, a0.y, b0.x, b0.y);
    p[h2] = make_uint4(a1.x, a1.y, b1.x, b1.y);
    p[2 * h2] = make_uint4(a2.x, a2.y, b2.x, b2.y);
    p[3 * h2] = make_uint4(a3.x, a3.y, b3.x, b3.y);
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ top layers, three per pass (tower)
// fft_top8_kernel (k_fft.cu) for GF(2^64): layers i+2, i+1, i per HBM round trip with the three G8
// tables of w(i+2, B), w(i+1, 2B), w(i, 4B); the sibling twiddles differ by subfield elements
// C2P(2m), m < 4, applied as byte-permute scalar products.
constexpr size_t kTop8Smem64 = kTop4Smem64 + sizeof(SmulTabs);
template <bool INV>
__global__ void __launch_bounds__(kTop4Threads64, 2) fft64_top8_kernel(uint2* __restrict__ ev, unsigned i, int opc,
                                                                       TwiddleSrc64 tw, uint2* __restrict__ ev2) {
  pdl_wait();
  extern __shared__ uint2 sm64[];
  uint2* rows = sm64 + 3 * kG8Uint2;   // 3 x kG8Rows
  uint2* to_r = rows + 3 * kG8Rows;    // conversion rows, to_r64_pad layout
  SmulTabs& stab = *reinterpret_cast<SmulTabs*>(reinterpret_cast<uint4*>(to_r + 72));
  const uint64_t h = (uint64_t)1 << i;
  const uint64_t oct0 = (uint64_t)blockIdx.x * opc;  // opc <= h
  const uint64_t B = oct0 >> i;
  const int tid = threadIdx.x, grp = tid >> 7, lt = tid & 127;
  const uint2 w = grp == 0 ? twiddle64(tw, i + 2, B) : grp == 1 ? twiddle64(tw, i + 1, 2 * B) : twiddle64(tw, i, 4 * B);
  smul_tabs_build(stab, tw.tau, tid);
  if (tid < 64) to_r[to_r64_pad(tid)] = __ldg(tw.to_r + tid);
  __syncthreads();
  {
    uint2* tab = sm64 + grp * kG8Uint2;
    uint2* rs = rows + grp * kG8Rows;
    rows_r64(rs, w, lt, to_r);
    __syncthreads();
    const int c = lt & 7;
    uint2 r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = rs[9 * c + j];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int sv = (lt >> 3) + 16 * half;
      uint2 t[8];
      t[0] = make_uint2(0, 0);
#pragma unroll
      for (int j = 0; j < 5; ++j)
        if (sv >> j & 1) t[0] = x2(t[0], r[3 + j]);
#pragma unroll
      for (int u = 1; u < 8; ++u) t[u] = x2(t[u & (u - 1)], r[(u & 1) ? 0 : (u & 2) ? 1 : 2]);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        uint2* e = tab + (8 * sv + u) * 16 + c;
        e[0] = t[u];
        e[8] = t[u];
      }
    }
    __syncthreads();
  }
  const int lane = tid & 31;
  const G8Base gb = g8_base(sm64, lane);
  constexpr uint32_t kT1 = kG8Uint2 * 8u, kT0 = 2u * kG8Uint2 * 8u;  // W1, W0 after W2
  auto mul = [&](uint2 u, uint32_t toff, int m) {
    uint2 r = g8_mul_r(gb, u, lane, toff);
    if (m) r = x2(r, smul_t2(u, smul_tab(stab, m)));
    return r;
  };
  auto oct = [&](uint2 (&a)[8]) {
    if (!INV) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[e] = x2(a[e], mul(a[e + 4], 0, 0));
        a[e + 4] = x2(a[e + 4], a[e]);
      }
#pragma unroll
      for (int hb = 0; hb < 2; ++hb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int u0 = 4 * hb + e, u1 = u0 + 2;
          a[u0] = x2(a[u0], mul(a[u1], kT1, hb));
          a[u1] = x2(a[u1], a[u0]);
        }
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        a[2 * m] = x2(a[2 * m], mul(a[2 * m + 1], kT0, m));
        a[2 * m + 1] = x2(a[2 * m + 1], a[2 * m]);
      }
    } else {
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        a[2 * m + 1] = x2(a[2 * m + 1], a[2 * m]);
        a[2 * m] = x2(a[2 * m], mul(a[2 * m + 1], kT0, m));
      }
#pragma unroll
      for (int hb = 0; hb < 2; ++hb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int u0 = 4 * hb + e, u1 = u0 + 2;
          a[u1] = x2(a[u1], a[u0]);
          a[u0] = x2(a[u0], mul(a[u1], kT1, hb));
        }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[e + 4] = x2(a[e + 4], a[e]);
        a[e] = x2(a[e], mul(a[e + 4], 0, 0));
      }
    }
  };
  const int no = ev2 ? 2 * opc : opc;
  const uint64_t off = (B << (i + 3)) + (oct0 & (h - 1));
#pragma unroll 1
  for (int k = tid; k < no; k += kTop4Threads64) {  // one octet per thread (8-byte accesses: no spills)
    uint2* p = (k < opc ? ev + k : ev2 + (k - opc)) + off;
    uint2 a[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] = p[e * h];
    oct(a);
#pragma unroll
    for (int e = 0; e < 8; ++e) p[e * h] = a[e];
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ tile layers (i < T)
#ifndef FPM_G8_LAYER
#define FPM_G8_LAYER 9
#endif
constexpr unsigned kTabLayer64 = FPM_G8_LAYER;  // layers >= 9: G8 tables (layer 8 on G4: 48.3 vs 49.0 ms)
// Layers [kG4Layer, kTabLayer64): 4-bit tables for up to 16 twiddles per round (gf64.cuh g4_*).
#ifndef FPM_G4_LAYER
#define FPM_G4_LAYER 6
#endif
constexpr unsigned kG4Layer = FPM_G4_LAYER;
#ifndef FPM_G8_LAYER2
#define FPM_G8_LAYER2 8
#endif
constexpr unsigned kTabLayer64_2 = FPM_G8_LAYER2;  // fft64_tile_fused2_kernel
// NT tiles sharing twiddles (both operands at one position) at s, s + 2^T (cf. k_fft.cu).
template <bool INV, int NT = 1, unsigned kTabLayer64 = kTabLayer64>
__device__ __forceinline__ void tile_layers64(uint2* __restrict__ s, unsigned T, uint64_t tile_idx,
                                              const TwiddleSrc64& tw, uint2* __restrict__ tab) {
  const int npairs = 1 << (T - 1), n = 1 << T;
  const int lane = threadIdx.x & 31;
  for (unsigned step = 0; step < T; ++step) {
    const unsigned i = INV ? step : T - 1 - step;
    const uint64_t bhi = tile_idx << (T - 1 - i);
    const uint2 Z = twiddle64(tw, i, bhi);  // w = Z ^ C2P(2 blk) (disjoint bit ranges, C2P linear)
    if (tab && i >= kG4Layer && i < kTabLayer64) {
      const int nblk = npairs >> i, G = nblk < 16 ? nblk : 16;
      const int gi = i + (G >= 16 ? 4 : G >= 8 ? 3 : G >= 4 ? 2 : G >= 2 ? 1 : 0);  // log2(G << i)
      for (int b0 = 0; b0 < nblk; b0 += G) {
        const uint2 w = x2(Z, c2p2_64(tw.c2p, (uint64_t)(b0 + (threadIdx.x >> 4))));
        __syncthreads();  // previous round's lookups done
        if (threadIdx.x < 16 * G) g4_build16(tab, w, threadIdx.x);
        __syncthreads();
        for (int pp = threadIdx.x; pp < (NT << gi); pp += blockDim.x) {
          const int p = NT == 1 ? pp : pp & ((1 << gi) - 1), tt = NT == 1 ? 0 : pp >> gi;
          const int t = p >> i, j = p & ((1 << i) - 1), blk = b0 + t;
          const int i0 = (blk << (i + 1)) + j + tt * n, i1 = i0 + (1 << i);
          const uint2* tb = tab + t * kG4TabUint2;
          uint2 u0 = s[i0], u1 = s[i1];
          if (!INV) {
            u0 = x2(u0, g4_mul(tb, u1, lane));
            u1 = x2(u1, u0);
          } else {
            u1 = x2(u1, u0);
            u0 = x2(u0, g4_mul(tb, u1, lane));
          }
          s[i0] = u0;
          s[i1] = u1;
        }
      }
      __syncthreads();
      continue;
    }
    if (tab && i >= kTabLayer64) {
      for (int blk = 0; blk < (npairs >> i); ++blk) {
        g8_build(tab, tab + kG8Uint2, x2(Z, c2p2_64(tw.c2p, (uint64_t)blk)), threadIdx.x);
        for (int jj = threadIdx.x; jj < (NT << i); jj += blockDim.x) {
          const int j = NT == 1 ? jj : jj & ((1 << i) - 1), tt = NT == 1 ? 0 : jj >> i;
          const int i0 = (blk << (i + 1)) + j + tt * n, i1 = i0 + (1 << i);
          uint2 u0 = s[i0], u1 = s[i1];
          if (!INV) {
            u0 = x2(u0, g8_mul(tab, u1, lane));
            u1 = x2(u1, u0);
          } else {
            u1 = x2(u1, u0);
            u0 = x2(u0, g8_mul(tab, u1, lane));
          }
          s[i0] = u0;
          s[i1] = u1;
        }
      }
      __syncthreads();
      continue;
    }
    if (tab && i >= 1 && (npairs >> i) * (int)sizeof(Gf64Prep) <= kG8Uint2 * (int)sizeof(uint2)) {
      // twiddle limbs prepared once per block in the idle table area (cf. k_fft.cu)
      Gf64Prep* prep = reinterpret_cast<Gf64Prep*>(tab);
      const int nblk = npairs >> i;
      for (int b = threadIdx.x; b < nblk; b += blockDim.x) prep[b] = gf64_prep(x2(Z, c2p2_64(tw.c2p, (uint64_t)b)));
      __syncthreads();
      for (int pp = threadIdx.x; pp < NT * npairs; pp += blockDim.x) {
        const int p = NT == 1 ? pp : pp & (npairs - 1), tt = NT == 1 ? 0 : pp >> (T - 1);
        const int blk = p >> i, j = p & ((1 << i) - 1);
        const int i0 = (blk << (i + 1)) + j + tt * n, i1 = i0 + (1 << i);
        const Gf64Prep w = prep[blk];
        uint2 u0 = s[i0], u1 = s[i1];
        if (!INV) {
          u0 = x2(u0, gf64_mul_prep(w, u1));
          u1 = x2(u1, u0);
        } else {
          u1 = x2(u1, u0);
          u0 = x2(u0, gf64_mul_prep(w, u1));
        }
        s[i0] = u0;
        s[i1] = u1;
      }
      __syncthreads();
      continue;
    }
    for (int pp = threadIdx.x; pp < NT * npairs; pp += blockDim.x) {
      const int p = NT == 1 ? pp : pp & (npairs - 1), tt = NT == 1 ? 0 : pp >> (T - 1);
      const int blk = p >> i, j = p & ((1 << i) - 1);
      const int i0 = (blk << (i + 1)) + j + tt * n, i1 = i0 + (1 << i);
      const uint2 w = x2(Z, c2p2_64(tw.c2p, (uint64_t)blk));
      uint2 u0 = s[i0], u1 = s[i1];
      if (!INV) {
        u0 = x2(u0, gf64_mul(w, u1));
        u1 = x2(u1, u0);
      } else {
        u1 = x2(u1, u0);
        u0 = x2(u0, gf64_mul(w, u1));
      }
      s[i0] = u0;
      s[i1] = u1;
    }
    __syncthreads();
  }
}

template <bool INV>
__global__ void __launch_bounds__(256, 3) fft64_tile_kernel(uint2* __restrict__ ev, unsigned l, unsigned T,
                                                         TwiddleSrc64 tw, int use_tab) {
  pdl_wait();
  extern __shared__ uint2 s64[];
  const int n = 1 << T;
  uint2* tab = use_tab ? s64 + n : nullptr;
  const uint64_t ntiles = ((uint64_t)1 << l) >> T;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    uint2* g = ev + (t << T);
    for (int k = threadIdx.x; k < n; k += blockDim.x) s64[k] = g[k];
    __syncthreads();
    tile_layers64<INV>(s64, T, t, tw, tab);
    for (int k = threadIdx.x; k < n; k += blockDim.x) g[k] = s64[k];
    __syncthreads();
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

__global__ void __launch_bounds__(256, 3) fft64_tile_fused_kernel(const uint2* __restrict__ ea, uint2* __restrict__ eb,
                                                               unsigned l, unsigned T, TwiddleSrc64 tw, int use_tab) {
  pdl_wait();
  extern __shared__ uint2 s64[];
  const int n = 1 << T;
  uint2* tab = use_tab ? s64 + n : nullptr;
  const uint64_t ntiles = ((uint64_t)1 << l) >> T;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    uint2* g = eb + (t << T);
    const uint2* ga = ea + (t << T);
    for (int k = threadIdx.x; k < n; k += blockDim.x) s64[k] = g[k];
    __syncthreads();
    tile_layers64<false>(s64, T, t, tw, tab);
    for (int k = threadIdx.x; k < n; k += blockDim.x) s64[k] = gf64_mul(ga[k], s64[k]);
    __syncthreads();
    tile_layers64<true>(s64, T, t, tw, tab);
    for (int k = threadIdx.x; k < n; k += blockDim.x) g[k] = s64[k];
    __syncthreads();
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// Both operands' tile layers in one CTA (shared tables / prepared twiddles), the pointwise product
// and the inverse tile layers (cf. k_fft.cu fft_tile_fused2_kernel).
__global__ void __launch_bounds__(256, 3) fft64_tile_fused2_kernel(const uint2* __restrict__ ea,
                                                                   uint2* __restrict__ eb, unsigned l, unsigned T,
                                                                   TwiddleSrc64 tw) {
  pdl_wait();
  extern __shared__ uint2 s64[];
  const int n = 1 << T;
  uint2* tab = s64 + 2 * n;
  const uint64_t ntiles = ((uint64_t)1 << l) >> T;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    uint2* g = eb + (t << T);
    const uint2* ga = ea + (t << T);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      s64[k] = ga[k];
      s64[n + k] = g[k];
    }
    __syncthreads();
    tile_layers64<false, 2, kTabLayer64_2>(s64, T, t, tw, tab);
    for (int k = threadIdx.x; k < n; k += blockDim.x) s64[k] = gf64_mul(s64[k], s64[n + k]);
    __syncthreads();
    tile_layers64<true, 1, kTabLayer64_2>(s64, T, t, tw, tab);
    for (int k = threadIdx.x; k < n; k += blockDim.x) g[k] = s64[k];
    __syncthreads();
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ tower-representation tiles
// fft64_tile_fused2_kernel on tiles in the GF(2^64) tower representation (tower.cuh; the algebra
// is k_fft.cu's fft_tile_tower_kernel): tile layers [P, T) as one G8 table per 128 blocks plus a
// GF(2^8)-scalar product by byte permutes, layers [0, P), the pointwise product and the inverse
// layers [0, P) in polynomial representation (gf64_mul), conversions by G8 tables of to_poly/to_r.
__host__ __device__ constexpr int tower64_groups(unsigned T, unsigned i) {
  return (1 << (T - 1 - i)) > 128 ? (1 << (T - 1 - i)) >> 7 : 1;
}
__host__ __device__ constexpr int tower64_tables(unsigned T) {
  int n = 0;
  for (unsigned i = 0; i < T; ++i) n += tower64_groups(T, i);
  return n;
}
__device__ __forceinline__ int tower64_wz_index(unsigned T, unsigned i, int g) {
  int k = 0;
  for (unsigned u = 0; u < i; ++u) k += tower64_groups(T, u);
  return k + g;
}
constexpr int kTower64MaxTables = tower64_tables(12);
struct TowerSmem64 {  // after the 2^(T+1) tile elements
  uint2 tab[kG8Uint2];
  uint2 rows[2][kG8Rows];
  uint2 to_r[72];              // rows_r64 conversion source, to_r64_pad layout
  uint2 rows_to_r[kG8Rows];    // g8 rows of poly -> R
  uint2 rows_to_poly[kG8Rows]; // g8 rows of R -> poly
  uint2 wz[kTower64MaxTables]; // table twiddles of the current tile (layer-ascending, groups ascending)
  SmulTabs stab;
};
// Tile element k at k ^ 15 [bit 4 of k]: a half-warp's 8-byte accesses at layers 0-3 reach 16
// distinct bank pairs.
__device__ __forceinline__ int tsw64(int k) { return k ^ (((k >> 4) & 1) * 15); }

template <bool INV, int NT>
__device__ __forceinline__ void tile_layers_r64(uint2* __restrict__ s, unsigned T, unsigned P, TowerSmem64& sm) {
  const int npairs = 1 << (T - 1), n = 1 << T, tid = threadIdx.x, lane = tid & 31;
  const int first = tower64_wz_index(T, P, 0), ntab = tower64_tables(T) - first;
  auto wz_of = [&](int k) -> int {
    if (INV) return first + k;
    int kk = 0;
    for (int i = (int)T - 1; i >= (int)P; --i) {
      const int g = tower64_groups(T, (unsigned)i);
      if (k < kk + g) return tower64_wz_index(T, (unsigned)i, k - kk);
      kk += g;
    }
    return 0;
  };
  rows_r64(sm.rows[0], sm.wz[wz_of(0)], tid, sm.to_r);
  __syncthreads();
  g8_expand(sm.tab, sm.rows[0], tid);
  __syncthreads();
  int k = 0;
  for (unsigned step = 0; step < T - P; ++step) {
    const unsigned i = INV ? P + step : T - 1 - step;
    const int nblk = npairs >> i;
    const int lg = (nblk < 128 ? T - 1 : 7 + i);
    for (int h = 0; h < nblk; h += 128, ++k) {
      if (k + 1 < ntab) rows_r64(sm.rows[(k + 1) & 1], sm.wz[wz_of(k + 1)], tid, sm.to_r);
      const G8Base gb = g8_base(sm.tab, lane);
      // pair indices as in tile_layers_r (k_fft.cu): i0 = p + (p & ~(2^i - 1)) + the group's base
      // (+ the operand's tile); the stride (256) keeps the low bits the swizzle looks at fixed
      const int mlg = (1 << lg) - 1, nmi = ~((1 << i) - 1), hb = h << (i + 1);
      const int pf = tid & mlg, i0f = hb + pf + (pf & nmi);
      const int sw0 = ((i0f >> 4) & 1) * 15, sw1 = (((i0f + (1 << i)) >> 4) & 1) * 15;
      for (int pp = tid; pp < (NT << lg); pp += blockDim.x) {
        const int p = pp & mlg;
        const int i0 = hb + p + (p & nmi) + (NT == 1 ? 0 : (pp >> lg) * n), i1 = i0 + (1 << i);
        const int d = (h + (p >> i)) & 127;
        const int x0 = i0 ^ sw0, x1 = i1 ^ sw1;
        uint2 u0 = s[x0], u1 = s[x1];
        if (!INV) {
          uint2 m = g8_mul_r(gb, u1, lane);
          if (d) m = x2(m, smul_t2(u1, smul_tab(sm.stab, d)));
          u0 = x2(u0, m);
          u1 = x2(u1, u0);
        } else {
          u1 = x2(u1, u0);
          uint2 m = g8_mul_r(gb, u1, lane);
          if (d) m = x2(m, smul_t2(u1, smul_tab(sm.stab, d)));
          u0 = x2(u0, m);
        }
        s[x0] = u0;
        s[x1] = u1;
      }
      __syncthreads();
      if (k + 1 < ntab) {
        g8_expand(sm.tab, sm.rows[(k + 1) & 1], tid);
        __syncthreads();
      }
    }
  }
}

template <bool INV>
__device__ __forceinline__ void tile_layers_poly64(uint2* __restrict__ s, unsigned T, unsigned P, uint64_t t,
                                                   const TwiddleSrc64& tw) {
  const int npairs = 1 << (T - 1), n = 1 << T;
  for (unsigned step = 0; step < P; ++step) {
    const unsigned i = INV ? step : P - 1 - step;
    const uint2 Z = twiddle64(tw, i, t << (T - 1 - i));
    for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
      const int blk = p >> i, j = p & ((1 << i) - 1);
      const int i0 = tsw64((blk << (i + 1)) + j), i1 = tsw64((blk << (i + 1)) + j + (1 << i));
      const uint2 w = x2(Z, c2p2_64(tw.c2p, (uint64_t)blk));
      if (!INV) {
        const Gf64Prep wp = gf64_prep(w);
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          uint2 u0 = s[i0 + tt * n], u1 = s[i1 + tt * n];
          u0 = x2(u0, gf64_mul_prep(wp, u1));
          u1 = x2(u1, u0);
          s[i0 + tt * n] = u0;
          s[i1 + tt * n] = u1;
        }
      } else {
        uint2 u0 = s[i0], u1 = s[i1];
        u1 = x2(u1, u0);
        u0 = x2(u0, gf64_mul(w, u1));
        s[i0] = u0;
        s[i1] = u1;
      }
    }
    __syncthreads();
  }
}

#ifndef FPM_TOWER64_POLY
#define FPM_TOWER64_POLY 2  // P = 1: 46.0 ms, 2: 45.34, 3: 45.39, 4: 45.86 (2^32-bit product)
#endif
constexpr unsigned kPolyLayers64 = FPM_TOWER64_POLY;
size_t tower64_smem(unsigned T) { return 2 * ((size_t)1 << T) * sizeof(uint2) + sizeof(TowerSmem64); }

// MODE as fft_tile_tower_kernel (k_fft.cu): 0 = the fused pass over tiles [tile0, ntiles); 2 = the
// pre-pass (forward R layers of one EvalVec's tiles, in place on eb); 1 = the fused pass over tiles
// whose operand-a tile the pre-pass already transformed.
template <int MODE>
__global__ void __launch_bounds__(256, 3) fft64_tile_tower_kernel(const uint2* __restrict__ ea, uint2* __restrict__ eb,
                                                                  unsigned l, unsigned T, TwiddleSrc64 tw,
                                                                  uint64_t tile0, uint64_t ntiles) {
  pdl_wait();
  extern __shared__ uint2 s64[];
  const int n = 1 << T, tid = threadIdx.x, lane = tid & 31;
  TowerSmem64& sm = *reinterpret_cast<TowerSmem64*>(s64 + 2 * n);
  smul_tabs_build(sm.stab, tw.tau, tid);
  if (tid < 64) {
    sm.to_r[to_r64_pad(tid)] = __ldg(tw.to_r + tid);
    sm.rows_to_r[tid + (tid >> 3)] = __ldg(tw.to_r + tid);
    sm.rows_to_poly[tid + (tid >> 3)] = __ldg(tw.to_poly + tid);
  }
  const int ntab = tower64_tables(T);
  for (uint64_t t = tile0 + blockIdx.x; t < ntiles; t += gridDim.x) {
    uint2* g = eb + (t << T);
    const uint2* ga = MODE == 2 ? nullptr : ea + (t << T);  // (the pre-pass has one EvalVec: eb)
    for (int k = tid; k < ntab; k += blockDim.x) {
      int i = 0, kk = k;
      while (kk >= tower64_groups(T, (unsigned)i)) kk -= tower64_groups(T, (unsigned)i++);
      sm.wz[k] = x2(twiddle64(tw, (unsigned)i, t << (T - 1 - i)), c2p2_64(tw.c2p, (uint64_t)kk << 7));
    }
    if constexpr (MODE == 2) {
      for (int k = tid; k < n; k += blockDim.x) s64[tsw64(k)] = g[k];
      __syncthreads();
      tile_layers_r64<false, 1>(s64, T, kPolyLayers64, sm);
      for (int k = tid; k < n; k += blockDim.x) g[k] = s64[tsw64(k)];
      __syncthreads();
    } else {
    for (int k = tid; k < n; k += blockDim.x) {
      s64[tsw64(k)] = ga[k];
      s64[n + tsw64(k)] = g[k];
    }
    __syncthreads();
    if (MODE == 1) tile_layers_r64<false, 1>(s64 + n, T, kPolyLayers64, sm);
    else tile_layers_r64<false, 2>(s64, T, kPolyLayers64, sm);
    g8_expand(sm.tab, sm.rows_to_poly, tid);
    __syncthreads();
    if (kPolyLayers64) {
      for (int k = tid; k < 2 * n; k += blockDim.x) s64[k] = g8_mul(sm.tab, s64[k], lane);
      __syncthreads();
      tile_layers_poly64<false>(s64, T, kPolyLayers64, t, tw);
      for (int k = tid; k < n; k += blockDim.x) s64[k] = gf64_mul(s64[k], s64[n + k]);
      __syncthreads();
      tile_layers_poly64<true>(s64, T, kPolyLayers64, t, tw);
    } else {
      for (int k = tid; k < n; k += blockDim.x)
        s64[k] = gf64_mul(g8_mul(sm.tab, s64[k], lane), g8_mul(sm.tab, s64[n + k], lane));
      __syncthreads();
    }
    g8_expand(sm.tab, sm.rows_to_r, tid);
    __syncthreads();
    for (int k = tid; k < n; k += blockDim.x) s64[k] = g8_mul(sm.tab, s64[k], lane);
    {  // the next tile's operands into L2 while this tile's inverse layers run
      const uint64_t tn = t + gridDim.x;
      const int lines = n * 8 / 128;
      if (tn < ntiles)
        for (int k = tid; k < 2 * lines; k += blockDim.x) {
          const char* p = reinterpret_cast<const char*>((k < lines ? ea : eb) + (tn << T)) + 128 * (k % lines);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
        }
    }
    tile_layers_r64<true, 1>(s64, T, kPolyLayers64, sm);
    for (int k = tid; k < n; k += blockDim.x) g[k] = s64[tsw64(k)];
    __syncthreads();
    }  // (MODE != 2)
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

__global__ void pointwise64_kernel(const uint2* __restrict__ u, const uint2* __restrict__ v, uint2* __restrict__ out,
                                   uint64_t n) {
  pdl_wait();
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
    out[k] = gf64_mul(u[k], v[k]);
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

int sms64() {
  int dev, n;
  FPM_CUDA(cudaGetDevice(&dev));
  FPM_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

template <class K>
void set_smem64(K kernel, size_t bytes) {
  FPM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

int tile_threads64(unsigned T) { return T >= 9 ? 256 : std::max(32, 1 << (T - 1)); }

struct TileCfg64 {
  int threads, use_tab;
  size_t smem;
};
TileCfg64 tile_cfg64(unsigned l, unsigned T) {
  TileCfg64 c;
  c.threads = tile_threads64(T);
  c.use_tab = T > kTabLayer64 && c.threads == 256;
  c.smem = ((size_t)1 << T) * sizeof(uint2) + (c.use_tab ? (kG8Uint2 + kG8Rows) * sizeof(uint2) : 0);
  return c;
}
constexpr size_t kTileSmemMax64 = ((size_t)1 << kTileMax64) * sizeof(uint2) + (kG8Uint2 + kG8Rows) * sizeof(uint2);

}  // namespace

// Tile depth for the GF(2^64) transforms (tuning override FPM_TILE_LOG2_64).
int tile_log2_knob64() {
  static const int knob = [] {
    const char* e = std::getenv("FPM_TILE_LOG2_64");
    return e ? std::max(8, std::min(kTileMax64, std::atoi(e))) : 0;
  }();
  return knob;
}

unsigned fft64_tile_log2(unsigned l) {
  const int knob = tile_log2_knob64();
  const unsigned cap = knob ? (unsigned)knob : (l >= 20 ? 12u : l >= 18 ? 10u : 8u);
  return l < cap ? l : cap;
}

// Both operands' tile layers in the fused pass (FPM_FUSE_AB=0 disables it).
bool tile64_fused2_enabled(unsigned T) {
  static const bool on = [] {
    const char* e = std::getenv("FPM_FUSE_AB");
    return !(e && e[0] == '0');
  }();
  return on && T >= 10 && T <= 12;
}

#ifndef FPM_TILE2_LOG2_64
#define FPM_TILE2_LOG2_64 11
#endif
unsigned pipeline64_tile_log2(unsigned l) {
  if (!tile_log2_knob64() && l >= 20 && tile64_fused2_enabled(FPM_TILE2_LOG2_64)) return FPM_TILE2_LOG2_64;
  return fft64_tile_log2(l);
}

void butterfly64_tile_fused2_device(const uint2* ea, uint2* eb, unsigned l, unsigned T, const TwiddleSrc64& tw,
                                    cudaStream_t s) {
  const size_t smem = (2 * ((size_t)1 << T) + kG8Uint2 + kG8Rows) * sizeof(uint2);
  static PerDeviceOnce attr;
  attr.run([&] { set_smem64(fft64_tile_fused2_kernel, (2 * ((size_t)1 << 12) + kG8Uint2 + kG8Rows) * sizeof(uint2)); });
  const int grid = resident_grid(fft64_tile_fused2_kernel, 256, smem, ((uint64_t)1 << l) >> T);
  launch_k(fft64_tile_fused2_kernel, dim3(grid), dim3(256), smem, s, ea, eb, l, T, tw);
  FPM_LAUNCH_CHECK();
}

// The tower tile pass for the GF(2^64) product pipeline (FPM_TOWER=0 disables it, as for GF(2^128)).
bool tile64_tower_enabled(unsigned T) {
  static const bool on = [] {
    const char* e = std::getenv("FPM_TOWER");
    return !(e && e[0] == '0');
  }();
  return on && T >= 10 && T <= 12;
}

void tower64_set_smem() {
  static PerDeviceOnce attr;
  attr.run([&] {
    set_smem64(fft64_tile_tower_kernel<0>, tower64_smem(12));
    set_smem64(fft64_tile_tower_kernel<1>, tower64_smem(12));
    set_smem64(fft64_tile_tower_kernel<2>, tower64_smem(12));
  });
}

// pre_tiles: operand a's tiles [0, pre_tiles) already hold their forward R layers
// (butterfly64_tile_tower_pre_device).
void butterfly64_tile_tower_device(const uint2* ea, uint2* eb, unsigned l, unsigned T, const TwiddleSrc64& tw,
                                   cudaStream_t s, uint64_t pre_tiles) {
  if (T < 10 || T > 12 || l < T) throw Error(kInvalid, "tower tile pass (GF(2^64)): T must be 10..12");
  tower64_set_smem();
  const size_t smem = tower64_smem(T);
  const uint64_t ntiles = ((uint64_t)1 << l) >> T;
  if (pre_tiles > ntiles) throw Error(kInvalid, "tower tile pass (GF(2^64)): more pre-passed tiles than tiles");
  if (pre_tiles) {
    const int g1 = resident_grid(fft64_tile_tower_kernel<1>, 256, smem, pre_tiles);
    launch_k(fft64_tile_tower_kernel<1>, dim3(g1), dim3(256), smem, s, ea, eb, l, T, tw, (uint64_t)0, pre_tiles);
    FPM_LAUNCH_CHECK();
    if (pre_tiles == ntiles) return;
  }
  const int grid = resident_grid(fft64_tile_tower_kernel<0>, 256, smem, ntiles - pre_tiles);
  launch_k(fft64_tile_tower_kernel<0>, dim3(grid), dim3(256), smem, s, ea, eb, l, T, tw, pre_tiles, ntiles);
  FPM_LAUNCH_CHECK();
}

// Host-buffer products (as tower_pre_tiles / butterfly_tile_tower_pre_device in k_fft.cu): the share
// of operand a's tiles whose forward R layers run while operand b is still being uploaded.
uint64_t tower64_pre_tiles(unsigned l, unsigned T) {
  static const double frac = [] {
    const char* e = std::getenv("FPM_PRE_A_FRAC");
    return e ? std::atof(e) : 0.5;
  }();
  static const unsigned min_l = [] {
    const char* e = std::getenv("FPM_PRE_A_MIN_L");
    return e ? (unsigned)std::atoi(e) : 27u;  // 2^33-bit products: l = 27 in GF(2^64)
  }();
  if (T < 10 || T > 12 || l < T || l < min_l || !(frac > 0)) return 0;
  tower64_set_smem();
  const uint64_t ntiles = ((uint64_t)1 << l) >> T;
  const uint64_t grid = (uint64_t)resident_grid(fft64_tile_tower_kernel<2>, 256, tower64_smem(T), ntiles);
  const uint64_t waves = (uint64_t)(std::min(frac, 1.0) * (double)ntiles / (double)grid);
  return std::min(ntiles, waves * grid);
}

void butterfly64_tile_tower_pre_device(uint2* ev, unsigned l, unsigned T, const TwiddleSrc64& tw, uint64_t pre_tiles,
                                       cudaStream_t s) {
  if (!pre_tiles) return;
  if (T < 10 || T > 12 || l < T || pre_tiles > (((uint64_t)1 << l) >> T))
    throw Error(kInvalid, "tower pre-pass (GF(2^64)): bad tile count");
  tower64_set_smem();
  const size_t smem = tower64_smem(T);
  const int grid = resident_grid(fft64_tile_tower_kernel<2>, 256, smem, pre_tiles);
  launch_k(fft64_tile_tower_kernel<2>, dim3(grid), dim3(256), smem, s, (const uint2*)nullptr, ev, l, T, tw, (uint64_t)0,
           pre_tiles);
  FPM_LAUNCH_CHECK();
}

TwiddleSrc64 make_twiddle_src64(int device, unsigned l, uint64_t base) {
  if (l > (unsigned)kMaxLayers) throw Error(kInvalid, "butterfly: too many layers");
  TwiddleSrc64 tw{};
  const DeviceTables& dt = device_tables(device);
  tw.c2p = dt.c2p64;
  tw.to_r = dt.to_r64;
  tw.to_poly = dt.to_poly64;
  const TowerTables& tt = tower_tables64();
  for (int b = 0; b < 8; ++b) tw.tau |= (uint64_t)tt.tau[b] << (8 * b);
  const FieldTables& ft = field_tables64();
  for (unsigned i = 0; i < l; ++i) {
    const U128 p = host_cantor_to_poly64(ft, base >> i);
    tw.layer[i] = make_uint2((uint32_t)p.lo, (uint32_t)(p.lo >> 32));
  }
  return tw;
}

template <bool R>
void top_passes64(uint2* ev, unsigned l, unsigned T, bool inverse, const TwiddleSrc64& tw, cudaStream_t s,
                  uint2* ev2 = nullptr) {
  const size_t smem = kG8Uint2 * sizeof(uint2);
  static PerDeviceOnce attr;
  attr.run([&] {
    set_smem64(fft64_top_kernel<false, R>, smem);
    set_smem64(fft64_top_kernel<true, R>, smem);
    set_smem64(fft64_top4_kernel<false, R>, kTop4Smem64);
    set_smem64(fft64_top4_kernel<true, R>, kTop4Smem64);
  });
  if (T < 8) throw Error(kInvalid, "butterfly_top: layer too small for the table layer kernel");
  const uint64_t pairs = ((uint64_t)1 << l) / 2;
  uint64_t ppc = 4096;
  while (ppc > 256 && pairs / ppc < (uint64_t)sms64() * 2) ppc /= 2;
  auto radix2 = [&](unsigned i) {
    const uint64_t p = std::min<uint64_t>(ppc, (uint64_t)1 << i);
    for (uint2* e : {ev, ev2}) {
      if (!e) continue;
      if (!inverse) launch_k(fft64_top_kernel<false, R>, dim3((unsigned)(pairs / p)), dim3(256), smem, s, e, i, (int)p, tw);
      else launch_k(fft64_top_kernel<true, R>, dim3((unsigned)(pairs / p)), dim3(256), smem, s, e, i, (int)p, tw);
      FPM_LAUNCH_CHECK();
    }
  };
  const uint64_t quads = ((uint64_t)1 << l) / 4;
#ifndef FPM_TOP4_QMAX64
#define FPM_TOP4_QMAX64 16384  // 40.12 -> 40.04 ms at 2^32 bits
#endif
  uint64_t qpc = FPM_TOP4_QMAX64;
  while (qpc > 1024 && quads / qpc < (uint64_t)sms64() * 4) qpc /= 2;
  auto radix4 = [&](unsigned i) {
    const unsigned q = (unsigned)std::min<uint64_t>(qpc, (uint64_t)1 << i);
    if (!inverse)
      launch_k(fft64_top4_kernel<false, R>, dim3((unsigned)(quads / q)), dim3(kTop4Threads64), kTop4Smem64, s, ev, i, (int)q, tw, ev2);
    else
      launch_k(fft64_top4_kernel<true, R>, dim3((unsigned)(quads / q)), dim3(kTop4Threads64), kTop4Smem64, s, ev, i, (int)q, tw, ev2);
    FPM_LAUNCH_CHECK();
  };
  const unsigned n = l - T;
#ifndef FPM_TOP8_64
#define FPM_TOP8_64 1
#endif
  if (R && FPM_TOP8_64 && n >= 3) {  // three layers per pass (fft64_top8_kernel), the remainder at the bottom
    static PerDeviceOnce attr8;
    attr8.run([&] {
      set_smem64(fft64_top8_kernel<false>, kTop8Smem64);
      set_smem64(fft64_top8_kernel<true>, kTop8Smem64);
    });
    const uint64_t octs = ((uint64_t)1 << l) / 8;
    uint64_t opc = FPM_TOP4_QMAX64 / 2;
    while (opc > 512 && octs / opc < (uint64_t)sms64() * 4) opc /= 2;
    auto radix8 = [&](unsigned i) {
      const unsigned o = (unsigned)std::min<uint64_t>(opc, (uint64_t)1 << i);
      if (!inverse)
        launch_k(fft64_top8_kernel<false>, dim3((unsigned)(octs / o)), dim3(kTop4Threads64), kTop8Smem64, s, ev, i, (int)o, tw, ev2);
      else
        launch_k(fft64_top8_kernel<true>, dim3((unsigned)(octs / o)), dim3(kTop4Threads64), kTop8Smem64, s, ev, i, (int)o, tw, ev2);
      FPM_LAUNCH_CHECK();
    };
    const unsigned rem = n % 3;
    if (!inverse) {
      for (unsigned k = 0; k + 3 <= n; k += 3) radix8(l - 3 - k);
      if (rem == 2) radix4(T);
      if (rem == 1) radix2(T);
    } else {
      if (rem == 2) radix4(T);
      if (rem == 1) radix2(T);
      for (unsigned i = T + rem; i + 3 <= l; i += 3) radix8(i);
    }
    return;
  }
  const bool odd = n & 1;
  if (!inverse) {
    for (unsigned k = 0; k + 1 < n; k += 2) radix4(l - 2 - k);
    if (odd) radix2(T);
  } else {
    if (odd) radix2(T);
    for (unsigned i = T + (odd ? 1 : 0); i + 1 < l; i += 2) radix4(i);
  }
}

void butterfly64_top_device(uint2* ev, unsigned l, unsigned T, bool inverse, const TwiddleSrc64& tw, cudaStream_t s,
                            bool tower, uint2* ev2) {
  if (l <= T) return;
  if (tower) top_passes64<true>(ev, l, T, inverse, tw, s, ev2);
  else top_passes64<false>(ev, l, T, inverse, tw, s, ev2);
}

void butterfly64_tile_device(uint2* ev, unsigned l, unsigned T, bool inverse, const TwiddleSrc64& tw, cudaStream_t s) {
  if (T == 0) return;
  static PerDeviceOnce attr;
  attr.run([&] {
    set_smem64(fft64_tile_kernel<false>, kTileSmemMax64);
    set_smem64(fft64_tile_kernel<true>, kTileSmemMax64);
  });
  const TileCfg64 c = tile_cfg64(l, T);
  const uint64_t ntiles = ((uint64_t)1 << l) >> T;
  if (!inverse)
    launch_k(fft64_tile_kernel<false>, dim3(resident_grid(fft64_tile_kernel<false>, c.threads, c.smem, ntiles)), dim3(c.threads), c.smem, s, ev, l, T, tw, c.use_tab);
  else
    launch_k(fft64_tile_kernel<true>, dim3(resident_grid(fft64_tile_kernel<true>, c.threads, c.smem, ntiles)), dim3(c.threads), c.smem, s, ev, l, T, tw, c.use_tab);
  FPM_LAUNCH_CHECK();
}

void butterfly64_tile_fused_device(const uint2* ea, uint2* eb, unsigned l, unsigned T, const TwiddleSrc64& tw,
                                   cudaStream_t s) {
  static PerDeviceOnce attr;
  attr.run([&] { set_smem64(fft64_tile_fused_kernel, kTileSmemMax64); });
  const TileCfg64 c = tile_cfg64(l, T);
  const int grid = resident_grid(fft64_tile_fused_kernel, c.threads, c.smem, ((uint64_t)1 << l) >> T);
  launch_k(fft64_tile_fused_kernel, dim3(grid), dim3(c.threads), c.smem, s, ea, eb, l, T, tw, c.use_tab);
  FPM_LAUNCH_CHECK();
}

void butterfly64_device(uint2* ev, unsigned l, uint64_t base, bool inverse, cudaStream_t s) {
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const TwiddleSrc64 tw = make_twiddle_src64(dev, l, base);
  const unsigned T = fft64_tile_log2(l);
  if (!inverse) {
    butterfly64_top_device(ev, l, T, false, tw, s);
    butterfly64_tile_device(ev, l, T, false, tw, s);
  } else {
    butterfly64_tile_device(ev, l, T, true, tw, s);
    butterfly64_top_device(ev, l, T, true, tw, s);
  }
}

void pointwise64_device(const uint2* u, const uint2* v, uint2* out, size_t n, cudaStream_t s) {
  if (!n) return;
  const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)sms64() * 16);
  launch_k(pointwise64_kernel, dim3(grid), dim3(256), 0, s, u, v, out, n);
  FPM_LAUNCH_CHECK();
}

}  // namespace fpm
