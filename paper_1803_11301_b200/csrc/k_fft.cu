// k_fft.cu -- LCH butterflies over GF(2^128) on sm_100a (north-star subsystems 2, 3, 4).
//
// Reference: proj/include/fpmul/detail/kernels_impl.hpp:29-123 and proj/src/butterfly.cpp.
// Layer i pairs p[j], p[j+2^i] inside blocks of 2^(i+1) elements; block b uses the twiddle
//     w(i, b) = C2P((base >> i) ^ 2b),  base = e_{l+64}  =>  w(i, b) = v_{l+64-i} ^ C2P(2b)
// (butterfly.cpp:45-49, encode.cpp:47).  Twiddles are generated on the fly from the Cantor basis
// and three 512-entry C2P tables (C2P is GF(2)-linear in b), so the reference's
// 2^l - 1 entry plan (1 GiB at l = 26) never exists on the GPU.
//   forward  p0 ^= w*p1; p1 ^= p0          inverse  p1 ^= p0; p0 ^= w*p1
//
// Kernels (T = fft_tile_log2(l): layers >= T are "top" layers, < T run in shared-memory tiles):
//  * fft_top4_kernel: top layers (i+1, i) per HBM round trip; the three twiddles of a block as M8
//    tables (gf128.cuh), one 768-thread CTA per SM; fft_top_kernel: a single top layer.
//  * fft_tile_kernel: layers [0, T) of a 2^T-element tile (one HBM read and write for T layers):
//    layers >= 9 via one M8 table per twiddle, layers 6-8 via M4 tables 8 twiddles at a time, lower
//    layers (twiddles vary per block) via the generic IMAD-hole gf_mul.
//  * fft_tile_fused_kernel: forward layers [0,T) of operand b, the pointwise product with operand
//    a (subsystem 3, kernels_impl.hpp:116-123), and inverse layers [0,T) in one tile pass.
//  * fft_tile_fused2_kernel (the product pipeline): forward layers [0,T) of BOTH operands (their
//    tiles share every twiddle, so each table serves both), the pointwise product and the inverse
//    layers [0,T) in one pass -- no separate tile pass for operand a.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "fpm_internal.h"
#include "gf128.cuh"
#include "tower.cuh"

namespace fpm {


namespace {

constexpr int kTileMax = 12;         // 2^12 elements x 16 B = 64 KiB tile
#ifndef FPM_TILE2_THREADS
#define FPM_TILE2_THREADS 256
#endif
constexpr int kTile2Threads = FPM_TILE2_THREADS;  // fft_tile_fused2_kernel
// M8 tables from this layer on in fft_tile_fused2_kernel (a table then serves both operands'
// butterflies in the forward layers): 57.27 ms at 2^32 bits vs 57.48 from layer 9.
#ifndef FPM_M8_LAYER2
#define FPM_M8_LAYER2 8
#endif
#ifndef FPM_M8_LAYER2_INV
#define FPM_M8_LAYER2_INV 8
#endif
constexpr unsigned kTabLayer2 = FPM_M8_LAYER2, kTabLayer2Inv = FPM_M8_LAYER2_INV;

__device__ __forceinline__ uint4 c2p2(const uint4* __restrict__ c2p, uint64_t b) {  // C2P(2b)
  uint4 r = c2p[b & 511];
  if (b >> 9) r = x4(r, c2p[512 + ((b >> 9) & 511)]);
  if (b >> 18) r = x4(r, c2p[1024 + ((b >> 18) & 511)]);
  if (b >> 27) r = x4(r, c2p[1536 + ((b >> 27) & 511)]);
  return r;
}

__device__ __forceinline__ uint4 twiddle(const TwiddleSrc& tw, unsigned l, unsigned i, uint64_t b) {
  return x4(tw.layer[i], c2p2(tw.c2p, b));
}

// ------------------------------------------------------------------ top layers (i >= T)
// R: elements in the tower representation (tower.cuh), the table built in R.
template <bool INV, bool R>
__global__ void __launch_bounds__(256) fft_top_kernel(uint4* __restrict__ ev, unsigned l, unsigned i, int ppc, TwiddleSrc tw) {
  pdl_wait();
  extern __shared__ uint4 tab[];            // kM8Uint4
  __shared__ uint4 rows[144];
  const uint64_t half = (uint64_t)1 << i;
  const uint64_t pair0 = (uint64_t)blockIdx.x * ppc;   // ppc <= 2^i: CTA pairs never straddle a block
  const uint64_t b = pair0 >> i;
  const uint4 w = twiddle(tw, l, i, b);
  if (R) {
    rows_r<false>(rows, w, threadIdx.x, tw.to_r);
    __syncthreads();
    m8_expand(tab, rows, threadIdx.x);
    __syncthreads();
  } else {
    m8_build(tab, rows, w, threadIdx.x);
  }
  const int copy = threadIdx.x & 7;
  uint4* base = ev + (b << (i + 1));
#pragma unroll 4
  for (int k = threadIdx.x; k < ppc; k += blockDim.x) {
    const uint64_t j = (pair0 & (half - 1)) + k;
    uint4 u0 = base[j], u1 = base[j + half];
    if (!INV) {
      u0 = x4(u0, m8_mul(tab, u1, copy));
      u1 = x4(u1, u0);
    } else {
      u1 = x4(u1, u0);
      u0 = x4(u0, m8_mul(tab, u1, copy));
    }
    base[j] = u0;
    base[j + half] = u1;
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ top layers, two per pass
// Layers i+1 and i in one HBM round trip.  A block of 2^(i+2) elements splits into quarters
// q0..q3 of h = 2^i; layer i+1 pairs (q0,q2), (q1,q3) with w(i+1, B); layer i pairs (q0,q1) with
// w(i, 2B) and (q2,q3) with w(i, 2B+1).  The three M8 tables (192 KiB) are built by three groups of
// 256 threads; one 768-thread CTA per SM then streams its quads.
constexpr int kTop4Threads = 768;
#ifndef FPM_TOP4_STREAM
#define FPM_TOP4_STREAM 1
#endif
__device__ __forceinline__ uint4 ld_na(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_cs(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
constexpr size_t kTop4Smem = (3 * (size_t)kM8Uint4 + 3 * 144 + 136) * sizeof(uint4);  // + to_r (tower)

// NT: 768 threads (80 registers; three table groups at once) or 512 (128 registers: the
// pre-rotated lookups in both directions; the third table in a second build round).
// ev2 (optional): a second evaluation vector at the same layers and twiddles (both operands of a
// product): every CTA runs its quads of both with one set of tables.
template <bool INV, bool R, int NT = kTop4Threads>
__global__ void __launch_bounds__(NT, 1) fft_top4_kernel(uint4* __restrict__ ev, unsigned l, unsigned i,
                                                          int qpc, TwiddleSrc tw, uint4* __restrict__ ev2) {
  pdl_wait();
  extern __shared__ uint4 sm4[];
  uint4* t1 = sm4;                   // w(i+1, B)
  uint4* t0a = sm4 + kM8Uint4;       // w(i, 2B)
  uint4* t0b = sm4 + 2 * kM8Uint4;   // w(i, 2B+1)
  uint4* rows = sm4 + 3 * kM8Uint4;  // 3 x 144
  uint4* to_r = rows + 3 * 144;      // tower: the conversion rows, to_r_pad layout
  const uint64_t h = (uint64_t)1 << i;
  const uint64_t quad0 = (uint64_t)blockIdx.x * qpc;  // qpc <= h: a CTA never straddles a block
  const uint64_t B = quad0 >> i;
  const int tid = threadIdx.x, grp = tid >> 8, lt = tid & 255;
  const int nq = ev2 ? 2 * qpc : qpc;
  // the twiddles (global loads) are issued before the to_r staging barrier: one L2 round trip, not two
  constexpr int kRounds = (3 + NT / 256 - 1) / (NT / 256);
  uint4 ws[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int g = r * (NT / 256) + grp;
    ws[r] = g == 0 ? twiddle(tw, l, i + 1, B)
                   : g == 1 ? twiddle(tw, l, i, 2 * B) : g == 2 ? twiddle(tw, l, i, 2 * B + 1) : make_uint4(0, 0, 0, 0);
  }
  if (R) {
    if (tid < 128) to_r[to_r_pad(tid)] = __ldg(tw.to_r + tid);
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int g = r * (NT / 256) + grp;
    const uint4 w = ws[r];
    uint4* tab = sm4 + g * kM8Uint4;
    uint4* rs = rows + g * 144;
    if (R) {
      if (g < 3) rows_r<true>(rs, w, lt, to_r);
    } else if (g < 3 && lt < 128) {
      rs[lt + (lt >> 3)] = gf_mul_xk(w, (unsigned)lt);
    }
    __syncthreads();
    if (g < 3) {
      const int c = lt & 15, sv = lt >> 4;
      uint4 r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = rs[9 * c + j];
      uint4 t[16];
      t[0] = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (sv >> j & 1) t[0] = x4(t[0], r[4 + j]);
#pragma unroll
      for (int u = 1; u < 16; ++u) t[u] = x4(t[u & (u - 1)], r[(u & 1) ? 0 : (u & 2) ? 1 : (u & 4) ? 2 : 3]);
      uint4* dst = tab + (c >> 3) * 2048 + 16 * sv * 8 + (c & 7);
#pragma unroll
      for (int u = 0; u < 16; ++u) dst[u * 8] = t[u];
    }
    __syncthreads();
  }
  const int q = tid & 7;
  const uint64_t off = (B << (i + 2)) + (quad0 & (h - 1));
  const M8Base mb = m8_base(t1, q);  // (inverse only)
  constexpr uint32_t kA = kM8Uint4 * 16u, kB = 2u * kM8Uint4 * 16u;  // t0a, t0b after t1
#pragma unroll 1
  for (int k = tid; k < nq; k += NT) {
    uint4* p = (k < qpc ? ev + k : ev2 + (k - qpc)) + off;
#if FPM_TOP4_STREAM
    // read-once / write-once quads: no L1 allocation (the L1TEX data path is the pass's binding unit)
    uint4 a0 = ld_na(p), a1 = ld_na(p + h), a2 = ld_na(p + 2 * h), a3 = ld_na(p + 3 * h);
#else
    uint4 a0 = p[0], a1 = p[h], a2 = p[2 * h], a3 = p[3 * h];
#endif
    if (!INV && NT == 768) {  // (m8_mul_r here spills at the 80 registers of a 768-thread CTA: 12.8 vs 11.3 ms)
      a0 = x4(a0, m8_mul(t1, a2, q));
      a1 = x4(a1, m8_mul(t1, a3, q));
      a2 = x4(a2, a0);
      a3 = x4(a3, a1);
      a0 = x4(a0, m8_mul(t0a, a1, q));
      a2 = x4(a2, m8_mul(t0b, a3, q));
      a1 = x4(a1, a0);
      a3 = x4(a3, a2);
    } else if (!INV) {
      a0 = x4(a0, m8_mul_r(mb, a2, q));
      a1 = x4(a1, m8_mul_r(mb, a3, q));
      a2 = x4(a2, a0);
      a3 = x4(a3, a1);
      a0 = x4(a0, m8_mul_r(mb, a1, q, kA));
      a2 = x4(a2, m8_mul_r(mb, a3, q, kB));
      a1 = x4(a1, a0);
      a3 = x4(a3, a2);
    } else {
      a1 = x4(a1, a0);
      a3 = x4(a3, a2);
      a0 = x4(a0, m8_mul_r(mb, a1, q, kA));
      a2 = x4(a2, m8_mul_r(mb, a3, q, kB));
      a2 = x4(a2, a0);
      a3 = x4(a3, a1);
      a0 = x4(a0, m8_mul_r(mb, a2, q));
      a1 = x4(a1, m8_mul_r(mb, a3, q));
    }
#if FPM_TOP4_STREAM
    st_cs(p, a0);
    st_cs(p + h, a1);
    st_cs(p + 2 * h, a2);
    st_cs(p + 3 * h, a3);
#else
    p[0] = a0;
    p[h] = a1;
    p[2 * h] = a2;
    p[3 * h] = a3;
#endif
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ top layers, three per pass (tower)
// Layers i+2, i+1 and i in one HBM round trip, elements in the tower representation R.  A block of
// 2^(i+3) elements splits into eighths a0..a7 of h = 2^i; layer i+2 pairs (a_k, a_k+4) with
// W2 = w(i+2, B); layer i+1 pairs (a0,a2), (a1,a3) with W1 = w(i+1, 2B) and (a4,a6), (a5,a7) with
// w(i+1, 2B+1) = W1 ^ C2P(2); layer i pairs (a_2m, a_2m+1) with w(i, 4B+m) = W0 ^ C2P(2m).  C2P(2m)
// (m < 4) lies in the subfield GF(2^8), so the three tables of radix-4 serve three layers: the
// sibling twiddles add a byte-permute scalar product (tower.cuh smul_t) instead of a table.
constexpr size_t kTop8Smem = kTop4Smem + sizeof(SmulTabs);
template <bool INV, int NT = 512>
__global__ void __launch_bounds__(NT, 1) fft_top8_kernel(uint4* __restrict__ ev, unsigned l, unsigned i, int opc,
                                                          TwiddleSrc tw, uint4* __restrict__ ev2) {
  pdl_wait();
  extern __shared__ uint4 sm8[];
  uint4* rows = sm8 + 3 * kM8Uint4;  // 3 x 144
  uint4* to_r = rows + 3 * 144;      // the conversion rows, to_r_pad layout
  SmulTabs& stab = *reinterpret_cast<SmulTabs*>(to_r + 136);
  const uint64_t h = (uint64_t)1 << i;
  const uint64_t oct0 = (uint64_t)blockIdx.x * opc;  // opc <= h: a CTA never straddles a block
  const uint64_t B = oct0 >> i;
  const int tid = threadIdx.x, grp = tid >> 8, lt = tid & 255;
  const int no = ev2 ? 2 * opc : opc;
  constexpr int kRounds = (3 + NT / 256 - 1) / (NT / 256);
  uint4 ws[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int g = r * (NT / 256) + grp;
    ws[r] = g == 0 ? twiddle(tw, l, i + 2, B)
                   : g == 1 ? twiddle(tw, l, i + 1, 2 * B) : g == 2 ? twiddle(tw, l, i, 4 * B) : make_uint4(0, 0, 0, 0);
  }
  smul_tabs_build(stab, tw.tau, tid);
  if (tid < 128) to_r[to_r_pad(tid)] = __ldg(tw.to_r + tid);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const int g = r * (NT / 256) + grp;
    uint4* tab = sm8 + g * kM8Uint4;
    uint4* rs = rows + g * 144;
    if (g < 3) rows_r<true>(rs, ws[r], lt, to_r);
    __syncthreads();
    if (g < 3) {
      const int c = lt & 15, sv = lt >> 4;
      uint4 rr[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) rr[j] = rs[9 * c + j];
      uint4 t[16];
      t[0] = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (sv >> j & 1) t[0] = x4(t[0], rr[4 + j]);
#pragma unroll
      for (int u = 1; u < 16; ++u) t[u] = x4(t[u & (u - 1)], rr[(u & 1) ? 0 : (u & 2) ? 1 : (u & 4) ? 2 : 3]);
      uint4* dst = tab + (c >> 3) * 2048 + 16 * sv * 8 + (c & 7);
#pragma unroll
      for (int u = 0; u < 16; ++u) dst[u * 8] = t[u];
    }
    __syncthreads();
  }
  const int q = tid & 7;
  const uint64_t off = (B << (i + 3)) + (oct0 & (h - 1));
  const M8Base mb = m8_base(sm8, q);
  constexpr uint32_t kT1 = kM8Uint4 * 16u, kT0 = 2u * kM8Uint4 * 16u;  // W1, W0 after W2
  // u * (table twiddle ^ d_m) with the scalar part d_m = R(C2P(2m)), m = 1..3
  auto mul = [&](uint4 u, uint32_t toff, int m) {
    uint4 r = m8_mul_r(mb, u, q, toff);
    if (m) r = x4(r, smul_t(u, smul_tab(stab, m)));
    return r;
  };
#pragma unroll 1
  for (int k = tid; k < no; k += NT) {
    uint4* p = (k < opc ? ev + k : ev2 + (k - opc)) + off;
    uint4 a[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] = ld_na(p + e * h);
    if (!INV) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {  // layer i+2
        a[e] = x4(a[e], mul(a[e + 4], 0, 0));
        a[e + 4] = x4(a[e + 4], a[e]);
      }
#pragma unroll
      for (int hb = 0; hb < 2; ++hb)  // layer i+1: blocks 2B (a0..a3), 2B+1 (a4..a7)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int u0 = 4 * hb + e, u1 = u0 + 2;
          a[u0] = x4(a[u0], mul(a[u1], kT1, hb));
          a[u1] = x4(a[u1], a[u0]);
        }
#pragma unroll
      for (int m = 0; m < 4; ++m) {  // layer i: blocks 4B + m
        a[2 * m] = x4(a[2 * m], mul(a[2 * m + 1], kT0, m));
        a[2 * m + 1] = x4(a[2 * m + 1], a[2 * m]);
      }
    } else {
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        a[2 * m + 1] = x4(a[2 * m + 1], a[2 * m]);
        a[2 * m] = x4(a[2 * m], mul(a[2 * m + 1], kT0, m));
      }
#pragma unroll
      for (int hb = 0; hb < 2; ++hb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int u0 = 4 * hb + e, u1 = u0 + 2;
          a[u1] = x4(a[u1], a[u0]);
          a[u0] = x4(a[u0], mul(a[u1], kT1, hb));
        }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a[e + 4] = x4(a[e + 4], a[e]);
        a[e] = x4(a[e], mul(a[e + 4], 0, 0));
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) st_cs(p + e * h, a[e]);
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ tile layers (i < T)
// Layers i >= kTabLayer of a 256-thread tile have <= 2 twiddles per tile, each shared by >= 512
// butterflies: those use an M8 table built in shared memory (tab != nullptr: 64 KiB + 144 rows
// after the tile) instead of the generic multiply.  (Layer 8's four twiddles per 2^11 tile: M4
// tables, 57.8 vs 58.3 ms at 2^32 bits; all tile layers on M4: 63.3 ms.)
#ifndef FPM_M8_LAYER
#define FPM_M8_LAYER 9
#endif
constexpr unsigned kTabLayer = FPM_M8_LAYER;
// Layers [kM4Layer, kTabLayer): rotated 4-bit tables for up to 8 twiddles at a time (gf128.cuh m4s_*).
#ifndef FPM_M4_LAYER
#define FPM_M4_LAYER 6
#endif
constexpr unsigned kM4Layer = FPM_M4_LAYER;
// Layers [kPrepLayer, kM4Layer): generic multiplies with the twiddle's limbs prepared once per block.
constexpr unsigned kPrepLayer = 1;
// NT tiles that share twiddles (operands a and b at the same position) lie at s, s + 2^T, ...:
// every table or prepared twiddle serves the butterflies of all of them.
template <bool INV, int NT = 1, unsigned kTabLayer = kTabLayer>
__device__ __forceinline__ void tile_layers(uint4* __restrict__ s, unsigned T, unsigned l, uint64_t tile_idx,
                                            const TwiddleSrc& tw, uint4* __restrict__ tab) {
  const int npairs = 1 << (T - 1), n = 1 << T;
  for (unsigned step = 0; step < T; ++step) {
    const unsigned i = INV ? step : T - 1 - step;
    const uint64_t bhi = tile_idx << (T - 1 - i);  // global block index of the tile's first block
    // w = v_{l+64-i} ^ C2P(2*(bhi + blk)) = Z ^ C2P(2*blk)  (bit ranges disjoint, C2P linear)
    const uint4 Z = twiddle(tw, l, i, bhi);
    if (tab && i >= kM4Layer && i < kTabLayer) {
      // 2^(T-1-i) twiddles of 2^i butterflies each: rotated 4-bit tables, up to 8 twiddles per round
      const int q = threadIdx.x & 7;
      const int nblk = npairs >> i, G = nblk < 8 ? nblk : 8;
      const int gi = i + (G >= 8 ? 3 : G >= 4 ? 2 : G >= 2 ? 1 : 0);  // log2(G << i)
      for (int b0 = 0; b0 < nblk; b0 += G) {
        const uint4 w = x4(Z, c2p2(tw.c2p, (uint64_t)(b0 + (threadIdx.x >> 5))));
        __syncthreads();  // previous round's lookups done
        if (threadIdx.x < 32 * G) m4s_build8(tab, w, threadIdx.x);
        __syncthreads();
        for (int pp = threadIdx.x; pp < (NT << gi); pp += blockDim.x) {
          const int p = pp & ((1 << gi) - 1), tt = pp >> gi;
          const int t = p >> i, j = p & ((1 << i) - 1), blk = b0 + t;
          const int i0 = (blk << (i + 1)) + j + tt * n, i1 = i0 + (1 << i);
          const uint4* tb = tab + t * kM4TabUint4;
          uint4 u0 = s[i0], u1 = s[i1];
          if (!INV) {
            u0 = x4(u0, m4s_mul(tb, u1, q));
            u1 = x4(u1, u0);
          } else {
            u1 = x4(u1, u0);
            u0 = x4(u0, m4s_mul(tb, u1, q));
          }
          s[i0] = u0;
          s[i1] = u1;
        }
      }
      __syncthreads();
      continue;
    }
    if (tab && i >= kTabLayer) {
      const int q = threadIdx.x & 7;
      for (int blk = 0; blk < (npairs >> i); ++blk) {
        m8_build(tab, tab + kM8Uint4, x4(Z, c2p2(tw.c2p, (uint64_t)blk)), threadIdx.x);
        for (int jj = threadIdx.x; jj < (NT << i); jj += blockDim.x) {
          const int j = jj & ((1 << i) - 1), tt = jj >> i;
          const int i0 = (blk << (i + 1)) + j + tt * n, i1 = i0 + (1 << i);
          uint4 u0 = s[i0], u1 = s[i1];
          if (!INV) {
            u0 = x4(u0, m8_mul(tab, u1, q));
            u1 = x4(u1, u0);
          } else {
            u1 = x4(u1, u0);
            u0 = x4(u0, m8_mul(tab, u1, q));
          }
          s[i0] = u0;
          s[i1] = u1;
        }
      }
      __syncthreads();
      continue;
    }
    if (tab && i >= kPrepLayer && (npairs >> i) * (int)sizeof(GfPrep) <= kM8Uint4 * (int)sizeof(uint4)) {
      // each twiddle serves 2^i butterflies: its masked Karatsuba limbs are prepared once, in the
      // (otherwise idle) table area
      GfPrep* prep = reinterpret_cast<GfPrep*>(tab);
      const int nblk = npairs >> i;
      for (int b = threadIdx.x; b < nblk; b += blockDim.x) prep[b] = gf_prep(x4(Z, c2p2(tw.c2p, (uint64_t)b)));
      __syncthreads();
      for (int pp = threadIdx.x; pp < NT * npairs; pp += blockDim.x) {
        const int p = pp & (npairs - 1), tt = pp >> (T - 1);
        const int blk = p >> i, j = p & ((1 << i) - 1);
        const int i0 = (blk << (i + 1)) + j + tt * n, i1 = i0 + (1 << i);
        const GfPrep w = prep[blk];
        uint4 u0 = s[i0], u1 = s[i1];
        if (!INV) {
          u0 = x4(u0, gf_mul_prep(w, u1));
          u1 = x4(u1, u0);
        } else {
          u1 = x4(u1, u0);
          u0 = x4(u0, gf_mul_prep(w, u1));
        }
        s[i0] = u0;
        s[i1] = u1;
      }
      __syncthreads();
      continue;
    }
    for (int pp = threadIdx.x; pp < NT * npairs; pp += blockDim.x) {
      const int p = pp & (npairs - 1), tt = pp >> (T - 1);
      const int blk = p >> i, j = p & ((1 << i) - 1);
      const int i0 = (blk << (i + 1)) + j + tt * n, i1 = i0 + (1 << i);
      const uint4 w = x4(Z, c2p2(tw.c2p, (uint64_t)blk));
      uint4 u0 = s[i0], u1 = s[i1];
      if (!INV) {
        u0 = x4(u0, gf_mul(w, u1));
        u1 = x4(u1, u0);
      } else {
        u1 = x4(u1, u0);
        u0 = x4(u0, gf_mul(w, u1));
      }
      s[i0] = u0;
      s[i1] = u1;
    }
    __syncthreads();
  }
}

template <bool INV>
__global__ void __launch_bounds__(256) fft_tile_kernel(uint4* __restrict__ ev, unsigned l, unsigned T, TwiddleSrc tw,
                                                       int use_tab) {
  pdl_wait();
  extern __shared__ uint4 s[];
  const int n = 1 << T;
  uint4* tab = use_tab ? s + n : nullptr;
  const uint64_t ntiles = ((uint64_t)1 << l) >> T;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    uint4* g = ev + (t << T);
    for (int k = threadIdx.x; k < n; k += blockDim.x) s[k] = g[k];
    __syncthreads();
    tile_layers<INV>(s, T, l, t, tw, tab);
    for (int k = threadIdx.x; k < n; k += blockDim.x) g[k] = s[k];
    __syncthreads();
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

__global__ void __launch_bounds__(256) fft_tile_fused_kernel(const uint4* __restrict__ ea, uint4* __restrict__ eb,
                                                             unsigned l, unsigned T, TwiddleSrc tw, int use_tab) {
  pdl_wait();
  extern __shared__ uint4 s[];
  const int n = 1 << T;
  uint4* tab = use_tab ? s + n : nullptr;
  const uint64_t ntiles = ((uint64_t)1 << l) >> T;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    uint4* g = eb + (t << T);
    const uint4* ga = ea + (t << T);
    for (int k = threadIdx.x; k < n; k += blockDim.x) s[k] = g[k];
    __syncthreads();
    tile_layers<false>(s, T, l, t, tw, tab);
    for (int k = threadIdx.x; k < n; k += blockDim.x) s[k] = gf_mul(ga[k], s[k]);
    __syncthreads();
    tile_layers<true>(s, T, l, t, tw, tab);
    for (int k = threadIdx.x; k < n; k += blockDim.x) g[k] = s[k];
    __syncthreads();
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// Both operands' tile layers in one CTA: the a and b tiles at the same position share every
// twiddle, so each M8/M4 table and prepared twiddle is built once for two butterflies; then the
// pointwise product and the inverse tile layers, as fft_tile_fused_kernel.  Saves operand a's
// separate tile pass (one HBM round trip of EvalVec a).
__global__ void __launch_bounds__(kTile2Threads, 512 / kTile2Threads) fft_tile_fused2_kernel(const uint4* __restrict__ ea,
                                                                          uint4* __restrict__ eb, unsigned l,
                                                                          unsigned T, TwiddleSrc tw) {
  pdl_wait();
  extern __shared__ uint4 s[];
  const int n = 1 << T;
  uint4* tab = s + 2 * n;
  const uint64_t ntiles = ((uint64_t)1 << l) >> T;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    uint4* g = eb + (t << T);
    const uint4* ga = ea + (t << T);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      s[k] = ga[k];
      s[n + k] = g[k];
    }
    __syncthreads();
    tile_layers<false, 2, kTabLayer2>(s, T, l, t, tw, tab);
    for (int k = threadIdx.x; k < n; k += blockDim.x) s[k] = gf_mul(s[k], s[n + k]);
    __syncthreads();
    tile_layers<true, 1, kTabLayer2Inv>(s, T, l, t, tw, tab);
    for (int k = threadIdx.x; k < n; k += blockDim.x) g[k] = s[k];
    __syncthreads();
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ tower-representation tiles
// Tile layers on R elements (tower.cuh).  Layer i's twiddle for tile block blk is
//   w = Z ^ C2P(2 (blk & ~127)) ^ C2P(2 (blk & 127)),  Z = twiddle(i, tile's first block);
// the first two terms are one M8 table per 128 blocks (layers 0 and 1 of a 2^10 tile need 4 and 2,
// every other layer one), the last is the subfield scalar d(blk & 127), applied by smul_t (byte permutes, tower.cuh).
// A table build is latency-bound (twiddle -> conversion -> shuffles -> xtimes -> 4096 stores), so:
// the tile's table twiddles are computed once per tile (wz, shared by both directions), the
// conversion rows stay in shared memory, and the rows of table k+1 are computed by warps 0-3 before
// their butterflies with table k (double-buffered rows), overlapping the other warps' work.
__host__ __device__ constexpr int tower_groups(unsigned T, unsigned i) {  // tables of layer i
  return (1 << (T - 1 - i)) > 128 ? (1 << (T - 1 - i)) >> 7 : 1;
}
__host__ __device__ constexpr int tower_tables(unsigned T) {
  int n = 0;
  for (unsigned i = 0; i < T; ++i) n += tower_groups(T, i);
  return n;
}
constexpr int kTowerMaxTables = tower_tables(12);  // 38

struct TowerSmem {  // after the 2^(T+1) tile elements
  uint4 tab[kM8Uint4];
  uint4 rows[2][144];
  uint4 to_r[128 + 8];        // rows_r conversion source, to_r_pad layout
  uint4 rows_to_r[144];       // m8 rows of poly -> R
  uint4 rows_to_poly[144];    // m8 rows of R -> poly
  uint4 wz[kTowerMaxTables];   // table twiddles of the current tile, layer-ascending, h ascending
  uint4 wzf[kTowerMaxTables];  // the same in the forward sequence (layers descending, h ascending)
  SmulTabs stab;              // subfield twiddle parts d(b) = R(C2P(2b)), b < 128 (tower.cuh)
};

// Tile element k lives at tsw(k) = k ^ 7 [bit 3 of k]: the butterflies of layers 0-2 (pairs at
// distance 1, 2, 4) then reach eight distinct 16-byte bank groups per quarter-warp (2-way bank
// conflicts otherwise); contiguous runs of 8 stay contiguous.
__device__ __forceinline__ int tsw(int k) { return k ^ (((k >> 3) & 1) * 7); }

// CTA shape per tile depth: T <= 11 -> 256 threads, 2 CTAs/SM (<= 140 KiB of shared memory each at
// T = 10); T = 12 (two 64 KiB tiles + the 64 KiB table, 207 KiB) -> 512 threads, 1 CTA/SM.
#ifndef FPM_TOWER_IDX2
#define FPM_TOWER_IDX2 1  // strength-reduced pair indices in tile_layers_r
#endif
#ifndef FPM_TOWER12_THREADS
#define FPM_TOWER12_THREADS 512
#endif
#ifndef FPM_TOWER_BIG_T
#define FPM_TOWER_BIG_T 12  // tile depths from here on: one 512-thread CTA per SM
#endif
__host__ __device__ constexpr int tower_threads(unsigned T) { return T >= FPM_TOWER_BIG_T ? FPM_TOWER12_THREADS : 256; }
__host__ __device__ constexpr int tower_min_blocks(unsigned T) { return T >= FPM_TOWER_BIG_T ? 1 : 2; }

// Index in wz of (layer i, group g): layers ascending.
__host__ __device__ constexpr int tower_wz_index(unsigned T, unsigned i, int g) {
  int k = 0;
  for (unsigned u = 0; u < i; ++u) k += tower_groups(T, u);
  return k + g;
}

// Layers [P, T) of the tile on R elements (forward: T-1 down to P; inverse: P up to T-1).  T and P
// are compile-time constants and the layer / group loops unroll, so every table index, block shift
// and pair count below folds to an immediate.
template <bool INV, int NT, unsigned T, unsigned P>
__device__ __forceinline__ void tile_layers_r(uint4* __restrict__ s, TowerSmem& sm) {
  constexpr int npairs = 1 << (T - 1), n = 1 << T;
  constexpr int ntab = tower_tables(T) - tower_wz_index(T, P, 0);
  const int tid = threadIdx.x, q = tid & 7;
  // table sequence k = 0..ntab-1: forward = wzf[k] (layers descending, h ascending), inverse =
  // wz[first + k] (layers ascending)
  constexpr int first = tower_wz_index(T, P, 0);
  auto wz_of = [&](int k) -> const uint4& { return INV ? sm.wz[first + k] : sm.wzf[k]; };
  rows_r<true>(sm.rows[0], wz_of(0), tid, sm.to_r);
  __syncthreads();
  m8_expand(sm.tab, sm.rows[0], tid);
  __syncthreads();
  int k = 0;
#pragma unroll
  for (unsigned step = 0; step < T - P; ++step) {
    const unsigned i = INV ? P + step : T - 1 - step;
    const int nblk = npairs >> i;
    const int lg = (nblk < 128 ? T - 1 : 7 + i);  // log2(pairs per table per tile)
#pragma unroll
    for (int h = 0; h < nblk; h += 128, ++k) {
      if (k + 1 < ntab) rows_r<true>(sm.rows[(k + 1) & 1], wz_of(k + 1), tid, sm.to_r);
      const M8Base mb = m8_base(sm.tab, q);
      // warps 0-3 computed the next table's rows: they take one pair fewer (c = pairs per thread:
      // threads 128..255 do c + 1, threads 0..127 do c - 1, threads >= 256 of a larger CTA do c;
      // consecutive threads keep consecutive pairs).  Fewer pairs than threads: threads >= 128 only.
      constexpr int NTH = tower_threads(T);
      const int total = NT << lg, c = total / NTH;
      int pp0, cnt, stride;
      if (c == 0) {
        pp0 = tid - 128, stride = 0, cnt = tid >= 128 && tid - 128 < total ? 1 : 0;
      } else if (tid < 128) {
        pp0 = 128 * (c + 1) + tid, stride = 128, cnt = c - 1;
      } else if (tid < 256) {
        pp0 = tid - 128, stride = 128, cnt = c + 1;
      } else {
        pp0 = 256 * c + tid - 256, stride = NTH - 256, cnt = c;
      }
#if FPM_TOWER_IDX2
      // i0 = (blk << (i + 1)) + j = p + (p & ~(2^i - 1)) (+ the group's base, + the operand's
      // tile); every stride is a multiple of 128, so the low four bits of i0 and i1 -- all the
      // swizzle looks at -- are the same for every r
      const int mlg = (1 << lg) - 1, nmi = ~((1 << i) - 1), hb = h << (i + 1);
      const int pf = pp0 & mlg, i0f = hb + pf + (pf & nmi);
      const int sw0 = ((i0f >> 3) & 1) * 7, sw1 = (((i0f + (1 << i)) >> 3) & 1) * 7;
#endif
      for (int r = 0; r < cnt; ++r) {
        const int pp = pp0 + stride * r;
#if FPM_TOWER_IDX2
        const int p = pp & mlg;
        const int i0 = hb + p + (p & nmi) + (NT == 1 ? 0 : (pp >> lg) * n), i1 = i0 + (1 << i);
        const int d = (h + (p >> i)) & 127;  // subfield part of the twiddle (zero iff d == 0)
        const int x0 = i0 ^ sw0, x1 = i1 ^ sw1;
        uint4 u0 = s[x0], u1 = s[x1];
#else
        const int p = pp & ((1 << lg) - 1), tt = pp >> lg;
        const int blk = h + (p >> i), j = p & ((1 << i) - 1);
        const int i0 = (blk << (i + 1)) + j + tt * n, i1 = i0 + (1 << i);
        const int d = blk & 127;  // subfield part of the twiddle (zero iff d == 0)
        const int x0 = tsw(i0), x1 = tsw(i1);
        uint4 u0 = s[x0], u1 = s[x1];
#endif
        if (!INV) {
          uint4 m = m8_mul_r(mb, u1, q);
#ifndef FPM_EXP_NO_SMUL
          if (d) m = x4(m, smul_t(u1, smul_tab(sm.stab, d)));
#endif
          u0 = x4(u0, m);
          u1 = x4(u1, u0);
        } else {
          u1 = x4(u1, u0);
          uint4 m = m8_mul_r(mb, u1, q);
#ifndef FPM_EXP_NO_SMUL
          if (d) m = x4(m, smul_t(u1, smul_tab(sm.stab, d)));
#endif
          u0 = x4(u0, m);
        }
        s[x0] = u0;
        s[x1] = u1;
      }
      __syncthreads();  // lookups of table k and this layer's butterflies done; rows of k+1 ready
      if (k + 1 < ntab) {
#ifndef FPM_EXP_NO_BUILD
        m8_expand(sm.tab, sm.rows[(k + 1) & 1], tid);
#endif
        __syncthreads();
      }
    }
  }
}

// Layers [0, P) of the tile in POLYNOMIAL representation with the IMAD-hole gf_mul (FMA pipe): these
// layers would need 2^(T-8-i) tables each in R, while the shared-memory pipe is the tower pass's
// bottleneck.  Forward: both tiles, one prepared twiddle per butterfly pair.
template <bool INV>
__device__ __forceinline__ void tile_layers_poly(uint4* __restrict__ s, unsigned T, unsigned P, unsigned l,
                                                 uint64_t t, const TwiddleSrc& tw) {
  const int npairs = 1 << (T - 1), n = 1 << T;
  for (unsigned step = 0; step < P; ++step) {
    const unsigned i = INV ? step : P - 1 - step;
    const uint4 Z = twiddle(tw, l, i, t << (T - 1 - i));
    for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
      const int blk = p >> i, j = p & ((1 << i) - 1);
      const int i0 = tsw((blk << (i + 1)) + j), i1 = tsw((blk << (i + 1)) + j + (1 << i));
      const uint4 w = x4(Z, c2p2(tw.c2p, (uint64_t)blk));
      if (!INV) {
        const GfPrep wp = gf_prep(w);
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          uint4 u0 = s[i0 + tt * n], u1 = s[i1 + tt * n];
          u0 = x4(u0, gf_mul_prep(wp, u1));
          u1 = x4(u1, u0);
          s[i0 + tt * n] = u0;
          s[i1 + tt * n] = u1;
        }
      } else {
        uint4 u0 = s[i0], u1 = s[i1];
        u1 = x4(u1, u0);
        u0 = x4(u0, gf_mul(w, u1));
        s[i0] = u0;
        s[i1] = u1;
      }
    }
    __syncthreads();
  }
}

#ifndef FPM_TOWER_FUSE_TOPOLY
#define FPM_TOWER_FUSE_TOPOLY 1
#endif
#ifndef FPM_TOWER_POLY
#define FPM_TOWER_POLY 1
#endif
constexpr unsigned kPolyLayers = FPM_TOWER_POLY;  // bottom tile layers in polynomial representation
size_t tower_smem(unsigned T) { return 2 * ((size_t)1 << T) * sizeof(uint4) + sizeof(TowerSmem); }

// fft_tile_fused2_kernel on R tiles: forward layers [0, T) of both operands (one table per layer
// serves both tiles), the pointwise product (R -> poly by an M8 table of to_poly, gf_mul, poly -> R
// by an M8 table of to_r) and the inverse layers [0, T).
// ntiles / tw_mask: a product's tiles (2^l >> T, each with its own twiddles: tw_mask = ~0), or a
// batch of independent products of 2^T positions each (l = T; ntiles = count, tw_mask = 0: every
// tile is a whole transform with tile 0's twiddles).
// MODE (host-buffer products, whose operand a arrives and is transformed while operand b is still
// being uploaded): 2 = the pre-pass -- forward R layers of the tiles [tile0, ntiles) of ONE EvalVec
// (eb), in place; 1 = the fused pass over tiles whose operand-a tile the pre-pass already
// transformed (forward R layers of operand b only); 0 = the fused pass.
template <unsigned T, int MODE = 0>
__global__ void __launch_bounds__(tower_threads(T), tower_min_blocks(T)) fft_tile_tower_kernel(const uint4* __restrict__ ea,
                                                                          uint4* __restrict__ eb, unsigned l,
                                                                          TwiddleSrc tw, uint64_t ntiles,
                                                                          uint64_t tw_mask, uint64_t tile0) {
  pdl_wait();
  extern __shared__ uint4 s[];
  constexpr int n = 1 << T;
  const int tid = threadIdx.x, q = tid & 7;
  TowerSmem& sm = *reinterpret_cast<TowerSmem*>(s + 2 * n);
  smul_tabs_build(sm.stab, tw.tau, tid);
  if (tid < 128) {
    sm.to_r[to_r_pad(tid)] = __ldg(tw.to_r + tid);
    sm.rows_to_r[tid + (tid >> 3)] = __ldg(tw.to_r + tid);
    sm.rows_to_poly[tid + (tid >> 3)] = __ldg(tw.to_poly + tid);
  }
  const int ntab = tower_tables(T);
  for (uint64_t t = tile0 + blockIdx.x; t < ntiles; t += gridDim.x) {
    uint4* g = eb + (t << T);
    const uint4* ga = MODE == 2 ? nullptr : ea + (t << T);  // (the pre-pass has one EvalVec: eb)
    const uint64_t tt = t & tw_mask;  // the tile's position in its transform (twiddles)
    if (tid < ntab) {  // wz[k]: layer i, group h of this tile: Z(i) ^ C2P(2 * 128 h)
      int i = 0, kk = tid;
      while (kk >= tower_groups(T, (unsigned)i)) kk -= tower_groups(T, (unsigned)i++);
      const uint4 w = x4(twiddle(tw, l, (unsigned)i, tt << (T - 1 - i)), c2p2(tw.c2p, (uint64_t)kk << 7));
      sm.wz[tid] = w;
      if (i >= (int)kPolyLayers) {  // forward sequence position: the groups of the layers above i first
        int pos = kk;
        for (int u = (int)T - 1; u > i; --u) pos += tower_groups(T, (unsigned)u);
        sm.wzf[pos] = w;
      }
    }
    if constexpr (MODE == 2) {  // pre-pass: this EvalVec's forward R layers only
      for (int k = tid; k < n; k += blockDim.x) s[tsw(k)] = g[k];
      __syncthreads();
      tile_layers_r<false, 1, T, kPolyLayers>(s, sm);
      for (int k = tid; k < n; k += blockDim.x) g[k] = s[tsw(k)];
      __syncthreads();
    } else {
    for (int k = tid; k < n; k += blockDim.x) {
      s[tsw(k)] = ga[k];
      s[n + tsw(k)] = g[k];
    }
    __syncthreads();
    if (MODE == 1) tile_layers_r<false, 1, T, kPolyLayers>(s + n, sm);
    else tile_layers_r<false, 2, T, kPolyLayers>(s, sm);
    m8_expand(sm.tab, sm.rows_to_poly, tid);
    __syncthreads();
    const M8Base mb = m8_base(sm.tab, q);
    if (kPolyLayers == 1) {
      // layer 0 forward on both operands, the pointwise product and inverse layer 0 act on the same
      // pair (2p, 2p+1) with the same twiddle: one register pass, one prepared twiddle
      // (FPM_TOWER_FUSE_TOPOLY: the R -> poly lookups of a pair run inside this loop, so that the
      // shared-memory lookups of some warps overlap the IMAD-pipe products of others instead of
      // forming a lookup-only pass with its own barrier)
#if !FPM_TOWER_FUSE_TOPOLY
      for (int k = tid; k < 2 * n; k += blockDim.x) s[k] = m8_mul_r(mb, s[k], q);
      __syncthreads();
#endif
      const uint4 Z = twiddle(tw, l, 0, tt << (T - 1));
      for (int p = tid; p < n / 2; p += blockDim.x) {
        const int i0 = tsw(2 * p), i1 = tsw(2 * p + 1);
        const GfPrep wp = gf_prep(x4(Z, c2p2(tw.c2p, (uint64_t)p)));
        uint4 a0 = s[i0], a1 = s[i1], b0 = s[n + i0], b1 = s[n + i1];
#if FPM_TOWER_FUSE_TOPOLY
        a0 = m8_mul_r(mb, a0, q);
        a1 = m8_mul_r(mb, a1, q);
        b0 = m8_mul_r(mb, b0, q);
        b1 = m8_mul_r(mb, b1, q);
#endif
        a0 = x4(a0, gf_mul_prep(wp, a1));
        a1 = x4(a1, a0);
        b0 = x4(b0, gf_mul_prep(wp, b1));
        b1 = x4(b1, b0);
        uint4 c0 = gf_mul(a0, b0), c1 = gf_mul(a1, b1);
        c1 = x4(c1, c0);
        c0 = x4(c0, gf_mul_prep(wp, c1));
        s[i0] = c0;
        s[i1] = c1;
      }
      __syncthreads();
    } else if (kPolyLayers) {
      for (int k = tid; k < 2 * n; k += blockDim.x) s[k] = m8_mul_r(mb, s[k], q);
      __syncthreads();
      tile_layers_poly<false>(s, T, kPolyLayers, l, tt, tw);
      for (int k = tid; k < n; k += blockDim.x) s[k] = gf_mul(s[k], s[n + k]);
      __syncthreads();
      tile_layers_poly<true>(s, T, kPolyLayers, l, tt, tw);
    } else {
      for (int k = tid; k < n; k += blockDim.x) s[k] = gf_mul(m8_mul_r(mb, s[k], q), m8_mul_r(mb, s[n + k], q));
      __syncthreads();
    }
    m8_expand(sm.tab, sm.rows_to_r, tid);
    __syncthreads();
    for (int k = tid; k < n; k += blockDim.x) s[k] = m8_mul_r(mb, s[k], q);
    {  // the next tile's operands into L2 while this tile's inverse layers run (128-byte lines)
      const uint64_t tn = t + gridDim.x;
      if (tn < ntiles) {
        constexpr int lines = n * 16 / 128;
        for (int k = tid; k < 2 * lines; k += blockDim.x) {
          const char* p = reinterpret_cast<const char*>((k < lines ? ea : eb) + (tn << T)) + 128 * (k % lines);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
        }
      }
    }
    // (tile_layers_r's first barrier orders these stores before its butterflies)
    tile_layers_r<true, 1, T, kPolyLayers>(s, sm);
    for (int k = tid; k < n; k += blockDim.x) g[k] = s[tsw(k)];
    __syncthreads();
    }  // (MODE != 2)
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// Exchanged layer of the sharded FFT: all local elements share one twiddle w (polynomial form);
// R: elements in the tower representation (table built in R).
template <bool INV, bool R>
// out: where the result goes -- `mine` itself after an NCCL exchange, or the other buffer of a
// ping-pong pair when `theirs` is the partner GPU's memory read over NVLink (fpm_bfly_pair_peer_dev:
// the exchange is these loads, fused with the butterfly; nothing is staged).
__global__ void __launch_bounds__(256) fft_pair_kernel(const uint4* mine, const uint4* __restrict__ theirs,
                                                       uint4* out, uint64_t n, uint4 w, int side, int ppc,
                                                       const uint4* to_r) {
  pdl_wait();
  extern __shared__ uint4 tab[];
  __shared__ uint4 rows[144];
  if (R) {
    rows_r<false>(rows, w, threadIdx.x, to_r);
    __syncthreads();
    m8_expand(tab, rows, threadIdx.x);
    __syncthreads();
  } else {
    m8_build(tab, rows, w, threadIdx.x);
  }
  const int copy = threadIdx.x & 7;
  const uint64_t k0 = (uint64_t)blockIdx.x * ppc;
  for (int k = threadIdx.x; k < ppc; k += blockDim.x) {
    const uint64_t e = k0 + k;
    if (e >= n) break;
    const uint4 a = mine[e], b = theirs[e];
    uint4 r;
    if (!INV) {  // p0' = p0 + w p1 ; p1' = p1 + p0'
      r = side == 0 ? x4(a, m8_mul(tab, b, copy)) : xor3(a, b, m8_mul(tab, a, copy));
    } else {     // p1' = p1 + p0 ; p0' = p0 + w p1'
      r = side == 0 ? x4(a, m8_mul(tab, x4(a, b), copy)) : x4(a, b);
    }
    out[e] = r;
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

__global__ void pointwise_kernel(const uint4* __restrict__ u, const uint4* __restrict__ v, uint4* __restrict__ out,
                                 uint64_t n) {
  pdl_wait();
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
    out[k] = gf_mul(u[k], v[k]);
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

int sms() {
  int dev, n;
  FPM_CUDA(cudaGetDevice(&dev));
  FPM_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

template <class K>
void set_smem(K kernel, size_t bytes) {
  FPM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

}  // namespace

// Tile depth: layers below T run in shared-memory tiles (generic multiplies, M8 tables for layers
// >= kTabLayer), layers >= T in radix-4 M8-table passes.  B200 sweeps (ms, T = 10 / 11):
// 2^26-bit 1.269 / 1.262, 2^28 4.375 / 4.320, 2^30 17.14 / 16.93, 2^32 73.0 / 71.8; 2^24 0.457 /
// 0.470; below 2^18 elements T = 8 keeps >= 2^10 tiles in flight.
bool tile_fused2_enabled(unsigned T);

int tile_log2_knob() {
  static const int knob = [] {
    const char* e = std::getenv("FPM_TILE_LOG2");  // tuning override (8..12)
    return e ? std::max(8, std::min(kTileMax, std::atoi(e))) : 0;
  }();
  return knob;
}

unsigned fft_tile_log2(unsigned l) {
  const int knob = tile_log2_knob();
  const unsigned cap = knob ? (unsigned)knob : (l >= 20 ? 11u : l >= 18 ? 10u : 8u);
  return l < cap ? l : cap;
}

// The product pipeline's tile depth: with both operands' tile layers fused (fft_tile_fused2_kernel,
// two 2^T tiles + tables per CTA) T = 10 keeps two CTAs per SM (2^32-bit product: 57.5 ms, vs
// 57.7 unfused at T = 11 and 60.1 fused at T = 11 with one CTA per SM).
// Round 2: on tower tiles, T = 12 (one 512-thread CTA per SM, 2^10 or more tiles) moves two layers
// out of the HBM-bound radix-4 passes and shares each layer-(>= 4) table over 4096 positions
// (2^32-bit product: 49.25 -> 46.97 ms).
unsigned pipeline_tile_log2(unsigned l) {
#ifndef FPM_TOWER_T
#define FPM_TOWER_T 12
#endif
  if (!tile_log2_knob() && l >= 22 && tile_tower_enabled(FPM_TOWER_T)) return FPM_TOWER_T;
  if (!tile_log2_knob() && l >= 20 && tile_fused2_enabled(10)) return 10;
  return fft_tile_log2(l);
}
bool pipeline_fuses_operands(unsigned T) { return tile_fused2_enabled(T) || (T == 12 && tile_tower_enabled(12)); }
bool pipeline_tower(unsigned T) { return pipeline_fuses_operands(T) && tile_tower_enabled(T); }

TwiddleSrc make_twiddle_src(int device, unsigned l, U128 base) {
  if (l > (unsigned)kMaxLayers) throw Error(kInvalid, "butterfly: too many layers");
  TwiddleSrc tw{};
  const DeviceTables& dt = device_tables(device);
  tw.c2p = dt.c2p;
  tw.to_r = dt.to_r;
  tw.to_poly = dt.to_poly;
  const TowerTables& tt = tower_tables();
  for (int b = 0; b < 8; ++b) tw.tau |= (uint64_t)tt.tau[b] << (8 * b);
  const FieldTables& ft = field_tables();
  for (unsigned i = 0; i < l; ++i) {
    U128 c;  // base >> i (Cantor coordinates)
    c.lo = i == 0 ? base.lo : (i < 64 ? (base.lo >> i) | (base.hi << (64 - i)) : base.hi >> (i - 64));
    c.hi = i < 64 ? (i == 0 ? base.hi : base.hi >> i) : 0;
    const U128 p = host_cantor_to_poly(ft, c);
    tw.layer[i] = make_uint4((uint32_t)p.lo, (uint32_t)(p.lo >> 32), (uint32_t)p.hi, (uint32_t)(p.hi >> 32));
  }
  return tw;
}

template <bool R>
void top_passes(uint4* ev, unsigned l, unsigned T, bool inverse, const TwiddleSrc& tw, cudaStream_t s,
                uint4* ev2 = nullptr) {
  const size_t smem = kM8Uint4 * sizeof(uint4);
  static PerDeviceOnce attr;
  attr.run([&] { set_smem(fft_top_kernel<false, R>, smem); set_smem(fft_top_kernel<true, R>, smem); });
  // Pairs per CTA: 4096 amortise the 64 KiB table build; smaller layers still fill 2 CTAs/SM.
  static PerDeviceOnce attr4;
  attr4.run([&] {
    set_smem(fft_top4_kernel<false, R>, kTop4Smem);
    set_smem(fft_top4_kernel<true, R>, kTop4Smem);
    set_smem(fft_top4_kernel<false, R, 512>, kTop4Smem);
    set_smem(fft_top4_kernel<true, R, 512>, kTop4Smem);
  });
  const uint64_t pairs = ((uint64_t)1 << l) / 2;
  uint64_t ppc = 4096;
  while (ppc > (l >= 16 ? 256u : 128u) && pairs / ppc < (uint64_t)sms() * 2) ppc /= 2;
  const uint64_t ctas = pairs / ppc;
  if (T < 8 || ctas == 0) throw Error(kInvalid, "butterfly_top: layer too small for the table layer kernel");
  auto radix2 = [&](unsigned i) {
    const uint64_t p = std::min<uint64_t>(ppc, (uint64_t)1 << i);  // a CTA stays inside one block
    for (uint4* e : {ev, ev2}) {
      if (!e) continue;
      if (!inverse) launch_k(fft_top_kernel<false, R>, dim3((unsigned)(pairs / p)), dim3(256), smem, s, e, l, i, (int)p, tw);
      else launch_k(fft_top_kernel<true, R>, dim3((unsigned)(pairs / p)), dim3(256), smem, s, e, l, i, (int)p, tw);
      FPM_LAUNCH_CHECK();
    }
  };
  // layer pairs (i+1, i) from the top down (forward) / bottom up (inverse); an odd count leaves
  // the lowest top layer T to the one-layer kernel.
  // Quads per CTA: up to 16384 amortise the three 64 KiB table builds at 2^32 bits; small transforms go
  // down to 128 quads so that the pass spreads over the SMs (at l = 14 a 1024-quad floor left 4 CTAs
  // per pass, ~10 us each, dominated by one CTA's table builds).
  const uint64_t quads = ((uint64_t)1 << l) / 4;
  const uint64_t qmin = l >= 16 ? 1024 : 128;  // l = 18: 1024 beats 128 (0.104 vs 0.154 ms of passes)
#ifndef FPM_TOP4_QMAX
#define FPM_TOP4_QMAX 16384  // 2^32-bit product: 46.09 -> 45.72 ms vs 8192 (half the table builds)
#endif
  uint64_t qpc = FPM_TOP4_QMAX;
#ifndef FPM_TOP4_WAVES
#define FPM_TOP4_WAVES 4
#endif
  while (qpc > qmin && quads / qpc < (uint64_t)sms() * FPM_TOP4_WAVES) qpc /= 2;
  auto radix4 = [&](unsigned i) {
    const unsigned q = (unsigned)std::min<uint64_t>(qpc, (uint64_t)1 << i);
    // forward: 512 threads (pre-rotated lookups without spills; 11.04 vs 11.22 ms at 2^32 bits);
    // inverse: 768 (5.48 vs 5.51).  FPM_TOP4_THREADS=512/768 forces one width for both.
    static const int knob = [] {
      const char* e = std::getenv("FPM_TOP4_THREADS");
      return e ? std::atoi(e) : 0;
    }();
    const int nt = knob == 512 || knob == 768 ? knob : (inverse ? kTop4Threads : 512);
    if (nt == 512) {
      if (!inverse) launch_k(fft_top4_kernel<false, R, 512>, dim3((unsigned)(quads / q)), dim3(512), kTop4Smem, s, ev, l, i, (int)q, tw, ev2);
      else launch_k(fft_top4_kernel<true, R, 512>, dim3((unsigned)(quads / q)), dim3(512), kTop4Smem, s, ev, l, i, (int)q, tw, ev2);
    } else {
      if (!inverse) launch_k(fft_top4_kernel<false, R>, dim3((unsigned)(quads / q)), dim3(kTop4Threads), kTop4Smem, s, ev, l, i, (int)q, tw, ev2);
      else launch_k(fft_top4_kernel<true, R>, dim3((unsigned)(quads / q)), dim3(kTop4Threads), kTop4Smem, s, ev, l, i, (int)q, tw, ev2);
    }
    FPM_LAUNCH_CHECK();
  };
  const unsigned n = l - T;
#ifndef FPM_TOP8
#define FPM_TOP8 1
#endif
  if (R && FPM_TOP8 && n >= 3) {
    // tower representation: three layers per pass (fft_top8_kernel), the remainder at the bottom
    static PerDeviceOnce attr8;
    attr8.run([&] {
      set_smem(fft_top8_kernel<false>, kTop8Smem);
      set_smem(fft_top8_kernel<true>, kTop8Smem);
    });
    const uint64_t octs = ((uint64_t)1 << l) / 8;
#ifndef FPM_TOP8_OMAX
#define FPM_TOP8_OMAX (FPM_TOP4_QMAX / 2)
#endif
    uint64_t opc = FPM_TOP8_OMAX;
    while (opc > 512 && octs / opc < (uint64_t)sms() * FPM_TOP4_WAVES) opc /= 2;
    auto radix8 = [&](unsigned i) {
      const unsigned o = (unsigned)std::min<uint64_t>(opc, (uint64_t)1 << i);
      if (!inverse) launch_k(fft_top8_kernel<false>, dim3((unsigned)(octs / o)), dim3(512), kTop8Smem, s, ev, l, i, (int)o, tw, ev2);
      else launch_k(fft_top8_kernel<true>, dim3((unsigned)(octs / o)), dim3(512), kTop8Smem, s, ev, l, i, (int)o, tw, ev2);
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

void butterfly_top_device(uint4* ev, unsigned l, unsigned T, bool inverse, const TwiddleSrc& tw, cudaStream_t s,
                          bool tower, uint4* ev2) {
  if (l <= T) return;
  if (tower) top_passes<true>(ev, l, T, inverse, tw, s, ev2);
  else top_passes<false>(ev, l, T, inverse, tw, s, ev2);
}

// One thread per butterfly of a tile layer (2^(T-1) pairs), at most 256: small tiles run more CTAs
// per SM instead of idling half the threads.
int tile_threads(unsigned T) { return T >= 9 ? 256 : std::max(32, 1 << (T - 1)); }

// Tile launch geometry: tables for layers >= kTabLayer when the tile runs 256 threads (T >= 9;
// FPM_TILE_TABLES=0 disables them for comparison).
struct TileCfg {
  int threads, use_tab;
  size_t smem;
};
TileCfg tile_cfg(unsigned l, unsigned T) {
  static const bool tables = [] {
    const char* e = std::getenv("FPM_TILE_TABLES");
    return !(e && e[0] == '0');
  }();
  TileCfg c;
  c.threads = tile_threads(T);
  c.use_tab = tables && T > kTabLayer && c.threads == 256;
  c.smem = ((size_t)1 << T) * sizeof(uint4) + (c.use_tab ? (kM8Uint4 + 144) * sizeof(uint4) : 0);
  return c;
}
constexpr size_t kTileSmemMax = ((size_t)1 << kTileMax << 4) + (kM8Uint4 + 144) * sizeof(uint4);

void butterfly_tile_device(uint4* ev, unsigned l, unsigned T, bool inverse, const TwiddleSrc& tw, cudaStream_t s) {
  if (T == 0) return;
  static PerDeviceOnce attr;
  attr.run([&] {
    set_smem(fft_tile_kernel<false>, kTileSmemMax);
    set_smem(fft_tile_kernel<true>, kTileSmemMax);
  });
  const TileCfg c = tile_cfg(l, T);
  const uint64_t ntiles = ((uint64_t)1 << l) >> T;
  if (!inverse)
    launch_k(fft_tile_kernel<false>, dim3(resident_grid(fft_tile_kernel<false>, c.threads, c.smem, ntiles)), dim3(c.threads), c.smem, s, ev, l, T, tw, c.use_tab);
  else
    launch_k(fft_tile_kernel<true>, dim3(resident_grid(fft_tile_kernel<true>, c.threads, c.smem, ntiles)), dim3(c.threads), c.smem, s, ev, l, T, tw, c.use_tab);
  FPM_LAUNCH_CHECK();
}

void butterfly_tile_fused_device(const uint4* ea, uint4* eb, unsigned l, unsigned T, const TwiddleSrc& tw,
                                 cudaStream_t s) {
  static PerDeviceOnce attr;
  attr.run([&] { set_smem(fft_tile_fused_kernel, kTileSmemMax); });
  const TileCfg c = tile_cfg(l, T);
  const int grid = resident_grid(fft_tile_fused_kernel, c.threads, c.smem, ((uint64_t)1 << l) >> T);
  launch_k(fft_tile_fused_kernel, dim3(grid), dim3(c.threads), c.smem, s, ea, eb, l, T, tw, c.use_tab);
  FPM_LAUNCH_CHECK();
}

// Both operands' tile layers + pointwise + inverse tile layers in one pass (fft_tile_fused2_kernel);
// T >= 10 (tables), FPM_FUSE_AB=0 disables it.
bool tile_fused2_enabled(unsigned T) {
  static const bool on = [] {
    const char* e = std::getenv("FPM_FUSE_AB");
    return !(e && e[0] == '0');
  }();
#ifndef FPM_FUSE2_MIN_T
#define FPM_FUSE2_MIN_T 8  // config 1 (T = 8): one launch fewer, 0.126 -> 0.124 ms
#endif
  return on && T >= FPM_FUSE2_MIN_T && T <= 11;
}

void butterfly_tile_fused2_device(const uint4* ea, uint4* eb, unsigned l, unsigned T, const TwiddleSrc& tw,
                                  cudaStream_t s) {
  const size_t smem = (2 * ((size_t)1 << T) + kM8Uint4 + 144) * sizeof(uint4);
  static PerDeviceOnce attr;
  attr.run([&] { set_smem(fft_tile_fused2_kernel, (2 * ((size_t)1 << 11) + kM8Uint4 + 144) * sizeof(uint4)); });
  const int grid = resident_grid(fft_tile_fused2_kernel, kTile2Threads, smem, ((uint64_t)1 << l) >> T);
  launch_k(fft_tile_fused2_kernel, dim3(grid), dim3(kTile2Threads), smem, s, ea, eb, l, T, tw);
  FPM_LAUNCH_CHECK();
}

// The tower tile pass (fft_tile_tower_kernel) for the product pipeline; FPM_TOWER=0 disables it.
bool tile_tower_enabled(unsigned T) {
  static const bool on = [] {
    const char* e = std::getenv("FPM_TOWER");
    return !(e && e[0] == '0');
  }();
  return on && T >= 10 && T <= 12;
}

void tower_set_smem() {
  static PerDeviceOnce attr;
  attr.run([&] {
    set_smem(fft_tile_tower_kernel<10>, tower_smem(10));
    set_smem(fft_tile_tower_kernel<11>, tower_smem(11));
    set_smem(fft_tile_tower_kernel<12>, tower_smem(12));
    set_smem(fft_tile_tower_kernel<12, 1>, tower_smem(12));
    set_smem(fft_tile_tower_kernel<12, 2>, tower_smem(12));
  });
}

// pre_tiles: operand a's tiles [0, pre_tiles) already hold their forward R layers
// (butterfly_tile_tower_pre_device); T = 12 only.
void butterfly_tile_tower_device(const uint4* ea, uint4* eb, unsigned l, unsigned T, const TwiddleSrc& tw,
                                 cudaStream_t s, uint64_t batch, uint64_t pre_tiles) {
  if (T < 10 || T > 12 || l < T) throw Error(kInvalid, "tower tile pass: T must be 10, 11 or 12");
  if (batch && l != T) throw Error(kInvalid, "tower tile pass: a batch of transforms needs l = T");
  tower_set_smem();
  const size_t smem = tower_smem(T);
  auto kern = T == 10 ? fft_tile_tower_kernel<10> : T == 11 ? fft_tile_tower_kernel<11> : fft_tile_tower_kernel<12>;
  const uint64_t ntiles = batch ? batch : ((uint64_t)1 << l) >> T;
  const uint64_t mask = batch ? (uint64_t)0 : ~(uint64_t)0;
  if (pre_tiles) {
    if (T != 12 || batch || pre_tiles > ntiles) throw Error(kInvalid, "tower tile pass: pre-passed tiles need T = 12");
    const int g1 = resident_grid(fft_tile_tower_kernel<12, 1>, tower_threads(T), smem, pre_tiles);
    launch_k(fft_tile_tower_kernel<12, 1>, dim3(g1), dim3(tower_threads(T)), smem, s, ea, eb, l, tw, pre_tiles, mask,
             (uint64_t)0);
    FPM_LAUNCH_CHECK();
    if (pre_tiles == ntiles) return;
  }
  const int grid = resident_grid(kern, tower_threads(T), smem, ntiles - pre_tiles);
  launch_k(kern, dim3(grid), dim3(tower_threads(T)), smem, s, ea, eb, l, tw, ntiles, mask, pre_tiles);
  FPM_LAUNCH_CHECK();
}

// Host-buffer products: the share of operand a's tiles whose forward R layers run ahead of the fused
// pass, in the window between the end of operand a's transforms and the arrival of operand b
// (FPM_PRE_A_FRAC, default 0.5; 0 disables).  A whole number of waves of the resident grid.
// Measured (host-buffer 2^33-bit products, tools/e2e_time.py): 75.0-75.2 ms without, 73.65-73.97
// with 0.5, 73.9-74.0 with 0.3 / 0.4, 74.5-74.6 with 0.6 / 0.7; no gain for 2^31- / 2^32-bit
// products (39.1-39.2 vs 39.4 ms, 19.5 vs 19.3-19.6), so only l >= 26 takes it (FPM_PRE_A_MIN_L).
uint64_t tower_pre_tiles(unsigned l, unsigned T) {
  static const unsigned min_l = [] {
    const char* e = std::getenv("FPM_PRE_A_MIN_L");
    return e ? (unsigned)std::atoi(e) : 26u;
  }();
  if (l < min_l) return 0;
  static const double frac = [] {
    const char* e = std::getenv("FPM_PRE_A_FRAC");
    return e ? std::atof(e) : 0.5;
  }();
  if (T != 12 || l < T || !(frac > 0)) return 0;
  tower_set_smem();
  const uint64_t ntiles = ((uint64_t)1 << l) >> T;
  const uint64_t grid = (uint64_t)resident_grid(fft_tile_tower_kernel<12, 2>, tower_threads(T), tower_smem(T), ntiles);
  const uint64_t waves = (uint64_t)(std::min(frac, 1.0) * (double)ntiles / (double)grid);
  return std::min(ntiles, waves * grid);
}

// Forward R layers of the tiles [0, pre_tiles) of one EvalVec, in place (fft_tile_tower_kernel<12, 2>).
void butterfly_tile_tower_pre_device(uint4* ev, unsigned l, unsigned T, const TwiddleSrc& tw, uint64_t pre_tiles,
                                     cudaStream_t s) {
  if (!pre_tiles) return;
  if (T != 12 || l < T || pre_tiles > (((uint64_t)1 << l) >> T)) throw Error(kInvalid, "tower pre-pass: T = 12 only");
  tower_set_smem();
  const size_t smem = tower_smem(T);
  const int grid = resident_grid(fft_tile_tower_kernel<12, 2>, tower_threads(T), smem, pre_tiles);
  launch_k(fft_tile_tower_kernel<12, 2>, dim3(grid), dim3(tower_threads(T)), smem, s, (const uint4*)nullptr, ev, l, tw,
           pre_tiles, ~(uint64_t)0, (uint64_t)0);
  FPM_LAUNCH_CHECK();
}

void butterfly_device(uint4* ev, unsigned l, U128 base, bool inverse, cudaStream_t s) {
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const TwiddleSrc tw = make_twiddle_src(dev, l, base);
  const unsigned T = fft_tile_log2(l);
  if (!inverse) {
    butterfly_top_device(ev, l, T, false, tw, s);
    butterfly_tile_device(ev, l, T, false, tw, s);
  } else {
    butterfly_tile_device(ev, l, T, true, tw, s);
    butterfly_top_device(ev, l, T, true, tw, s);
  }
}

void bfly_pair_device(uint4* mine, const uint4* theirs, uint64_t n, U128 w, int side, bool inverse, cudaStream_t s,
                      bool tower, uint4* out) {
  if (!out) out = mine;
  if (!n) return;
  const size_t smem = kM8Uint4 * sizeof(uint4);
  static PerDeviceOnce attr;
  attr.run([&] {
    set_smem(fft_pair_kernel<false, false>, smem);
    set_smem(fft_pair_kernel<true, false>, smem);
    set_smem(fft_pair_kernel<false, true>, smem);
    set_smem(fft_pair_kernel<true, true>, smem);
  });
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const uint4* to_r = device_tables(dev).to_r;
  uint64_t ppc = 4096;
  while (ppc > 256 && n / ppc < (uint64_t)sms() * 2) ppc /= 2;
  const unsigned ctas = (unsigned)((n + ppc - 1) / ppc);
  const uint4 w4 = make_uint4((uint32_t)w.lo, (uint32_t)(w.lo >> 32), (uint32_t)w.hi, (uint32_t)(w.hi >> 32));
  if (tower) {
    if (!inverse) launch_k(fft_pair_kernel<false, true>, dim3(ctas), dim3(256), smem, s, mine, theirs, out, n, w4, side, (int)ppc, to_r);
    else launch_k(fft_pair_kernel<true, true>, dim3(ctas), dim3(256), smem, s, mine, theirs, out, n, w4, side, (int)ppc, to_r);
  } else {
    if (!inverse) launch_k(fft_pair_kernel<false, false>, dim3(ctas), dim3(256), smem, s, mine, theirs, out, n, w4, side, (int)ppc, to_r);
    else launch_k(fft_pair_kernel<true, false>, dim3(ctas), dim3(256), smem, s, mine, theirs, out, n, w4, side, (int)ppc, to_r);
  }
  FPM_LAUNCH_CHECK();
}

void pointwise_device(const uint4* u, const uint4* v, uint4* out, size_t n, cudaStream_t s) {
  if (!n) return;
  const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)sms() * 16);
  launch_k(pointwise_kernel, dim3(grid), dim3(256), 0, s, u, v, out, n);
  FPM_LAUNCH_CHECK();
}

}  // namespace fpm
