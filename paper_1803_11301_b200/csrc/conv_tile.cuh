// conv_tile.cuh -- basis conversion of 2^r-bit chunks (r <= 16) inside one 8 KiB shared-memory tile.
//
// The reference conversion (proj/src/basis_convert.cpp) is build_schedule's fold-pass list; its
// recursion is  conv(2^r) = C_rows(conv(256)) o C_cols(conv(D)) o L1(256, D)  with the chunk seen as
// D = 2^(r-8) rows of 256 bits.  L1 (the level passes, a radix-y Taylor expansion, y = x^256 + x)
// has the closed form (Lucas' theorem; verified against the pass list in tools/models/bc_model.py):
//     G_k = sum_{d superset of k} x^(d-k) F_d ,   g_k = (G_k mod x^256) + x (G_k div x^256) + (G_{k-1} div x^256)
// and its inverse  F'_d = sum_{k superset of d} x^(k-d) g_k ,  F_d = (F'_d mod x^256) + (F'_{d-1} div x^256).
// Skewing row d left by d bits turns the shifted subset sums into plain XOR butterflies over the row
// index (shuffles for row distances < 32, shared memory above).  C_cols is conv(D) with whole rows
// as units (pure row XORs), run as conv_regs on the columns of the transposed tile; C_rows is
// conv(256) in registers (conv_regs_gen.cuh).
//
// Tile layout: 256 rows x 8 words (row-major); thread t owns row t.  A tile holds 2^(16-r)
// independent chunks (r >= 8) or 256 rows each holding 2^(8-r) chunks (r < 8).
#pragma once
#include <cstdint>

#include "conv_regs_gen.cuh"
#include "warp_bits.cuh"

namespace fpm {

constexpr int kTileRows = 256;
#ifndef FPM_UNIT_CONV_TILE
#define FPM_UNIT_CONV_TILE 0  // measured: forward 2.29 -> 2.23 ms, inverse 1.56 -> 1.92 ms (off)
#endif
constexpr bool kUnitConvTile = FPM_UNIT_CONV_TILE;
constexpr int kScPitch = 17;  // scratch row pitch (words) for 512-bit widened rows

// 16-word registers shifted by whole words (ws < 16), left (towards higher words) or right, by
// three/four conditional stages: no local memory, no shared-memory round trip.  ws is
// warp-uniform in the callers (d >> 5 with 32 consecutive rows per warp).
__device__ __forceinline__ void words_shl16(uint32_t (&t)[16], int ws) {
#pragma unroll
  for (int st = 8; st >= 1; st >>= 1)
    if (ws & st) {
#pragma unroll
      for (int i = 15; i >= 0; --i) t[i] = i >= st ? t[i - st] : 0u;
    }
}
__device__ __forceinline__ void words_shr16(uint32_t (&t)[16], int ws) {
#pragma unroll
  for (int st = 8; st >= 1; st >>= 1)
    if (ws & st) {
#pragma unroll
      for (int i = 0; i < 16; ++i) t[i] = i + st < 16 ? t[i + st] : 0u;
    }
}

// L1(256, 2^g) forward (carry) or inverse (overflow) on the chunk rows; m = this thread's row.
template <bool INV>
__device__ __forceinline__ void l1_tile(uint32_t (&m)[8], uint32_t* sc, int g, int d) {
  const int tid = threadIdx.x;
  uint32_t* my = sc + tid * kScPitch;
  const int ws = d >> 5, bs = d & 31;
  // skew: the row m << d -- the bit part (bs) in registers, the word part (ws) as the store offset
  // into the 16-word shared row (no register shuffling)
  uint32_t W9[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) W9[i] = __funnelshift_l(i ? m[i - 1] : 0u, i < 8 ? m[i] : 0u, bs);
  // subset-zeta over the g low row bits (rows with bit b clear ^= row | 2^b), as register-local
  // stages in two transposed mappings with shared-memory exchanges (row-major sc, pitch 17):
  //   A: thread (c = tid & 15, r0 = tid >> 4) holds word c of rows r0 + 16k -> row bits 4..7 local
  //   B: thread (c, r1 = tid >> 4) holds word c of rows 16 r1 + k         -> row bits 0..3 local
  // Chunk boundaries (2^g rows) are respected by running only stages b < g.
  {
    const int c = tid & 15, rr = tid >> 4;
    uint32_t v[16];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 16; ++i) my[i] = 0u;
#pragma unroll
    for (int i = 0; i < 9; ++i) my[ws + i] = W9[i];
    __syncthreads();
    if (g > 4) {
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = sc[(rr + 16 * k) * kScPitch + c];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (4 + j < g) {
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (!(k >> j & 1)) v[k] ^= v[k | (1 << j)];
        }
#pragma unroll
      for (int k = 0; k < 16; ++k) sc[(rr + 16 * k) * kScPitch + c] = v[k];
      __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = sc[(16 * rr + k) * kScPitch + c];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < g) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (!(k >> j & 1)) v[k] ^= v[k | (1 << j)];
      }
#pragma unroll
    for (int k = 0; k < 16; ++k) sc[(16 * rr + k) * kScPitch + c] = v[k];
    __syncthreads();
  }
  // unskew: G = (skewed row) >> d -- the word part as the load offset, the bit part in registers
  uint32_t G[16];
  {
    uint32_t U[17];
#pragma unroll
    for (int j = 0; j < 17; ++j) U[j] = j + ws < 16 ? my[j + ws] : 0u;
#pragma unroll
    for (int i = 0; i < 16; ++i) G[i] = __funnelshift_r(U[i], U[i + 1], bs);
  }
  // carry (forward) / overflow (inverse) with the previous row's high half H_{d-1}
  // (no barrier before these stores: since the last one every thread has read only its own row)
#pragma unroll
  for (int i = 0; i < 8; ++i) my[i] = G[8 + i];
  __syncthreads();
  uint32_t prevH[8];
  const uint32_t* pr = sc + (tid - 1) * kScPitch;
#pragma unroll
  for (int i = 0; i < 8; ++i) prevH[i] = d >= 1 ? pr[i] : 0u;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t v = G[i] ^ prevH[i];
    if (!INV) v ^= (G[8 + i] << 1) | (i ? (G[7 + i] >> 31) : 0u);  // x * H_d
    m[i] = v;
  }
}

// conv(2^g) over the chunk's rows (rows as units): pass (S, D) -> rows q of each S-span with
// q in [S/2-D, S-D) get row q+D (and row q+2D if q+2D < S, forward).
// rowpasses over W adjacent 8-word columns at once (W * 32 B per row and barrier); tile is
// 256 x kRowPitchW(W) words (one uint4 of padding keeps the 16 B stores conflict-free).
template <int W>
constexpr int kRowPitchW = 8 * W + 4;
template <bool INV, int W>
__device__ __forceinline__ void rowpasses_w(uint32_t (&m)[W][8], uint32_t* tile, int g, int d) {
  const int tid = threadIdx.x;
  const int n = kRowSchedN[g];
  constexpr int P = kRowPitchW<W>;
  for (int kk = 0; kk < n; ++kk) {
    const int k = INV ? n - 1 - kk : kk;
    const int S = kRowSchedS[g][k], D = kRowSchedD[g][k];
    __syncthreads();
    uint4* my4 = reinterpret_cast<uint4*>(tile + tid * P);
#pragma unroll
    for (int c = 0; c < W; ++c) {
      my4[2 * c] = make_uint4(m[c][0], m[c][1], m[c][2], m[c][3]);
      my4[2 * c + 1] = make_uint4(m[c][4], m[c][5], m[c][6], m[c][7]);
    }
    __syncthreads();
    const int q = d & (S - 1);
    if (q >= S / 2 - D && q < S - D) {
      const uint4* s1 = reinterpret_cast<const uint4*>(tile + (tid + D) * P);
      const uint4* s2 = reinterpret_cast<const uint4*>(tile + (tid + 2 * D) * P);
      const bool two = !INV && q + 2 * D < S;
#pragma unroll
      for (int c = 0; c < W; ++c) {
        uint4 a = s1[2 * c], b = s1[2 * c + 1];
        if (two) {
          const uint4 e = s2[2 * c], f = s2[2 * c + 1];
          a.x ^= e.x; a.y ^= e.y; a.z ^= e.z; a.w ^= e.w;
          b.x ^= f.x; b.y ^= f.y; b.z ^= f.z; b.w ^= f.w;
        }
        m[c][0] ^= a.x; m[c][1] ^= a.y; m[c][2] ^= a.z; m[c][3] ^= a.w;
        m[c][4] ^= b.x; m[c][5] ^= b.y; m[c][6] ^= b.z; m[c][7] ^= b.w;
      }
    }
  }
}

// conv16 over 16 register values (build_schedule(16): (16,6), (8,3), (16,4), (4,1)); increasing q
// reads every source before it is overwritten (sources sit above their targets).
template <int S, int D, bool INV>
__device__ __forceinline__ void conv_pass16(uint32_t (&x)[16]) {
#pragma unroll
  for (int base = 0; base < 16; base += S)
#pragma unroll
    for (int q = S / 2 - D; q < S - D; ++q) {
      uint32_t v = x[base + q + D];
      if (!INV && q + 2 * D < S) v ^= x[base + q + 2 * D];
      x[base + q] ^= v;
    }
}
template <bool INV>
__device__ __forceinline__ void conv16_vals(uint32_t (&x)[16]) {
  if (!INV) {
    conv_pass16<16, 6, false>(x);
    conv_pass16<8, 3, false>(x);
    conv_pass16<16, 4, false>(x);
    conv_pass16<4, 1, false>(x);
  } else {
    conv_pass16<4, 1, true>(x);
    conv_pass16<16, 4, true>(x);
    conv_pass16<8, 3, true>(x);
    conv_pass16<16, 6, true>(x);
  }
}

// zeta over the 4 digit bits (superset sums): x[d] ^= x[d | 2^b] for d without bit b.
__device__ __forceinline__ void zeta16_vals(uint32_t (&x)[16]) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int d = 0; d < 16; ++d)
      if (!(d >> j & 1)) x[d] ^= x[d | (1 << j)];
}

// conv(256) over the tile's 256 sub-rows as units (C_cols at g = 8) WITHOUT transposing the tile:
// the unit-level recursion conv(256) = C_rows(conv16 over v) o C_cols(conv16 over d) o L1(16, 16)
// (units u = 16 d + v, unit skew), as conv256_units_kernel, on 16-bit half-columns: thread
// (r = tid / 16, hc = tid % 16) holds half-word hc of 16 units per phase.  tile: >= 2048 words;
// z: >= 4096 words (16 x 32 slots x 16 half-words).  All 256 threads call it.
template <bool INV>
__device__ __forceinline__ void unitconv256_tile(uint32_t (&m)[8], uint32_t* tile, uint32_t* z) {
  const int tid = threadIdx.x, r = tid >> 4, hc = tid & 15;
  uint16_t* t16 = reinterpret_cast<uint16_t*>(tile);  // [unit][16 half-words]
  uint16_t* Z = reinterpret_cast<uint16_t*>(z);       // [d][32 slots][16]
  auto zi = [&](int d, int s) { return (d * 32 + s) * 16 + hc; };
  __syncthreads();
  {
    uint4* t4 = reinterpret_cast<uint4*>(tile + tid * 8);
    t4[0] = make_uint4(m[0], m[1], m[2], m[3]);
    t4[1] = make_uint4(m[4], m[5], m[6], m[7]);
  }
  __syncthreads();
  uint32_t x[16];
  if (!INV) {
    uint32_t y[16];
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      const int v0 = r - d, v1 = r + 16 - d;
      x[d] = v0 >= 0 ? t16[(16 * d + v0) * 16 + hc] : 0u;
      y[d] = v1 < 16 ? t16[(16 * d + v1) * 16 + hc] : 0u;
    }
    zeta16_vals(x);
    zeta16_vals(y);
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      Z[zi(d, r)] = (uint16_t)x[d];
      Z[zi(d, r + 16)] = (uint16_t)y[d];
    }
    __syncthreads();
    const int v = r;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      uint32_t g = Z[zi(k, v + k)];
      if (v >= 1 && 15 + v + k < 31) g ^= Z[zi(k, 15 + v + k)];
      if (k >= 1 && 15 + v + k < 31) g ^= Z[zi(k - 1, 15 + v + k)];
      x[k] = g;
    }
    conv16_vals<false>(x);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) Z[zi(k, v)] = (uint16_t)x[k];
    __syncthreads();
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) x[vv] = Z[zi(r, vv)];
    conv16_vals<false>(x);
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) t16[(16 * r + vv) * 16 + hc] = (uint16_t)x[vv];
  } else {
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) x[vv] = t16[(16 * r + vv) * 16 + hc];
    conv16_vals<true>(x);
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) Z[zi(r, vv)] = (uint16_t)x[vv];
    __syncthreads();
    const int v = r;
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = Z[zi(k, v)];
    conv16_vals<true>(x);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) Z[zi(k, v + k)] = (uint16_t)x[k];
    __syncthreads();
    uint32_t y[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x[k] = (r >= k) ? Z[zi(k, r)] : 0u;
      y[k] = (r < k) ? Z[zi(k, r + 16)] : 0u;
    }
    zeta16_vals(x);
    zeta16_vals(y);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      Z[zi(k, r)] = (uint16_t)x[k];
      Z[zi(k, r + 16)] = (uint16_t)y[k];
    }
    __syncthreads();
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) {
      uint32_t f = Z[zi(r, vv + r)];
      if (r >= 1 && 15 + vv + r < 31) f ^= Z[zi(r - 1, 15 + vv + r)];
      t16[(16 * r + vv) * 16 + hc] = (uint16_t)f;
    }
  }
  __syncthreads();
  {
    const uint4* t4 = reinterpret_cast<const uint4*>(tile + tid * 8);
    const uint4 a = t4[0], b = t4[1];
    m[0] = a.x; m[1] = a.y; m[2] = a.z; m[3] = a.w; m[4] = b.x; m[5] = b.y; m[6] = b.z; m[7] = b.w;
  }
}

// 256 x 256-bit tile transpose (an involution): thread t's row t <-> thread c's column c (word w
// of a column = rows 32w .. 32w+31).  Each warp transposes its eight 32 x 32 blocks in registers
// (Transpose32), then the blocks change warps through shared memory (pitch 9: conflict-free).
// sm: >= 256 x 9 words; all 256 threads call it (two barriers).
__device__ __forceinline__ void tile_transpose(uint32_t (&m)[8], uint32_t* sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Transpose32 tr(lane);
  uint32_t x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = tr(m[j]);  // lane l: column 32j + l of rows 32 warp ..
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 8; ++j) sm[(32 * j + lane) * 9 + warp] = x[j];
  __syncthreads();
#pragma unroll
  for (int w = 0; w < 8; ++w) m[w] = sm[tid * 9 + w];
}

// conv(2^g) over the tile's rows as units (C_cols): a GF(2)-linear map applied identically to
// every bit column, so in the transposed tile it is conv_regs on each column word -- two
// transposes instead of kRowSchedN[g] shared-memory row passes (12 passes, 24 barriers at g = 8).
template <bool INV>
__device__ __forceinline__ void colconv_tile(uint32_t (&m)[8], uint32_t* sm, int g) {
  tile_transpose(m, sm);
  conv_regs<INV>(g, m);
  tile_transpose(m, sm);
}

// Converts every aligned 2^r-bit chunk of the tile (thread t's row in m), r in [1, 16].
// tile: 256 x kRowPitchW<1> words of shared memory; sc: 256 x kScPitch words of shared memory.
// All 256 threads must call it (barriers inside when r > 8).
template <bool INV>
__device__ __forceinline__ void conv_tile(uint32_t (&m)[8], uint32_t* tile, uint32_t* sc, int r) {
  if (r <= 8) {
    conv_regs<INV>(r, m);
    return;
  }
  const int g = r - 8, d = threadIdx.x & ((1 << g) - 1);
  // full 2^16-bit rows: the sub-row conversion on 16-bit half-columns (no transposes)
  const bool units = g == 8 && kUnitConvTile;
  if (!INV) {
    l1_tile<false>(m, sc, g, d);
    if (units) unitconv256_tile<false>(m, tile, sc);
    else colconv_tile<false>(m, tile, g);
    conv_regs<false>(8, m);
  } else {
    conv_regs<true>(8, m);
    if (units) unitconv256_tile<true>(m, tile, sc);
    else colconv_tile<true>(m, tile, g);
    l1_tile<true>(m, sc, g, d);
  }
}

}  // namespace fpm
