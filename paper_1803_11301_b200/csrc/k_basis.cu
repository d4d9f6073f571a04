// k_basis.cu -- monomial <-> novel-polynomial basis conversion (Taylor expansion) on sm_100a.
//
// Reference: proj/src/basis_convert.cpp -- the fixed fold-pass list of build_schedule (:53-67),
//     forward  y[q] = x[q] ^ x[q+D] ^ (q+2D < S ? x[q+2D] : 0)   q in [S/2-D, S-D) of each S-span
//     inverse  x[q] = y[q] ^ y[q+D]                              (reverse pass order)
// applied one pass per sweep (81 sweeps for a 2^33-bit array).  Here the same linear map is
// evaluated in a handful of HBM sweeps, using the schedule's recursion
//     conv(2^K) = C_rows(conv(t)) o C_cols(conv(D)) o L1(t, D),  t = 2^16, D = 2^(K-16)  (17 <= K <= 32)
// with L1 in closed form (see conv_tile.cuh; model check: tools/models/bc_model.py):
//   Z     zeta_kernel       skew row d by d bits (fused into the load) and XOR-butterfly the row index
//                           over 256-row groups (stride 1, then stride 256): pure streaming XOR tiles
//   C     carry_rows_kernel unskew + single carry level, then conv(2^16) of the row in shared memory
//                           (forward; the inverse uses overflow_kernel and a separate row pass)
//   C_D   conv over the row index: D <= 256 -> slab tiles of D rows x 1024 bits (row XOR passes);
//         D > 256 -> the same recursion one level up with whole rows as units (row-skewed zeta,
//         unit carry fused with the row passes over the high digit, slab passes over the low one)
// HBM traffic at K = 32: ~9 GiB (vs ~70 GiB for 48 separate passes).  Arrays of <= 2^16 bits run in
// one shared-memory tile; > 2^32 bits run their top passes with the generic in-place pass kernel
// and recurse per 2^32-bit block.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "basis_dev.cuh"
#include "conv_tile.cuh"
#include "gf128.cuh"
#include "gf64.cuh"
#include "warp_bits.cuh"
#include "fpm_internal.h"

namespace fpm {
namespace {

constexpr int kTLog2 = 16;                  // digit size t = 2^16 bits for 2^17..2^32-bit arrays
constexpr uint64_t kT = (uint64_t)1 << kTLog2;
constexpr int kTWords = (int)(kT / 32);     // 2048
constexpr size_t kTileSmem = (kTileRows * kRowPitchW<1> + kTileRows * kScPitch) * sizeof(uint32_t);

__device__ __forceinline__ uint4 x4v(uint4 a, uint4 b) { return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w); }

int sm_count() {
  int dev, n;
  FPM_CUDA(cudaGetDevice(&dev));
  FPM_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

// ------------------------------------------------------------------ generic in-place pass (K > 32)
__global__ void bc_pass_kernel(uint32_t* __restrict__ w, uint64_t nwords, uint64_t S, uint64_t D, int inverse,
                               uint64_t w_first, uint64_t nw_span, uint64_t nspans, uint64_t rlo, uint64_t rhi,
                               uint64_t live_bits) {
  pdl_wait();
  const uint64_t total = nw_span * nspans;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t span = k / nw_span;
    const uint64_t base = span * S;
    if (!inverse && base + S / 2 >= live_bits) continue;
    const uint64_t wi = (base >> 5) + w_first + (k - span * nw_span);
    w[wi] = fold_word(w, nwords, wi, S, D, inverse != 0, rlo, rhi);
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ small arrays (< 2^8 bits)
__global__ void bc_small_kernel(uint32_t* __restrict__ w, int words, PassList pl, int inverse) {
  pdl_wait();
  extern __shared__ uint32_t sm[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) sm[i] = w[i];
  __syncthreads();
  const uint32_t* a = smem_passes(sm, sm + words, words, pl, inverse != 0);
  for (int i = threadIdx.x; i < words; i += blockDim.x) w[i] = a[i];
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ conv of 2^r-bit chunks, 8 KiB tiles
template <bool INV>
__global__ void __launch_bounds__(256) conv_rows_kernel(uint32_t* __restrict__ data, uint64_t nwords, int r) {
  pdl_wait();
  extern __shared__ uint32_t smem[];
  uint32_t* tile = smem;
  uint32_t* sc = smem + kTileRows * kRowPitchW<1>;
  const int tid = threadIdx.x;
  const uint64_t tile_words = nwords < 2048 ? nwords : 2048;
  const uint64_t ntiles = nwords / tile_words;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t off = t * tile_words + (uint64_t)tid * 8;
    uint32_t m[8];
    const bool valid = (uint64_t)tid * 8 < tile_words;
    if (valid) {
      const uint4 a = reinterpret_cast<const uint4*>(data + off)[0];
      const uint4 b = reinterpret_cast<const uint4*>(data + off)[1];
      m[0] = a.x; m[1] = a.y; m[2] = a.z; m[3] = a.w; m[4] = b.x; m[5] = b.y; m[6] = b.z; m[7] = b.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) m[i] = 0;
    }
    conv_tile<INV>(m, tile, sc, r);
    if (valid) {
      reinterpret_cast<uint4*>(data + off)[0] = make_uint4(m[0], m[1], m[2], m[3]);
      reinterpret_cast<uint4*>(data + off)[1] = make_uint4(m[4], m[5], m[6], m[7]);
    }
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ Z: subset-zeta over row bits
// Tile = 256 tile rows x 32 words (one 128 B line per row): tile row R = s * 2^nb + j is row
// d = base + j * 2^b0 of the group, window wi = wb * (256 >> nb) + s.  Two thread mappings make
// every butterfly stage register-local with ONE shared-memory exchange between them:
//   A: thread t holds word t&31 of tile rows (t>>5) + 8k, k < 32   -> row bits 3..7 local
//   B: thread t holds words 4(t&7).. of tile rows 8(t>>3) + k, k < 8 -> row bits 0..2 local
// Skew: source row d is read at bit offset -(((d >> lo) & mask) << log) (mask 0: no skew).  The
// L1 skew by d bits is split over the two launches of a 2^16-row conversion: the first skews by
// the low digit d & 255 (rows grow by 256 bits only), the second by 256 * (d >> 8) bits, which is
// word aligned; whole-row (unit) skews use log = 16.
struct Skew {
  uint64_t mask = 0;
  int lo = 0, log = 0;
};
constexpr int kZW = 32;
constexpr int kZP = 36;  // shared row pitch (16 B aligned, conflict-free for both mappings)
// BITSKEW: the bit-granular skew path (neighbour words by shuffle) needs the registers of 2 CTAs/SM;
// word-aligned or no skew runs at 3 CTAs/SM.
template <bool BITSKEW, bool FULL = false>  // FULL: bit skew over complete 256-row groups (nb = 8)
__global__ void __launch_bounds__(256, BITSKEW ? (FULL ? 3 : 2) : 4) zeta_kernel(const uint32_t* __restrict__ src, uint64_t src_pitch,
                                                   uint32_t* __restrict__ dst, uint64_t dst_pitch, uint64_t D,
                                                   int b0, int nb, Skew skew, uint64_t src_row_words,
                                                   uint64_t windows) {
  pdl_wait();
  extern __shared__ __align__(16) uint32_t sx[];  // 256 x kZP
  const int tid = threadIdx.x;
  const int wpc = 256 >> nb;  // windows per CTA
  const uint64_t groups = D >> nb;
  const uint64_t wblocks = (windows + wpc - 1) / wpc;
  const uint64_t items = groups * wblocks;
  const uint64_t lowmask = ((uint64_t)1 << b0) - 1;
  for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const uint64_t gid = it / wblocks, wb = it - gid * wblocks;
    const uint64_t base = (gid & lowmask) | ((gid >> b0) << (b0 + nb));
    // ---- mapping A: load, stages on tile-row bits 3..7
    const int c = tid & 31;
    uint32_t a[32];
    if (!BITSKEW && nb == 8) {  // full 256-row groups: one window per CTA, rows at a fixed stride
      // Within a full group the skew is affine in the row (its digit never wraps): the word offset
      // advances by a constant per 8 rows, so addresses are one add per load.
      const uint64_t dstep = (uint64_t)8 << b0;
      const uint64_t d0 = base + ((uint64_t)(tid >> 5) << b0);
      auto skw = [&](uint64_t d) -> int64_t {
        return skew.mask ? (int64_t)((((d >> skew.lo) & skew.mask) << skew.log) >> 5) : 0;
      };
      const int64_t s0 = skw(d0), sstep = skw(d0 + dstep) - s0;
      const uint32_t* p = src + d0 * src_pitch + wb * kZW + c - s0;   // row d0, word iw
      int64_t iw = (int64_t)(wb * kZW) + c - s0;
      const int64_t pstep = (int64_t)(dstep * src_pitch) - sstep;
#pragma unroll
      for (int k = 0; k < 32; ++k, p += pstep, iw -= sstep)
        a[k] = (iw >= 0 && iw < (int64_t)src_row_words) ? __ldg(p) : 0u;
    } else if (!BITSKEW && skew.mask) {  // word-aligned skew: plain coalesced loads
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int R = (tid >> 5) + 8 * k;
        const uint64_t d = base + ((uint64_t)(R & ((1 << nb) - 1)) << b0);
        const uint64_t wi = wb * wpc + (R >> nb);
        const int64_t iw = (int64_t)(wi * kZW) - (int64_t)((((d >> skew.lo) & skew.mask) << skew.log) >> 5) + c;
        a[k] = (wi < windows && iw >= 0 && iw < (int64_t)src_row_words) ? __ldg(src + d * src_pitch + iw) : 0u;
      }
    } else if (BITSKEW) {
      // R (so d, wi, the shift) is warp-uniform: one coalesced word per lane and row, all rows'
      // loads in flight at once (lane 31 also fetches the word after the window), then the
      // neighbour word comes by shuffle and a funnel shift aligns the window.
      if (FULL) {
        // full group: skew bits affine in the row (d & 255 = R, base 256-aligned): per load one add.
        // The word after row k's window (lane 31's funnel input) is loaded by lane k and
        // broadcast: one register instead of 32 (and the shifts recomputed), for the occupancy.
        const uint64_t dstep = (uint64_t)8 << b0;
        const uint64_t d0 = base + ((uint64_t)(tid >> 5) << b0);
        const int64_t s0 = (int64_t)(((d0 >> skew.lo) & skew.mask) << skew.log);
        const int64_t sstep = (int64_t)((((d0 + dstep) >> skew.lo) & skew.mask) << skew.log) - s0;
        // 32-bit window arithmetic (rows < 2^31 bits); one unsigned compare bounds a word index
        const int32_t pos0 = (int32_t)((int64_t)(wb * 32 * kZW) - s0), ss = (int32_t)sstep;
        const uint32_t rows_w = (uint32_t)src_row_words;
        const uint32_t* row0 = src + d0 * src_pitch;
        const uint64_t rstep = dstep * src_pitch;
        const uint32_t* row = row0;
#pragma unroll
        for (int k = 0; k < 32; ++k, row += rstep) {
          const uint32_t iw = (uint32_t)(((pos0 - k * ss) >> 5) + c);
          a[k] = iw < rows_w ? __ldg(row + iw) : 0u;
        }
        const uint32_t iwe = (uint32_t)(((pos0 - c * ss) >> 5) + 32);
        const uint32_t ext = iwe < rows_w ? __ldg(row0 + c * rstep + iwe) : 0u;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const uint32_t nx = __shfl_down_sync(0xFFFFFFFFu, a[k], 1);
          const uint32_t ek = __shfl_sync(0xFFFFFFFFu, ext, k);
          a[k] = __funnelshift_r(a[k], c == 31 ? ek : nx, (pos0 - k * ss) & 31);
        }
      } else {
      uint32_t e[32];
      int sh[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int R = (tid >> 5) + 8 * k;
        const uint64_t d = base + ((uint64_t)(R & ((1 << nb) - 1)) << b0);
        const uint64_t wi = wb * wpc + (R >> nb);
        const uint32_t* row = src + d * src_pitch;
        const int64_t pos0 = (int64_t)(wi * 32 * kZW) - (int64_t)(((d >> skew.lo) & skew.mask) << skew.log);
        const int64_t iw = (pos0 >> 5) + c;
        sh[k] = (int)(pos0 & 31);
        const bool ok = wi < windows;
        a[k] = (ok && iw >= 0 && iw < (int64_t)src_row_words) ? __ldg(row + iw) : 0u;
        e[k] = (ok && c == 31 && iw + 1 >= 0 && iw + 1 < (int64_t)src_row_words) ? __ldg(row + iw + 1) : 0u;
      }
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const uint32_t nx = __shfl_down_sync(0xFFFFFFFFu, a[k], 1);
        a[k] = __funnelshift_r(a[k], c == 31 ? e[k] : nx, sh[k]);
      }
      }
    } else {
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int R = (tid >> 5) + 8 * k;
        const uint64_t d = base + ((uint64_t)(R & ((1 << nb) - 1)) << b0);
        const uint64_t wi = wb * wpc + (R >> nb);
        a[k] = wi < windows ? __ldg(src + d * src_pitch + wi * kZW + c) : 0u;
      }
    }
#pragma unroll
    for (int b = 3; b < 8; ++b) {
      if (b < nb) {
        const int kb = 1 << (b - 3);
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (!(k & kb)) a[k] ^= a[k | kb];
      }
    }
#pragma unroll
    for (int k = 0; k < 32; ++k) sx[((tid >> 5) + 8 * k) * kZP + c] = a[k];
    __syncthreads();
    // ---- mapping B: stages on tile-row bits 0..2, store
    const int q = tid & 7, R0 = 8 * (tid >> 3);
    uint4 bq[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) bq[k] = *reinterpret_cast<const uint4*>(sx + (R0 + k) * kZP + 4 * q);
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      if (b < nb) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (!(k & (1 << b))) bq[k] = make_uint4(bq[k].x ^ bq[k | (1 << b)].x, bq[k].y ^ bq[k | (1 << b)].y,
                                                   bq[k].z ^ bq[k | (1 << b)].z, bq[k].w ^ bq[k | (1 << b)].w);
      }
    }
    if (nb == 8) {  // one window, rows base + (R0 + k) << b0
      uint32_t* p = dst + (base + ((uint64_t)R0 << b0)) * dst_pitch + wb * kZW + 4 * q;
      const uint64_t step = ((uint64_t)1 << b0) * dst_pitch;
#pragma unroll
      for (int k = 0; k < 8; ++k) *reinterpret_cast<uint4*>(p + k * step) = bq[k];
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int R = R0 + k;
        const uint64_t d = base + ((uint64_t)(R & ((1 << nb) - 1)) << b0);
        const uint64_t wi = wb * wpc + (R >> nb);
        if (wi < windows) *reinterpret_cast<uint4*>(dst + d * dst_pitch + wi * kZW + 4 * q) = bq[k];
      }
    }
    __syncthreads();
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}
// ------------------------------------------------------------------ C: carry + unskew + conv(2^16)
// g_k[p] = Gs[k][p+k] ^ (p >= 1 ? Gs[k][t+p-1+k] : 0) ^ (k >= 1 ? Gs[k-1][t+p+k-1] : 0), then conv(g_k).
// kmask: the digit index of row k is k & kmask (all-ones: one Taylor step over all D rows; 255: the
// chunk-local step L1_inner of conv2d, whose digits restart every 256 rows).
__global__ void __launch_bounds__(256, 4) carry_rows_kernel(const uint32_t* __restrict__ gs, uint64_t gs_pitch,
                                                         uint32_t* __restrict__ out, uint64_t D, uint64_t kmask) {
  pdl_wait();
  extern __shared__ uint32_t smem[];
  uint32_t* tile = smem;
  uint32_t* sc = smem + kTileRows * kRowPitchW<1>;
  const int tid = threadIdx.x;
  // Staging (aliases the conversion tile): the two source spans of the row, word w at w + w/8 so
  // that thread t's 9-word window starting at 8t is bank-conflict free.
  uint32_t* sa = smem;                    // Gs[k] words a0 .. a0 + 2048      (L part, bit offset k)
  uint32_t* sh = smem + 2312;             // Gs[k] ^ Gs[k-1], words b0 ..     (H parts, t + k - 1)
  auto pad = [](int w) { return w + (w >> 3); };
  // coalesced: 2049 words per span; the next row's spans are loaded (into registers) while this
  // row converts
  uint32_t va[9], vh[9];
  auto fetch = [&](uint64_t kr) {
    if (kr >= D) return;
    const uint64_t k = kr & kmask;
    const uint32_t* rk = gs + kr * gs_pitch;
    const uint32_t* rk1 = gs + (kr - (k ? 1 : 0)) * gs_pitch;
    const uint64_t a0 = k >> 5, b0 = (kT + k - 1) >> 5;
    uint32_t vb[9], vc[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      const int w = tid + 256 * j;
      const uint64_t wb = b0 + w;
      const bool in = w <= kTWords;
      va[j] = in ? __ldg(rk + a0 + w) : 0u;
      vb[j] = in && wb < gs_pitch ? __ldg(rk + wb) : 0u;
      vc[j] = in && wb < gs_pitch && k ? __ldg(rk1 + wb) : 0u;
    }
#pragma unroll
    for (int j = 0; j < 9; ++j) vh[j] = vb[j] ^ vc[j];
  };
  fetch(blockIdx.x);
  for (uint64_t kr = blockIdx.x; kr < D; kr += gridDim.x) {
    const uint64_t k = kr & kmask;
    const uint32_t* rk = gs + kr * gs_pitch;
    const int sA = (int)(k & 31), sB = (int)((kT + k - 1) & 31);
    __syncthreads();  // the previous row's conversion is done with the shared tile
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      const int w = tid + 256 * j;
      if (w <= kTWords) {
        sa[pad(w)] = va[j];
        sh[pad(w)] = vh[j];
      }
    }
    fetch(kr + gridDim.x);
    __syncthreads();
    uint32_t m[8];
    {
      uint32_t wa[9], wh[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        wa[j] = sa[pad(8 * tid + j)];
        wh[j] = sh[pad(8 * tid + j)];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) m[i] = __funnelshift_r(wa[i], wa[i + 1], sA) ^ __funnelshift_r(wh[i], wh[i + 1], sB);
    }
    if (tid == 0) {  // g_k[0] takes no x * H_k term ([p >= 1]): undo bit 0 of Gs[k]'s H contribution
      const uint64_t pos = kT + k - 1;
      m[0] ^= __funnelshift_r(__ldg(rk + (pos >> 5)), (pos >> 5) + 1 < gs_pitch ? __ldg(rk + (pos >> 5) + 1) : 0u,
                              (int)(pos & 31)) & 1u;
    }
    conv_tile<false>(m, tile, sc, kTLog2);
    uint4* o = reinterpret_cast<uint4*>(out + kr * kTWords + tid * 8);
    o[0] = make_uint4(m[0], m[1], m[2], m[3]);
    o[1] = make_uint4(m[4], m[5], m[6], m[7]);
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ O: overflow + unskew (inverse)
// F_d[p] = Gs[d][p+d] ^ (d >= 1 ? Gs[d-1][t+p+d-1] : 0)
// top (optional): the single inverse top pass of a 2^33-bit array fused in when `out` is the lower
// 2^32-bit block: out bit q (q >= 1) ^= top bit q - 1, top = the (final) upper block.
__global__ void __launch_bounds__(256) overflow_kernel(const uint32_t* __restrict__ gs, uint64_t gs_pitch,
                                                       uint32_t* __restrict__ out, uint64_t D,
                                                       const uint32_t* __restrict__ top, uint64_t kmask) {
  pdl_wait();
  // One row per CTA iteration: the shifts and row pointers are row-invariant; thread t produces
  // words t, t + 256, ... (a warp covers 32 consecutive words: one coalesced load per lane, the
  // funnel's upper word from the next lane, lane 31 loads its own).  Only the first words of a row
  // receive the previous row's overflow (its skewed row ends t + 1024 bits in).
  const int tid = threadIdx.x, lane = tid & 31;
  for (uint64_t dr = blockIdx.x; dr < D; dr += gridDim.x) {
    const uint32_t d = (uint32_t)(dr & kmask);
    const uint32_t* r0 = gs + dr * gs_pitch;
    const uint32_t sh0 = d & 31, a0 = d >> 5;
    const uint32_t pos = (uint32_t)kT + d - 1, sh1 = pos & 31, b0 = pos >> 5;
    uint32_t* o = out + dr * kTWords;
    const uint32_t* tp = top ? top + dr * kTWords : nullptr;
    uint32_t x[8], y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // all eight loads in flight
      const uint32_t ia = tid + 256 * i + a0;
      x[i] = __ldg(r0 + ia);
      y[i] = lane == 31 && ia + 1 < gs_pitch ? __ldg(r0 + ia + 1) : 0u;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t w = tid + 256 * i;
      const uint32_t nx = __shfl_down_sync(0xFFFFFFFFu, x[i], 1);
      uint32_t v = __funnelshift_r(x[i], lane == 31 ? y[i] : nx, sh0);
      if (d && (w - lane) + b0 < gs_pitch) {  // warp-uniform: the previous row's overflow reaches
        const uint32_t ib = w + b0;               // only the first words of the row
        const uint32_t xb = ib < gs_pitch ? __ldg(r0 - gs_pitch + ib) : 0u;
        uint32_t yb = __shfl_down_sync(0xFFFFFFFFu, xb, 1);
        if (lane == 31) yb = ib + 1 < gs_pitch ? __ldg(r0 - gs_pitch + ib + 1) : 0u;
        v ^= __funnelshift_r(xb, yb, sh1);
      }
      if (tp) v ^= (tp[w] << 1) | ((dr || w) ? tp[(int64_t)w - 1] >> 31 : 0u);
      o[w] = v;
    }
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ L1_inner + T_r, one pipelined pass
// The chunk-local step L1_inner (256-row skewed zeta, zeta_kernel) and the per-row T_r (carry +
// conv(2^16), carry_rows_kernel; inverse: conv_rows, zeta, overflow) in ONE persistent kernel whose
// CTAs claim work items in a fixed order from an atomic counter: per chunk c (256 rows of 2^16
// bits), Z(c) = its 65 zeta windows and C(c) = its 256 rows, interleaved with a lag of kPipeLag
// chunks (forward: Z(0) Z(1) [Z(2) C(0)] [Z(3) C(1)] ...; inverse R(c) = the rows' conv^-1 first,
// then Z, then O = the overflow rows).  A consumer item waits (spinning on a per-chunk counter) for
// its chunk's producer items, which were all claimed before it: claimed items only ever wait on
// earlier claims, so the pipeline makes progress with any number of resident CTAs (no co-residency
// assumption, safe next to other kernels).  The skewed rows live in a ring of kPipeSlots chunk
// slots (16 MiB instead of a 520 MiB scratch array) that stays in L2: HBM sees one read and one
// write of the block instead of three of each.
#ifndef FPM_PIPE_LAG
#define FPM_PIPE_LAG 8
#endif
constexpr int kPipeLag = FPM_PIPE_LAG;  // chunks between a chunk's producer and consumer items
constexpr int kPipeSlots = 2 * FPM_PIPE_LAG;  // skewed-row ring (chunks); > kPipeLag
constexpr int kPipeZW = 65;    // zeta windows per skewed row: (2^16 + 1024) / 1024
constexpr int kPipeORows = 4;  // overflow rows per item (inverse, no T_r^-1)
constexpr uint64_t kPipeP1 = (kT + 32 * kZW) / 32;  // skewed row pitch (words)
// CTAs per SM: forward (zeta + carry / T_r) 3 at 80 registers; inverse (zeta + overflow) 4 at 64
// without spills (inverse conversions of a 2^33-bit product 5.55 -> 5.46 ms; forward unchanged at 4)
#ifndef FPM_PIPE_CTAS
#define FPM_PIPE_CTAS 3
#endif
#ifndef FPM_PIPE_CTAS_INV
#define FPM_PIPE_CTAS_INV 4
#endif
constexpr int pipe_ctas(bool inv) { return inv ? FPM_PIPE_CTAS_INV : FPM_PIPE_CTAS; }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// thread 0 waits until *cnt >= target, then the whole CTA proceeds
__device__ __forceinline__ void pipe_wait(const int* cnt, int target) {
  if (threadIdx.x == 0)
    while (ld_acquire(cnt) < target) __nanosleep(64);
  __syncthreads();
}
// after the item's stores (all threads): publish `units` of progress on *cnt (release: the CTA's
// stores, ordered before it by the barrier, are visible to whoever acquires the count)
__device__ __forceinline__ void pipe_done(int* cnt, int units = 1) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(cnt), "r"(units) : "memory");
}

// One L1_inner window: rows j < 256 of a chunk (src, pitch kTWords) skewed left by j bits, words
// [32 wb, 32 wb + 32) of the skewed rows, superset zeta over j -> dst rows (pitch kPipeP1).  The
// full-group bit-skew path of zeta_kernel<true, true> with the group fixed to one chunk.  CG: load
// through L2 only (src written by another CTA of the same kernel).
template <bool CG>
__device__ __forceinline__ void pipe_zeta_item(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int wb,
                                               uint32_t* sx) {
  const int tid = threadIdx.x, c = tid & 31, j0 = tid >> 5;
  auto ld = [](const uint32_t* p) { return CG ? __ldcg(p) : __ldg(p); };
  uint32_t a[32];
  {
    const int32_t pos0 = wb * 32 * kZW - j0;  // skew of row j0 + 8k: j0 + 8k bits
    const uint32_t* row0 = src + (uint64_t)j0 * kTWords;
    constexpr uint64_t rstep = 8 * (uint64_t)kTWords;
    const uint32_t* row = row0;
#pragma unroll
    for (int k = 0; k < 32; ++k, row += rstep) {
      const uint32_t iw = (uint32_t)(((pos0 - 8 * k) >> 5) + c);
      a[k] = iw < (uint32_t)kTWords ? ld(row + iw) : 0u;
    }
    const uint32_t iwe = (uint32_t)(((pos0 - 8 * c) >> 5) + 32);
    const uint32_t ext = iwe < (uint32_t)kTWords ? ld(row0 + c * rstep + iwe) : 0u;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const uint32_t nx = __shfl_down_sync(0xFFFFFFFFu, a[k], 1);
      const uint32_t ek = __shfl_sync(0xFFFFFFFFu, ext, k);
      a[k] = __funnelshift_r(a[k], c == 31 ? ek : nx, (pos0 - 8 * k) & 31);
    }
  }
#pragma unroll
  for (int b = 3; b < 8; ++b) {
    const int kb = 1 << (b - 3);
#pragma unroll
    for (int k = 0; k < 32; ++k)
      if (!(k & kb)) a[k] ^= a[k | kb];
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) sx[(j0 + 8 * k) * kZP + c] = a[k];
  __syncthreads();
  const int q = tid & 7, R0 = 8 * (tid >> 3);
  uint4 bq[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) bq[k] = *reinterpret_cast<const uint4*>(sx + (R0 + k) * kZP + 4 * q);
#pragma unroll
  for (int b = 0; b < 3; ++b)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (!(k & (1 << b))) bq[k] = x4v(bq[k], bq[k | (1 << b)]);
  uint32_t* p = dst + (uint64_t)R0 * kPipeP1 + wb * kZW + 4 * q;
#pragma unroll
  for (int k = 0; k < 8; ++k) *reinterpret_cast<uint4*>(p + k * kPipeP1) = bq[k];
}

// One forward T_r row: carry from the skewed rows (row k of the chunk and k - 1; carry_rows_kernel's
// g_k formula) + conv(2^16) of the row in shared memory -> out (kTWords words).
__device__ __forceinline__ void pipe_carry_row(const uint32_t* __restrict__ gs, int k, uint32_t* __restrict__ out,
                                               uint32_t* smem) {
  uint32_t* tile = smem;
  uint32_t* sc = smem + kTileRows * kRowPitchW<1>;
  const int tid = threadIdx.x;
  uint32_t* sa = smem;
  uint32_t* sh = smem + 2312;
  auto pad = [](int w) { return w + (w >> 3); };
  const uint32_t* rk = gs + (uint64_t)k * kPipeP1;
  const uint32_t* rk1 = gs + (uint64_t)(k ? k - 1 : 0) * kPipeP1;
  const int a0 = k >> 5, b0 = (int)((kT + k - 1) >> 5);
  uint32_t va[9], vh[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    const int w = tid + 256 * j;
    const int wb = b0 + w;
    const bool in = w <= kTWords;
    va[j] = in ? __ldcg(rk + a0 + w) : 0u;
    const uint32_t vb = in && wb < (int)kPipeP1 ? __ldcg(rk + wb) : 0u;
    const uint32_t vc = in && wb < (int)kPipeP1 && k ? __ldcg(rk1 + wb) : 0u;
    vh[j] = vb ^ vc;
  }
  const int sA = k & 31, sB = (int)((kT + k - 1) & 31);
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    const int w = tid + 256 * j;
    if (w <= kTWords) {
      sa[pad(w)] = va[j];
      sh[pad(w)] = vh[j];
    }
  }
  __syncthreads();
  uint32_t m[8];
  {
    uint32_t wa[9], wh[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      wa[j] = sa[pad(8 * tid + j)];
      wh[j] = sh[pad(8 * tid + j)];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = __funnelshift_r(wa[i], wa[i + 1], sA) ^ __funnelshift_r(wh[i], wh[i + 1], sB);
  }
  if (tid == 0) {  // g_k[0] takes no x * H_k term: undo bit 0 of Gs[k]'s H contribution
    const uint32_t pos = (uint32_t)(kT + k - 1);
    m[0] ^= __funnelshift_r(__ldcg(rk + (pos >> 5)), (pos >> 5) + 1 < kPipeP1 ? __ldcg(rk + (pos >> 5) + 1) : 0u,
                            (int)(pos & 31)) & 1u;
  }
  conv_tile<false>(m, tile, sc, kTLog2);  // (its first barrier orders the staging reads above)
  uint4* o = reinterpret_cast<uint4*>(out + tid * 8);
  o[0] = make_uint4(m[0], m[1], m[2], m[3]);
  o[1] = make_uint4(m[4], m[5], m[6], m[7]);
}

// One inverse T_r row in place: conv(2^16)^-1.
__device__ __forceinline__ void pipe_iconv_row(uint32_t* __restrict__ row, uint32_t* smem) {
  uint32_t* tile = smem;
  uint32_t* sc = smem + kTileRows * kRowPitchW<1>;
  const int tid = threadIdx.x;
  const uint4 a = reinterpret_cast<const uint4*>(row + tid * 8)[0];
  const uint4 b = reinterpret_cast<const uint4*>(row + tid * 8)[1];
  uint32_t m[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  conv_tile<true>(m, tile, sc, kTLog2);
  reinterpret_cast<uint4*>(row + tid * 8)[0] = make_uint4(m[0], m[1], m[2], m[3]);
  reinterpret_cast<uint4*>(row + tid * 8)[1] = make_uint4(m[4], m[5], m[6], m[7]);
}

// One inverse overflow row (overflow_kernel with the chunk-local digit d = row & 255): F_d[p] =
// Gs[d][p+d] ^ (d >= 1 ? Gs[d-1][t+p+d-1] : 0), gs = the chunk's skewed rows (ring slot).
__device__ __forceinline__ void pipe_overflow_row(const uint32_t* __restrict__ gs, int d, uint32_t* __restrict__ o,
                                                  const uint32_t* __restrict__ tp, bool first_row) {
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t* r0 = gs + (uint64_t)d * kPipeP1;
  const uint32_t sh0 = d & 31, a0 = d >> 5;
  const uint32_t pos = (uint32_t)kT + d - 1, sh1 = pos & 31, b0 = pos >> 5;
  uint32_t x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t ia = tid + 256 * i + a0;
    x[i] = __ldcg(r0 + ia);
    y[i] = lane == 31 && ia + 1 < kPipeP1 ? __ldcg(r0 + ia + 1) : 0u;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t w = tid + 256 * i;
    const uint32_t nx = __shfl_down_sync(0xFFFFFFFFu, x[i], 1);
    uint32_t v = __funnelshift_r(x[i], lane == 31 ? y[i] : nx, sh0);
    if (d && (w - lane) + b0 < kPipeP1) {
      const uint32_t ib = w + b0;
      const uint32_t xb = ib < kPipeP1 ? __ldcg(r0 - kPipeP1 + ib) : 0u;
      uint32_t yb = __shfl_down_sync(0xFFFFFFFFu, xb, 1);
      if (lane == 31) yb = ib + 1 < kPipeP1 ? __ldcg(r0 - kPipeP1 + ib + 1) : 0u;
      v ^= __funnelshift_r(xb, yb, sh1);
    }
    if (tp) v ^= (tp[w] << 1) | ((!first_row || w) ? tp[(int64_t)w - 1] >> 31 : 0u);
    o[w] = v;
  }
}

// Work item k of the pipelined pass over nch chunks: (kind, chunk, sub).  Kinds in claim order per
// step s: [forward] Z(s), C(s - lag); [inverse] R(s), Z(s - lag), O(s - 2 lag).
struct PipeItem {
  int kind, chunk, sub;  // kind: 0 = zeta window, 1 = carry / overflow row, 2 = inverse conv row
};
template <bool INV, bool ICONV>
__device__ __forceinline__ PipeItem pipe_item(int k, int nch) {
  // Step s holds, in order, the items of the kinds j whose chunk s - j * lag is in [0, nch).  The
  // per-step count only changes at the steps j * lag and nch + j * lag: walk those phases.
  constexpr int nk = ICONV ? 3 : 2;
  constexpr int kinds[3] = {ICONV ? 2 : 0, ICONV ? 0 : 1, 1};
  constexpr int sizes[3] = {ICONV ? 256 : kPipeZW, ICONV ? kPipeZW : (INV ? 256 / kPipeORows : 256), 256};
  int b[2 * nk];
#pragma unroll
  for (int j = 0; j < nk; ++j) {
    b[j] = j * kPipeLag;
    b[nk + j] = nch + j * kPipeLag;
  }
#pragma unroll
  for (int i = 1; i < 2 * nk; ++i)  // insertion sort (<= 6 values)
#pragma unroll
    for (int j = i; j > 0; --j)
      if (b[j] < b[j - 1]) {
        const int t = b[j];
        b[j] = b[j - 1];
        b[j - 1] = t;
      }
  for (int i = 0; i + 1 < 2 * nk; ++i) {
    const int s0 = b[i], steps = b[i + 1] - s0;
    if (steps <= 0) continue;
    int per = 0;
#pragma unroll
    for (int j = 0; j < nk; ++j) {
      const int ch = s0 - j * kPipeLag;
      if (ch >= 0 && ch < nch) per += sizes[j];
    }
    if (k < per * steps) {
      const int s = s0 + k / per;
      int r = k % per;
#pragma unroll
      for (int j = 0; j < nk; ++j) {
        const int ch = s - j * kPipeLag;
        if (ch < 0 || ch >= nch) continue;
        if (r < sizes[j]) return PipeItem{kinds[j], ch, r};
        r -= sizes[j];
      }
    }
    k -= per * steps;
  }
  return PipeItem{-1, 0, 0};
}

// cnt: 3 * nch + 1 zeroed ints: [0, nch) zeta windows done per chunk, [nch, 2 nch) rows done per
// chunk (carry / overflow), [2 nch, 3 nch) inverse conv rows done per chunk, [3 nch] the claim
// counter.  w: the block (nch * 256 rows of kTWords words); src: the rows the zeta reads (forward:
// the unconverted rows, may be w; inverse: w); ring: kPipeSlots chunks of 256 skewed rows (pitch
// kPipeP1); top: as overflow_kernel.  INV: zeta + overflow (L1_inner^-1); ICONV: with the rows'
// conv(2^16)^-1 (T_r^-1) first.
template <bool INV, bool ICONV>
__global__ void __launch_bounds__(256, pipe_ctas(INV)) l1_inner_rows_kernel(const uint32_t* src, uint32_t* w, uint32_t* ring,
                                                                int nch, int* cnt, const uint32_t* __restrict__ top) {
  pdl_wait();
  extern __shared__ __align__(16) uint32_t smem[];  // max(zeta 256 x kZP, row tile kTileSmem)
  __shared__ int s_item[2];
  const int total = nch * (kPipeZW + (INV && !ICONV ? 256 / kPipeORows : 256) + (ICONV ? 256 : 0));
  int* zdone = cnt;
  int* rdone = cnt + nch;
  int* idone = cnt + 2 * nch;
  int* claim = cnt + 3 * nch;
  if (threadIdx.x == 0) s_item[0] = atomicAdd(claim, 1);
  __syncthreads();
  int buf = 0;
  for (int cur = s_item[0]; cur < total; cur = s_item[buf]) {
    if (threadIdx.x == 0) s_item[buf ^ 1] = atomicAdd(claim, 1);  // next claim in flight
    const PipeItem it = pipe_item<INV, ICONV>(cur, nch);
    const int c = it.chunk;
    uint32_t* slot = ring + (uint64_t)(c % kPipeSlots) * 256 * kPipeP1;
    uint32_t* wc = w + (uint64_t)c * 256 * kTWords;
    if (it.kind == 0) {  // zeta window
      if (ICONV) pipe_wait(idone + c, 256);                       // the chunk's rows are conv^-1'ed
      if (c >= kPipeSlots) pipe_wait(rdone + c - kPipeSlots, 256);  // the slot's previous chunk is consumed
      if (ICONV) pipe_zeta_item<true>(wc, slot, it.sub, smem);
      else pipe_zeta_item<false>(src + (uint64_t)c * 256 * kTWords, slot, it.sub, smem);
      pipe_done(zdone + c);
    } else if (it.kind == 1) {  // carry (forward) / overflow (inverse) row
      pipe_wait(zdone + c, kPipeZW);
      if (!INV) {
        pipe_carry_row(slot, it.sub, wc + (uint64_t)it.sub * kTWords, smem);
        pipe_done(rdone + c);
      } else {
        constexpr int nr = ICONV ? 1 : kPipeORows;
#pragma unroll 1
        for (int r = 0; r < nr; ++r) {
          const int d = it.sub * nr + r;
          const uint64_t row = (uint64_t)c * 256 + d;
          pipe_overflow_row(slot, d, wc + (uint64_t)d * kTWords, top ? top + row * kTWords : nullptr, row == 0);
        }
        pipe_done(rdone + c, nr);
      }
    } else if (it.kind == 2) {  // inverse conv row
      pipe_iconv_row(wc + (uint64_t)it.sub * kTWords, smem);
      pipe_done(idone + c);
    }
    buf ^= 1;  // (s_item[buf] was written before pipe_done's barrier)
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// Bit 0 of the upper 2^32-bit block ^= its last bit (the fused 2^33-bit top pass's target 2^32).
__global__ void top_bit_fix_kernel(uint32_t* __restrict__ hi_block, uint64_t block_words) {
  pdl_wait();
  if (threadIdx.x == 0) hi_block[0] ^= hi_block[block_words - 1] >> 31;
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ C_D for D <= 256: slab tiles
// Tile = (256 / D) slabs x D rows x 8 words; rows of the array are t bits (kTWords words) apart.
// Generalised: rows r = outer * (Dr * rstride) + d * rstride + inner, inner < rstride (row units of
// kTWords words); a slab = (outer, inner, 8W-word column) -- conv over d at row stride rstride.
constexpr int kSlabW = 4;  // 128 B of each row per slab: full lines, 4x fewer barriers
template <bool INV>
__global__ void __launch_bounds__(256) slab_kernel(uint32_t* __restrict__ data, int g, uint64_t rstride,
                                                   uint64_t nslabs) {
  pdl_wait();
  extern __shared__ __align__(16) uint32_t tile[];  // 256 x kRowPitchW<kSlabW>
  constexpr int W = kSlabW, cpr = kTWords / (8 * W);  // slabs per row
  const int tid = threadIdx.x;
  const int Dr = 1 << g;
  const int d = tid & (Dr - 1), slot = tid >> g;
  const int spc = 256 >> g;  // slabs per CTA
  for (uint64_t sb = (uint64_t)blockIdx.x * spc; sb < nslabs; sb += (uint64_t)gridDim.x * spc) {
    const uint64_t slab = sb + slot;
    const uint64_t col = slab % cpr, rest = slab / cpr;
    const uint64_t inner = rest % rstride, outer = rest / rstride;
    const uint64_t row = outer * ((uint64_t)Dr * rstride) + (uint64_t)d * rstride + inner;
    uint4* p = reinterpret_cast<uint4*>(data + row * kTWords + col * 8 * W);
    const bool valid = slab < nslabs;
    uint32_t m[W][8];
#pragma unroll
    for (int c = 0; c < W; ++c) {
      uint4 a = make_uint4(0, 0, 0, 0), b = a;
      if (valid) { a = p[2 * c]; b = p[2 * c + 1]; }
      m[c][0] = a.x; m[c][1] = a.y; m[c][2] = a.z; m[c][3] = a.w;
      m[c][4] = b.x; m[c][5] = b.y; m[c][6] = b.z; m[c][7] = b.w;
    }
    rowpasses_w<INV, W>(m, tile, g, d);
    if (valid) {
#pragma unroll
      for (int c = 0; c < W; ++c) {
        p[2 * c] = make_uint4(m[c][0], m[c][1], m[c][2], m[c][3]);
        p[2 * c + 1] = make_uint4(m[c][4], m[c][5], m[c][6], m[c][7]);
      }
    }
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ conv(256) over units, by L1(16, 16)
// conv(256) of 256 units (8 KiB rows; unit u = 16 d + v) evaluated per bit column by the same
// recursion as the whole conversion one level down: C_rows(conv16 over v) o C_cols(conv16 over d)
// o L1(16, 16), with the L1 skew in units.  A CTA of 16 x kC256Cols threads owns kC256Cols words of each
// of the 256 units; thread (r = tid / cols, c = tid % cols).  Three register-local phases (zeta over d,
// conv16 over k, conv16 over v) with shared-memory exchanges between them: 28 B of shared traffic
// per word instead of the ~80 B of the 12 row passes.  Skewed rows Z[d][s] (s < 32 unit slots):
// Z[d][v + d] = F_d[v].
// kC256Cols words of each unit per CTA (16 x kC256Cols threads, 2 CTAs/SM: one CTA's load phase
// overlaps the other's shared-memory phases).
constexpr int kC256Cols = 16;
constexpr int kC256Threads = 16 * kC256Cols;
// Z[16][33][cols]: the digit stride padded by one slot row, so that the two half-warps of a phase
// that differ in d (512 words apart unpadded) land in different banks.
constexpr size_t kC256Smem = 16 * 33 * kC256Cols * sizeof(uint32_t);

// Units of CTA slab `blk`: unit u of group `grp` is row grp_base + u * ustride (rows of kTWords
// words); the CTA takes word columns [c0, c0 + 32).
struct UnitMap {
  uint64_t ustride, gstride, ngroups;  // group g's unit u at row g_row(g) + u * ustride
  // conv256_units_tma_kernel only: column items [col_lo, col_lo + ncols) of every group (ncols = 0:
  // all kTWords / kCT of them) -- a rank's column share in the sharded conversion
  uint32_t col_lo = 0, ncols = 0;
  __device__ __forceinline__ uint64_t row(uint64_t grp, int u) const {
    // groups: (ngroups) groups; group index -> base row = (grp % gstride) + (grp / gstride) * 256 * gstride
    return (grp % gstride) + (grp / gstride) * 256 * gstride + (uint64_t)u * ustride;
  }
};

// Optional fused input stage (forward only): the units are the unit-level L1 carry of a
// unit-skewed zeta output gs (digit rows of gs_pitch words, 256 + 256 units):
//   unit kh of group v = gs[kh][v+kh] ^ [v>=1] gs[kh][255+v+kh] ^ [kh>=1] gs[kh-1][255+v+kh]
// (the last two only while 255 + v + kh < 512, the stored width; digit count 256)
struct CarrySrc {
  const uint32_t* gs = nullptr;
  uint64_t gs_pitch = 0;
};

template <bool INV>
__global__ void __launch_bounds__(kC256Threads, INV ? 3 : 4) conv256_units_kernel(uint32_t* __restrict__ data, UnitMap um,
                                                                        uint64_t nitems, CarrySrc cs) {
  pdl_wait();
  extern __shared__ uint32_t Z[];  // [d][s][c], d < 16, s < 32, c < 32
  const int tid = threadIdx.x, c = tid % kC256Cols, r = tid / kC256Cols;
  constexpr int kCols = kTWords / kC256Cols;  // column blocks per unit
  auto zi = [](int d, int s, int cc) { return (d * 33 + s) * kC256Cols + cc; };
  for (uint64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const uint64_t grp = it / kCols;
    const uint64_t colw = (it % kCols) * kC256Cols + c;
    uint32_t* const gbase = data + um.row(grp, 0) * kTWords + colw;
    const uint32_t ustep = (uint32_t)(um.ustride * kTWords);  // 256 units x ustep < 2^32 words
    auto at = [&](int u) -> uint32_t* { return gbase + (uint32_t)u * ustep; };
    auto src = [&](int u) -> uint32_t {  // input unit u of this group
      if (!cs.gs) return *at(u);
      const uint64_t v = grp;  // group = offset v within the digit, unit = digit kh
      const uint32_t* rk = cs.gs + (uint64_t)u * cs.gs_pitch + colw;
      uint32_t g = rk[(v + u) * kTWords];
      if (v + u < 257) {  // units >= 256 + 256 of a skewed digit row are zero (not stored)
        if (v >= 1) g ^= rk[(255 + v + u) * kTWords];
        if (u >= 1) g ^= rk[(255 + v + u) * kTWords - cs.gs_pitch];
      }
      return g;
    };
    uint32_t x[16];
    if (!INV) {
      // ---- skewed load (thread = slot pair {r, r+16}) + zeta over d
      uint32_t y[16];
#pragma unroll
      for (int d = 0; d < 16; ++d) {
        const int v0 = r - d, v1 = r + 16 - d;
        x[d] = v0 >= 0 ? src(16 * d + v0) : 0u;
        y[d] = v1 < 16 ? src(16 * d + v1) : 0u;
      }
      zeta16_vals(x);
      zeta16_vals(y);
      __syncthreads();  // previous item's readers of Z are done
#pragma unroll
      for (int d = 0; d < 16; ++d) {
        Z[zi(d, r, c)] = x[d];
        Z[zi(d, r + 16, c)] = y[d];
      }
      __syncthreads();
      // ---- carry + unskew (thread = v = r): g_k[v] = Z[k][v+k] ^ Z[k][15+v+k] ^ Z[k-1][15+v+k]
      const int v = r;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        uint32_t g = Z[zi(k, v + k, c)];
        if (v >= 1 && 15 + v + k < 31) g ^= Z[zi(k, 15 + v + k, c)];
        if (k >= 1 && 15 + v + k < 31) g ^= Z[zi(k - 1, 15 + v + k, c)];
        x[k] = g;
      }
      conv16_vals<false>(x);  // C_cols: conv16 over k
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) Z[zi(k, v, c)] = x[k];
      __syncthreads();
      // ---- C_rows: conv16 over v (thread = k = r)
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) x[vv] = Z[zi(r, vv, c)];
      conv16_vals<false>(x);
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) *at(16 * r + vv) = x[vv];
    } else {
      // ---- C_rows^-1 over v (thread = k = r)
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) x[vv] = *at(16 * r + vv);
      conv16_vals<true>(x);
      __syncthreads();
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) Z[zi(r, vv, c)] = x[vv];
      __syncthreads();
      // ---- C_cols^-1 over k (thread = v = r), then skew: Z[k][v + k]
      const int v = r;
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = Z[zi(k, v, c)];
      conv16_vals<true>(x);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) Z[zi(k, v + k, c)] = x[k];
      __syncthreads();
      // ---- zeta over k on the skewed rows (thread = slot pair {r, r+16}); row k holds slots k..k+15
      uint32_t y[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        x[k] = (r >= k) ? Z[zi(k, r, c)] : 0u;
        y[k] = (r + 16 < k + 16) ? Z[zi(k, r + 16, c)] : 0u;
      }
      zeta16_vals(x);
      zeta16_vals(y);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        Z[zi(k, r, c)] = x[k];
        Z[zi(k, r + 16, c)] = y[k];
      }
      __syncthreads();
      // ---- overflow + unskew (thread = d = r): F_d[v] = Z[d][v+d] ^ Z[d-1][15+v+d]
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) {
        uint32_t f = Z[zi(r, vv + r, c)];
        if (r >= 1 && 15 + vv + r < 31) f ^= Z[zi(r - 1, 15 + vv + r, c)];
        *at(16 * r + vv) = f;
      }
    }
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ---- the same conv(256) over units with TMA-fed staging (no fused carry input): 128 B of each of
// the 256 units per item (a warp = one unit row x 32 words), moved global -> shared by 256
// cp.async.bulk copies completing on an mbarrier, double-buffered so item k+2's copies run while
// item k computes; 512 threads, one CTA per SM (2 x 32 KiB staging + 66 KiB of Z).  The register
// phases are those of conv256_units_kernel.
#ifndef FPM_CT_WORDS
#define FPM_CT_WORDS 32
#endif
constexpr int kCT = FPM_CT_WORDS;            // words of each unit per item (16: 3 CTAs/SM, 32: 1)
constexpr int kCTMinBlocks = kCT == 16 ? 3 : 1;
constexpr int kCTThreads = 16 * kCT;         // (r, c), r < 16
constexpr size_t kCTStage = 256 * kCT * 4;   // bytes per staging buffer
constexpr size_t kCTSmem = 2 * kCTStage + 16 * 33 * kCT * 4 + 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
template <bool INV>
__global__ void __launch_bounds__(kCTThreads, kCTMinBlocks) conv256_units_tma_kernel(uint32_t* data, UnitMap um, uint64_t nitems,
                                                                          const __grid_constant__ CUtensorMap tmap) {
  pdl_wait();
  extern __shared__ __align__(128) uint32_t sm_ct[];
  auto stage = [&](int st) { return sm_ct + st * (256 * kCT); };
  uint32_t* Z = sm_ct + 2 * 256 * kCT;  // [d][33][kCT]
  uint64_t* bar = reinterpret_cast<uint64_t*>(Z + 16 * 33 * kCT);
  const int tid = threadIdx.x, c = tid % kCT, r = tid / kCT;
  constexpr int kCols = kTWords / kCT;
  const uint64_t nc = um.ncols ? um.ncols : kCols;  // column items per group
  auto zi = [](int d, int s, int cc) { return (d * 33 + s) * kCT + cc; };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // one TMA box per item: 32 words x 1 x 256 units of the (word, group-in-stride, unit-row) view
  auto issue = [&](uint64_t it, int st) {
    if (tid != 0 || it >= nitems) return;
    mbar_expect_tx(&bar[st], (uint32_t)kCTStage);
    const uint64_t grp = it / nc;
    const int c0 = (int)((um.col_lo + it % nc) * kCT), c1 = (int)(grp % um.gstride), c2 = (int)((grp / um.gstride) * 256);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(stage(st))),
        "l"(&tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(&bar[st]))
        : "memory");
  };
  uint32_t phases = 0;  // bit st: parity of stage st's next completion
  issue(blockIdx.x, 0);
  issue(blockIdx.x + gridDim.x, 1);
  int st = 0;
  for (uint64_t it = blockIdx.x; it < nitems; it += gridDim.x, st ^= 1) {
    const uint64_t grp = it / nc, colw = (um.col_lo + it % nc) * kCT + c;
    uint32_t* const gbase = data + um.row(grp, 0) * kTWords + colw;
    const uint32_t ustep = (uint32_t)(um.ustride * kTWords);
    auto at = [&](int u) -> uint32_t* { return gbase + (uint32_t)u * ustep; };
    const uint32_t* sg = stage(st);
    mbar_wait(&bar[st], (phases >> st) & 1u);
    phases ^= 1u << st;
    uint32_t x[16];
    if (!INV) {
      uint32_t y[16];
#pragma unroll
      for (int d = 0; d < 16; ++d) {
        const int v0 = r - d, v1 = r + 16 - d;
        x[d] = v0 >= 0 ? sg[(16 * d + v0) * kCT + c] : 0u;
        y[d] = v1 < 16 ? sg[(16 * d + v1) * kCT + c] : 0u;
      }
      __syncthreads();  // staging consumed: refill it with item + 2 while this item computes
      if (tid == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(it + 2 * (uint64_t)gridDim.x, st);
      zeta16_vals(x);
      zeta16_vals(y);
#pragma unroll
      for (int d = 0; d < 16; ++d) {
        Z[zi(d, r, c)] = x[d];
        Z[zi(d, r + 16, c)] = y[d];
      }
      __syncthreads();
      const int v = r;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        uint32_t g = Z[zi(k, v + k, c)];
        if (v >= 1 && 15 + v + k < 31) g ^= Z[zi(k, 15 + v + k, c)];
        if (k >= 1 && 15 + v + k < 31) g ^= Z[zi(k - 1, 15 + v + k, c)];
        x[k] = g;
      }
      conv16_vals<false>(x);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) Z[zi(k, v, c)] = x[k];
      __syncthreads();
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) x[vv] = Z[zi(r, vv, c)];
      conv16_vals<false>(x);
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) *at(16 * r + vv) = x[vv];
    } else {
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) x[vv] = sg[(16 * r + vv) * kCT + c];
      __syncthreads();
      if (tid == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(it + 2 * (uint64_t)gridDim.x, st);
      conv16_vals<true>(x);
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) Z[zi(r, vv, c)] = x[vv];
      __syncthreads();
      const int v = r;
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = Z[zi(k, v, c)];
      conv16_vals<true>(x);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) Z[zi(k, v + k, c)] = x[k];
      __syncthreads();
      uint32_t y[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        x[k] = (r >= k) ? Z[zi(k, r, c)] : 0u;
        y[k] = (r + 16 < k + 16) ? Z[zi(k, r + 16, c)] : 0u;
      }
      zeta16_vals(x);
      zeta16_vals(y);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        Z[zi(k, r, c)] = x[k];
        Z[zi(k, r + 16, c)] = y[k];
      }
      __syncthreads();
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) {
        uint32_t f = Z[zi(r, vv + r, c)];
        if (r >= 1 && 15 + vv + r < 31) f ^= Z[zi(r - 1, 15 + vv + r, c)];
        *at(16 * r + vv) = f;
      }
    }
    __syncthreads();  // Z reuse by the next item
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ---- the last step of a forward 2^32-bit conversion fused with the Frobenius-partition encode
// (encode.cpp:165-193): conv(256) over the digit A of the rows B + 256 A (one item = a fixed B and
// 32 words of every row), then, instead of writing the converted rows back, the item's 4096 encode
// elements: element i = a 2^24 + B 2^16 + 1024 cb + e (a < 4, e < 1024) takes bit j < 64 (the
// operand's live partition rows) from converted row A = 4 j + a, bit 32 col + lane of the item's
// words -- rows 4j + a of the item are exactly a 64 x 1024-bit encode slab.  The slab goes through
// the warp transpose and the 8 byte-chunk lookups of encode_kernel<64>; the converted operand never
// reaches HBM (its write and the separate encode sweep's read disappear).
// GF(2^64) (M = 64, l = 27): 32 live partition rows of 2^27 bits, so converted row A = 8 j + a
// (a < 8, j < 32) and 4 byte-chunk G8 lookups per element (encode64_kernel<32>).  Rows of sub-slab
// a are stored at (A % S) (256 / S) + A / S, S = the number of sub-slabs (4 or 8): consecutive j,
// conflict-free transposes.
constexpr size_t kCTEncSmem = kCTSmem + 32768;  // + the x*E table (M8 chunks 0..7 / G8 chunks 0..3)
template <int M>
__global__ void __launch_bounds__(kCTThreads, 1) conv256_a_encode_kernel(const uint32_t* data, UnitMap um,
                                                                         uint64_t nitems,
                                                                         const __grid_constant__ CUtensorMap tmap,
                                                                         const void* __restrict__ tab_g,
                                                                         void* __restrict__ ev_out) {
  pdl_wait();
  using E = std::conditional_t<M == 128, uint4, uint2>;
  constexpr int S = M == 128 ? 4 : 8, RPS = 256 / S;  // sub-slabs, rows per sub-slab
  E* ev = static_cast<E*>(ev_out);
  extern __shared__ __align__(128) uint32_t sm_ct[];
  auto stage = [&](int st) { return sm_ct + st * (256 * kCT); };
  uint32_t* Z = sm_ct + 2 * 256 * kCT;  // [d][33][kCT]; after the conv: the converted rows [A][33]
  uint64_t* bar = reinterpret_cast<uint64_t*>(Z + 16 * 33 * kCT);
  uint4* tab = reinterpret_cast<uint4*>(sm_ct + (kCTSmem / 4));  // x*E byte-chunk table, 32 KiB
  const int tid = threadIdx.x, c = tid % kCT, r = tid / kCT, lane = tid & 31, warp = tid >> 5;
  constexpr int kCols = kTWords / kCT;
  auto zi = [](int d, int s, int cc) { return (d * 33 + s) * kCT + cc; };
  for (int i = tid; i < 32768 / 16; i += kCTThreads) tab[i] = static_cast<const uint4*>(tab_g)[i];
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](uint64_t it, int st) {
    if (tid != 0 || it >= nitems) return;
    mbar_expect_tx(&bar[st], (uint32_t)kCTStage);
    const uint64_t grp = it / kCols;
    const int c0 = (int)((it % kCols) * kCT), c1 = (int)(grp % um.gstride), c2 = (int)((grp / um.gstride) * 256);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(stage(st))),
        "l"(&tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(&bar[st]))
        : "memory");
  };
  const int q8 = lane & 7;
  const Transpose32 tr(lane);
  uint32_t phases = 0;
  issue(blockIdx.x, 0);
  issue(blockIdx.x + gridDim.x, 1);
  int st = 0;
  for (uint64_t it = blockIdx.x; it < nitems; it += gridDim.x, st ^= 1) {
    const uint64_t B = it / kCols, cb = it % kCols;  // groups = B (um.gstride = 256)
    const uint32_t* sg = stage(st);
    mbar_wait(&bar[st], (phases >> st) & 1u);
    phases ^= 1u << st;
    uint32_t x[16], y[16];
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      const int v0 = r - d, v1 = r + 16 - d;
      x[d] = v0 >= 0 ? sg[(16 * d + v0) * kCT + c] : 0u;
      y[d] = v1 < 16 ? sg[(16 * d + v1) * kCT + c] : 0u;
    }
    __syncthreads();
    if (tid == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue(it + 2 * (uint64_t)gridDim.x, st);
    zeta16_vals(x);
    zeta16_vals(y);
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      Z[zi(d, r, c)] = x[d];
      Z[zi(d, r + 16, c)] = y[d];
    }
    __syncthreads();
    const int v = r;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      uint32_t g = Z[zi(k, v + k, c)];
      if (v >= 1 && 15 + v + k < 31) g ^= Z[zi(k, 15 + v + k, c)];
      if (k >= 1 && 15 + v + k < 31) g ^= Z[zi(k - 1, 15 + v + k, c)];
      x[k] = g;
    }
    conv16_vals<false>(x);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) Z[zi(k, v, c)] = x[k];
    __syncthreads();
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) x[vv] = Z[zi(r, vv, c)];
    conv16_vals<false>(x);
    __syncthreads();  // every thread's conv input read from Z: Z now holds the converted rows
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) {  // row A = 16 r + vv stored at (A % S) RPS + A / S: the
      const int A = 16 * r + vv;        // encode's slab rows A = S j + a are then consecutive
      Z[((A % S) * RPS + A / S) * 33 + c] = x[vv];
    }
    __syncthreads();
    // encode: (a, col) pairs, 256 / 16 warps each; slab row j of sub-slab a is converted row S j + a
    const uint64_t e0 = B * 65536 + cb * 1024;
    constexpr int kPairsPerWarp = S * 32 / 16;
#pragma unroll 1
    for (int k = 0; k < kPairsPerWarp; ++k) {
      const int pair = warp * kPairsPerWarp + k, a = pair >> 5, col = pair & 31;
      const uint64_t ei = (uint64_t)a * (1u << 24) + e0 + 32 * col + lane;
      const uint32_t x0 = tr(Z[(a * RPS + lane) * 33 + col]);  // rows j = lane
      if constexpr (M == 128) {
        const uint32_t x1 = tr(Z[(a * RPS + 32 + lane) * 33 + col]);  // rows j = 32 + lane
        uint4 acc0 = make_uint4(0, 0, 0, 0), acc1 = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int kk = 0; kk < 8; kk += 2) {
          const int k0 = (kk + q8) & 7, k1 = (kk + 1 + q8) & 7;
          const uint32_t b0 = __byte_perm(k0 < 4 ? x0 : x1, 0, 0x4440u | (uint32_t)(k0 & 3));
          const uint32_t b1 = __byte_perm(k1 < 4 ? x0 : x1, 0, 0x4440u | (uint32_t)(k1 & 3));
          acc0 = x4v(acc0, tab[b0 * 8 + k0]);
          acc1 = x4v(acc1, tab[b1 * 8 + k1]);
        }
        ev[ei] = x4v(acc0, acc1);
      } else {  // G8 layout: entry (chunk c, value v, copy h) at v * 16 + 8 h + c (gf64.cuh)
        const uint2* t2 = reinterpret_cast<const uint2*>(tab);
        const int h8 = lane & 8;
        uint2 acc0 = make_uint2(0, 0), acc1 = make_uint2(0, 0);
#pragma unroll
        for (int kk = 0; kk < 4; kk += 2) {
          const int k0 = (kk + q8) & 3, k1 = (kk + 1 + q8) & 3;
          const uint32_t b0 = __byte_perm(x0, 0, 0x4440u | (uint32_t)k0);
          const uint32_t b1 = __byte_perm(x0, 0, 0x4440u | (uint32_t)k1);
          acc0 = x2(acc0, t2[b0 * 16 + h8 + k0]);
          acc1 = x2(acc1, t2[b1 * 16 + h8 + k1]);
        }
        ev[ei] = x2(acc0, acc1);
      }
    }
    __syncthreads();  // Z reuse by the next item
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ---- the first step of a 2^33-bit inverse conversion fused with the decode (encode.cpp:195-220):
// one item = a fixed row offset B and 32 words of every row, for BOTH 2^32-bit blocks.  The item's
// 4096 elements i = a 2^24 + B 2^16 + 1024 cb + e (a < 4) are decoded (16 byte-chunk lookups of
// x*E^-1, the warp transpose of decode_kernel), which yields, for block b, the rows A = 4 j + a
// (j = partition row - 64 b) of the item; then conv(256)^-1 over A (the inverse register phases of
// conv256_units_kernel) runs on each block's 256 rows and the results are stored.  The decoded
// product array never reaches HBM.
// GF(2^64) (M = 64): 64 partition rows of 2^27 bits, 32 per block; row A = 8 (j % 32) + a (a < 8);
// 8 G8 lookups per element (decode64_kernel).
constexpr size_t kDecRows = 256 * 33;  // one block's rows of an item, [A][33]
constexpr size_t kDecSmem = (size_t)kM8Uint4 * sizeof(uint4) + (2 * kDecRows + 16 * 33 * kCT) * sizeof(uint32_t);
template <int M>
__global__ void __launch_bounds__(kCTThreads, 1) decode_conv_a_kernel(const void* __restrict__ ev_in,
                                                                      const void* __restrict__ tab_g,
                                                                      uint32_t* __restrict__ w_lo,
                                                                      uint32_t* __restrict__ w_hi, uint64_t nitems) {
  pdl_wait();
  using E = std::conditional_t<M == 128, uint4, uint2>;
  constexpr int S = M == 128 ? 4 : 8, RPS = 256 / S;
  constexpr int kTabUint4 = M == 128 ? kM8Uint4 : kG8Uint2 / 2;
  const E* ev = static_cast<const E*>(ev_in);
  extern __shared__ __align__(16) uint4 sm_dc[];
  uint4* tab = sm_dc;  // x*E^-1 byte-chunk tables (gf128.cuh m8 / gf64.cuh g8 layout)
  uint32_t* Rw = reinterpret_cast<uint32_t*>(sm_dc + kM8Uint4);  // [block][A][33]
  uint32_t* Z = Rw + 2 * kDecRows;                                // [d][33][kCT]
  const int tid = threadIdx.x, c = tid % kCT, r = tid / kCT, lane = tid & 31, warp = tid >> 5;
  constexpr int kCols = kTWords / kCT;
  auto zi = [](int d, int s, int cc) { return (d * 33 + s) * kCT + cc; };
  for (int i = tid; i < kTabUint4; i += kCTThreads) tab[i] = static_cast<const uint4*>(tab_g)[i];
  const int q8 = lane & 7;
  const Transpose32 tr(lane);
  __syncthreads();
  constexpr int kPairsPerWarp = S * 32 / 16;
  for (uint64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const uint64_t B = it / kCols, cb = it % kCols;
    const uint64_t e0 = B * 65536 + cb * 1024;
    // ---- decode: (a, col) pairs; all the warp's elements' loads first
    E f[kPairsPerWarp];
#pragma unroll
    for (int k = 0; k < kPairsPerWarp; ++k) {
      const int pair = warp * kPairsPerWarp + k, a = pair >> 5, col = pair & 31;
      f[k] = __ldg(ev + (uint64_t)a * (1u << 24) + e0 + 32 * col + lane);
    }
#pragma unroll
    for (int k = 0; k < kPairsPerWarp; ++k) {
      const int pair = warp * kPairsPerWarp + k, a = pair >> 5, col = pair & 31;
      if constexpr (M == 128) {
        const uint4 y = m8_mul(tab, f[k], q8);
        // word q of y: partition rows 32q + lane after the transpose; block q >> 1, row A = 4 j + a
        const uint32_t yw[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = 32 * (q & 1) + lane;
          Rw[(q >> 1) * kDecRows + (a * RPS + j) * 33 + col] = tr(yw[q]);  // row A = S j + a
        }
      } else {
        const uint2 y = g8_mul(reinterpret_cast<const uint2*>(tab), f[k], lane);
        Rw[(a * RPS + lane) * 33 + col] = tr(y.x);             // rows 0..31: block 0
        Rw[kDecRows + (a * RPS + lane) * 33 + col] = tr(y.y);  // rows 32..63: block 1
      }
    }
    __syncthreads();
    // ---- conv(256)^-1 over A, each block (inverse phases of conv256_units_kernel)
#pragma unroll 1
    for (int blk = 0; blk < 2; ++blk) {
      const uint32_t* Rb = Rw + blk * kDecRows;
      uint32_t* const gbase = (blk ? w_hi : w_lo) + B * kTWords + cb * kCT + c;
      auto at = [&](int u) -> uint32_t* { return gbase + (uint64_t)u * 256 * kTWords; };
      uint32_t x[16];
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) {
        const int A = 16 * r + vv;
        x[vv] = Rb[((A % S) * RPS + A / S) * 33 + c];
      }
      conv16_vals<true>(x);
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) Z[zi(r, vv, c)] = x[vv];
      __syncthreads();
      const int v = r;
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = Z[zi(k, v, c)];
      conv16_vals<true>(x);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) Z[zi(k, v + k, c)] = x[k];
      __syncthreads();
      uint32_t y[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        x[k] = (r >= k) ? Z[zi(k, r, c)] : 0u;
        y[k] = (r + 16 < k + 16) ? Z[zi(k, r + 16, c)] : 0u;
      }
      zeta16_vals(x);
      zeta16_vals(y);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        Z[zi(k, r, c)] = x[k];
        Z[zi(k, r + 16, c)] = y[k];
      }
      __syncthreads();
#pragma unroll
      for (int vv = 0; vv < 16; ++vv) {
        uint32_t fv = Z[zi(r, vv + r, c)];
        if (r >= 1 && 15 + vv + r < 31) fv ^= Z[zi(r - 1, 15 + vv + r, c)];
        *at(16 * r + vv) = fv;
      }
      __syncthreads();  // Z reuse
    }
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// One block of decode_conv_a_kernel (GF(2^128), tower representation): the 64 product rows of the
// block only (16 LDS.64 lookups per element in dec_half_r[HALF], conflict-free), then conv(256)^-1
// over A for that block.  The upper block's copy-out can start after half the decode work.
constexpr size_t kDecHalfSmem = 4096 * sizeof(uint2) + (kDecRows + 16 * 33 * kCT) * sizeof(uint32_t);
template <int HALF>
__global__ void __launch_bounds__(kCTThreads, 1) decode_half_conv_a_kernel(const uint4* __restrict__ ev,
                                                                           const uint2* __restrict__ tab_g,
                                                                           uint32_t* __restrict__ w, uint64_t nitems) {
  pdl_wait();
  constexpr int S = 4, RPS = 256 / S;
  extern __shared__ __align__(16) uint2 sm_dh[];
  uint2* tab = sm_dh;                                              // [v][16 byte indices]
  uint32_t* Rw = reinterpret_cast<uint32_t*>(sm_dh + 4096);      // [A][33]
  uint32_t* Z = Rw + kDecRows;                                     // [d][33][kCT]
  const int tid = threadIdx.x, c = tid % kCT, r = tid / kCT, lane = tid & 31, warp = tid >> 5;
  constexpr int kCols = kTWords / kCT;
  auto zi = [](int d, int s, int cc) { return (d * 33 + s) * kCT + cc; };
  for (int i = tid; i < 4096; i += kCTThreads) tab[i] = tab_g[i];
  const int q16 = lane & 15;
  const Transpose32 tr(lane);
  __syncthreads();
  constexpr int kPairsPerWarp = S * 32 / 16;
  const uint32_t tbase = (uint32_t)__cvta_generic_to_shared(tab);
  for (uint64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const uint64_t B = it / kCols, cb = it % kCols;
    const uint64_t e0 = B * 65536 + cb * 1024;
    uint4 f[kPairsPerWarp];
#pragma unroll
    for (int k = 0; k < kPairsPerWarp; ++k) {
      const int pair = warp * kPairsPerWarp + k, a = pair >> 5, col = pair & 31;
      f[k] = __ldg(ev + (uint64_t)a * (1u << 24) + e0 + 32 * col + lane);
    }
#pragma unroll
    for (int k = 0; k < kPairsPerWarp; ++k) {
      const int pair = warp * kPairsPerWarp + k, a = pair >> 5, col = pair & 31;
      const uint32_t fw[4] = {f[k].x, f[k].y, f[k].z, f[k].w};
      uint2 y0 = make_uint2(0, 0), y1 = make_uint2(0, 0);
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const int cc = (kk + q16) & 15;  // byte index: lanes l and l + 16 share it, but read one bank pair each
        const uint32_t v = __byte_perm(fw[cc >> 2], 0, 0x4440u | (uint32_t)(cc & 3));
        uint2 e;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(e.x), "=r"(e.y) : "r"(tbase + 8u * (16u * v + (uint32_t)cc)));
        if (kk & 1) { y1.x ^= e.x; y1.y ^= e.y; } else { y0.x ^= e.x; y0.y ^= e.y; }
      }
      const uint32_t yw[2] = {y0.x ^ y1.x, y0.y ^ y1.y};
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int j = 32 * q + lane;
        Rw[(a * RPS + j) * 33 + col] = tr(yw[q]);  // row A = S j + a of this block
      }
    }
    __syncthreads();
    // ---- conv(256)^-1 over A (as decode_conv_a_kernel)
    uint32_t* const gbase = w + B * kTWords + cb * kCT + c;
    auto at = [&](int u) -> uint32_t* { return gbase + (uint64_t)u * 256 * kTWords; };
    uint32_t x[16];
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) {
      const int A = 16 * r + vv;
      x[vv] = Rw[((A % S) * RPS + A / S) * 33 + c];
    }
    conv16_vals<true>(x);
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) Z[zi(r, vv, c)] = x[vv];
    __syncthreads();
    const int v = r;
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = Z[zi(k, v, c)];
    conv16_vals<true>(x);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) Z[zi(k, v + k, c)] = x[k];
    __syncthreads();
    uint32_t y[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x[k] = (r >= k) ? Z[zi(k, r, c)] : 0u;
      y[k] = (r + 16 < k + 16) ? Z[zi(k, r + 16, c)] : 0u;
    }
    zeta16_vals(x);
    zeta16_vals(y);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      Z[zi(k, r, c)] = x[k];
      Z[zi(k, r + 16, c)] = y[k];
    }
    __syncthreads();
#pragma unroll
    for (int vv = 0; vv < 16; ++vv) {
      uint32_t fv = Z[zi(r, vv + r, c)];
      if (r >= 1 && 15 + vv + r < 31) fv ^= Z[zi(r - 1, 15 + vv + r, c)];
      *at(16 * r + vv) = fv;
    }
    __syncthreads();  // Rw / Z reuse
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ unit-level L1 carry + C_cols
// Rows of t bits are units; row d = 256 * dh + v (digit dh, offset v).  After the unit-skewed zeta,
// Gs[kh] holds units u = 0 .. 256+Dd-1 (pitch gs_pitch words).  Output unit (kh, v):
//   g = Gs[kh][v+kh] ^ (v >= 1 ? Gs[kh][256+v-1+kh] : 0) ^ (kh >= 1 ? Gs[kh-1][256+v+kh-1] : 0)
// followed by conv(Dd) over kh (C_cols, row passes in shared memory).  Item = (v, 8-word column).
__global__ void __launch_bounds__(256) unit_carry_cols_kernel(const uint32_t* __restrict__ gs, uint64_t gs_pitch,
                                                              uint32_t* __restrict__ out, int gd, uint64_t items) {
  pdl_wait();
  extern __shared__ __align__(16) uint32_t tile[];  // 256 x kRowPitchW<kSlabW>
  constexpr int W = kSlabW, cpr = kTWords / (8 * W);
  const int tid = threadIdx.x;
  const int kh = tid & ((1 << gd) - 1), slot = tid >> gd;
  const int ipc = 256 >> gd;
  const uint64_t Dd = (uint64_t)1 << gd;
  for (uint64_t ib = (uint64_t)blockIdx.x * ipc; ib < items; ib += (uint64_t)gridDim.x * ipc) {
    const uint64_t item = ib + slot;
    const uint64_t v = item / cpr, col = item % cpr;
    uint32_t m[W][8];
#pragma unroll
    for (int c = 0; c < W; ++c)
#pragma unroll
      for (int k = 0; k < 8; ++k) m[c][k] = 0;
    if (item < items) {
      auto add = [&](const uint32_t* p) {
        const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
        for (int c = 0; c < W; ++c) {
          const uint4 a = q[2 * c], b = q[2 * c + 1];
          m[c][0] ^= a.x; m[c][1] ^= a.y; m[c][2] ^= a.z; m[c][3] ^= a.w;
          m[c][4] ^= b.x; m[c][5] ^= b.y; m[c][6] ^= b.z; m[c][7] ^= b.w;
        }
      };
      // units >= 256 + Dd of a skewed digit row are zero (not stored)
      const uint32_t* rk = gs + (uint64_t)kh * gs_pitch + col * 8 * W;
      add(rk + (v + kh) * kTWords);
      if (v >= 1 && v - 1 + kh < Dd) add(rk + (256 + v - 1 + kh) * kTWords);
      if (kh >= 1 && v + kh - 1 < Dd) add(rk - gs_pitch + (256 + v + kh - 1) * kTWords);
    }
    rowpasses_w<false, W>(m, tile, gd, kh);
    if (item < items) {
      uint4* o = reinterpret_cast<uint4*>(out + ((uint64_t)kh * 256 + v) * kTWords + col * 8 * W);
#pragma unroll
      for (int c = 0; c < W; ++c) {
        o[2 * c] = make_uint4(m[c][0], m[c][1], m[c][2], m[c][3]);
        o[2 * c + 1] = make_uint4(m[c][4], m[c][5], m[c][6], m[c][7]);
      }
    }
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// Unit-level L1 inverse tail: F[256 dh + v] = Gs[dh][v+dh] ^ (dh >= 1 ? Gs[dh-1][256+v+dh-1] : 0).
__global__ void unit_overflow_kernel(const uint32_t* __restrict__ gs, uint64_t gs_pitch, uint32_t* __restrict__ out,
                                     uint64_t Dd) {
  pdl_wait();
  const uint64_t q_per_row = kTWords / 4;
  const uint64_t total = Dd * 256 * q_per_row;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = k / q_per_row, q = k % q_per_row;
    const uint64_t dh = row >> 8, v = row & 255;
    uint4 a = reinterpret_cast<const uint4*>(gs + dh * gs_pitch + (v + dh) * kTWords)[q];
    if (dh && v + dh - 1 < Dd) {
      const uint4 b = reinterpret_cast<const uint4*>(gs + (dh - 1) * gs_pitch + (256 + v + dh - 1) * kTWords)[q];
      a.x ^= b.x; a.y ^= b.y; a.z ^= b.z; a.w ^= b.w;
    }
    reinterpret_cast<uint4*>(out)[k] = a;
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ L1_outer: Taylor step in z = y^256
// L1 (the Taylor expansion in y = x^t + x over D = 2^lgD rows, t = 2^16) factors as L1_inner o L1_outer
// with z = y^256 = x^(2^24) + x^256 (tools/models/bc2_model.py): L1_outer expands the array in z over
// DA = D / 256 chunks of 2^24 bits (digits c, skew 256 c bits = 8 c words: word aligned, so the
// absolute-frame windows read and write the same words and the step runs IN PLACE); L1_inner is then
// the 256-row step inside every chunk (skew < 256 bits).  Generic two-term step, R = 2^nb digits:
//   forward  G_e = sum_{c superset e} x^(256(c-e)) f_c ;  F_e = (G_e mod x^T) + x^256 (G_e div x^T) + (G_{e-1} div x^T)
//   inverse  F'_c = sum_{e superset c} x^(256(e-c)) F_e ;  f_c = (F'_c mod x^T) + (F'_{c-1} div x^T)
// Both are the same superset zeta in the absolute frame (row c read at word offset -8c); every row's
// part beyond its own 2^19-word window goes to `side` (R rows x 8R words) and is folded into the first
// 8R words of rows e and e+1 (forward) / c+1 (inverse) by outer_fix_kernel.
// top (inverse, 2^33-bit arrays): the single top pass fused into the lower block's stores, as in
// overflow_kernel.
constexpr uint64_t kChunkWords = (uint64_t)1 << 19;
// Geometry of one generic two-term step: `groups` independent groups (group_words apart), each of
// R = 2^nb digit rows of row_words words (rows row_words apart), skew skew_words per digit (a
// multiple of 4 words); side: per group R rows x R*skew_words words.
struct StepGeom {
  uint64_t row_words, skew_words, group_words;
  int nb;
  uint64_t side_pitch() const { return skew_words << nb; }
  uint64_t windows() const { return (row_words + skew_words * (((uint64_t)1 << nb) - 1) + kZW - 1) / kZW; }
};
// NB = log2 R (template: the tile-row -> (row, window) split is then compile-time and every load /
// store address is one add from a per-thread base).
// The window blocks (wpc windows each) a launch processes: wb = lo + period (j / n) + first + j % n for
// j < count, wb < hi -- all of them by default; a contiguous range (L1_outer) or the blocks of one
// column range (T_d steps: the column of a block is wb mod period) for a rank of the sharded
// conversion.
struct WinSel {
  uint64_t lo = 0, hi = ~(uint64_t)0, count = 0;  // count = 0: every block of [0, wblocks)
  uint32_t period = 1, first = 0, n = 1;
};
template <int NB>
__global__ void __launch_bounds__(256, 3) outer_zeta_kernel(const uint32_t* src, uint32_t* dst, const StepGeom gm,
                                                            uint64_t windows, uint64_t groups,
                                                            uint32_t* __restrict__ side,
                                                            const uint32_t* __restrict__ top, const WinSel sel) {
  pdl_wait();
  extern __shared__ __align__(16) uint32_t sx[];  // 256 x kZP
  constexpr int R = 1 << NB, wpc = 256 >> NB;
  const int tid = threadIdx.x, c = tid & 31, w8 = tid >> 5;
  const uint64_t wblocks = (windows + wpc - 1) / wpc;
  const uint64_t side_pitch = gm.skew_words << NB;
  const int64_t rw = (int64_t)gm.row_words, sk = (int64_t)gm.skew_words;
  const uint64_t nsel = sel.count ? sel.count : wblocks;
  const uint64_t items = nsel * groups;
  for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const uint64_t grp = it / nsel, j = it - grp * nsel;
    const uint64_t wb = sel.count ? sel.lo + sel.period * (j / sel.n) + sel.first + j % sel.n : j;
    if (wb >= wblocks || wb >= sel.hi) continue;
    const uint32_t* gsrc = src + grp * gm.group_words;
    const int64_t wi0 = (int64_t)(wb * wpc);
    // mapping A: word c of tile rows TR = w8 + 8k; row j = TR % R, window slot TR / R
    uint32_t a[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int TR = w8 + 8 * k, j = TR & (R - 1), slot = TR >> NB;
      const int64_t wi = wi0 + slot;
      const int64_t iw = wi * kZW + c - sk * j;
      a[k] = (wi < (int64_t)windows && iw >= 0 && iw < rw) ? gsrc[j * rw + iw] : 0u;
    }
#pragma unroll
    for (int b = 3; b < 8; ++b) {
      if (b < NB) {
        const int kb = 1 << (b - 3);
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (!(k & kb)) a[k] ^= a[k | kb];
      }
    }
#pragma unroll
    for (int k = 0; k < 32; ++k) sx[(w8 + 8 * k) * kZP + c] = a[k];
    __syncthreads();
    const int q = tid & 7, R0 = 8 * (tid >> 3);
    uint4 bq[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) bq[k] = *reinterpret_cast<const uint4*>(sx + (R0 + k) * kZP + 4 * q);
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      if (b < NB) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (!(k & (1 << b))) bq[k] = make_uint4(bq[k].x ^ bq[k | (1 << b)].x, bq[k].y ^ bq[k | (1 << b)].y,
                                                   bq[k].z ^ bq[k | (1 << b)].z, bq[k].w ^ bq[k | (1 << b)].w);
      }
    }
    uint32_t* gdst = dst + grp * gm.group_words;
    uint32_t* gside = side + grp * (side_pitch << NB);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int TR = R0 + k, j = TR & (R - 1), slot = TR >> NB;
      const int64_t wi = wi0 + slot;
      const int64_t iw = wi * kZW + 4 * q - sk * j;  // 4 words, one region (all multiples of 4)
      if (wi >= (int64_t)windows || iw < 0) continue;
      uint4 v = bq[k];
      if (iw < rw) {
        const uint64_t g = (uint64_t)(j * rw + iw);
        if (top) {
          const uint64_t G = grp * gm.group_words + g;
          const uint4 t4 = *reinterpret_cast<const uint4*>(top + G);
          const uint32_t tp = G ? top[G - 1] : 0u;
          v.x ^= (t4.x << 1) | (tp >> 31);
          v.y ^= (t4.y << 1) | (t4.x >> 31);
          v.z ^= (t4.z << 1) | (t4.y >> 31);
          v.w ^= (t4.w << 1) | (t4.z >> 31);
        }
        *reinterpret_cast<uint4*>(gdst + g) = v;
      } else if ((uint64_t)(iw - rw) < side_pitch) {
        *reinterpret_cast<uint4*>(gside + (uint64_t)j * side_pitch + (uint64_t)(iw - rw)) = v;
      }
    }
    __syncthreads();
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// Folds the beyond-window parts into the first R*skew words of the rows (row e's side holds
// skew*(R-1-e) meaningful words): forward F_e[p] ^= side_e[p-skew] ^ side_{e-1}[p];
// inverse f_c[p] ^= side_{c-1}[p].  Four words per thread.
// FixSel: rows e in [e_lo, e_hi) and words p with (p mod 2048) - col_lo < col_n (a rank's chunks /
// columns in the sharded conversion; default all).
struct FixSel {
  uint32_t e_lo = 0, e_hi = ~0u, col_lo = 0, col_n = 2048;
};
template <bool INV>
__global__ void outer_fix_kernel(uint32_t* __restrict__ dst, const uint32_t* __restrict__ side, const StepGeom gm,
                                 uint64_t groups, const FixSel fs) {
  pdl_wait();
  const uint64_t R = (uint64_t)1 << gm.nb, P = gm.skew_words << gm.nb, S = gm.skew_words, per_group = R * P / 4;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < groups * per_group;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t grp = k / per_group, r = k % per_group;
    const uint64_t e = r / (P / 4), p = 4 * (r % (P / 4));
    if (e < fs.e_lo || e >= fs.e_hi || (uint32_t)((p & 2047) - fs.col_lo) >= fs.col_n) continue;
    const uint32_t* gs = side + grp * R * P;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (!INV && p >= S && p - S < S * (R - 1 - e)) v = *reinterpret_cast<const uint4*>(gs + e * P + p - S);
    if (e >= 1 && p < S * (R - e)) v = x4v(v, *reinterpret_cast<const uint4*>(gs + (e - 1) * P + p));
    if (v.x | v.y | v.z | v.w) {
      uint4* d = reinterpret_cast<uint4*>(dst + grp * gm.group_words + e * gm.row_words + p);
      *d = x4v(*d, v);
    }
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ host orchestration
void set_smem_attr() {
  static PerDeviceOnce once;
  once.run([] {
    FPM_CUDA(cudaFuncSetAttribute(conv_rows_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmem));
    FPM_CUDA(cudaFuncSetAttribute(conv_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmem));
    FPM_CUDA(cudaFuncSetAttribute(carry_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmem));
  });
}

int grid_cap(uint64_t items, int per_sm) {
  const uint64_t g = std::min<uint64_t>(items, (uint64_t)sm_count() * per_sm);
  return (int)(g ? g : 1);
}

void conv_rows(uint32_t* data, uint64_t nwords, int r, bool inv, cudaStream_t s) {
  const uint64_t tiles = nwords < 2048 ? 1 : nwords / 2048;
  if (inv) launch_k(conv_rows_kernel<true>, dim3(grid_cap(tiles, 7)), dim3(256), kTileSmem, s, data, nwords, r);
  else launch_k(conv_rows_kernel<false>, dim3(grid_cap(tiles, 7)), dim3(256), kTileSmem, s, data, nwords, r);
  FPM_LAUNCH_CHECK();
}

// src_row_words: words of one source row (reads beyond are zeros).
void zeta(const uint32_t* src, uint64_t src_pitch, uint32_t* dst, uint64_t dst_pitch, uint64_t D, int b0, int nb,
          Skew skew, uint64_t windows, cudaStream_t s, uint64_t src_row_words) {
  if (nb <= 0) return;
  const int wpc = 256 >> nb;
  const uint64_t items = (D >> nb) * ((windows + wpc - 1) / wpc);
  if (skew.mask && skew.log < 5)
    if (nb == 8)
      launch_k(zeta_kernel<true, true>, dim3(grid_cap(items, 3)), dim3(256), 256 * kZP * sizeof(uint32_t), s, src, src_pitch, dst, dst_pitch, D, b0, nb, skew, src_row_words, windows);
    else
      launch_k(zeta_kernel<true>, dim3(grid_cap(items, 4)), dim3(256), 256 * kZP * sizeof(uint32_t), s, src, src_pitch, dst, dst_pitch, D, b0, nb, skew, src_row_words, windows);
  else
    launch_k(zeta_kernel<false>, dim3(grid_cap(items, 4)), dim3(256), 256 * kZP * sizeof(uint32_t), s, src, src_pitch, dst, dst_pitch, D, b0, nb, skew, src_row_words, windows);
  FPM_LAUNCH_CHECK();
}

constexpr size_t kSlabSmem = 256 * kRowPitchW<kSlabW> * sizeof(uint32_t);
// nslabs counts 8-word columns (callers' unit); the kernels take kSlabW of them per slab.
// conv(256) over groups of 256 units: group g's unit u is row base(g) + u * ustride, base(g) =
// (g % gstride) + (g / gstride) * 256 * gstride.
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    FPM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw Error(kCuda, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// The unit view of conv256_units as a 3-D uint32 tensor: (word of a row, group index within the
// stride, unit row), box 32 x 1 x 256.
CUtensorMap unit_tensor_map(uint32_t* w, uint64_t rows, uint64_t gstride) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {(cuuint64_t)kTWords, (cuuint64_t)gstride, (cuuint64_t)(rows / gstride)};
  const cuuint64_t strides[2] = {(cuuint64_t)kTWords * 4, (cuuint64_t)kTWords * 4 * gstride};
  const cuuint32_t box[3] = {(cuuint32_t)kCT, 1, 256};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, w, dims, strides, box, estr,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(kCuda, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

bool tma_units_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FPM_TMA_UNITS");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

void conv256_units(uint32_t* w, uint64_t ngroups, uint64_t ustride, uint64_t gstride, bool inv, cudaStream_t s,
                   CarrySrc cs = CarrySrc{}, int q = 0, int Q = 1) {
  static PerDeviceOnce attr;
  attr.run([&] {
    FPM_CUDA(cudaFuncSetAttribute(conv256_units_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kC256Smem));
    FPM_CUDA(cudaFuncSetAttribute(conv256_units_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kC256Smem));
  });
  UnitMap um{ustride, gstride, ngroups};
  if (Q > 1) {  // a rank's column items (TMA path only)
    if (cs.gs || !tma_units_enabled()) throw Error(kInvalid, "conv256_units: column shares need the TMA path");
    um.ncols = (uint32_t)(kTWords / kCT / Q);
    um.col_lo = (uint32_t)(q * um.ncols);
  }
  if (!cs.gs && tma_units_enabled()) {
    static PerDeviceOnce tattr;
    tattr.run([&] {
      FPM_CUDA(cudaFuncSetAttribute(conv256_units_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCTSmem));
      FPM_CUDA(cudaFuncSetAttribute(conv256_units_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCTSmem));
    });
    const uint64_t titems = ngroups * (um.ncols ? um.ncols : kTWords / kCT);
    // groups of 256 units: (ustride, gstride) = (1, 1) consecutive rows, or (g, g) rows g apart
    if (ustride != gstride) throw Error(kInvalid, "conv256_units: unit stride must equal the group stride");
    const CUtensorMap tm = unit_tensor_map(w, ngroups * 256, gstride);
    if (inv) launch_k(conv256_units_tma_kernel<true>, dim3(grid_cap(titems, kCTMinBlocks)), dim3(kCTThreads), kCTSmem, s, w, um, titems, tm);
    else launch_k(conv256_units_tma_kernel<false>, dim3(grid_cap(titems, kCTMinBlocks)), dim3(kCTThreads), kCTSmem, s, w, um, titems, tm);
    FPM_LAUNCH_CHECK();
    return;
  }
  const uint64_t items = ngroups * (kTWords / kC256Cols);
  if (inv) launch_k(conv256_units_kernel<true>, dim3(grid_cap(items, 3)), dim3(kC256Threads), kC256Smem, s, w, um, items, cs);
  else launch_k(conv256_units_kernel<false>, dim3(grid_cap(items, 4)), dim3(kC256Threads), kC256Smem, s, w, um, items, cs);
  FPM_LAUNCH_CHECK();
}

void slab(uint32_t* w, int g, uint64_t rstride, uint64_t nslabs, bool inv, cudaStream_t s) {
  static_assert(kSlabSmem <= 48 * 1024, "slab tile fits the default dynamic smem limit");
  nslabs /= kSlabW;
  const int spc = 256 >> g;
  const uint64_t ctas = (nslabs + spc - 1) / spc;
  if (inv) launch_k(slab_kernel<true>, dim3(grid_cap(ctas, 6)), dim3(256), kSlabSmem, s, w, g, rstride, nslabs);
  else launch_k(slab_kernel<false>, dim3(grid_cap(ctas, 6)), dim3(256), kSlabSmem, s, w, g, rstride, nslabs);
  FPM_LAUNCH_CHECK();
}

void unit_carry_cols(const uint32_t* gs, uint64_t gs_pitch, uint32_t* out, int gd, cudaStream_t s) {
  const uint64_t items = 256 * (kTWords / (8 * kSlabW));
  const int spc = 256 >> gd;
  launch_k(unit_carry_cols_kernel, dim3(grid_cap((items + spc - 1) / spc, 6)), dim3(256), kSlabSmem, s, gs, gs_pitch, out, gd, items);
  FPM_LAUNCH_CHECK();
}

void unit_overflow(const uint32_t* gs, uint64_t gs_pitch, uint32_t* out, uint64_t Dd, cudaStream_t s) {
  const uint64_t total = Dd * 256 * (kTWords / 4);
  launch_k(unit_overflow_kernel, dim3(grid_cap((total + 255) / 256, 16)), dim3(256), 0, s, gs, gs_pitch, out, Dd);
  FPM_LAUNCH_CHECK();
}

// conv over the row index (D rows of t bits), forward or inverse.
void conv_cols(uint32_t* w, uint32_t* scratch, int lgD, bool inv, cudaStream_t s) {
  if (lgD <= 1) return;  // conv(2) is the identity (no passes)
  if (lgD <= 8) {
    slab(w, lgD, 1, kTWords / 8, inv, s);
    return;
  }
  // D > 256 rows: conv(2^lgD) over the row index with whole rows as units, by the same recursion
  // one level up: digits of 256 rows, Dd = D / 256 digits.
  //   forward  L1(256, Dd) over units (row-skew + zeta, then carry fused with C_cols), C_rows
  //   inverse  C_rows^-1, C_cols^-1, L1^-1 (row-skew + zeta, then overflow)
  const int gd = lgD - 8;
  const uint64_t Dd = (uint64_t)1 << gd;
  const uint64_t su = 256 + std::max<uint64_t>(Dd, 1);           // skewed units per digit row
  const uint64_t sk_pitch = su * kTWords;                         // words
  const uint64_t windows = sk_pitch / kZW;
  Skew unit_skew;  // digit row dh read at offset -dh whole rows
  unit_skew.mask = ~(uint64_t)0;
  unit_skew.log = kTLog2;
  if (!inv) {
    zeta(w, 256 * (uint64_t)kTWords, scratch, sk_pitch, Dd, 0, gd, unit_skew, windows, s, 256 * (uint64_t)kTWords);
    if (gd == 8) {  // carry fused into the conv(256) over the high digit (row stride 256)
      CarrySrc cs;
      cs.gs = scratch;
      cs.gs_pitch = sk_pitch;
      conv256_units(w, 256, 256, 256, false, s, cs);
    } else {
      unit_carry_cols(scratch, sk_pitch, w, gd, s);
    }
    conv256_units(w, Dd, 1, 1, false, s);                         // C_rows: conv(256) over consecutive rows
  } else {
    conv256_units(w, Dd, 1, 1, true, s);
    if (gd == 8) conv256_units(w, 256, 256, 256, true, s);        // C_cols^-1: conv(Dd) at row stride 256
    else slab(w, gd, 256, 256 * (kTWords / 8), true, s);
    zeta(w, 256 * (uint64_t)kTWords, scratch, sk_pitch, Dd, 0, gd, unit_skew, windows, s, 256 * (uint64_t)kTWords);
    unit_overflow(scratch, sk_pitch, w, Dd, s);
  }
}

// conv(2^K) for 17 <= K <= 32 on w (2^K bits).  scratch >= 2^(K-16) * (2^16 + max(2^(K-16), 1024)) bits.
// src (forward only, may be null): read the unconverted rows from src instead of w (w is first
// written by the carry pass, so an input buffer need not be copied into w beforehand).
// top (inverse only): fuse the 2^33-bit top pass into this (lower) block's last kernel.
void conv2d(uint32_t* w, int K, bool inv, uint32_t* scratch, cudaStream_t s, const uint32_t* src = nullptr,
            const uint32_t* top = nullptr) {
  const int lgD = K - kTLog2;
  const uint64_t D = (uint64_t)1 << lgD;
  const uint64_t wsk_bits = kT + std::max<uint64_t>(D, 32 * kZW);
  const uint64_t wsk = wsk_bits / 32;  // skewed row pitch (words)
  const uint64_t windows = wsk / kZW;
  const int nb_lo = std::min(lgD, 8), nb_hi = lgD - nb_lo;
  // first launch: skew by the low 8 digit bits into rows of t + 1024 bits (scratch tail), second:
  // the word-aligned 256 * (d >> 8) skew, into full skewed rows (scratch head)
  const uint64_t w1 = (kT + 32 * kZW) / 32;
  uint32_t* s1 = nb_hi ? scratch + D * wsk : scratch;
  const uint64_t p1 = nb_hi ? w1 : wsk;
  Skew lo_skew, hi_skew;
  lo_skew.mask = 255;
  hi_skew.mask = ~(uint64_t)0; hi_skew.lo = 8; hi_skew.log = 8;
  auto l1_zeta = [&](const uint32_t* src) {
    zeta(src, kTWords, s1, p1, D, 0, nb_lo, lo_skew, p1 / kZW, s, kTWords);
    if (nb_hi) zeta(s1, w1, scratch, wsk, D, 8, nb_hi, hi_skew, windows, s, w1);
  };
  if (!inv) {
    l1_zeta(src ? src : w);
    launch_k(carry_rows_kernel, dim3(grid_cap(D, 7)), dim3(256), kTileSmem, s, scratch, wsk, w, D, ~(uint64_t)0);
    FPM_LAUNCH_CHECK();
    conv_cols(w, scratch, lgD, false, s);
  } else {
    conv_rows(w, D * kTWords, kTLog2, true, s);
    conv_cols(w, scratch, lgD, true, s);
    l1_zeta(w);
    launch_k(overflow_kernel, dim3(grid_cap(D, 8)), dim3(256), 0, s, scratch, wsk, w, D, top, ~(uint64_t)0);
    FPM_LAUNCH_CHECK();
  }
}

// conv(2^K), 17 <= K <= 32, with L1 factored as L1_inner o L1_outer (see outer_zeta_kernel):
//   forward  [K > 24: L1_outer in place + fix-up] -> L1_inner (256-row skewed zeta -> scratch, then
//            chunk-local carry fused with conv(2^16) of every row) -> C_cols = conv(D) over the rows
//   inverse  C_cols^-1 -> conv(2^16)^-1 of every row -> L1_inner^-1 (zeta -> scratch, chunk-local
//            overflow) -> [K > 24: L1_outer^-1 in place (+ the fused 2^33 top pass) + fix-up]
// No step writes a skewed array wider than t + 1024 bits per row (the single-step L1 of conv2d skews
// rows by up to D = t bits: 2x the array).  scratch >= D * (t + 1024) bits and the C_cols scratch.
// One generic two-term step (outer_zeta_kernel + fix-up), in place on w (or from src).
void outer_fix(uint32_t* w, const uint32_t* side, StepGeom gm, uint64_t groups, bool inv, cudaStream_t s,
               FixSel fs = FixSel{}) {
  const uint64_t fix = groups * (gm.side_pitch() << gm.nb) / 4;
  if (inv) launch_k(outer_fix_kernel<true>, dim3(grid_cap((fix + 255) / 256, 8)), dim3(256), 0, s, w, side, gm, groups, fs);
  else launch_k(outer_fix_kernel<false>, dim3(grid_cap((fix + 255) / 256, 8)), dim3(256), 0, s, w, side, gm, groups, fs);
  FPM_LAUNCH_CHECK();
}

// The zeta half of a two-term step over the selected window blocks (no fix-up).
void outer_zeta(const uint32_t* src, uint32_t* w, StepGeom gm, uint64_t groups, uint32_t* side, cudaStream_t s,
                const uint32_t* top = nullptr, WinSel sel = WinSel{}) {
  const int wpc = 256 >> gm.nb;
  const uint64_t wblocks = (gm.windows() + wpc - 1) / wpc;
  const uint64_t items = (sel.count ? sel.count : wblocks) * groups;
  const size_t smem = 256 * kZP * sizeof(uint32_t);  // 36 KiB: under the default dynamic limit
  const int grid = grid_cap(items, 3);
  switch (gm.nb) {
#define FPM_OUTER(NB) \
    case NB: launch_k(outer_zeta_kernel<NB>, dim3(grid), dim3(256), smem, s, src, w, gm, gm.windows(), groups, side, top, sel); break;
    FPM_OUTER(1) FPM_OUTER(2) FPM_OUTER(3) FPM_OUTER(4) FPM_OUTER(5) FPM_OUTER(6) FPM_OUTER(7) FPM_OUTER(8)
#undef FPM_OUTER
    default: throw Error(kInvalid, "two-term step: 1..8 digit bits");
  }
  FPM_LAUNCH_CHECK();
}

// Column selection of a T_d step for rank q of Q (Q | 4): window blocks of wpc windows cover
// 32 wpc words of a 2048-word row; the blocks of columns [q 2048/Q, (q+1) 2048/Q).
WinSel column_sel(StepGeom gm, int q, int Q) {
  WinSel sel;
  if (Q <= 1) return sel;
  const uint64_t wpc = 256 >> gm.nb, bw = 32 * wpc;  // words per window block
  if (2048 % bw || (2048 / bw) % (uint64_t)Q) throw Error(kInvalid, "column_sel: unsupported step geometry");
  const uint64_t per_row = 2048 / bw, wblocks = (gm.windows() + wpc - 1) / wpc;
  sel.period = (uint32_t)per_row;
  sel.n = (uint32_t)(per_row / Q);
  sel.first = (uint32_t)(q * sel.n);
  sel.count = (wblocks + per_row - 1) / per_row * sel.n;
  return sel;
}

void two_term_step(const uint32_t* src, uint32_t* w, StepGeom gm, uint64_t groups, uint32_t* side, bool inv,
                   cudaStream_t s, const uint32_t* top = nullptr, int q = 0, int Q = 1) {
  outer_zeta(src, w, gm, groups, side, s, top, column_sel(gm, q, Q));
  FixSel fs;
  if (Q > 1) {
    fs.col_lo = (uint32_t)(q * (2048 / Q));
    fs.col_n = (uint32_t)(2048 / Q);
  }
  outer_fix(w, side, gm, groups, inv, s, fs);
}

// Side words the split steps need for D = 2^lgD rows (max over the steps, per call).
uint64_t split_side_words(int lgD) {
  uint64_t m = 0;
  if (lgD > 8) m = std::max<uint64_t>(m, (uint64_t)8 << (2 * (lgD - 8)));  // L1_outer
  const int gd = lgD - 8;
  if (gd > 4) {  // T_d's w^(2^k) and w steps
    const int k = gd / 2;
    m = std::max<uint64_t>(m, ((uint64_t)kTWords << k) << (2 * (gd - k)));
    m = std::max<uint64_t>(m, ((uint64_t)kTWords << (2 * k)) << (gd - k));
  } else if (gd > 0) {
    m = std::max<uint64_t>(m, (uint64_t)kTWords << (2 * gd));
  }
  return m;
}

// C_cols = conv(D) over the row index (rows of t bits as units), D = 2^lgD, without any skewed copy:
// lgD <= 8: slab passes; else (digits of 256 rows, Dd = D/256 of them):
//   L1_d (Taylor in w = y^256 + y over the row index, unit skews) as two in-place steps, w^(2^k)
//   over Dd/2^k digits of 256*2^k rows (skew 2^k rows) then w inside each chunk (skew 1 row)
//   (tools/models/bc2_model.py), then conv(Dd) over the digit (rows 256 apart) and conv(256) over
//   the row within the digit.  The inverse runs the same in reverse.
void conv256_a_encode(uint32_t* w, const EncodeSink& enc, cudaStream_t s) {
  static PerDeviceOnce attr;
  attr.run([] {
    FPM_CUDA(cudaFuncSetAttribute(conv256_a_encode_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCTEncSmem));
    FPM_CUDA(cudaFuncSetAttribute(conv256_a_encode_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCTEncSmem));
  });
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const DeviceTables& dt = device_tables(dev);
  UnitMap um{256, 256, 256};
  const uint64_t items = 256 * (kTWords / kCT);
  const CUtensorMap tm = unit_tensor_map(w, 65536, 256);
  const int grid = grid_cap(items, 1);
  if (enc.m == 64)
    launch_k(conv256_a_encode_kernel<64>, dim3(grid), dim3(kCTThreads), kCTEncSmem, s, w, um, items, tm, enc.tower ? dt.enc_g8r : dt.enc_g8,
                                                                     enc.ev);
  else
    launch_k(conv256_a_encode_kernel<128>, dim3(grid), dim3(kCTThreads), kCTEncSmem, s, w, um, items, tm, enc.tower ? dt.enc_m8r : dt.enc_m8,
                                                                      enc.ev);
  FPM_LAUNCH_CHECK();
}

// skip_a (inverse, 2^32-bit blocks): conv(Dd)^-1 over the digit already ran (decode_conv_a_kernel).
// q, Q: only rank q's column share (columns [q 2048/Q, (q+1) 2048/Q) of every row; the sharded
// conversion, lgD = 16, no fused encode).
void conv_cols_split(uint32_t* w, uint32_t* side, int lgD, bool inv, cudaStream_t s, const EncodeSink* enc = nullptr,
                     bool skip_a = false, int q = 0, int Q = 1) {
  if (Q > 1 && (lgD != 16 || enc)) throw Error(kInvalid, "conv_cols_split: column shares for 2^32-bit blocks only");
  if (lgD <= 1) return;
  if (lgD <= 8) {
    slab(w, lgD, 1, kTWords / 8, inv, s);
    return;
  }
  const int gd = lgD - 8;
  const uint64_t Dd = (uint64_t)1 << gd;
  const uint64_t unit = kTWords;  // words per row
  auto l1d = [&](bool fwd) {
    if (gd <= 4) {
      two_term_step(w, w, StepGeom{256 * unit, unit, 0, gd}, 1, side, !fwd, s, nullptr, q, Q);
      return;
    }
    const int k = gd / 2;
    const StepGeom outer{(256 * unit) << k, unit << k, 0, gd - k};
    const StepGeom inner{256 * unit, unit, (256 * unit) << k, k};
    if (fwd) {
      two_term_step(w, w, outer, 1, side, false, s, nullptr, q, Q);
      two_term_step(w, w, inner, (uint64_t)1 << (gd - k), side, false, s, nullptr, q, Q);
    } else {
      two_term_step(w, w, inner, (uint64_t)1 << (gd - k), side, true, s, nullptr, q, Q);
      two_term_step(w, w, outer, 1, side, true, s, nullptr, q, Q);
    }
  };
  auto over_digit = [&](bool iv) {  // conv(Dd) over rows 256 apart
    if (gd == 8) conv256_units(w, 256, 256, 256, iv, s, CarrySrc{}, q, Q);
    else slab(w, gd, 256, 256 * (kTWords / 8), iv, s);
  };
  if (!inv) {
    l1d(true);
    if (enc && gd == 8 && tma_units_enabled()) {  // conv over B, then conv over A fused with the encode
      conv256_units(w, Dd, 1, 1, false, s);
      conv256_a_encode(w, *enc, s);
      return;
    }
    over_digit(false);
    conv256_units(w, Dd, 1, 1, false, s, CarrySrc{}, q, Q);
  } else {
    // (conv over the digit and conv over the row within it commute: the digit one runs first so
    // that it can be fused with the decode)
    if (!skip_a) over_digit(true);
    conv256_units(w, Dd, 1, 1, true, s, CarrySrc{}, q, Q);
    l1d(false);
  }
}

// FPM_L1_PIPE: 0 = separate kernels (zeta -> 520 MiB skewed copy -> carry_rows / overflow); 1
// (default) = the pipelined pass for the forward zeta + carry/T_r and for the inverse zeta +
// overflow, T_r^-1 staying a separate conv_rows pass; 2 = T_r^-1 inside the pipelined pass too.
// Measured at 2^32 bits (two blocks per direction, bench stage times): forward 5.70 (0) / 5.68 ms
// (1), inverse 5.65 / 5.65 / 6.04 (2: conv^-1 at 3 CTAs/SM instead of 6).  The gain is memory: the
// skewed rows need a 32 MiB ring instead of a 520 MiB scratch array, and HBM traffic drops by the
// skewed copy's write + read (ncu: 2.0 -> 1.1 GB per forward block).
int l1_pipe_mode() {
  static const int m = [] {
    const char* e = std::getenv("FPM_L1_PIPE");
    return e ? std::atoi(e) : 1;
  }();
  return m;
}
// Skewed-row scratch words the L1_inner step needs for D rows: the pipelined pass keeps a ring of
// kPipeSlots chunks, the separate kernels a skewed copy of every row.
uint64_t l1_scratch_words(uint64_t D, bool inverse) {
  (void)inverse;  // both directions use the ring
  const bool ring = D >= 256 && l1_pipe_mode() >= 1;
  const uint64_t rows = ring ? std::min<uint64_t>(D, (uint64_t)kPipeSlots * 256) : D;
  return rows * kPipeP1;
}

// L1_inner (+ T_r) as one pipelined pass (l1_inner_rows_kernel) over the D = 256 nch rows of w:
// mode 0 forward zeta + carry/T_r; 1 inverse zeta + overflow; 2 inverse T_r^-1 + zeta + overflow.
void l1_inner_rows(const uint32_t* src, uint32_t* w, uint32_t* ring, uint64_t D, int mode, const uint32_t* top,
                   cudaStream_t s) {
  static PerDeviceOnce attr;
  constexpr size_t smem = 256 * kZP * sizeof(uint32_t);
  static_assert(smem >= kTileSmem, "the zeta tile is the larger shared-memory user");
  attr.run([] {
    FPM_CUDA(cudaFuncSetAttribute(l1_inner_rows_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FPM_CUDA(cudaFuncSetAttribute(l1_inner_rows_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FPM_CUDA(cudaFuncSetAttribute(l1_inner_rows_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  const int nch = (int)(D / 256);
  DevBuf cnt((3 * nch + 1) * sizeof(int), s);
  FPM_CUDA(cudaMemsetAsync(cnt.p, 0, (3 * nch + 1) * sizeof(int), s));
  const int items = nch * (kPipeZW + (mode == 1 ? 256 / kPipeORows : 256) + (mode == 2 ? 256 : 0));
  const int grid = grid_cap((uint64_t)items, pipe_ctas(mode != 0));
  if (mode == 2) launch_k(l1_inner_rows_kernel<true, true>, dim3(grid), dim3(256), smem, s, src, w, ring, nch, cnt.as<int>(), top);
  else if (mode == 1) launch_k(l1_inner_rows_kernel<true, false>, dim3(grid), dim3(256), smem, s, src, w, ring, nch, cnt.as<int>(), top);
  else launch_k(l1_inner_rows_kernel<false, false>, dim3(grid), dim3(256), smem, s, src, w, ring, nch, cnt.as<int>(), top);
  FPM_LAUNCH_CHECK();
}

void conv2d_split(uint32_t* w, int K, bool inv, uint32_t* scratch, uint32_t* side, cudaStream_t s,
                  const uint32_t* src = nullptr, const uint32_t* top = nullptr, const EncodeSink* enc = nullptr,
                  bool skip_a = false, cudaEvent_t top_ready = nullptr) {
  const int lgD = K - kTLog2;
  const uint64_t D = (uint64_t)1 << lgD;
  const int nb_in = std::min(lgD, 8), nb_out = lgD - nb_in;
  const uint64_t p1 = (kT + 32 * kZW) / 32;  // skewed row pitch of L1_inner (t + 1024 bits)
  Skew lo_skew;
  lo_skew.mask = 255;
  auto outer = [&](const uint32_t* from, const uint32_t* tp) {
    two_term_step(from, w, StepGeom{kChunkWords, 8, 0, nb_out}, 1, side, inv, s, tp);
  };
  if (!inv) {
    const uint32_t* in = src ? src : w;
    if (nb_out) {
      outer(in, nullptr);
      in = w;
    }
    if (nb_in == 8 && l1_pipe_mode() >= 1) {
      l1_inner_rows(in, w, scratch, D, 0, nullptr, s);
    } else {
      zeta(in, kTWords, scratch, p1, D, 0, nb_in, lo_skew, p1 / kZW, s, kTWords);
      launch_k(carry_rows_kernel, dim3(grid_cap(D, 7)), dim3(256), kTileSmem, s, scratch, p1, w, D, 255);
      FPM_LAUNCH_CHECK();
    }
    conv_cols_split(w, side, lgD, false, s, enc);
  } else {
    conv_cols_split(w, side, lgD, true, s, nullptr, skip_a);
    if (nb_in == 8 && l1_pipe_mode() == 2) {
      l1_inner_rows(w, w, scratch, D, 2, nb_out ? nullptr : top, s);
    } else if (nb_in == 8 && l1_pipe_mode() == 1) {
      conv_rows(w, D * kTWords, kTLog2, true, s);
      l1_inner_rows(w, w, scratch, D, 1, nb_out ? nullptr : top, s);
    } else {
      conv_rows(w, D * kTWords, kTLog2, true, s);
      zeta(w, kTWords, scratch, p1, D, 0, nb_in, lo_skew, p1 / kZW, s, kTWords);
      launch_k(overflow_kernel, dim3(grid_cap(D, 8)), dim3(256), 0, s, scratch, p1, w, D, nb_out ? nullptr : top, 255);
      FPM_LAUNCH_CHECK();
    }
    if (top_ready) FPM_CUDA(cudaStreamWaitEvent(s, top_ready, 0));  // (the top pass reads the final upper block)
    if (nb_out) outer(w, top);
  }
}

bool split_l1_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FPM_BASIS");
    return !(e && std::string(e) == "single");
  }();
  return on;
}

void run_big_pass(uint32_t* w, uint64_t nwords, Pass p, bool inverse, uint64_t live_bits, cudaStream_t s) {
  const uint64_t S = p.span, D = p.shift;
  const uint64_t nspans = (nwords * 32) / S;
  const uint64_t regions[2][2] = {{S / 2 - D, S / 2}, {S / 2, S - D}};
  for (int ph = 0; ph < 2; ++ph) {
    const uint64_t rlo = regions[ph][0], rhi = regions[ph][1];
    if (rhi <= rlo) continue;
    const uint64_t w_first = rlo / 32, w_last = (rhi + 31) / 32;
    const uint64_t nw_span = w_last - w_first;
    const uint64_t total = nw_span * nspans;
    launch_k(bc_pass_kernel, dim3(grid_cap((total + 255) / 256, 32)), dim3(256), 0, s, w, nwords, S, D, inverse ? 1 : 0, w_first,
                                                                     nw_span, nspans, rlo, rhi, live_bits);
    FPM_LAUNCH_CHECK();
  }
}

using Scratch = DevBuf;

}  // namespace

// One 2^32-bit block of a 2^33-bit array's inverse conversion, on its own: conv(2^32)^-1 of w, then
// (top != null: the lower block) the array's single top pass x[q] ^= top[q - 1] fused in -- top is the
// final upper block, possibly in a peer GPU's memory.  The upper block's own bit 0 fix-up is
// top_bit_fix_device, to be ordered after the lower block's conversion (it reads the pre-fix bit).
void basis_cvt_block32_inverse(uint32_t* w, const uint32_t* top, cudaStream_t s) {
  set_smem_attr();
  const uint64_t D = (uint64_t)1 << 16;
  const bool split = split_l1_enabled();
  const size_t scr_bytes = split ? l1_scratch_words(D, true) * sizeof(uint32_t)
                                 : D * (kT + std::max<uint64_t>(D, 32 * kZW)) / 8 + D * (kT + 32 * kZW) / 8;
  Scratch scr(scr_bytes, s), side_buf(split ? split_side_words(16) * sizeof(uint32_t) : 0, s);

  if (split) conv2d_split(w, 32, true, static_cast<uint32_t*>(scr.p), static_cast<uint32_t*>(side_buf.p), s, nullptr, top);
  else conv2d(w, 32, true, static_cast<uint32_t*>(scr.p), s, nullptr, top);
}

void top_bit_fix_device(uint32_t* hi_block, cudaStream_t s) {
  launch_k(top_bit_fix_kernel, dim3(1), dim3(32), 0, s, hi_block, ((uint64_t)1 << 32) / 32);
  FPM_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ the sharded 2^32-bit conversion
// fpm_polymul_multi at P >= 4 converts each 2^32-bit block (an operand, or a block of the 2^33-bit
// product) on Q = P/2 ranks holding full-size replicas, one phase of build_schedule's recursion at a
// time, each phase split the way its data dependencies allow (
// proj/src/basis_convert.cpp:60-67 the phases, :278-327 the tiling):
//   L1_outer   (z over the 256 chunks)      by L1_outer window: rank q the windows [q wpr, (q+1) wpr)
//   L1_inner + T_r (chunk-local)             by chunk: rank q the chunks [q 256/Q, (q+1) 256/Q)
//   T_d        (conv over the row index)     by column: rank q the words [q 2048/Q, ...) of every row
// Between two phases every rank pulls the 16-byte groups it owns next from their previous owners'
// replicas (regather_kernel, peer loads over NVLink); all replicas use the same word offsets.
namespace {

constexpr uint64_t kB32Words = (uint64_t)1 << 27;                          // 32-bit words per block
constexpr uint64_t kB32Windows = (kChunkWords + 8 * 255 + kZW - 1) / kZW;  // L1_outer windows (16448)

__device__ __forceinline__ int dist_owner(int dist, uint64_t wi, int lgq, uint64_t wpr) {
  if (dist == kDistChunk) return (int)((wi >> 19) >> (8 - lgq));
  if (dist == kDistColumn) return (int)((wi & (kTWords - 1)) >> (11 - lgq));
  const uint64_t c = wi >> 19, o = wi & (kChunkWords - 1);
  return (int)(((o + 8 * c) >> 5) / wpr);
}

// The k-th 16-byte group rank q owns under distribution `dist` (n_owned(dist) of them), or ~0 for a
// padding index (window ranges are clipped per chunk).
__device__ __forceinline__ uint64_t dist_group(int dist, uint64_t k, int q, int lgq, uint64_t wpr) {
  const int Q = 1 << lgq;
  if (dist == kDistChunk) return ((uint64_t)q << (25 - lgq)) + k;
  if (dist == kDistColumn) {
    const uint64_t per = 512 >> lgq;  // of a row's 512 groups
    return (k / per) * 512 + (uint64_t)q * per + k % per;
  }
  const uint64_t span = 8 * wpr, c = k / span, u = k % span;
  const int64_t lo = (int64_t)(8 * (uint64_t)q * wpr) - 2 * (int64_t)c;
  const uint64_t whi = q + 1 == Q ? kB32Windows : (uint64_t)(q + 1) * wpr;
  const int64_t hi = std::min<int64_t>((int64_t)1 << 17, (int64_t)(8 * whi) - 2 * (int64_t)c);
  const int64_t v = std::max<int64_t>(lo, 0) + (int64_t)u;
  return v < hi ? (c << 17) + (uint64_t)v : ~(uint64_t)0;
}
__host__ __device__ __forceinline__ uint64_t dist_count(int dist, int lgq, uint64_t wpr) {
  return dist == kDistWindow ? 256 * 8 * wpr : (uint64_t)1 << (25 - lgq);
}

__global__ void regather_kernel(uint32_t* __restrict__ dst, const RankPtrs src, int from, int to, int q, int lgq,
                                uint64_t wpr) {
  pdl_wait();
  const uint64_t n = dist_count(to, lgq, wpr);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = dist_group(to, k, q, lgq, wpr);
    if (v == ~(uint64_t)0) continue;
    const int o = dist_owner(from, 4 * v, lgq, wpr);
    if (o != q) d4[v] = __ldcg(reinterpret_cast<const uint4*>(src.p[o]) + v);
  }
  pdl_trigger();
}

// The 2^33-bit array's single top pass on rank q's window groups of the lower block: bit b ^= bit
// b - 1 of the upper block (read from its window owners).
__global__ void top_pass_windows_kernel(uint32_t* __restrict__ lo, const RankPtrs hi, int q, int lgq, uint64_t wpr) {
  pdl_wait();
  const uint64_t n = dist_count(kDistWindow, lgq, wpr);
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = dist_group(kDistWindow, k, q, lgq, wpr);
    if (v == ~(uint64_t)0) continue;
    const uint64_t G = 4 * v;
    const uint4 t4 = __ldcg(reinterpret_cast<const uint4*>(hi.p[dist_owner(kDistWindow, G, lgq, wpr)]) + v);
    const uint32_t tp = G ? __ldcg(hi.p[dist_owner(kDistWindow, G - 1, lgq, wpr)] + G - 1) : 0u;
    uint4 x = reinterpret_cast<uint4*>(lo)[v];
    x.x ^= (t4.x << 1) | (tp >> 31);
    x.y ^= (t4.y << 1) | (t4.x >> 31);
    x.z ^= (t4.z << 1) | (t4.y >> 31);
    x.w ^= (t4.w << 1) | (t4.z >> 31);
    reinterpret_cast<uint4*>(lo)[v] = x;
  }
  pdl_trigger();
}

__global__ void top_bit_fix_peer_kernel(uint32_t* __restrict__ hi0, const uint32_t* __restrict__ hi_last) {
  pdl_wait();
  if (threadIdx.x == 0) hi0[0] ^= __ldcg(hi_last + kB32Words - 1) >> 31;
  pdl_trigger();
}

uint64_t b32_wpr(int Q) { return (kB32Windows + Q - 1) / Q; }

}  // namespace

void b32_regather(uint32_t* dst, const RankPtrs& src, int from, int to, int q, int Q, cudaStream_t s) {
  const int lgq = __builtin_ctz((unsigned)Q);
  if (Q < 2 || Q > 4 || (Q & (Q - 1))) throw Error(kInvalid, "regather: 2 or 4 ranks per block");
  const uint64_t n = dist_count(to, lgq, b32_wpr(Q));
  launch_k(regather_kernel, dim3(grid_cap((n + 255) / 256, 8)), dim3(256), 0, s, dst, src, from, to, q, lgq, b32_wpr(Q));
  FPM_LAUNCH_CHECK();
}

void b32_l1_outer(const uint32_t* src, uint32_t* w, uint32_t* side, bool inv, int q, int Q, cudaStream_t s) {
  const StepGeom gm{kChunkWords, 8, 0, 8};
  WinSel sel;
  const uint64_t wpr = b32_wpr(Q);
  sel.lo = (uint64_t)q * wpr;
  sel.hi = std::min<uint64_t>(kB32Windows, sel.lo + wpr);
  sel.count = sel.hi - sel.lo;
  (void)inv;  // the zeta half is the same superset zeta in both directions
  outer_zeta(src, w, gm, 1, side, s, nullptr, sel);
}

void b32_l1_outer_fix(uint32_t* w, const uint32_t* side, bool inv, uint32_t e_lo, uint32_t e_hi, cudaStream_t s) {
  FixSel fs;
  fs.e_lo = e_lo;
  fs.e_hi = e_hi;
  outer_fix(w, side, StepGeom{kChunkWords, 8, 0, 8}, 1, inv, s, fs);
}

void b32_rows(uint32_t* w_rows, uint64_t rows, bool inv, cudaStream_t s) {
  if (rows % 256) throw Error(kInvalid, "b32_rows: whole chunks");
  set_smem_attr();
  const uint64_t ring_rows = std::min<uint64_t>(rows, (uint64_t)kPipeSlots * 256);
  DevBuf ring(ring_rows * kPipeP1 * sizeof(uint32_t), s);
  if (inv) conv_rows(w_rows, rows * kTWords, kTLog2, true, s);
  l1_inner_rows(w_rows, w_rows, ring.as<uint32_t>(), rows, inv ? 1 : 0, nullptr, s);
}

void b32_cols(uint32_t* w, bool inv, int q, int Q, cudaStream_t s) {
  DevBuf side(split_side_words(16) * sizeof(uint32_t), s);
  conv_cols_split(w, side.as<uint32_t>(), 16, inv, s, nullptr, false, q, Q);
}

void b32_top_pass(uint32_t* lo, const RankPtrs& hi, int q, int Q, cudaStream_t s) {
  const int lgq = __builtin_ctz((unsigned)Q);
  const uint64_t n = dist_count(kDistWindow, lgq, b32_wpr(Q));
  launch_k(top_pass_windows_kernel, dim3(grid_cap((n + 255) / 256, 8)), dim3(256), 0, s, lo, hi, q, lgq, b32_wpr(Q));
  FPM_LAUNCH_CHECK();
}

void b32_top_bit_fix(uint32_t* hi0, const uint32_t* hi_last_owner, cudaStream_t s) {
  launch_k(top_bit_fix_peer_kernel, dim3(1), dim3(32), 0, s, hi0, hi_last_owner);
  FPM_LAUNCH_CHECK();
}

// Rank q's 32-bit word ranges of a block under the window distribution (for the copy to the host).
std::vector<std::pair<uint64_t, uint64_t>> b32_window_ranges(int q, int Q) {
  std::vector<std::pair<uint64_t, uint64_t>> r;
  const uint64_t wpr = b32_wpr(Q), wlo = (uint64_t)q * wpr, whi = std::min<uint64_t>(kB32Windows, wlo + wpr);
  for (uint64_t c = 0; c < 256; ++c) {
    const int64_t lo = std::max<int64_t>(0, (int64_t)(32 * wlo) - (int64_t)(8 * c));
    const int64_t hi = std::min<int64_t>((int64_t)kChunkWords, (int64_t)(32 * whi) - (int64_t)(8 * c));
    if (lo < hi) r.emplace_back(c * kChunkWords + (uint64_t)lo, c * kChunkWords + (uint64_t)hi);
  }
  return r;
}

// conv(2^16) (inverse: conv(2^16)^-1) of every 2048-word row of data (a batch of 2^16-bit arrays).
void conv_rows_batch16(uint32_t* data, uint64_t nwords, bool inv, cudaStream_t s) {
  set_smem_attr();
  conv_rows(data, nwords, kTLog2, inv, s);
}

bool basis_cvt_can_decode(size_t n_bits) {
  return n_bits == ((size_t)1 << 33) && split_l1_enabled();
}

void decode_conv_a(const DecodeSource& dec, uint32_t* w_lo, uint32_t* w_hi, cudaStream_t s) {
  static PerDeviceOnce attr;
  attr.run([] {
    FPM_CUDA(cudaFuncSetAttribute(decode_conv_a_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDecSmem));
    FPM_CUDA(cudaFuncSetAttribute(decode_conv_a_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDecSmem));
  });
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const DeviceTables& dt = device_tables(dev);
  const uint64_t items = 256 * (kTWords / kCT);
  const int grid = grid_cap(items, 1);
  if (dec.m == 64)
    launch_k(decode_conv_a_kernel<64>, dim3(grid), dim3(kCTThreads), kDecSmem, s, dec.ev, dec.tower ? dt.dec_g8r : dt.dec_g8, w_lo, w_hi,
                                                                items);
  else
    launch_k(decode_conv_a_kernel<128>, dim3(grid), dim3(kCTThreads), kDecSmem, s, dec.ev, dec.tower ? dt.dec_m8r : dt.dec_m8, w_lo, w_hi,
                                                                 items);
  FPM_LAUNCH_CHECK();
}

// One 2^32-bit block of the fused 2^33-bit decode (GF(2^128) in the tower representation): half = 0
// the lower block (product rows 0..63), 1 the upper (rows 64..127).
bool decode_halves_ok(const DecodeSource& dec) { return dec.m == 128 && dec.tower; }
void decode_half_conv_a(const DecodeSource& dec, int half, uint32_t* w_block, cudaStream_t s) {
  static PerDeviceOnce attr;
  attr.run([] {
    FPM_CUDA(cudaFuncSetAttribute(decode_half_conv_a_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDecHalfSmem));
    FPM_CUDA(cudaFuncSetAttribute(decode_half_conv_a_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDecHalfSmem));
  });
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const DeviceTables& dt = device_tables(dev);
  const uint64_t items = 256 * (kTWords / kCT);
  const int grid = grid_cap(items, 1);
  const uint4* ev = static_cast<const uint4*>(dec.ev);
  if (half) launch_k(decode_half_conv_a_kernel<1>, dim3(grid), dim3(kCTThreads), kDecHalfSmem, s, ev, dt.dec_half_r[1], w_block, items);
  else launch_k(decode_half_conv_a_kernel<0>, dim3(grid), dim3(kCTThreads), kDecHalfSmem, s, ev, dt.dec_half_r[0], w_block, items);
  FPM_LAUNCH_CHECK();
}

bool basis_cvt_can_encode(size_t n_bits, bool tower) {
  (void)tower;
  return n_bits == ((size_t)1 << 32) && split_l1_enabled() && tma_units_enabled();
}

// A second stream per device for the concurrent conversions (operand b beside operand a, the lower
// inverse block beside the upper one); forked from and joined to the caller's stream with events.
cudaStream_t side_stream(int dev) {
  static cudaStream_t ss[64] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (!ss[dev & 63]) FPM_CUDA(cudaStreamCreateWithFlags(&ss[dev & 63], cudaStreamNonBlocking));
  return ss[dev & 63];
}

bool concurrent_blocks_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FPM_CONCURRENT_BLOCKS");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

void basis_cvt_device(uint32_t* w, size_t n_bits, size_t live_bits, bool inverse, cudaStream_t s,
                      const FinalFn* on_final, const uint32_t* src, const EncodeSink* enc, const DecodeSource* dec,
                      bool concurrent) {
  if (enc && (inverse || !basis_cvt_can_encode(n_bits, enc->tower)))
    throw Error(kInvalid, "basis_cvt: the fused encode needs a forward 2^32-bit conversion");
  if (dec && (!inverse || !basis_cvt_can_decode(n_bits)))
    throw Error(kInvalid, "basis_cvt: the fused decode needs an inverse 2^33-bit conversion");
  if (n_bits < 4 || (n_bits & (n_bits - 1))) throw Error(kInvalid, "basis_cvt: length must be a power of two >= 4");
  set_smem_attr();
  int K = 0;
  while (((size_t)1 << K) < n_bits) ++K;
  const uint64_t nwords = n_bits < 32 ? 1 : n_bits / 32;
  if (K < 8) {  // < 256 bits: the pass list directly, in shared memory
    Pass sched[64];
    size_t np = 0;
    build_schedule(sched, &np, n_bits, 1);
    std::vector<Pass> v(sched, sched + np);
    if (inverse) v = std::vector<Pass>(sched, sched + np), v = std::vector<Pass>(v.rbegin(), v.rend());
    const PassList pl = make_passlist(v, inverse);
    launch_k(bc_small_kernel, dim3(1), dim3(32), 2 * nwords * sizeof(uint32_t), s, w, (int)nwords, pl, inverse ? 1 : 0);
    FPM_LAUNCH_CHECK();
    if (inverse && on_final) (*on_final)(0, nwords);
    return;
  }
  if (src && (inverse || K <= kTLog2 || K > 32))
    throw Error(kInvalid, "basis_cvt: a separate source is supported for forward 2^17..2^32-bit arrays");
  if (K <= kTLog2) {
    conv_rows(w, nwords, K, inverse, s);
    if (inverse && on_final) (*on_final)(0, nwords);
    return;
  }
  const int Kb = std::min(K, 32);
  const uint64_t lgD = Kb - kTLog2, D = (uint64_t)1 << lgD;
  // skewed rows (t + max(D, 1024) bits) + the first zeta's rows (t + 1024 bits) when D > 256; the
  // split L1 needs the C_cols scratch (2 Dd x (256 + Dd) rows) and the outer step's side rows
  const bool split = split_l1_enabled();

  const size_t scr_bytes = split ? l1_scratch_words(D, inverse) * sizeof(uint32_t)
                                 : D * (kT + std::max<uint64_t>(D, 32 * kZW)) / 8 + (D > 256 ? D * (kT + 32 * kZW) / 8 : 0);
  Scratch scr(scr_bytes, s), side_buf(split ? split_side_words((int)lgD) * sizeof(uint32_t) : 0, s);
  uint32_t* scratch = static_cast<uint32_t*>(scr.p);
  uint32_t* side = static_cast<uint32_t*>(side_buf.p);
  auto conv_block = [&](uint32_t* blk, const uint32_t* from, const uint32_t* tp) {
    if (split) conv2d_split(blk, Kb, inverse, scratch, side, s, from, tp, enc, dec != nullptr);
    else conv2d(blk, Kb, inverse, scratch, s, from, tp);
  };
  const uint64_t block_words = ((uint64_t)1 << Kb) / 32;
  // fused decode (2^33-bit inverse): decode + conv^-1 over the digit of both blocks in one pass; each
  // block's conversion then skips that step
  static const bool halves_on = [] {
    const char* e = std::getenv("FPM_DECODE_HALVES");
    return !(e && std::string(e) == "0");
  }();
  // (the split decode serves the host-buffer path: the upper block's copy-out starts after half the
  // decode; device-resident products decode both blocks at once -- 5.55 vs 5.99 ms of inverse
  // conversion with the halves on two streams, while e2e gains 74.69 -> 74.35 ms)
  const bool halves = dec && halves_on && !concurrent && decode_halves_ok(*dec);
  if (dec && !halves) decode_conv_a(*dec, w, w + block_words, s);
  // Arrays above 2^32 bits: their passes with S > 2^32 come first (forward) / last (inverse);
  // what remains is conv(2^32) of every 2^32-bit block (build_schedule's per-digit recursion).
  std::vector<Pass> top;
  if (K > 32) {
    static thread_local Pass sched[512];
    size_t np = 0;
    build_schedule(sched, &np, n_bits, 1);
    for (size_t k = 0; k < np; ++k)
      if (sched[k].span > ((size_t)1 << 32)) top.push_back(sched[k]);
  }
  const uint64_t nblocks = nwords / block_words;
  if (!inverse) {
    for (const Pass& p : top) run_big_pass(w, nwords, p, false, live_bits, s);
    for (uint64_t b = 0; b < nblocks; ++b) {
      if (b * block_words * 32 >= live_bits) continue;  // all-zero block stays zero
      conv_block(w + b * block_words, src ? src + b * block_words : nullptr, nullptr);
    }
    return;
  }
  // Inverse: per-block conversions, then the top passes.  With a single top pass (2^33 bits: S =
  // 2^33, D = 2^32 - 1) the pass rewrites bits [S/2 - D, S - D) = [1, 2^32 + 1) only, so the upper
  // block is final, but for its first word, once its own conversion is done: convert it first.
  uint64_t early_from = nwords;  // words >= early_from are final after their block's conversion
  if (top.size() == 1 && nblocks == 2) {
    const uint64_t hi_bit = top[0].span - top[0].shift;  // exclusive end of the rewritten bits
    early_from = (hi_bit + 31) / 32;
  }
  // 2^33 bits: that single pass is fused into the lower block's overflow kernel (bits [1, 2^32)),
  // and its last target bit 2^32 (= upper bit 0 ^= bit 2^33 - 1) is one word fixed afterwards.
  const bool fuse_top = top.size() == 1 && nblocks == 2 && top[0].shift == block_words * 32 - 1;
  if (concurrent && fuse_top && split && concurrent_blocks_enabled()) {
    // the lower block on a second stream (own scratch) beside the upper block on s; its last step
    // (L1_outer^-1 with the fused top pass) waits for the final upper block
    int dev;
    FPM_CUDA(cudaGetDevice(&dev));
    const cudaStream_t t = side_stream(dev);
    Ev fork, hi_done, lo_done;
    FPM_CUDA(cudaEventRecord(fork.e, s));
    FPM_CUDA(cudaStreamWaitEvent(t, fork.e, 0));
    {
      Scratch scr2(scr_bytes, t), side2(split_side_words((int)lgD) * sizeof(uint32_t), t);
      if (halves) {
        decode_half_conv_a(*dec, 1, w + block_words, s);
        decode_half_conv_a(*dec, 0, w, t);
      }
      conv2d_split(w + block_words, Kb, true, scratch, side, s, nullptr, nullptr, nullptr, dec != nullptr);
      FPM_CUDA(cudaEventRecord(hi_done.e, s));
      conv2d_split(w, Kb, true, static_cast<uint32_t*>(scr2.p), static_cast<uint32_t*>(side2.p), t, nullptr,
                   w + block_words, nullptr, dec != nullptr, hi_done.e);
    }  // (scratch of t freed in t's order)
    FPM_CUDA(cudaEventRecord(lo_done.e, t));
    FPM_CUDA(cudaStreamWaitEvent(s, lo_done.e, 0));
    for (uint64_t b = nblocks; b-- > 0;) {  // (as the sequential loop below)
      const uint64_t w0 = std::max(b * block_words, early_from), w1 = (b + 1) * block_words;
      if (on_final && w0 < w1) (*on_final)(w0, w1);
    }
    launch_k(top_bit_fix_kernel, dim3(1), dim3(32), 0, s, w + block_words, block_words);
    FPM_LAUNCH_CHECK();
    if (on_final) (*on_final)(0, std::min<uint64_t>(early_from, nwords));
    return;
  }
  for (uint64_t b = nblocks; b-- > 0;) {
    if (halves) decode_half_conv_a(*dec, (int)b, w + b * block_words, s);  // (upper block first)
    conv_block(w + b * block_words, nullptr, fuse_top && b == 0 ? w + block_words : nullptr);
    const uint64_t w0 = std::max(b * block_words, early_from), w1 = (b + 1) * block_words;
    if (on_final && w0 < w1) (*on_final)(w0, w1);
  }
  if (fuse_top) {
    launch_k(top_bit_fix_kernel, dim3(1), dim3(32), 0, s, w + block_words, block_words);
    FPM_LAUNCH_CHECK();
  } else {
    for (size_t k = top.size(); k-- > 0;) run_big_pass(w, nwords, top[k], true, n_bits, s);
  }
  if (on_final) (*on_final)(0, std::min<uint64_t>(early_from, nwords));
}

}  // namespace fpm
