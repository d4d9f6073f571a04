// k_codec.cu -- Frobenius-partition encode / decode on sm_100a (north-star subsystems 1 and 5).
//
// Reference: proj/src/encode.cpp.  Element i of the EvalVec is f_i = x_i * E where bit j of x_i is
// coefficient a_{j*n_p+i} (gather_columns :108-129, encode :165-193); decode is y_i = f_i * E^{-1}
// scattered back to a_{j*n_p+i} (:195-220).
//
// Layout insight: row j of the polynomial (n_p consecutive bits) already holds bit j of every
// element, so 32 consecutive elements are one 32-bit word per row.  A CTA stages a 1024-element
// slab (32 words x 64|128 rows, coalesced 128 B row segments) in padded shared memory, each warp
// turns 32x32 bit blocks into per-lane column words with a 5-step __shfl_xor_sync transpose, and
// the matrix product x*E runs as byte-chunk lookups in a lane-rotated, bank-conflict-free shared
// table (gf128.cuh M8 layout; GF(2^64): gf64.cuh G8 layout).  Decode runs the same steps in reverse.
#include <cuda_runtime.h>

#include <mutex>

#include "fpm_internal.h"
#include "gf128.cuh"
#include "gf64.cuh"
#include "warp_bits.cuh"

namespace fpm {
namespace {

constexpr int kSlabWords = 32;                 // words per row per CTA slab -> 1024 elements
constexpr int kPad = kSlabWords + 1;

// polys: the operand, or (sharded conversion) the replicas of the 2^(11 - lgq)-word column owners:
// a 32-word slab's column (word index mod 2048) selects polys.p[column >> (11 - lgq)].
template <int ROWS>  // 64: rows >= 64 are known zero (pipeline); 128: general encode
// slab_stride: words between consecutive slabs' first rows (kSlabWords: one polynomial's columns;
// a batch of independent polynomials of 32-word rows: the polynomials' stride).
__global__ void __launch_bounds__(256) encode_kernel(const RankPtrs polys, int lgq, uint64_t row_words,
                                                     uint64_t col0_words, uint64_t nslabs,
                                                     const uint4* __restrict__ tab_g, uint4* __restrict__ ev,
                                                     uint64_t slab_stride) {
  pdl_wait();
  extern __shared__ uint4 smem4[];
  // rotated 8-bit table of x*E (gf128.cuh m8 layout): chunks 0..7 (ROWS = 64) or all 16
  constexpr int kTab = ROWS == 64 ? kM8Uint4 / 2 : kM8Uint4;
  uint4* tab = smem4;
  uint32_t* slab = reinterpret_cast<uint32_t*>(smem4 + kTab);  // ROWS x kPad
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kTab; i += blockDim.x) tab[i] = tab_g[i];
  const int q8 = lane & 7;
  const Transpose32 tr(lane);
  // Each thread's share of the next slab is loaded into registers while the current one is
  // transformed (software pipelining across slabs).
  constexpr int kPer = ROWS * kSlabWords / 256;
  uint32_t nx[kPer];
  auto fetch = [&](uint64_t sl) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = tid + 256 * j, r = i / kSlabWords, c = i % kSlabWords;
      const uint64_t wc = col0_words + sl * slab_stride;
      const uint32_t* poly = polys.p[lgq ? (int)((wc & 2047) >> (11 - lgq)) : 0];
      nx[j] = sl < nslabs ? __ldg(poly + (uint64_t)r * row_words + wc + c) : 0u;
    }
  };
  fetch(blockIdx.x);
  for (uint64_t sl = blockIdx.x; sl < nslabs; sl += gridDim.x) {
    const uint64_t w0 = sl * kSlabWords;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = tid + 256 * j, r = i / kSlabWords, c = i % kSlabWords;
      slab[r * kPad + c] = nx[j];
    }
    __syncthreads();
    fetch(sl + gridDim.x);
#pragma unroll 1
    for (int k = 0; k < kSlabWords / 8; ++k) {
      const int col = warp * (kSlabWords / 8) + k;
      uint32_t xw[4];
#pragma unroll
      for (int q = 0; q < ROWS / 32; ++q) xw[q] = tr(slab[(q * 32 + lane) * kPad + col]);
      uint4 f;
      if (ROWS == 64) {  // 8 byte chunks, lane-rotated order: conflict-free LDS.128
        uint4 acc0 = make_uint4(0, 0, 0, 0), acc1 = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int kk = 0; kk < 8; kk += 2) {
          const int c0 = (kk + q8) & 7, c1 = (kk + 1 + q8) & 7;
          const uint32_t b0 = __byte_perm(c0 < 4 ? xw[0] : xw[1], 0, 0x4440u | (uint32_t)(c0 & 3));
          const uint32_t b1 = __byte_perm(c1 < 4 ? xw[0] : xw[1], 0, 0x4440u | (uint32_t)(c1 & 3));
          acc0 = x4(acc0, tab[b0 * 8 + c0]);
          acc1 = x4(acc1, tab[b1 * 8 + c1]);
        }
        f = x4(acc0, acc1);
      } else {
        f = m8_mul(tab, make_uint4(xw[0], xw[1], xw[ROWS / 32 > 2 ? 2 : 0], xw[ROWS / 32 > 3 ? 3 : 0]), q8);
      }
      ev[(w0 + col) * 32 + lane] = f;
    }
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// Rows 0..63 go to poly (pitch row_words), rows 64..127 to poly_hi (same pitch); column word offset
// of slab sl: col0w + sl * kSlabWords.  Sharded conversion (lgq > 0): the slab's column (word index
// mod 2048) selects the owner replica polys.p / polys_hi.p[column >> (11 - lgq)].
__global__ void __launch_bounds__(256) decode_kernel(const uint4* __restrict__ ev, uint64_t nslabs,
                                                     uint64_t row_words,
                                                     const uint4* __restrict__ tab_g, const RankPtrs polys,
                                                     const RankPtrs polys_hi, int lgq, uint64_t col0w,
                                                     uint64_t slab_stride) {
  pdl_wait();
  extern __shared__ uint4 smem4[];
  uint4* tab = smem4;  // rotated 8-bit table of x*E^-1 (gf128.cuh m8 layout)
  uint32_t* slab = reinterpret_cast<uint32_t*>(smem4 + kM8Uint4);  // 128 x kPad
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kM8Uint4; i += blockDim.x) tab[i] = tab_g[i];
  const int q8 = lane & 7;
  const Transpose32 tr(lane);
  __syncthreads();
  // The warp's four elements of the next slab are loaded while this slab is transformed and
  // stored (software pipelining across slabs).
  constexpr int kCols = kSlabWords / 8;
  uint4 nx[kCols];
  auto fetch = [&](uint64_t sl) {
#pragma unroll
    for (int k = 0; k < kCols; ++k)
      nx[k] = sl < nslabs ? __ldg(ev + (sl * kSlabWords + warp * kCols + k) * 32 + lane) : make_uint4(0, 0, 0, 0);
  };
  fetch(blockIdx.x);
  for (uint64_t sl = blockIdx.x; sl < nslabs; sl += gridDim.x) {
    uint4 cur[kCols];
#pragma unroll
    for (int k = 0; k < kCols; ++k) cur[k] = nx[k];
    fetch(sl + gridDim.x);
#pragma unroll
    for (int k = 0; k < kCols; ++k) {
      const int col = warp * kCols + k;
      const uint4 y = m8_mul(tab, cur[k], q8);
      slab[(0 * 32 + lane) * kPad + col] = tr(y.x);
      slab[(1 * 32 + lane) * kPad + col] = tr(y.y);
      slab[(2 * 32 + lane) * kPad + col] = tr(y.z);
      slab[(3 * 32 + lane) * kPad + col] = tr(y.w);
    }
    __syncthreads();
    const uint64_t wc = col0w + sl * slab_stride;
    const int own = lgq ? (int)((wc & 2047) >> (11 - lgq)) : 0;
    uint32_t* const poly = polys.p[own];
    uint32_t* const poly_hi = polys_hi.p[own];
    for (int i = tid; i < 128 * kSlabWords; i += blockDim.x) {
      const int r = i / kSlabWords, c = i % kSlabWords;
      uint32_t* base = r < 64 ? poly + (uint64_t)r * row_words : poly_hi + (uint64_t)(r - 64) * row_words;
      base[wc + c] = slab[r * kPad + c];
    }
    __syncthreads();
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// Tiny shapes (n_p < 1024): one thread per element, direct row products (encode.cpp:172-181).
__global__ void encode_small_kernel(const uint32_t* __restrict__ poly, uint64_t n_p, const uint4* __restrict__ rows,
                                    uint4* __restrict__ ev) {
  pdl_wait();
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_p) return;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int j = 0; j < 128; ++j) {
    const uint64_t k = (uint64_t)j * n_p + i;
    if ((poly[k >> 5] >> (k & 31)) & 1u) acc = x4(acc, rows[j]);
  }
  ev[i] = acc;
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

__global__ void decode_small_kernel(const uint4* __restrict__ ev, uint64_t n_p, const uint4* __restrict__ inv_rows,
                                    uint32_t* __restrict__ poly) {
  pdl_wait();
  // one thread per output word of the 128*n_p-bit polynomial
  const uint64_t wi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nwords = (128 * n_p + 31) / 32;
  if (wi >= nwords) return;
  uint32_t out = 0;
  for (int b = 0; b < 32; ++b) {
    const uint64_t k = wi * 32 + b;
    if (k >= 128 * n_p) break;
    const uint64_t j = k / n_p, i = k % n_p;
    // bit j of y_i = parity(<f_i, column j of E^{-1}>) = XOR over bits t of f_i of inv_rows[t] bit j
    const uint4 f = ev[i];
    const uint32_t fw[4] = {f.x, f.y, f.z, f.w};
    uint32_t acc = 0;
    for (int t = 0; t < 128; ++t)
      if ((fw[t >> 5] >> (t & 31)) & 1u) {
        const uint4 r = inv_rows[t];
        const uint32_t rw[4] = {r.x, r.y, r.z, r.w};
        acc ^= (rw[j >> 5] >> (j & 31)) & 1u;
      }
    out |= acc << b;
  }
  poly[wi] = out;
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ GF(2^64) (m = 64)
// Element i of EvalVec<gf64> is x_i * E with x_i = (a_{j*n_p+i})_{j<64} (encode.cpp:165-193 at
// m = 64).  Same slab scheme as above: ROWS (32: pipeline operands, rows >= 32 zero; 64: general)
// rows x 1024 elements, warp transposes, then x*E by 4 or 8 G8 lookups (gf64.cuh layout).
template <int ROWS>
__global__ void __launch_bounds__(256) encode64_kernel(const uint32_t* __restrict__ poly, uint64_t row_words,
                                                       uint64_t nslabs, const uint2* __restrict__ tab_g,
                                                       uint2* __restrict__ ev) {
  pdl_wait();
  extern __shared__ uint2 smem2[];
  uint2* tab = smem2;                                               // kG8Uint2
  uint32_t* slab = reinterpret_cast<uint32_t*>(smem2 + kG8Uint2);  // ROWS x kPad
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kG8Uint2; i += blockDim.x) tab[i] = tab_g[i];
  const Transpose32 tr(lane);
  const int q = lane & 7, h8 = lane & 8;
  constexpr int kPer = ROWS * kSlabWords / 256;  // next-slab register prefetch, as encode_kernel
  uint32_t nx[kPer];
  auto fetch = [&](uint64_t sl) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = tid + 256 * j, r = i / kSlabWords, c = i % kSlabWords;
      nx[j] = sl < nslabs ? __ldg(poly + (uint64_t)r * row_words + sl * kSlabWords + c) : 0u;
    }
  };
  fetch(blockIdx.x);
  for (uint64_t sl = blockIdx.x; sl < nslabs; sl += gridDim.x) {
    const uint64_t w0 = sl * kSlabWords;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = tid + 256 * j, r = i / kSlabWords, c = i % kSlabWords;
      slab[r * kPad + c] = nx[j];
    }
    __syncthreads();
    fetch(sl + gridDim.x);
#pragma unroll 1
    for (int k = 0; k < kSlabWords / 8; ++k) {
      const int col = warp * (kSlabWords / 8) + k;
      uint2 x;
      x.x = tr(slab[lane * kPad + col]);
      x.y = ROWS == 64 ? tr(slab[(32 + lane) * kPad + col]) : 0u;
      uint2 acc0 = make_uint2(0, 0), acc1 = make_uint2(0, 0);
      constexpr int kChunks = ROWS / 8;
#pragma unroll
      for (int kk = 0; kk < kChunks; kk += 2) {
        const int c0 = (kk + q) % kChunks, c1 = (kk + 1 + q) % kChunks;
        const uint32_t b0 = __byte_perm(c0 < 4 ? x.x : x.y, 0, 0x4440u | (uint32_t)(c0 & 3));
        const uint32_t b1 = __byte_perm(c1 < 4 ? x.x : x.y, 0, 0x4440u | (uint32_t)(c1 & 3));
        acc0 = x2(acc0, tab[b0 * 16 + h8 + c0]);
        acc1 = x2(acc1, tab[b1 * 16 + h8 + c1]);
      }
      ev[(w0 + col) * 32 + lane] = x2(acc0, acc1);
    }
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

__global__ void __launch_bounds__(256) decode64_kernel(const uint2* __restrict__ ev, uint64_t nslabs,
                                                       uint64_t row_words, const uint2* __restrict__ tab_g,
                                                       uint32_t* __restrict__ poly) {
  pdl_wait();
  extern __shared__ uint2 smem2[];
  uint2* tab = smem2;
  uint32_t* slab = reinterpret_cast<uint32_t*>(smem2 + kG8Uint2);  // 64 x kPad
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kG8Uint2; i += blockDim.x) tab[i] = tab_g[i];
  const Transpose32 tr(lane);
  __syncthreads();
  constexpr int kCols = kSlabWords / 8;  // next-slab register prefetch, as decode_kernel
  uint2 nx[kCols];
  auto fetch = [&](uint64_t sl) {
#pragma unroll
    for (int k = 0; k < kCols; ++k)
      nx[k] = sl < nslabs ? __ldg(ev + (sl * kSlabWords + warp * kCols + k) * 32 + lane) : make_uint2(0, 0);
  };
  fetch(blockIdx.x);
  for (uint64_t sl = blockIdx.x; sl < nslabs; sl += gridDim.x) {
    const uint64_t w0 = sl * kSlabWords;
    uint2 cur[kCols];
#pragma unroll
    for (int k = 0; k < kCols; ++k) cur[k] = nx[k];
    fetch(sl + gridDim.x);
#pragma unroll
    for (int k = 0; k < kCols; ++k) {
      const int col = warp * kCols + k;
      const uint2 y = g8_mul(tab, cur[k], lane);
      slab[lane * kPad + col] = tr(y.x);
      slab[(32 + lane) * kPad + col] = tr(y.y);
    }
    __syncthreads();
    for (int i = tid; i < 64 * kSlabWords; i += blockDim.x) {
      const int r = i / kSlabWords, c = i % kSlabWords;
      poly[(uint64_t)r * row_words + w0 + c] = slab[r * kPad + c];
    }
    __syncthreads();
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// Tiny shapes: one thread per element / output word, direct row products.
__global__ void encode64_small_kernel(const uint32_t* __restrict__ poly, uint64_t n_p, const uint2* __restrict__ rows,
                                      uint2* __restrict__ ev) {
  pdl_wait();
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_p) return;
  uint2 acc = make_uint2(0, 0);
  for (int j = 0; j < 64; ++j) {
    const uint64_t k = (uint64_t)j * n_p + i;
    if ((poly[k >> 5] >> (k & 31)) & 1u) acc = x2(acc, rows[j]);
  }
  ev[i] = acc;
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

__global__ void decode64_small_kernel(const uint2* __restrict__ ev, uint64_t n_p, const uint2* __restrict__ inv_rows,
                                      uint32_t* __restrict__ poly) {
  pdl_wait();
  const uint64_t wi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nwords = (64 * n_p + 31) / 32;
  if (wi >= nwords) return;
  uint32_t out = 0;
  for (int b = 0; b < 32; ++b) {
    const uint64_t k = wi * 32 + b;
    if (k >= 64 * n_p) break;
    const uint64_t j = k / n_p, i = k % n_p;
    const uint64_t f = ev[i].x | ((uint64_t)ev[i].y << 32);
    uint32_t acc = 0;
    for (int t = 0; t < 64; ++t)
      if ((f >> t) & 1u) {
        const uint64_t r = inv_rows[t].x | ((uint64_t)inv_rows[t].y << 32);
        acc ^= (uint32_t)(r >> j) & 1u;
      }
    out |= acc << b;
  }
  poly[wi] = out;
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// Device copies of the plain row tables for the tiny-shape kernels.
struct RowTables {
  uint4* rows = nullptr;
  uint4* inv = nullptr;
};
const RowTables& row_tables(int dev) {
  static std::mutex mu;
  static RowTables t[64];
  static bool have[64];
  if (dev < 0 || dev >= 64) throw Error(kInvalid, "device ordinal out of range");
  std::lock_guard<std::mutex> lock(mu);
  if (!have[dev]) {
    const FieldTables& ft = field_tables();
    FPM_CUDA(cudaMalloc(&t[dev].rows, 128 * 16));
    FPM_CUDA(cudaMalloc(&t[dev].inv, 128 * 16));
    FPM_CUDA(cudaMemcpy(t[dev].rows, ft.enc_rows, 128 * 16, cudaMemcpyHostToDevice));
    FPM_CUDA(cudaMemcpy(t[dev].inv, ft.inv_rows, 128 * 16, cudaMemcpyHostToDevice));
    have[dev] = true;
  }
  return t[dev];
}

__device__ __forceinline__ void flip_bit0(uint32_t* w) { *w ^= 1u; }
__global__ void flip_encode_tables_kernel(uint32_t* small128, uint32_t* m8, uint32_t* m8r, uint32_t* rows64,
                                          uint32_t* g8, uint32_t* g8r) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  // The forward tables' entry for "row 0 alone" (the reference flips bit 0 of tab_[1], chunk 0 /
  // value 1, encode.hpp:70-71): the tiny-shape row table, the M8 / G8 tables (entry (c=0, v=1);
  // both G8 copies) and their tower-representation twins.
  flip_bit0(small128);
  flip_bit0(m8 + 4 * (1 * 8 + 0));
  flip_bit0(m8r + 4 * (1 * 8 + 0));
  flip_bit0(rows64);
  flip_bit0(g8 + 2 * (1 * 16 + 0));
  flip_bit0(g8 + 2 * (1 * 16 + 8));
  flip_bit0(g8r + 2 * (1 * 16 + 0));
  flip_bit0(g8r + 2 * (1 * 16 + 8));
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

}  // namespace

// Test hook (EncodeMatrix::corrupt_for_test, proj/include/fpmul/encode.hpp:70-71): flips one bit of
// the DEVICE copies of the forward encode tables of both fields; a second call restores them.
void flip_encode_tables(int dev, cudaStream_t s) {
  const DeviceTables& dt = device_tables(dev);
  launch_k(flip_encode_tables_kernel, dim3(1), dim3(32), 0, s, reinterpret_cast<uint32_t*>(row_tables(dev).rows),
                                             reinterpret_cast<uint32_t*>(dt.enc_m8), reinterpret_cast<uint32_t*>(dt.enc_m8r),
                                             reinterpret_cast<uint32_t*>(dt.rows64), reinterpret_cast<uint32_t*>(dt.enc_g8),
                                             reinterpret_cast<uint32_t*>(dt.enc_g8r));
  FPM_LAUNCH_CHECK();
  FPM_CUDA(cudaStreamSynchronize(s));
}

// Column range [col0, col0 + ncols) of the 128-row partition matrix (row pitch n_p bits) -> ncols
// elements.  rows_live: 64 when rows >= 64 are known zero (pipeline operands), else 128.
void encode_cols_device(const uint32_t* poly, unsigned l, uint64_t col0, uint64_t ncols, uint4* ev, int rows_live,
                        cudaStream_t s, bool tower) {
  RankPtrs one{};
  one.p[0] = const_cast<uint32_t*>(poly);
  encode_cols_owners(one, 1, l, col0, ncols, ev, rows_live, s, tower);
}

// polys: Q = 1, 2 or 4 replicas, replica q holding the columns [q 2048/Q, (q+1) 2048/Q) of every 2048-word
// row (the sharded conversion's column owners; Q > 1 needs rows of >= 2048 words).
void encode_cols_owners(const RankPtrs& polys, int Q, unsigned l, uint64_t col0, uint64_t ncols, uint4* ev,
                        int rows_live, cudaStream_t s, bool tower) {
  const uint32_t* poly = polys.p[0];
  const int lgq = __builtin_ctz((unsigned)Q);
  if (Q > 1 && (((uint64_t)1 << l) / 32) % 2048) throw Error(kInvalid, "encode: column owners need 2048-word rows");
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const uint64_t n_p = (uint64_t)1 << l;
  if (n_p < 1024) {
    if (col0 != 0 || ncols != n_p || tower) throw Error(kInvalid, "encode: column ranges need n_p >= 1024");
    launch_k(encode_small_kernel, dim3((unsigned)((n_p + 127) / 128)), dim3(128), 0, s, poly, n_p, row_tables(dev).rows, ev);
    FPM_LAUNCH_CHECK();
    return;
  }
  if (col0 % 1024 || ncols % 1024 || col0 + ncols > n_p) throw Error(kInvalid, "encode: column range not 1024-aligned");
  const DeviceTables& dt = device_tables(dev);
  const uint4* tab = tower ? dt.enc_m8r : dt.enc_m8;
  const uint64_t nslabs = ncols / 32 / kSlabWords;
  if (rows_live == 64) {
    const size_t smem = kM8Uint4 / 2 * sizeof(uint4) + 64 * kPad * sizeof(uint32_t);
    static PerDeviceOnce attr;
    attr.run([&] { FPM_CUDA(cudaFuncSetAttribute(encode_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); });
    launch_k(encode_kernel<64>, dim3(resident_grid(encode_kernel<64>, 256, smem, nslabs)), dim3(256), smem, s, polys, lgq, n_p / 32, col0 / 32, nslabs, tab, ev,
             (uint64_t)kSlabWords);
  } else {
    const size_t smem = kM8Uint4 * sizeof(uint4) + 128 * kPad * sizeof(uint32_t);
    static PerDeviceOnce attr;
    attr.run([&] { FPM_CUDA(cudaFuncSetAttribute(encode_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); });
    launch_k(encode_kernel<128>, dim3(resident_grid(encode_kernel<128>, 256, smem, nslabs)), dim3(256), smem, s, polys, lgq, n_p / 32, col0 / 32, nslabs, tab, ev,
             (uint64_t)kSlabWords);
  }
  FPM_LAUNCH_CHECK();
}

// A batch of count independent 2^16-bit operands (l = 10: 64 live rows of 32 words each, operands
// stride_words apart) -> count EvalVecs of 1024 elements in the tower representation, back to back.
void encode_batch_r(const uint32_t* polys, uint64_t count, uint64_t stride_words, uint4* ev, cudaStream_t s) {
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const DeviceTables& dt = device_tables(dev);
  RankPtrs one{};
  one.p[0] = const_cast<uint32_t*>(polys);
  const size_t smem = kM8Uint4 / 2 * sizeof(uint4) + 64 * kPad * sizeof(uint32_t);
  static PerDeviceOnce attr;
  attr.run([&] { FPM_CUDA(cudaFuncSetAttribute(encode_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); });
  launch_k(encode_kernel<64>, dim3(resident_grid(encode_kernel<64>, 256, smem, count)), dim3(256), smem, s, one, 0,
           (uint64_t)32, (uint64_t)0, count, dt.enc_m8r, ev, stride_words);
  FPM_LAUNCH_CHECK();
}

// count tower-representation EvalVecs of 1024 elements -> count 2^17-bit products (128 rows of 32
// words), stride_words apart.
void decode_batch_r(const uint4* ev, uint64_t count, uint32_t* out, uint64_t stride_words, cudaStream_t s) {
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const DeviceTables& dt = device_tables(dev);
  const size_t smem = kM8Uint4 * sizeof(uint4) + 128 * kPad * sizeof(uint32_t);
  static PerDeviceOnce attr;
  attr.run([&] { FPM_CUDA(cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); });
  RankPtrs lo{}, hi{};
  lo.p[0] = out;
  hi.p[0] = out + 64 * 32;
  launch_k(decode_kernel, dim3(resident_grid(decode_kernel, 256, smem, count)), dim3(256), smem, s, ev, count, (uint64_t)32,
           dt.dec_m8r, lo, hi, 0, (uint64_t)0, stride_words);
  FPM_LAUNCH_CHECK();
}

void encode_device_rows(const uint32_t* poly, unsigned l, uint4* ev, int rows_live, cudaStream_t s, bool tower) {
  encode_cols_device(poly, l, 0, (uint64_t)1 << l, ev, rows_live, s, tower);
}

void encode_device(const uint32_t* poly, unsigned l, uint4* ev, cudaStream_t s) {
  encode_device_rows(poly, l, ev, 128, s);
}

// ncols elements -> a 128-row x ncols-bit slice (row pitch ncols bits).
void decode_cols_device(const uint4* ev, uint64_t ncols, uint32_t* slice, cudaStream_t s, bool tower) {
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  if (ncols < 1024) {
    if ((ncols & (ncols - 1)) || tower) throw Error(kInvalid, "decode: element count must be a power of two");
    const uint64_t nwords = (128 * ncols + 31) / 32;
    launch_k(decode_small_kernel, dim3((unsigned)((nwords + 127) / 128)), dim3(128), 0, s, ev, ncols, row_tables(dev).inv, slice);
    FPM_LAUNCH_CHECK();
    return;
  }
  if (ncols % 1024) throw Error(kInvalid, "decode: column count not 1024-aligned");
  const DeviceTables& dt = device_tables(dev);
  const size_t smem = kM8Uint4 * sizeof(uint4) + 128 * kPad * sizeof(uint32_t);
  static PerDeviceOnce attr;
  attr.run([&] { FPM_CUDA(cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); });
  const uint64_t nslabs = ncols / 32 / kSlabWords;
  RankPtrs lo{}, hi{};
  lo.p[0] = slice;
  hi.p[0] = slice + 64 * (ncols / 32);
  launch_k(decode_kernel, dim3(resident_grid(decode_kernel, 256, smem, nslabs)), dim3(256), smem, s, ev, nslabs, ncols / 32, tower ? dt.dec_m8r : dt.dec_m8, lo, hi, 0,
           (uint64_t)0, (uint64_t)kSlabWords);
  FPM_LAUNCH_CHECK();
}

void decode_cols_split_device(const uint4* ev, uint64_t ncols, uint64_t col0, uint64_t row_bits, uint32_t* lo,
                              uint32_t* hi, cudaStream_t s, bool tower) {
  RankPtrs l{}, h{};
  l.p[0] = lo;
  h.p[0] = hi;
  decode_cols_owners(ev, ncols, col0, row_bits, l, h, 1, s, tower);
}

// The sharded variant: rows 0..63 into the column owners los.p[q], rows 64..127 into his.p[q] (Q
// replicas as encode_cols_owners).
void decode_cols_owners(const uint4* ev, uint64_t ncols, uint64_t col0, uint64_t row_bits, const RankPtrs& los,
                        const RankPtrs& his, int Q, cudaStream_t s, bool tower) {
  const int lgq = __builtin_ctz((unsigned)Q);
  if (Q > 1 && (row_bits / 32) % 2048) throw Error(kInvalid, "decode: column owners need 2048-word rows");
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  if (ncols % 1024 || col0 % 1024 || row_bits % 1024 || col0 + ncols > row_bits)
    throw Error(kInvalid, "decode: split column ranges need 1024-aligned columns");
  const DeviceTables& dt = device_tables(dev);
  const size_t smem = kM8Uint4 * sizeof(uint4) + 128 * kPad * sizeof(uint32_t);
  static PerDeviceOnce attr;
  attr.run([&] { FPM_CUDA(cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); });
  const uint64_t nslabs = ncols / 32 / kSlabWords;
  launch_k(decode_kernel, dim3(resident_grid(decode_kernel, 256, smem, nslabs)), dim3(256), smem, s, ev, nslabs, row_bits / 32, tower ? dt.dec_m8r : dt.dec_m8, los, his, lgq,
           col0 / 32, (uint64_t)kSlabWords);
  FPM_LAUNCH_CHECK();
}

void encode64_device(const uint32_t* poly, unsigned l, uint2* ev, int rows_live, cudaStream_t s, bool tower) {
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const DeviceTables& dt = device_tables(dev);
  const uint64_t n_p = (uint64_t)1 << l;
  if (n_p < 1024) {
    if (tower) throw Error(kInvalid, "encode64: the tower representation needs n_p >= 1024");
    launch_k(encode64_small_kernel, dim3((unsigned)((n_p + 127) / 128)), dim3(128), 0, s, poly, n_p, dt.rows64, ev);
    FPM_LAUNCH_CHECK();
    return;
  }
  const uint64_t nslabs = n_p / 32 / kSlabWords;
  if (rows_live <= 32) {
    const size_t smem = kG8Uint2 * sizeof(uint2) + 32 * kPad * sizeof(uint32_t);
    launch_k(encode64_kernel<32>, dim3(resident_grid(encode64_kernel<32>, 256, smem, nslabs)), dim3(256), smem, s, poly, n_p / 32, nslabs, tower ? dt.enc_g8r : dt.enc_g8, ev);
  } else {
    const size_t smem = kG8Uint2 * sizeof(uint2) + 64 * kPad * sizeof(uint32_t);
    launch_k(encode64_kernel<64>, dim3(resident_grid(encode64_kernel<64>, 256, smem, nslabs)), dim3(256), smem, s, poly, n_p / 32, nslabs, tower ? dt.enc_g8r : dt.enc_g8, ev);
  }
  FPM_LAUNCH_CHECK();
}

void decode64_device(const uint2* ev, unsigned l, uint32_t* poly, cudaStream_t s, bool tower) {
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const DeviceTables& dt = device_tables(dev);
  const uint64_t n_p = (uint64_t)1 << l;
  if (n_p < 1024) {
    if (tower) throw Error(kInvalid, "decode64: the tower representation needs n_p >= 1024");
    const uint64_t nwords = (64 * n_p + 31) / 32;
    launch_k(decode64_small_kernel, dim3((unsigned)((nwords + 127) / 128)), dim3(128), 0, s, ev, n_p, dt.inv64, poly);
    FPM_LAUNCH_CHECK();
    return;
  }
  const uint64_t nslabs = n_p / 32 / kSlabWords;
  const size_t smem = kG8Uint2 * sizeof(uint2) + 64 * kPad * sizeof(uint32_t);
  launch_k(decode64_kernel, dim3(resident_grid(decode64_kernel, 256, smem, nslabs)), dim3(256), smem, s, ev, nslabs, n_p / 32, tower ? dt.dec_g8r : dt.dec_g8, poly);
  FPM_LAUNCH_CHECK();
}

void decode_device(const uint4* ev, unsigned l, uint32_t* poly, cudaStream_t s, bool tower) {
  decode_cols_device(ev, (uint64_t)1 << l, poly, s, tower);
}

}  // namespace fpm
