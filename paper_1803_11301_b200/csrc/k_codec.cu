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
// the 128-bit matrix product x*E runs as M4R lookups in an 8x-replicated, bank-conflict-free
// shared table.  Decode runs the same steps in reverse.
#include <cuda_runtime.h>

#include "fpm_internal.h"
#include "gf128.cuh"

namespace fpm {
namespace {

constexpr int kSlabWords = 32;                 // words per row per CTA slab -> 1024 elements
constexpr int kPad = kSlabWords + 1;

// 32x32 bit transpose across a warp: on entry lane r holds row r (bit c = M[r][c]); on exit lane c
// holds column c (bit r = M[r][c]).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  const uint32_t masks[5] = {0xFFFF0000u, 0xFF00FF00u, 0xF0F0F0F0u, 0xCCCCCCCCu, 0xAAAAAAAAu};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int s = 16 >> k;
    const uint32_t m = masks[k];
    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, s);
    if (lane & s) x = (x & m) | ((y >> s) & ~m);
    else x = (x & ~m) | ((y << s) & m);
  }
  return x;
}

template <int ROWS>  // 64: rows >= 64 are known zero (pipeline); 128: general encode
__global__ void __launch_bounds__(256) encode_kernel(const uint32_t* __restrict__ poly, uint64_t row_words,
                                                     uint64_t col0_words, uint64_t nslabs,
                                                     const uint4* __restrict__ tab_g, uint4* __restrict__ ev) {
  extern __shared__ uint4 smem4[];
  uint4* tab = smem4;                                           // (ROWS/4) chunks x 16 x 8 copies
  uint32_t* slab = reinterpret_cast<uint32_t*>(smem4 + (ROWS / 4) * 16 * kM4RCopies);  // ROWS x kPad
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < (ROWS / 4) * 16 * kM4RCopies; i += blockDim.x) tab[i] = tab_g[i];
  const int copy = lane & 7;
  for (uint64_t sl = blockIdx.x; sl < nslabs; sl += gridDim.x) {
    const uint64_t w0 = sl * kSlabWords;
    __syncthreads();
    for (int i = tid; i < ROWS * kSlabWords; i += blockDim.x) {
      const int r = i / kSlabWords, c = i % kSlabWords;
      slab[r * kPad + c] = poly[(uint64_t)r * row_words + col0_words + w0 + c];
    }
    __syncthreads();
#pragma unroll 1
    for (int k = 0; k < kSlabWords / 8; ++k) {
      const int col = warp * (kSlabWords / 8) + k;
      uint32_t xw[4];
#pragma unroll
      for (int q = 0; q < ROWS / 32; ++q) xw[q] = warp_transpose32(slab[(q * 32 + lane) * kPad + col], lane);
      uint4 f;
      if (ROWS == 64) {
        // x has 64 bits -> 16 nibble chunks
        uint4 acc0 = make_uint4(0, 0, 0, 0), acc1 = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int s = 0; s < 8; s += 2) {
            const int c0 = q * 8 + s;
            acc0 = x4(acc0, tab[((c0 * 16 + ((xw[q] >> (4 * s)) & 15u)) << 3) + copy]);
            acc1 = x4(acc1, tab[(((c0 + 1) * 16 + ((xw[q] >> (4 * s + 4)) & 15u)) << 3) + copy]);
          }
        f = x4(acc0, acc1);
      } else {
        f = m4r_mul(tab, make_uint4(xw[0], xw[1], xw[ROWS / 32 > 2 ? 2 : 0], xw[ROWS / 32 > 3 ? 3 : 0]), copy);
      }
      ev[(w0 + col) * 32 + lane] = f;
    }
  }
}

__global__ void __launch_bounds__(256) decode_kernel(const uint4* __restrict__ ev, uint64_t nslabs,
                                                     uint64_t row_words,
                                                     const uint4* __restrict__ tab_g, uint32_t* __restrict__ poly) {
  extern __shared__ uint4 smem4[];
  uint4* tab = smem4;  // 32 chunks x 16 x 8 copies
  uint32_t* slab = reinterpret_cast<uint32_t*>(smem4 + kM4RUint4);  // 128 x kPad
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kM4RUint4; i += blockDim.x) tab[i] = tab_g[i];
  const int copy = lane & 7;
  __syncthreads();
  for (uint64_t sl = blockIdx.x; sl < nslabs; sl += gridDim.x) {
    const uint64_t w0 = sl * kSlabWords;
#pragma unroll 1
    for (int k = 0; k < kSlabWords / 8; ++k) {
      const int col = warp * (kSlabWords / 8) + k;
      const uint4 y = m4r_mul(tab, ev[(w0 + col) * 32 + lane], copy);
      slab[(0 * 32 + lane) * kPad + col] = warp_transpose32(y.x, lane);
      slab[(1 * 32 + lane) * kPad + col] = warp_transpose32(y.y, lane);
      slab[(2 * 32 + lane) * kPad + col] = warp_transpose32(y.z, lane);
      slab[(3 * 32 + lane) * kPad + col] = warp_transpose32(y.w, lane);
    }
    __syncthreads();
    for (int i = tid; i < 128 * kSlabWords; i += blockDim.x) {
      const int r = i / kSlabWords, c = i % kSlabWords;
      poly[(uint64_t)r * row_words + w0 + c] = slab[r * kPad + c];
    }
    __syncthreads();
  }
}

// Tiny shapes (n_p < 1024): one thread per element, direct row products (encode.cpp:172-181).
__global__ void encode_small_kernel(const uint32_t* __restrict__ poly, uint64_t n_p, const uint4* __restrict__ rows,
                                    uint4* __restrict__ ev) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_p) return;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int j = 0; j < 128; ++j) {
    const uint64_t k = (uint64_t)j * n_p + i;
    if ((poly[k >> 5] >> (k & 31)) & 1u) acc = x4(acc, rows[j]);
  }
  ev[i] = acc;
}

__global__ void decode_small_kernel(const uint4* __restrict__ ev, uint64_t n_p, const uint4* __restrict__ inv_rows,
                                    uint32_t* __restrict__ poly) {
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
}

// Device copies of the plain row tables for the tiny-shape kernels.
struct RowTables {
  uint4* rows = nullptr;
  uint4* inv = nullptr;
};
const RowTables& row_tables(int dev) {
  static RowTables t[64];
  static bool have[64];
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

int grid_for(uint64_t work, int per_sm) {
  int dev, sms;
  FPM_CUDA(cudaGetDevice(&dev));
  FPM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const uint64_t g = std::min<uint64_t>(work, (uint64_t)sms * per_sm);
  return (int)(g ? g : 1);
}

}  // namespace

// Column range [col0, col0 + ncols) of the 128-row partition matrix (row pitch n_p bits) -> ncols
// elements.  rows_live: 64 when rows >= 64 are known zero (pipeline operands), else 128.
void encode_cols_device(const uint32_t* poly, unsigned l, uint64_t col0, uint64_t ncols, uint4* ev, int rows_live,
                        cudaStream_t s) {
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const uint64_t n_p = (uint64_t)1 << l;
  if (n_p < 1024) {
    if (col0 != 0 || ncols != n_p) throw Error(kInvalid, "encode: column ranges need n_p >= 1024");
    encode_small_kernel<<<(unsigned)((n_p + 127) / 128), 128, 0, s>>>(poly, n_p, row_tables(dev).rows, ev);
    FPM_LAUNCH_CHECK();
    return;
  }
  if (col0 % 1024 || ncols % 1024 || col0 + ncols > n_p) throw Error(kInvalid, "encode: column range not 1024-aligned");
  const DeviceTables& dt = device_tables(dev);
  const uint64_t nslabs = ncols / 32 / kSlabWords;
  if (rows_live == 64) {
    const size_t smem = 16 * 16 * kM4RCopies * sizeof(uint4) + 64 * kPad * sizeof(uint32_t);
    static bool attr = false;
    if (!attr) { FPM_CUDA(cudaFuncSetAttribute(encode_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); attr = true; }
    encode_kernel<64><<<grid_for(nslabs, 4), 256, smem, s>>>(poly, n_p / 32, col0 / 32, nslabs, dt.enc_m4r, ev);
  } else {
    const size_t smem = 32 * 16 * kM4RCopies * sizeof(uint4) + 128 * kPad * sizeof(uint32_t);
    static bool attr = false;
    if (!attr) { FPM_CUDA(cudaFuncSetAttribute(encode_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); attr = true; }
    encode_kernel<128><<<grid_for(nslabs, 2), 256, smem, s>>>(poly, n_p / 32, col0 / 32, nslabs, dt.enc_m4r, ev);
  }
  FPM_LAUNCH_CHECK();
}

void encode_device_rows(const uint32_t* poly, unsigned l, uint4* ev, int rows_live, cudaStream_t s) {
  encode_cols_device(poly, l, 0, (uint64_t)1 << l, ev, rows_live, s);
}

void encode_device(const uint32_t* poly, unsigned l, uint4* ev, cudaStream_t s) {
  encode_device_rows(poly, l, ev, 128, s);
}

// ncols elements -> a 128-row x ncols-bit slice (row pitch ncols bits).
void decode_cols_device(const uint4* ev, uint64_t ncols, uint32_t* slice, cudaStream_t s) {
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  if (ncols < 1024) {
    if (ncols & (ncols - 1)) throw Error(kInvalid, "decode: element count must be a power of two");
    const uint64_t nwords = (128 * ncols + 31) / 32;
    decode_small_kernel<<<(unsigned)((nwords + 127) / 128), 128, 0, s>>>(ev, ncols, row_tables(dev).inv, slice);
    FPM_LAUNCH_CHECK();
    return;
  }
  if (ncols % 1024) throw Error(kInvalid, "decode: column count not 1024-aligned");
  const DeviceTables& dt = device_tables(dev);
  const size_t smem = kM4RUint4 * sizeof(uint4) + 128 * kPad * sizeof(uint32_t);
  static bool attr = false;
  if (!attr) { FPM_CUDA(cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); attr = true; }
  const uint64_t nslabs = ncols / 32 / kSlabWords;
  decode_kernel<<<grid_for(nslabs, 2), 256, smem, s>>>(ev, nslabs, ncols / 32, dt.dec_m4r, slice);
  FPM_LAUNCH_CHECK();
}

void decode_device(const uint4* ev, unsigned l, uint32_t* poly, cudaStream_t s) {
  decode_cols_device(ev, (uint64_t)1 << l, poly, s);
}

}  // namespace fpm
