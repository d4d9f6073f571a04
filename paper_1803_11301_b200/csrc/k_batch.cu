// k_batch.cu -- whole small products, one CTA each, entirely in shared memory.
//
// Serves (a) BASELINE config 2 (4096 independent 2^16 x 2^16-bit products, n = 2^17, l = 10) and
// (b) every product whose padded length n <= 2^17 bits (l <= 10).  The CTA runs the complete
// reference pipeline run_pipeline<gf128> (proj/src/polymul.cpp:78-135) on its product:
//   basis_cvt(a), encode, forward butterflies; same for b; pointwise; inverse butterflies;
//   decode; i_basis_cvt; trim to len_a + len_b - 1 (polymul.cpp:237)
// with no HBM traffic besides reading a, b and writing c.  Products share every table, so the
// batch is sharded across GPUs (and CTAs) with no exchange.
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>
#include <vector>

#include "basis_dev.cuh"
#include "conv_tile.cuh"
#include "fpm_internal.h"
#include "gf128.cuh"
#include "warp_bits.cuh"

namespace fpm {


namespace {

constexpr int kBatchMaxLog2N = 17;

__device__ __forceinline__ uint4 c2p2b(const uint4* __restrict__ c2p, uint64_t b) {
  uint4 r = c2p[b & 511];
  if (b >> 9) r = x4(r, c2p[512 + ((b >> 9) & 511)]);
  return r;
}


// Basis conversion of a <= 2^16-bit array W (2^K bits) in place, as one conversion tile
// (conv_tile.cuh: L1 + row passes + register passes; zero-padded to the 8 KiB tile).
// scratch: >= kTileRows * (kRowPitchW<1> + kScPitch) words, disjoint from W.
template <bool INV>
__device__ __forceinline__ void conv_small(uint32_t* W, int K, uint32_t* scratch) {
  const int tid = threadIdx.x;
  const int words = K >= 5 ? 1 << (K - 5) : 1;
  uint32_t m[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) m[j] = 8 * tid + j < words ? W[8 * tid + j] : 0u;
  conv_tile<INV>(m, scratch, scratch + kTileRows * kRowPitchW<1>, K);
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (8 * tid + j < words) W[8 * tid + j] = m[j];
  __syncthreads();
}

// Inverse conversion of the 2^17-bit product array: conv(2^16)^-1 of both halves, then the inverse
// of the single top pass (S = 2^17, D = 2^16 - 1: bits [1, 2^16] ^= bits [2^16, 2^17 - 1], from the
// pre-pass values; build_schedule at 2^17, basis_convert.cpp:53-67).
__device__ __forceinline__ void i_conv_17(uint32_t* W, uint32_t* scratch) {
  conv_small<true>(W, 16, scratch);
  conv_small<true>(W + 2048, 16, scratch);
  const int tid = threadIdx.x;
  uint32_t t[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int w = tid + 256 * k;  // target words 0 .. 2048
    t[k] = 0;
    if (w <= 2048) {
      const uint32_t lo = W[w + 2047], hi = w + 2048 < 4096 ? W[w + 2048] : 0u;
      t[k] = __funnelshift_r(lo, hi, 31);
      if (w == 0) t[k] &= ~1u;
      if (w == 2048) t[k] &= 1u;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int w = tid + 256 * k;
    if (w <= 2048) W[w] ^= t[k];
  }
  __syncthreads();
}

// Forward transform of one operand: W0 <- x (n/2 bits), basis conversion, encode into E, butterflies.
__device__ void transform_operand(const uint64_t* __restrict__ x, uint64_t x_bits, uint32_t* W0, uint32_t* scratch,
                                  uint4* E, unsigned l, int half_words, const uint4* __restrict__ enc_m8,
                                  const uint4* __restrict__ enc_rows, const TwiddleSrc& tw) {
  const int tid = threadIdx.x;
  const uint32_t* x32 = reinterpret_cast<const uint32_t*>(x);
  for (int i = tid; i < half_words; i += blockDim.x) {
    const uint64_t bit0 = (uint64_t)i * 32;
    uint32_t v = 0;
    if (bit0 < x_bits) {
      v = x32[i];
      if (x_bits - bit0 < 32) v &= (1u << (x_bits - bit0)) - 1u;
    }
    W0[i] = v;
  }
  __syncthreads();
  const int Kh = l + 6;  // the operand half: 2^(l+6) bits
  conv_small<false>(W0, Kh, scratch);
  const uint32_t* P = W0;
  // encode: f_i = sum_j a_{j n_p + i} r_j, rows j < 64 (the upper half is zero padding): 8 byte
  // lookups in the rotated 8-bit table of x*E (read through L1)
  const int n_p = 1 << l;
  const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  if (n_p >= 32) {
    const Transpose32 tr(lane);
    const int q8 = lane & 7;
    const int row_words = n_p / 32;
    for (int col = warp; col < row_words; col += nwarps) {
      const uint32_t lo = tr(P[lane * row_words + col]);
      const uint32_t hi = tr(P[(lane + 32) * row_words + col]);
      uint4 f = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int c = (k + q8) & 7;
        const uint32_t byte = __byte_perm(c < 4 ? lo : hi, 0, 0x4440u | (uint32_t)(c & 3));
        f = x4(f, __ldg(enc_m8 + byte * 8 + c));
      }
      E[col * 32 + lane] = f;
    }
  } else {
    for (int i = tid; i < n_p; i += blockDim.x) {
      uint4 f = make_uint4(0, 0, 0, 0);
      for (int j = 0; j < 64; ++j) {
        const int k = j * n_p + i;
        if ((P[k >> 5] >> (k & 31)) & 1u) f = x4(f, enc_rows[j]);
      }
      E[i] = f;
    }
  }
  __syncthreads();
  // forward butterflies, layers l-1 .. 0 (kernels_impl.hpp:29-47)
  for (int i = (int)l - 1; i >= 0; --i) {
    const uint4 vbase = tw.layer[i];
    for (int p = tid; p < n_p / 2; p += blockDim.x) {
      const int blk = p >> i, j = p & ((1 << i) - 1);
      const int i0 = (blk << (i + 1)) + j, i1 = i0 + (1 << i);
      const uint4 w = x4(vbase, c2p2b(tw.c2p, (uint64_t)blk));
      uint4 u0 = E[i0], u1 = E[i1];
      u0 = x4(u0, gf_mul(w, u1));
      u1 = x4(u1, u0);
      E[i0] = u0;
      E[i1] = u1;
    }
    __syncthreads();
  }
}

// Shared memory (fixed l = 10 layout, 64 KiB): EA | EB | W0 | W1, 16 KiB each.  The bit arrays
// (operand halves, then the product) live in W1; EB..W0 (32 KiB, contiguous) is the conversion
// tile's scratch whenever it is not holding data (EB is only written by the second encode, after
// that operand's conversion).
constexpr int kBatchSmemUint4 = 4 * 1024;
__global__ void __launch_bounds__(256) batch_kernel(const uint64_t* __restrict__ a, uint64_t a_bits, uint64_t a_stride,
                                                    const uint64_t* __restrict__ b, uint64_t b_bits, uint64_t b_stride,
                                                    uint64_t* __restrict__ c, uint64_t c_stride, unsigned l,
                                                    const uint4* __restrict__ enc_m8, const uint4* __restrict__ dec_m8,
                                                    const uint4* __restrict__ enc_rows,
                                                    const uint4* __restrict__ inv_rows, TwiddleSrc tw) {
  pdl_wait();
  extern __shared__ uint4 sm[];
  const int n_p = 1 << l;
  const int n_words = n_p * 4;  // n = 128 n_p bits
  uint4* EA = sm;
  uint4* EB = sm + 1024;
  uint32_t* W1 = reinterpret_cast<uint32_t*>(sm + 3 * 1024);
  uint32_t* scratch = reinterpret_cast<uint32_t*>(EB);  // EB + W0: 8192 words
  const uint64_t prod = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

  transform_operand(a + prod * a_stride, a_bits, W1, scratch, EA, l, n_words / 2, enc_m8, enc_rows, tw);
  transform_operand(b + prod * b_stride, b_bits, W1, scratch, EB, l, n_words / 2, enc_m8, enc_rows, tw);
  for (int i = tid; i < n_p; i += blockDim.x) EA[i] = gf_mul(EA[i], EB[i]);
  __syncthreads();
  // inverse butterflies, layers 0 .. l-1 (kernels_impl.hpp:48-61)
  for (unsigned i = 0; i < l; ++i) {
    const uint4 vbase = tw.layer[i];
    for (int p = tid; p < n_p / 2; p += blockDim.x) {
      const int blk = p >> i, j = p & ((1 << i) - 1);
      const int i0 = (blk << (i + 1)) + j, i1 = i0 + (1 << i);
      const uint4 w = x4(vbase, c2p2b(tw.c2p, (uint64_t)blk));
      uint4 u0 = EA[i0], u1 = EA[i1];
      u1 = x4(u1, u0);
      u0 = x4(u0, gf_mul(w, u1));
      EA[i0] = u0;
      EA[i1] = u1;
    }
    __syncthreads();
  }
  // decode: y_i = f_i E^{-1} (16 byte lookups in the rotated table, through L1); bit j of y_i ->
  // c_{j n_p + i} by warp transposes (encode.cpp:195-220)
  if (n_p >= 32) {
    const Transpose32 tr(lane);
    const int q8 = lane & 7;
    const int row_words = n_p / 32;
    for (int col = warp; col < row_words; col += nwarps) {
      const uint4 f = EA[col * 32 + lane];
      uint4 y = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int cc = (k + q8) & 7;
        const uint32_t lo = __byte_perm(cc < 4 ? f.x : f.y, 0, 0x4440u | (uint32_t)(cc & 3));
        const uint32_t hi = __byte_perm(cc < 4 ? f.z : f.w, 0, 0x4440u | (uint32_t)(cc & 3));
        y = x4(y, __ldg(dec_m8 + lo * 8 + cc));
        y = x4(y, __ldg(dec_m8 + 2048 + hi * 8 + cc));
      }
      W1[(0 * 32 + lane) * row_words + col] = tr(y.x);
      W1[(1 * 32 + lane) * row_words + col] = tr(y.y);
      W1[(2 * 32 + lane) * row_words + col] = tr(y.z);
      W1[(3 * 32 + lane) * row_words + col] = tr(y.w);
    }
  } else {
    for (int wi = tid; wi < n_words; wi += blockDim.x) {
      uint32_t out = 0;
      for (int bb = 0; bb < 32; ++bb) {
        const int k = wi * 32 + bb, j = k / n_p, i = k % n_p;
        const uint4 f = EA[i];
        const uint32_t fw[4] = {f.x, f.y, f.z, f.w};
        uint32_t acc = 0;  // bit j of f E^{-1}
        for (int t = 0; t < 128; ++t)
          if ((fw[t >> 5] >> (t & 31)) & 1u) {
            const uint4 r = inv_rows[t];
            const uint32_t rw[4] = {r.x, r.y, r.z, r.w};
            acc ^= (rw[j >> 5] >> (j & 31)) & 1u;
          }
        out |= acc << bb;
      }
      W1[wi] = out;
    }
  }
  __syncthreads();
  // inverse basis conversion of the n-bit product (n = 2^(l+7))
  if (l + 7 <= 16) conv_small<true>(W1, l + 7, scratch);
  else i_conv_17(W1, scratch);
  // trim to len_a + len_b - 1 bits and write 64-bit words
  const uint64_t out_bits = a_bits + b_bits - 1;
  const uint64_t out_words = (out_bits + 63) / 64;
  uint64_t* cc = c + prod * c_stride;
  for (uint64_t k = tid; k < out_words; k += blockDim.x) {
    uint64_t v = (uint64_t)W1[2 * k] | ((uint64_t)W1[2 * k + 1] << 32);
    if (k == out_words - 1 && (out_bits & 63)) v &= (((uint64_t)1) << (out_bits & 63)) - 1;
    cc[k] = v;
  }
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

// ------------------------------------------------------------------ config 2 in the tower representation
// Batches of 2^17-bit products (l = 10) as a handful of batch-wide kernels instead of one CTA per
// product: operands padded to 2^16 bits, conv(2^16) of every operand (conv_rows), encode into the
// tower representation, the tower tile pass with ONE tile per product (a whole 2^10-element
// transform of both operands, the pointwise product and the inverse; every table serves both
// operands and is built per product instead of the generic multiplies of batch_kernel), decode,
// conv(2^16)^-1 of both halves and the single top pass of the 2^17-bit inverse, then the trimmed
// product words.
__global__ void batch_load_kernel(const uint64_t* __restrict__ x, uint64_t x_bits, uint64_t x_stride,
                                  uint64_t* __restrict__ w, uint64_t count) {
  pdl_wait();
  constexpr uint64_t kWords = 1024;  // 2^16 bits
  const uint64_t xw = (x_bits + 63) / 64;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count * kWords; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = k / kWords, i = k % kWords;
    uint64_t v = 0;
    if (i < xw) {
      v = x[p * x_stride + i];
      if (i == xw - 1 && (x_bits & 63)) v &= ((uint64_t)1 << (x_bits & 63)) - 1;
    }
    w[k] = v;
  }
  pdl_trigger();
}

// Per product (one CTA): the inverse of the 2^17-bit array's single top pass (bits [1, 2^16] ^= bits
// [2^16, 2^17 - 1], from the pre-pass values; as i_conv_17), then the product trimmed to out_bits into
// c (c_stride words apart).
__global__ void __launch_bounds__(256) batch_fold_store_kernel(const uint32_t* __restrict__ W, uint64_t* __restrict__ c,
                                                               uint64_t c_stride, uint64_t out_bits, uint64_t count) {
  pdl_wait();
  __shared__ uint32_t t[2049];
  const int tid = threadIdx.x;
  const uint64_t out_words = (out_bits + 63) / 64;
  for (uint64_t p = blockIdx.x; p < count; p += gridDim.x) {
    const uint32_t* w = W + p * 4096;
    for (int k = tid; k <= 2048; k += blockDim.x) {
      const uint32_t lo = w[k + 2047], hi = k + 2048 < 4096 ? w[k + 2048] : 0u;
      uint32_t v = __funnelshift_r(lo, hi, 31);
      if (k == 0) v &= ~1u;
      if (k == 2048) v &= 1u;
      t[k] = v;
    }
    __syncthreads();
    uint64_t* cc = c + p * c_stride;
    for (uint64_t k = tid; k < out_words; k += blockDim.x) {
      const uint32_t x0 = w[2 * k] ^ (2 * k <= 2048 ? t[2 * k] : 0u);
      const uint32_t x1 = w[2 * k + 1] ^ (2 * k + 1 <= 2048 ? t[2 * k + 1] : 0u);
      uint64_t v = (uint64_t)x0 | ((uint64_t)x1 << 32);
      if (k == out_words - 1 && (out_bits & 63)) v &= (((uint64_t)1) << (out_bits & 63)) - 1;
      cc[k] = v;
    }
    __syncthreads();
  }
  pdl_trigger();
}

}  // namespace

bool batch_tower_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FPM_BATCH_TOWER");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

void polymul_batch_device(const uint64_t* a, size_t a_bits, size_t a_stride_words, const uint64_t* b, size_t b_bits,
                          size_t b_stride_words, uint64_t* c, size_t c_stride_words, size_t count, cudaStream_t s) {
  if (!count) return;
  const size_t mx = a_bits > b_bits ? a_bits : b_bits;
  size_t n = 1;
  while (n < 2 * mx) n <<= 1;
  if (n < 128) n = 128;
  unsigned logn = 0;
  while (((size_t)1 << logn) < n) ++logn;
  if (logn > (unsigned)kBatchMaxLog2N) throw Error(kInvalid, "polymul_batch: product longer than 2^17 bits");
  const unsigned l = logn - 7;
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  if (l == 10 && count >= 64 && batch_tower_enabled()) {  // config 2: the tower-representation batch pipeline
    const TwiddleSrc tw = make_twiddle_src(dev, l, partition_base(l));
    DevBuf WA(count * 8192, s), WB(count * 8192, s), EA(count * 1024 * 16, s), EB(count * 1024 * 16, s);
    const int g1 = (int)std::min<uint64_t>((count * 1024 + 255) / 256, 148u * 16u);
    launch_k(batch_load_kernel, dim3(g1), dim3(256), 0, s, a, (uint64_t)a_bits, (uint64_t)a_stride_words, WA.as<uint64_t>(), (uint64_t)count);
    FPM_LAUNCH_CHECK();
    launch_k(batch_load_kernel, dim3(g1), dim3(256), 0, s, b, (uint64_t)b_bits, (uint64_t)b_stride_words, WB.as<uint64_t>(), (uint64_t)count);
    FPM_LAUNCH_CHECK();
    conv_rows_batch16(WA.as<uint32_t>(), count * 2048, false, s);
    conv_rows_batch16(WB.as<uint32_t>(), count * 2048, false, s);
    encode_batch_r(WA.as<uint32_t>(), count, 2048, EA.as<uint4>(), s);
    encode_batch_r(WB.as<uint32_t>(), count, 2048, EB.as<uint4>(), s);
    butterfly_tile_tower_device(EA.as<uint4>(), EB.as<uint4>(), l, l, tw, s, count);
    // the 2^17-bit products (4096 words each) reuse WA + WB (contiguous in the pool? not assumed:
    // a separate array)
    DevBuf WC(count * 16384, s);
    decode_batch_r(EB.as<uint4>(), count, WC.as<uint32_t>(), 4096, s);
    conv_rows_batch16(WC.as<uint32_t>(), count * 4096, true, s);
    launch_k(batch_fold_store_kernel, dim3((unsigned)std::min<uint64_t>(count, 148u * 8u)), dim3(256), 0, s, WC.as<uint32_t>(), c,
             (uint64_t)c_stride_words, (uint64_t)(a_bits + b_bits - 1), (uint64_t)count);
    FPM_LAUNCH_CHECK();
    return;
  }
  const DeviceTables& dt = device_tables(dev);
  const size_t smem = kBatchSmemUint4 * sizeof(uint4);
  static PerDeviceOnce attr;
  attr.run([&] {
    FPM_CUDA(cudaFuncSetAttribute(batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  for (size_t off = 0; off < count; off += 65535u * 16u) {
    const size_t cnt = std::min<size_t>(count - off, 65535u * 16u);
    launch_k(batch_kernel, dim3((unsigned)cnt), dim3(256), smem, s, a + off * a_stride_words, a_bits, a_stride_words,
                                                  b + off * b_stride_words, b_bits, b_stride_words,
                                                  c + off * c_stride_words, c_stride_words, l, dt.enc_m8, dt.dec_m8,
                                                  dt.enc_rows, dt.inv_rows, make_twiddle_src(dev, l, partition_base(l)));
    FPM_LAUNCH_CHECK();
  }
}

}  // namespace fpm
