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

#include <vector>

#include "basis_dev.cuh"
#include "fpm_internal.h"
#include "gf128.cuh"

namespace fpm {


namespace {

constexpr int kBatchMaxLog2N = 17;

__device__ __forceinline__ uint4 c2p2b(const uint4* __restrict__ c2p, uint64_t b) {
  uint4 r = c2p[b & 511];
  if (b >> 9) r = x4(r, c2p[512 + ((b >> 9) & 511)]);
  return r;
}

__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
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

// Forward transform of one operand: W0 <- x (n/2 bits), basis conversion, encode into E, butterflies.
__device__ void transform_operand(const uint64_t* __restrict__ x, uint64_t x_bits, uint32_t* W0, uint32_t* W1,
                                  uint4* E, unsigned l, int half_words, const PassList& pl_half,
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
  const uint32_t* P = smem_passes(W0, W1, half_words, pl_half, false);
  // encode: f_i = sum_j a_{j n_p + i} r_j, rows j < 64 (the upper half is zero padding)
  const int n_p = 1 << l;
  const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  if (n_p >= 32) {
    const int row_words = n_p / 32;
    for (int col = warp; col < row_words; col += nwarps) {
      const uint32_t lo = transpose32(P[lane * row_words + col], lane);
      const uint32_t hi = transpose32(P[(lane + 32) * row_words + col], lane);
      uint4 f = make_uint4(0, 0, 0, 0);
      for (int j = 0; j < 32; ++j) {
        if (lo >> j & 1u) f = x4(f, enc_rows[j]);
        if (hi >> j & 1u) f = x4(f, enc_rows[32 + j]);
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

__global__ void __launch_bounds__(256) batch_kernel(const uint64_t* __restrict__ a, uint64_t a_bits, uint64_t a_stride,
                                                    const uint64_t* __restrict__ b, uint64_t b_bits, uint64_t b_stride,
                                                    uint64_t* __restrict__ c, uint64_t c_stride, unsigned l,
                                                    PassList pl_half, PassList pl_full_inv,
                                                    const uint4* __restrict__ enc_rows,
                                                    const uint4* __restrict__ inv_rows, TwiddleSrc tw) {
  extern __shared__ uint4 sm[];
  const int n_p = 1 << l;
  const int n_words = n_p * 4;  // n = 128 n_p bits
  uint4* EA = sm;
  uint4* EB = sm + n_p;
  uint32_t* W0 = reinterpret_cast<uint32_t*>(sm + 2 * n_p);
  uint32_t* W1 = W0 + n_words;
  const uint64_t prod = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

  transform_operand(a + prod * a_stride, a_bits, W0, W1, EA, l, n_words / 2, pl_half, enc_rows, tw);
  transform_operand(b + prod * b_stride, b_bits, W0, W1, EB, l, n_words / 2, pl_half, enc_rows, tw);
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
  // decode: y_i = f_i E^{-1}; bit j of y_i -> c_{j n_p + i}  (encode.cpp:195-220)
  for (int i = tid; i < n_p; i += blockDim.x) {
    const uint4 f = EA[i];
    const uint32_t fw[4] = {f.x, f.y, f.z, f.w};
    uint4 y = make_uint4(0, 0, 0, 0);
    for (int t = 0; t < 128; ++t)
      if ((fw[t >> 5] >> (t & 31)) & 1u) y = x4(y, inv_rows[t]);
    EB[i] = y;  // EB is free now
  }
  __syncthreads();
  if (n_p >= 32) {
    const int row_words = n_p / 32;
    for (int col = warp; col < row_words; col += nwarps) {
      const uint4 y = EB[col * 32 + lane];
      W0[(0 * 32 + lane) * row_words + col] = transpose32(y.x, lane);
      W0[(1 * 32 + lane) * row_words + col] = transpose32(y.y, lane);
      W0[(2 * 32 + lane) * row_words + col] = transpose32(y.z, lane);
      W0[(3 * 32 + lane) * row_words + col] = transpose32(y.w, lane);
    }
  } else {
    for (int wi = tid; wi < n_words; wi += blockDim.x) {
      uint32_t out = 0;
      for (int bb = 0; bb < 32; ++bb) {
        const int k = wi * 32 + bb, j = k / n_p, i = k % n_p;
        const uint4 y = EB[i];
        const uint32_t yw[4] = {y.x, y.y, y.z, y.w};
        out |= ((yw[j >> 5] >> (j & 31)) & 1u) << bb;
      }
      W0[wi] = out;
    }
  }
  __syncthreads();
  const uint32_t* C = smem_passes(W0, W1, n_words, pl_full_inv, true);
  // trim to len_a + len_b - 1 bits and write 64-bit words
  const uint64_t out_bits = a_bits + b_bits - 1;
  const uint64_t out_words = (out_bits + 63) / 64;
  uint64_t* cc = c + prod * c_stride;
  for (uint64_t k = tid; k < out_words; k += blockDim.x) {
    uint64_t v = (uint64_t)C[2 * k] | ((uint64_t)C[2 * k + 1] << 32);
    if (k == out_words - 1 && (out_bits & 63)) v &= (((uint64_t)1) << (out_bits & 63)) - 1;
    cc[k] = v;
  }
}

}  // namespace

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
  Pass sched[128];
  size_t np = 0;
  build_schedule(sched, &np, n / 2, 1);
  const PassList pl_half = make_passlist(std::vector<Pass>(sched, sched + np), false);
  np = 0;
  build_schedule(sched, &np, n, 1);
  std::vector<Pass> inv(sched, sched + np);
  std::vector<Pass> rinv(inv.rbegin(), inv.rend());
  const PassList pl_full_inv = make_passlist(rinv, true);
  int dev;
  FPM_CUDA(cudaGetDevice(&dev));
  const DeviceTables& dt = device_tables(dev);
  const size_t n_p = (size_t)1 << l;
  const size_t smem = 2 * n_p * sizeof(uint4) + 2 * (n / 8);
  static bool attr = false;
  if (!attr) {
    FPM_CUDA(cudaFuncSetAttribute(batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 1024 * 16 + 2 * (1 << 14)));
    attr = true;
  }
  for (size_t off = 0; off < count; off += 65535u * 16u) {
    const size_t cnt = std::min<size_t>(count - off, 65535u * 16u);
    batch_kernel<<<(unsigned)cnt, 256, smem, s>>>(a + off * a_stride_words, a_bits, a_stride_words,
                                                  b + off * b_stride_words, b_bits, b_stride_words,
                                                  c + off * c_stride_words, c_stride_words, l, pl_half, pl_full_inv,
                                                  dt.enc_rows, dt.inv_rows, make_twiddle_src(dev, l, partition_base(l)));
    FPM_LAUNCH_CHECK();
  }
}

}  // namespace fpm
