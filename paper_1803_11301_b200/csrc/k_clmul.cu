// k_clmul.cu -- word-level carry-less product on sm_100a: the reference's Karatsuba / schoolbook
// path.
//
// Reference: proj/src/polymul.cpp:156-183 (kara_words), :268-282 (karatsuba_mul), :223-231
// (fp_polymul takes it in auto mode below fft_threshold_bits = 4096), and
// proj/include/fpmul/detail/kernels_impl.hpp:125-137 (naive_mul_words_kernel: out[i+j] ^= lo,
// out[i+j+1] ^= hi of clmul64(a[i], b[j])).  Over GF(2) every exact product algorithm gives the
// same words, so the GPU computes the schoolbook sum directly, tiled for shared memory:
//   * CTA (x, y) owns output words [256x, 256x + 256) and the a-words of chunk range y;
//   * per a-chunk of 256 words it stages a[i0 .. i0+256) and the b-window b[k0-i0-256 .. k0-i0+256)
//     in shared memory; thread t (output word k = k0 + t) XORs lo(a_i b_{k-i}) into its word and
//     hi(a_i b_{k-i}) into the next one (kept in a second accumulator, passed down at the end);
//   * each 64 x 64 carry-less product is clmul64 of gf128.cuh (Karatsuba over three IMAD-hole
//     32 x 32 products, no carry-less multiply instruction on the GPU);
//   * chunk ranges (gridDim.y > 1) combine by atomicXor into the zero-filled output.
// Work: wa * wb clmul64 (~2.3 clk each per SM); it serves short products and the independent
// cross-check of the FFT path (karatsuba_mul / naive_mul, polymul.hpp:83-87).
#include <cuda_runtime.h>

#include <algorithm>

#include "fpm_internal.h"
#include "gf128.cuh"

namespace fpm {
namespace {

constexpr int kClTile = 256;

__global__ void __launch_bounds__(kClTile) clmul_words_kernel(const uint64_t* __restrict__ a, uint64_t wa,
                                                               const uint64_t* __restrict__ b, uint64_t wb,
                                                               uint64_t* __restrict__ out, uint64_t wout,
                                                               uint64_t chunks_per_y) {
  pdl_wait();
  __shared__ uint64_t sa[kClTile];
  __shared__ uint64_t sb[2 * kClTile];
  __shared__ uint64_t carry[kClTile];
  const int t = threadIdx.x;
  const uint64_t k0 = (uint64_t)blockIdx.x * kClTile, k = k0 + t;
  const uint64_t nchunks = (wa + kClTile - 1) / kClTile;
  const uint64_t c_begin = (uint64_t)blockIdx.y * chunks_per_y;
  const uint64_t c_end = std::min<uint64_t>(nchunks, c_begin + chunks_per_y);
  uint64_t lo = 0, hi = 0;  // contributions to out[k] and out[k + 1]
  for (uint64_t c = c_begin; c < c_end; ++c) {
    const uint64_t i0 = c * kClTile;
    // output words of this tile need b_j with j = k - i in (k0 - i0 - 256, k0 - i0 + 256)
    if (k0 + kClTile <= i0 || k0 >= i0 + kClTile + wb) continue;  // uniform across the CTA
    __syncthreads();
    sa[t] = i0 + t < wa ? a[i0 + t] : 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = (int64_t)k0 - (int64_t)i0 - kClTile + h * kClTile + t;  // sb[x] = b[k0 - i0 - 256 + x]
      sb[h * kClTile + t] = j >= 0 && (uint64_t)j < wb ? b[j] : 0;
    }
    __syncthreads();
#pragma unroll 4
    for (int ii = 0; ii < kClTile; ++ii) {
      const uint64_t x = sa[ii];                 // a[i0 + ii]
      const uint64_t y = sb[kClTile + t - ii];   // b[k - i0 - ii]
      uint64_t plo, phi;
      clmul64(x, y, plo, phi);
      lo ^= plo;
      hi ^= phi;
    }
  }
  // out[k] = lo(k) ^ hi(k - 1): the previous word's high half comes from thread t - 1, or for
  // t == 0 from the previous tile (whose thread 255 adds it there by atomicXor).
  carry[t] = hi;
  __syncthreads();
  uint64_t v = lo ^ (t ? carry[t - 1] : 0);
  if (k < wout && v) atomicXor(reinterpret_cast<unsigned long long*>(out + k), (unsigned long long)v);
  if (t == kClTile - 1 && k + 1 < wout && hi)
    atomicXor(reinterpret_cast<unsigned long long*>(out + k + 1), (unsigned long long)hi);
  pdl_trigger();  // (late: the next kernel is scheduled as this grid drains)
}

}  // namespace

// out[0 .. wa + wb) = a * b (carry-less), stream-ordered.
void clmul_words_device(const uint64_t* a, uint64_t wa, const uint64_t* b, uint64_t wb, uint64_t* out,
                        cudaStream_t s) {
  const uint64_t wout = wa + wb;
  if (!wout) return;
  FPM_CUDA(cudaMemsetAsync(out, 0, wout * 8, s));
  if (!wa || !wb) return;
  if (wa < wb) {  // fewer a-chunks: less staging
    std::swap(a, b);
    std::swap(wa, wb);
  }
  const uint64_t tiles = (wout + kClTile - 1) / kClTile;
  const uint64_t nchunks = (wa + kClTile - 1) / kClTile;
  int dev, sms;
  FPM_CUDA(cudaGetDevice(&dev));
  FPM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // split the a-chunks over gridDim.y until the grid covers ~8 CTAs per SM
  uint64_t ys = 1;
  while (tiles * ys < (uint64_t)sms * 8 && ys < nchunks && ys < 65535) ys *= 2;
  ys = std::min<uint64_t>(ys, nchunks);
  const uint64_t per_y = (nchunks + ys - 1) / ys;
  ys = (nchunks + per_y - 1) / per_y;
  if (tiles > 0x7FFFFFFFull) throw Error(kInvalid, "clmul_words: product too long");
  launch_k(clmul_words_kernel, dim3(dim3((unsigned)tiles, (unsigned)ys)), dim3(kClTile), 0, s, a, wa, b, wb, out, wout, per_y);
  FPM_LAUNCH_CHECK();
}

}  // namespace fpm
