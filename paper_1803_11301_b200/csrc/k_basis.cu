// k_basis.cu -- monomial <-> novel-polynomial basis conversion (Taylor expansion) on sm_100a.
//
// Reference: proj/src/basis_convert.cpp.  The conversion is the fixed sequence of fold passes of
// build_schedule (:53-67); pass (S, D) acts on every aligned S-bit span:
//     forward  y[q] = x[q] ^ x[q+D] ^ (q+2D < S ? x[q+2D] : 0)      q in [S/2-D, S-D)
//     inverse  x[q] = y[q] ^ y[q+D]                                 (reverse pass order)
// with all right-hand sides pre-pass values (:34-46).
//
// GPU structure (HBM-bound work; bytes only):
//  * bc_tile_kernel: the maximal run of passes with S <= 2^16 at the end of the forward schedule
//    (start of the inverse) -- the per-digit conversion build_schedule(2^16, 1) -- runs on 8 KiB
//    tiles double-buffered in shared memory: one HBM read + one write for ~32 passes.
//  * bc_pass_kernel: each larger pass as an in-place sweep in two race-free phases:
//    region L = [S/2-D, S/2) (reads the pre-pass upper half), then U = [S/2, S-D) (reads only
//    [S/2+D, S), never written by the pass).  Spans whose sources lie in the zero tail are skipped
//    (the reference's content_bits skip, :167).
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "basis_dev.cuh"
#include "fpm_internal.h"

namespace fpm {
namespace {

constexpr int kTileLog2 = 16;                // 2^16-bit tiles (8 KiB)

// ------------------------------------------------------------------ big passes, in place
__global__ void bc_pass_kernel(uint32_t* __restrict__ w, uint64_t nwords, uint64_t S, uint64_t D, int inverse,
                               uint64_t w_first, uint64_t nw_span, uint64_t nspans, uint64_t rlo, uint64_t rhi,
                               uint64_t live_bits) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t total = nw_span * nspans;
  for (uint64_t k = t; k < total; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t span = k / nw_span;
    const uint64_t base = span * S;
    if (!inverse && base + S / 2 >= live_bits) continue;  // sources in the zero tail
    const uint64_t wi = (base >> 5) + w_first + (k - span * nw_span);
    const uint32_t nv = fold_word(w, nwords, wi, S, D, inverse != 0, rlo, rhi);
    w[wi] = nv;
  }
}

// ------------------------------------------------------------------ small passes, SMEM tiles
__global__ void __launch_bounds__(256) bc_tile_kernel(uint32_t* __restrict__ w, uint64_t nwords, int tile_words,
                                                      PassList pl, int inverse, uint64_t live_words) {
  extern __shared__ uint32_t sm[];
  uint32_t* bufA = sm;
  uint32_t* bufB = sm + tile_words;
  const uint64_t ntiles = nwords / tile_words;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t off = tile * tile_words;
    if (!inverse && off >= live_words) continue;  // all-zero tile stays zero
    for (int i = threadIdx.x; i < tile_words; i += blockDim.x) bufA[i] = w[off + i];
    __syncthreads();
    const uint32_t* a = smem_passes(bufA, bufB, tile_words, pl, inverse != 0);
    for (int i = threadIdx.x; i < tile_words; i += blockDim.x) w[off + i] = a[i];
    __syncthreads();
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev;
    FPM_CUDA(cudaGetDevice(&dev));
    FPM_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

void run_tile_passes(uint32_t* w, uint64_t nwords, const std::vector<Pass>& passes, bool inverse, uint64_t live_bits,
                     cudaStream_t s) {
  if (passes.empty()) return;
  const PassList pl = make_passlist(passes, inverse);
  uint64_t tile_bits = 32;
  for (const Pass& p : passes) tile_bits = std::max<uint64_t>(tile_bits, p.span);
  // Tile: at least 256 words (one per thread), at most the array.
  uint64_t tile_words = tile_bits / 32;
  if (tile_words < 256) tile_words = 256;
  if (tile_words > nwords) tile_words = nwords;
  const size_t smem = 2 * tile_words * sizeof(uint32_t);
  const uint64_t ntiles = nwords / tile_words;
  const uint64_t live_words = (live_bits + 31) / 32;
  const int grid = (int)std::min<uint64_t>(ntiles, (uint64_t)sm_count() * 8);
  bc_tile_kernel<<<grid, 256, smem, s>>>(w, nwords, (int)tile_words, pl, inverse ? 1 : 0, live_words);
  FPM_LAUNCH_CHECK();
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
    const int threads = 256;
    const uint64_t blocks = std::min<uint64_t>((total + threads - 1) / threads, (uint64_t)sm_count() * 32);
    bc_pass_kernel<<<(unsigned)blocks, threads, 0, s>>>(w, nwords, S, D, inverse ? 1 : 0, w_first, nw_span, nspans,
                                                       rlo, rhi, live_bits);
    FPM_LAUNCH_CHECK();
  }
}

}  // namespace

void basis_cvt_device(uint32_t* w, size_t n_bits, size_t live_bits, bool inverse, cudaStream_t s) {
  if (n_bits < 32 || (n_bits & (n_bits - 1))) throw Error(kInvalid, "basis_cvt: length must be a power of two >= 32");
  static thread_local Pass sched[512];
  size_t np = 0;
  build_schedule(sched, &np, n_bits, 1);
  // Split: [big passes][maximal suffix with S <= 2^16].
  size_t split = np;
  while (split > 0 && sched[split - 1].span <= ((size_t)1 << kTileLog2)) --split;
  std::vector<Pass> big(sched, sched + split), small(sched + split, sched + np);
  const uint64_t nwords = n_bits / 32;
  if (!inverse) {
    for (const Pass& p : big) run_big_pass(w, nwords, p, false, live_bits, s);
    run_tile_passes(w, nwords, small, false, live_bits, s);
  } else {
    std::vector<Pass> rsmall(small.rbegin(), small.rend());
    run_tile_passes(w, nwords, rsmall, true, n_bits, s);
    for (size_t k = big.size(); k-- > 0;) run_big_pass(w, nwords, big[k], true, n_bits, s);
  }
}

}  // namespace fpm
